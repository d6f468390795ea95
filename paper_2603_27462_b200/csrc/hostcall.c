/* hostcall.c -- CPython fast-call binding of the two host-buffer entry points
 * of librsr_b200.so (rsr_matvec_host, rsr_fused_matvec_host).
 *
 * The numpy path of rsr_matvec / rsr_matvec_fused is a ~50 us host-in,
 * host-out round trip; a ctypes call plus `ndarray.ctypes.data` costs ~3-4 us
 * of it.  This module takes the function address from the ctypes handle, the
 * vector as any C-contiguous buffer and the rest as integers, and calls
 * through with the GIL released.  It carries no logic of its own: kernels.py
 * falls back to the ctypes call when the module is not built.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stddef.h>

typedef int (*matvec_host_fn)(const void *, const void *, int, void *, void *, void *, void *,
                              size_t, void *);
typedef int (*fused_host_fn)(const void *, const void *, int, double, void *, void *, void *,
                             void *, size_t, void *);

static int as_ptr(PyObject *o, void **out) {
    *out = PyLong_AsVoidPtr(o);
    return !(*out == NULL && PyErr_Occurred());
}

/* matvec_host(fn, view, v, dtype, y, dv, dy, ws, wsb, stream) -> status */
static PyObject *matvec_host(PyObject *self, PyObject *const *a, Py_ssize_t n) {
    (void)self;
    if (n != 10) {
        PyErr_SetString(PyExc_TypeError, "matvec_host takes 10 arguments");
        return NULL;
    }
    void *fn, *view, *y, *dv, *dy, *ws, *stream;
    if (!as_ptr(a[0], &fn) || !as_ptr(a[1], &view) || !as_ptr(a[4], &y) || !as_ptr(a[5], &dv) ||
        !as_ptr(a[6], &dy) || !as_ptr(a[7], &ws) || !as_ptr(a[9], &stream))
        return NULL;
    const long dtype = PyLong_AsLong(a[3]);
    const size_t wsb = PyLong_AsSize_t(a[8]);
    if (PyErr_Occurred()) return NULL;
    Py_buffer vb;
    if (PyObject_GetBuffer(a[2], &vb, PyBUF_C_CONTIGUOUS) != 0) return NULL;
    int st;
    Py_BEGIN_ALLOW_THREADS
    st = ((matvec_host_fn)fn)(view, vb.buf, (int)dtype, y, dv, dy, ws, wsb, stream);
    Py_END_ALLOW_THREADS
    PyBuffer_Release(&vb);
    return PyLong_FromLong(st);
}

/* fused_host(fn, view, v, dtype, beta, y, dv, dy, ws, wsb, stream) -> status */
static PyObject *fused_host(PyObject *self, PyObject *const *a, Py_ssize_t n) {
    (void)self;
    if (n != 11) {
        PyErr_SetString(PyExc_TypeError, "fused_host takes 11 arguments");
        return NULL;
    }
    void *fn, *view, *y, *dv, *dy, *ws, *stream;
    if (!as_ptr(a[0], &fn) || !as_ptr(a[1], &view) || !as_ptr(a[5], &y) || !as_ptr(a[6], &dv) ||
        !as_ptr(a[7], &dy) || !as_ptr(a[8], &ws) || !as_ptr(a[10], &stream))
        return NULL;
    const long dtype = PyLong_AsLong(a[3]);
    const double beta = PyFloat_AsDouble(a[4]);
    const size_t wsb = PyLong_AsSize_t(a[9]);
    if (PyErr_Occurred()) return NULL;
    Py_buffer vb;
    if (PyObject_GetBuffer(a[2], &vb, PyBUF_C_CONTIGUOUS) != 0) return NULL;
    int st;
    Py_BEGIN_ALLOW_THREADS
    st = ((fused_host_fn)fn)(view, vb.buf, (int)dtype, beta, y, dv, dy, ws, wsb, stream);
    Py_END_ALLOW_THREADS
    PyBuffer_Release(&vb);
    return PyLong_FromLong(st);
}

static PyMethodDef methods[] = {
    {"matvec_host", (PyCFunction)(void (*)(void))matvec_host, METH_FASTCALL,
     "rsr_matvec_host through a function address"},
    {"fused_host", (PyCFunction)(void (*)(void))fused_host, METH_FASTCALL,
     "rsr_fused_matvec_host through a function address"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_hostcall", NULL, -1, methods};

PyMODINIT_FUNC PyInit__hostcall(void) { return PyModule_Create(&mod); }
