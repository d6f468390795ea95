"""Online multiply API on the GPU (operator API of reference kernels.py).

Same names, arguments, dtypes and errors as pkg/src/rsrmv/kernels.py:
``rsr_matvec`` (int8 -> exact int32; real -> float32), ``rsr_matvec_fused``
(ternary only; quantize -> exact int multiply -> f32(f64(y)*beta/scale)),
``batched_preprocess``, ``Multiplier`` / ``multiplier_multiply`` and
``OpCounter``.  Every multiply runs the sm_100a kernels of
csrc/rsr_matvec.cu through the C ABI; there is no CPU path.

Vectors may be numpy arrays (copied to the artifact's device, result copied
back -- the reference-facing, host-buffer call) or CUDA tensors (result stays
on the device, nothing synchronizes).
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionMismatch, HeterogeneousSiblings
from .matcore import (BINARY, TERNARY, PackedMatrix, _is_torch, dense_device,
                      naive_matvec, quantize_activations)
from .preproc import RsrArtifact, preprocess

NAIVE_F32 = "NaiveF32"
NAIVE_I8 = "NaiveI8"
RSR_BINARY = "RsrBinary"
RSR_TERNARY = "RsrTernary"
KINDS = (NAIVE_F32, NAIVE_I8, RSR_BINARY, RSR_TERNARY)


@dataclass
class OpCounter:
    """Add/visit counts over one or more multiplies (reference kernels.py:30-36)."""
    gather_adds: int = 0
    scatter_adds: int = 0
    groups_visited: int = 0


def thread_count() -> int:
    """RSR_THREADS (reference kernels.py:39-45).  Kept for API compatibility:
    the GPU kernels ignore it (the whole device is used)."""
    try:
        t = int(os.environ.get("RSR_THREADS", "1"))
    except ValueError:
        return 1
    return max(1, t)


def _count(a: RsrArtifact, counter: OpCounter | None):
    if counter is not None:
        g, s, ng = a.op_totals()
        counter.gather_adds += g
        counter.scatter_adds += s
        counter.groups_visited += ng


class _Workspace:
    """Scratch for tile partials, one buffer per (device, stream), grown on
    demand.  Keyed by stream so multiplies running concurrently on different
    streams never share partials; a superseded buffer is simply released
    (torch's caching allocator only hands its block to later work on the
    same stream, i.e. after the kernels that used it)."""
    _bufs: dict = {}
    _lock = threading.Lock()

    @classmethod
    def get(cls, device, nbytes: int, stream: int = 0):
        import torch
        if nbytes <= 0:
            return None, 0
        key = (str(device), int(stream))
        with cls._lock:
            b = cls._bufs.get(key)
            if b is None or b.numel() < nbytes:
                b = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8, device=device)
                cls._bufs[key] = b
        return b, nbytes


def _prepare_vec(a: RsrArtifact, v):
    """-> (device tensor, is_host, kind) with kind 'int' or 'float'."""
    import torch
    host = not _is_torch(v)
    if host:
        vn = np.asarray(v)
        if vn.ndim != 1 or vn.shape[0] != a.n:
            raise DimensionMismatch(f"vector of length {vn.size} against {a.n} columns")
        if np.issubdtype(vn.dtype, np.integer):
            if vn.dtype != np.int8:
                raise DimensionMismatch("integer vectors must be int8")
            t = torch.from_numpy(np.ascontiguousarray(vn))
        else:
            t = torch.from_numpy(np.ascontiguousarray(vn.astype(np.float32, copy=False)))
        return t.to(a.device, non_blocking=False), True
    t = v
    if t.dim() != 1 or t.shape[0] != a.n:
        raise DimensionMismatch(f"vector of length {t.numel()} against {a.n} columns")
    if not (t.is_floating_point() or t.is_complex()):
        if t.dtype != torch.int8:
            raise DimensionMismatch("integer vectors must be int8")
    elif t.dtype not in (torch.float32, torch.bfloat16, torch.float16):
        t = t.to(torch.float32)
    if t.device != a.device:
        t = t.to(a.device)
    return t.contiguous(), False


class _ViewLaunch:
    """Per-view launch state cached on first use (ctypes byref + workspace
    size); the workspace itself is looked up per stream."""
    __slots__ = ("ref", "wsb", "device")

    def __init__(self, a: RsrArtifact, vw):
        import ctypes
        self.ref = ctypes.byref(vw)
        self.wsb = int(_lib.lib().rsr_matvec_workspace_bytes(self.ref))
        self.device = a.device

    def workspace(self, stream: int):
        if self.wsb <= 0:
            return 0, 0
        ws, wsb = _Workspace.get(self.device, self.wsb, stream)
        return _lib.ptr(ws), wsb


def _launch_state(a: RsrArtifact, view) -> _ViewLaunch:
    vw = a._view if view is None else view
    cache = a.__dict__.setdefault("_launch_cache", {})
    st = cache.get(id(vw))
    if st is None or st.ref._obj is not vw:
        st = _ViewLaunch(a, vw)
        cache[id(vw)] = st
    return st


def matvec_into(a: RsrArtifact, vt, y, accumulate: bool = False, view=None, stream=None):
    """Launch the multiply on device tensors: y (+)= A.v (no checks, no sync).

    vt: int8 -> y int32; float32/bfloat16/float16 -> y float32.
    """
    from .matcore import _dtype_code
    st = _launch_state(a, view)
    s = _lib.current_stream_ptr(a.device) if stream is None else stream
    ws, wsb = st.workspace(s) if st.wsb else (0, 0)
    _lib.check(_lib.lib().rsr_matvec(st.ref, vt.data_ptr(), _dtype_code(vt), y.data_ptr(),
                                     int(accumulate), ws, wsb, s), "rsr_matvec")
    return y


def matvec_peers_into(a: RsrArtifact, vt, peer_rows, npeers: int, view=None, stream=None):
    """Multiply and all-gather in one launch (rsr_matvec_peers): every output
    row is stored to each of `npeers` buffers.  peer_rows: int64 device
    tensor of npeers addresses, each this artifact's row 0 inside one rank's
    full output (peer memory mapped here, e.g. symmetric memory).  The caller
    synchronizes the ranks before reading (shard.ShardedMatrix does)."""
    from .matcore import _dtype_code
    st = _launch_state(a, view)
    s = _lib.current_stream_ptr(a.device) if stream is None else stream
    ws, wsb = st.workspace(s) if st.wsb else (0, 0)
    _lib.check(_lib.lib().rsr_matvec_peers(st.ref, vt.data_ptr(), _dtype_code(vt),
                                           peer_rows.data_ptr(), int(npeers), ws, wsb, s),
               "rsr_matvec_peers")


def fused_into(a: RsrArtifact, vt, out, beta: float | None = None, view=None, stream=None,
               scale_out=None, row_beta=None):
    """Launch the fused quantize/multiply/dequantize kernel on device tensors.

    out: float32 or bfloat16.  row_beta: optional float64 device tensor of
    per-row betas (stacked siblings)."""
    import torch
    from .matcore import _dtype_code
    st = _launch_state(a, view)
    s = _lib.current_stream_ptr(a.device) if stream is None else stream
    b = float(a.weight_scale) if beta is None else float(beta)
    odt = _lib.RSR_BF16 if out.dtype == torch.bfloat16 else _lib.RSR_F32
    ws, wsb = st.workspace(s) if st.wsb else (0, 0)
    _lib.check(_lib.lib().rsr_fused_matvec(st.ref, vt.data_ptr(), _dtype_code(vt), b,
                                           _lib.ptr(row_beta), out.data_ptr(), odt,
                                           _lib.ptr(scale_out), ws, wsb, s),
               "rsr_matvec_fused")
    return out


def fused_norm_into(a: RsrArtifact, vt, out, norm_w, norm_eps: float, beta: float | None = None,
                    row_beta=None, stream=None):
    """BitLinear in one launch: the fused kernel of the RMS-normalized bf16
    vector (HF BitNetRMSNorm with weight norm_w and eps; rsr_fused_matvec_norm).
    Raises CorruptArtifact (invalid argument) when the shape has no register-
    staged prologue (several tiles, n % 8 != 0, n > 10240)."""
    import torch
    from .matcore import _dtype_code
    st = _launch_state(a, None)
    s = _lib.current_stream_ptr(a.device) if stream is None else stream
    b = float(a.weight_scale) if beta is None else float(beta)
    odt = _lib.RSR_BF16 if out.dtype == torch.bfloat16 else _lib.RSR_F32
    ws, wsb = st.workspace(s) if st.wsb else (0, 0)
    _lib.check(_lib.lib().rsr_fused_matvec_norm(st.ref, vt.data_ptr(), _dtype_code(vt),
                                                norm_w.data_ptr(), float(norm_eps), b,
                                                _lib.ptr(row_beta), out.data_ptr(), odt, ws, wsb,
                                                s), "rsr_fused_matvec_norm")
    return out


def fused_rows_into(a: RsrArtifact, V, out, beta: float | None = None, row_beta=None,
                    stream=None, norm_w=None, norm_eps: float = 0.0):
    """The fused quantize/multiply/dequantize path for T activation rows at
    once (prefill): out[t] = rsr_matvec_fused(a, V[t]) bit for bit, computed
    as one per-row quantization launch, one batched exact int8 multiply
    (matmul_into) and one dequantization launch.  V: [T, n] f32/bf16/f16;
    out: [T, m] float32 or bfloat16; row_beta as fused_into; norm_w / norm_eps
    as fused_norm_into (bf16 rows).  From TC_MIN_BATCH rows the multiply and
    the dequantization are one int8 tensor-core launch."""
    import torch
    from .matcore import _dtype_code
    T = int(V.shape[0])
    if T == 0:
        return out
    V = V.contiguous()
    dev = a.device
    s = _lib.current_stream_ptr(dev) if stream is None else stream
    L = _lib.lib()
    # pitch a multiple of 16 bytes: the int8 tensor-core path loads rows by TMA
    Q = torch.empty(T, -(-a.n // 16) * 16, dtype=torch.int8, device=dev)[:, :a.n]
    scales = torch.empty(T, dtype=torch.float64, device=dev)
    _lib.check(L.rsr_absmax_quantize_rows(V.data_ptr(), _dtype_code(V), V.stride(0), T, a.n,
                                          _lib.ptr(norm_w), float(norm_eps), Q.data_ptr(),
                                          Q.stride(0), scales.data_ptr(), s),
               "quantize rows")
    b = float(a.weight_scale) if beta is None else float(beta)
    odt = _lib.RSR_BF16 if out.dtype == torch.bfloat16 else _lib.RSR_F32
    if TC_MIN_BATCH <= T <= 256 and a.keymat("i8") is not None:
        # int8 tensor cores with the dequantization in the epilogue: one launch
        vw = a._view
        wsb = int(L.rsr_matmul_tc_workspace_bytes(a.m, a.n, a.k, vw.row_begin_block,
                                                  vw.n_blocks, T))
        ws, wsb = _Workspace.get(dev, wsb, s)
        with torch.cuda.device(dev):
            _lib.check(L.rsr_matmul_tc_i8_dequant(
                _lib.ptr(a.keymat("i8")), a.m, a.n, vw.bitwidth, a.k, vw.row_begin_block,
                vw.n_blocks, Q.data_ptr(), Q.stride(0), T, scales.data_ptr(),
                _lib.ptr(row_beta), b, out.data_ptr(), odt, out.stride(0), _lib.ptr(ws), wsb, s),
                "rsr_matmul_tc_i8_dequant")
        return out
    Y = torch.empty(T, a.m, dtype=torch.int32, device=dev)
    matmul_into(a, Q, Y, stream=s)
    _lib.check(L.rsr_dequant_rows(Y.data_ptr(), Y.stride(0), T, a.m, scales.data_ptr(),
                                  _lib.ptr(row_beta), b, out.data_ptr(), odt, out.stride(0), s),
               "dequant rows")
    return out


def rsr_matvec(a: RsrArtifact, v, counter: OpCounter | None = None,
               threads: int | None = None):
    """Multiply a preprocessed matrix by v on the GPU (reference kernels.py:59-102).

    int8 vectors take the exact integer path (int32 result); real vectors
    the float path (float32 result, fp32 accumulation -- see DESIGN.md for
    the stated tolerance).  ``threads`` is accepted for API compatibility.
    Host vectors (numpy float32 / int8, or a CPU torch bfloat16 tensor --
    numpy has no bf16) return a numpy result; device tensors stay on the
    device.
    """
    if type(v) is np.ndarray and v.ndim == 1 and v.shape[0] == a.n and \
            (v.dtype == np.float32 or v.dtype == np.int8):
        if counter is not None:
            _count(a, counter)
        return _matvec_host(a, v if v.flags.c_contiguous else np.ascontiguousarray(v))
    import torch
    if not _is_torch(v):
        vn = np.asarray(v)
        if vn.ndim == 1 and vn.shape[0] == a.n and vn.dtype in (np.int8, np.float32):
            _count(a, counter)
            return _matvec_host(a, np.ascontiguousarray(vn))
    elif v.device.type == "cpu" and v.dtype == torch.bfloat16 and v.dim() == 1 \
            and v.shape[0] == a.n:
        # a bf16 host vector (numpy has no bf16): host in, host out in one C
        # call, the bf16 kernel reading the halfwords as they are
        _count(a, counter)
        with _host_lock(a):
            return _matvec_host_locked(a, v.contiguous().view(torch.int16).numpy(), bf16=True)
    vt, host = _prepare_vec(a, v)
    _count(a, counter)
    if vt.dtype == torch.int8:
        y = torch.empty(a.m, dtype=torch.int32, device=a.device)
    else:
        y = torch.empty(a.m, dtype=torch.float32, device=a.device)
    matvec_into(a, vt, y)
    return y.cpu().numpy() if host else y


try:  # CPython fast-call binding of the host round trips (csrc/hostcall.c)
    from . import _hostcall
except ImportError:  # not built: the same C entry points through ctypes
    _hostcall = None

_FN_ADDR: dict = {}


def _fn_addr(fn) -> int:
    a = _FN_ADDR.get(id(fn))
    if a is None:
        a = _FN_ADDR[id(fn)] = ctypes.cast(fn, ctypes.c_void_p).value
    return a


def _host_lock(a: RsrArtifact) -> threading.Lock:
    lk = a.__dict__.get("_host_lock")
    if lk is None:
        with _HOST_LOCKS_GUARD:
            lk = a.__dict__.setdefault("_host_lock", threading.Lock())
    return lk


_HOST_LOCKS_GUARD = threading.Lock()


def _matvec_host(a: RsrArtifact, vn: np.ndarray) -> np.ndarray:
    """numpy in, numpy out in one C call (H2D, multiply, D2H, sync) using
    device buffers cached on the artifact.  The call's constant arguments
    are bound once per (artifact, dtype); per call only the vector pointer
    and the current stream are read (the host-in/host-out latency is a few
    tens of microseconds, so Python overhead is a visible share of it).
    The C call releases the GIL, so the cached buffers are guarded by a
    per-artifact lock held until the result has been copied out: threads
    sharing an artifact serialize (as the reference's GIL-held cores do)."""
    with _host_lock(a):
        return _matvec_host_locked(a, vn)


def _matvec_host_locked(a: RsrArtifact, vn: np.ndarray, bf16: bool = False) -> np.ndarray:
    is_int = vn.dtype == np.int8
    key = "_host_call_i8" if is_int else ("_host_call_bf16" if bf16 else "_host_call_f32")
    hc = a.__dict__.get(key)
    if hc is None or hc[0] is not a._view:
        import torch
        dv = torch.empty(a.n, dtype=torch.int8 if is_int else
                         (torch.bfloat16 if bf16 else torch.float32), device=a.device)
        ydt = torch.int32 if is_int else torch.float32
        dy = torch.empty(a.m, dtype=ydt, device=a.device)
        # pinned landing buffer: mapped into the device address space, the
        # result is written by a copy kernel (page-locked, so no staging);
        # the caller gets a private copy
        hy = torch.empty(a.m, dtype=ydt, pin_memory=True).numpy()
        st = _launch_state(a, None)
        dev_idx = torch.device(a.device).index
        if dev_idx is None:
            dev_idx = torch.cuda.current_device()
        hc = a.__dict__[key] = (
            a._view, _lib.lib().rsr_matvec_host, st.ref,
            _lib.RSR_I8 if is_int else (_lib.RSR_BF16 if bf16 else _lib.RSR_F32),
            hy, hy.ctypes.data, dv.data_ptr(), dy.data_ptr(), st,
            torch._C._cuda_getCurrentRawStream, dev_idx, (dv, dy))
    _, fn, ref, code, hy, hyp, dvp, dyp, st, cur_stream, dev_idx, _keep = hc
    s = cur_stream(dev_idx)
    ws, wsb = st.workspace(s) if st.wsb else (0, 0)
    if _hostcall is not None:
        status = _hostcall.matvec_host(_fn_addr(fn), ctypes.addressof(a._view), vn, code, hyp,
                                       dvp, dyp, ws or 0, wsb, s)
    else:
        status = fn(ref, vn.ctypes.data, code, hyp, dvp, dyp, ws, wsb, s)
    if status:
        _lib.check(status, "rsr_matvec")
    return hy.copy()


def rsr_matvec_fused(a: RsrArtifact, v, counter: OpCounter | None = None):
    """Quantize v to int8, multiply exactly, rescale by weight_scale/scale
    (reference kernels.py:105-125), in one kernel launch."""
    if a.bitwidth != TERNARY:
        raise ValueError("fused path requires a ternary artifact")
    if type(v) is np.ndarray and v.ndim == 1 and v.shape[0] == a.n and v.dtype == np.float32:
        if counter is not None:
            _count(a, counter)
        return _fused_host(a, v if v.flags.c_contiguous else np.ascontiguousarray(v))
    import torch
    vt, host = _prepare_vec(a, v)
    _count(a, counter)
    if vt.dtype == torch.int8:
        vt = vt.to(torch.float32)
    out = torch.empty(a.m, dtype=torch.float32, device=a.device)
    fused_into(a, vt, out)
    return out.cpu().numpy() if host else out


def _fused_host(a: RsrArtifact, vn: np.ndarray) -> np.ndarray:
    """numpy float32 in, numpy float32 out through rsr_fused_matvec_host (one
    C call, constant arguments bound once per artifact; see _matvec_host)."""
    with _host_lock(a):
        return _fused_host_locked(a, vn)


def _fused_host_locked(a: RsrArtifact, vn: np.ndarray) -> np.ndarray:
    hc = a.__dict__.get("_host_call_fused")
    if hc is None or hc[0] is not a._view or hc[2] != float(a.weight_scale):
        import torch
        dv = torch.empty(a.n, dtype=torch.float32, device=a.device)
        dy = torch.empty(a.m, dtype=torch.float32, device=a.device)
        hy = torch.empty(a.m, dtype=torch.float32, pin_memory=True).numpy()
        st = _launch_state(a, None)
        dev_idx = torch.device(a.device).index
        if dev_idx is None:
            dev_idx = torch.cuda.current_device()
        hc = a.__dict__["_host_call_fused"] = (
            a._view, _lib.lib().rsr_fused_matvec_host, float(a.weight_scale), st.ref, hy,
            hy.ctypes.data, dv.data_ptr(), dy.data_ptr(), st,
            torch._C._cuda_getCurrentRawStream, dev_idx, (dv, dy))
    _, fn, beta, ref, hy, hyp, dvp, dyp, st, cur_stream, dev_idx, _keep = hc
    s = cur_stream(dev_idx)
    ws, wsb = st.workspace(s) if st.wsb else (0, 0)
    if _hostcall is not None:
        status = _hostcall.fused_host(_fn_addr(fn), ctypes.addressof(a._view), vn, _lib.RSR_F32,
                                      beta, hyp, dvp, dyp, ws or 0, wsb, s)
    else:
        status = fn(ref, vn.ctypes.data, _lib.RSR_F32, beta, hyp, dvp, dyp, ws, wsb, s)
    if status:
        _lib.check(status, "rsr_matvec_fused")
    return hy.copy()


# auto policy (measured at C4, ternary 8192^2 k=5, tools/bench_batched.py):
# bf16 and int8 batches from TC_MIN_BATCH on go to the tensor cores (bf16:
# 15.0 us at B=2 vs 21.7 for two single-vector calls); other batches of up to
# SINGLE_MAX_BATCH vectors take the single-vector kernel per column; the
# CUDA-core batched stream kernel covers the rest
SINGLE_MAX_BATCH = 2
TC_MIN_BATCH = 2
# bf16 batches up to this size take the 256-column-step kernel (N <= 32);
# RSR_TC_WIDE=0 turns it off (A/B experiments)
TC_WIDE_MAX_BATCH = int(os.environ.get("RSR_TC_WIDE_MAX", "32")) \
    if os.environ.get("RSR_TC_WIDE", "1") != "0" else 0


def matmul_into(a: RsrArtifact, Vt, Y, view=None, stream=None, method: str = "auto"):
    """Batched multiply on device tensors: Y[b] = A . Vt[b].

    Vt: [B, n] (int8 -> Y int32; float32/bfloat16/float16 -> Y float32), rows
    contiguous; Y: [B, rows].  method: "tc" (bf16 batches on tcgen05
    kind::f16, int8 batches on kind::i8 -- exact int32 -- via the code
    matrix), "stream" (CUDA-core kernel on the chunk stream) or "auto" (tc
    for bf16 / int8 batches of TC_MIN_BATCH .. 256 vectors, else the
    single-vector kernel per column up to SINGLE_MAX_BATCH, else stream).  Streams without a
    batched kernel (u32 format, > 2187 pattern keys, tiles above ~13k
    columns) run the single-vector kernel column by column.
    """
    import ctypes
    import torch
    from .matcore import _dtype_code
    B = int(Vt.shape[0])
    tc_dtype = Vt.dtype in (torch.bfloat16, torch.int8)
    use_tc = method == "tc" or (method == "auto" and tc_dtype and TC_MIN_BATCH <= B <= 256)
    i8 = Vt.dtype == torch.int8
    if use_tc and tc_dtype and B <= 256 and a.keymat("i8" if i8 else "bf16") is not None:
        vw = a._view if view is None else view
        align = 16 if i8 else 8  # TMA: rows 16-byte aligned
        if Vt.stride(0) % align or Vt.data_ptr() % 16:
            Vp = torch.empty(B, -(-a.n // align) * align, dtype=Vt.dtype, device=Vt.device)
            Vp[:, :a.n].copy_(Vt)
            Vt = Vp[:, :a.n]
        s = _lib.current_stream_ptr(a.device) if stream is None else stream
        L = _lib.lib()
        wsb = int(L.rsr_matmul_tc_workspace_bytes(a.m, a.n, a.k, vw.row_begin_block,
                                                  vw.n_blocks, B))
        ws, wsb = _Workspace.get(a.device, wsb, s)
        with torch.cuda.device(a.device):  # raw-pointer entry point: no view device
            if i8:
                _lib.check(L.rsr_matmul_tc_i8(_lib.ptr(a.keymat("i8")), a.m, a.n, vw.bitwidth,
                                              a.k, vw.row_begin_block, vw.n_blocks,
                                              Vt.data_ptr(), Vt.stride(0), B, Y.data_ptr(),
                                              Y.stride(0), _lib.ptr(ws), wsb, s),
                           "rsr_matmul_tc_i8")
            elif B <= TC_WIDE_MAX_BATCH:
                # 256-column steps over the wide code matrix (N = 16)
                _lib.check(L.rsr_matmul_tc_wide(_lib.ptr(a.keymat("wide")), a.m, a.n,
                                                vw.bitwidth, a.k, vw.row_begin_block,
                                                vw.n_blocks, Vt.data_ptr(), _lib.RSR_BF16,
                                                Vt.stride(0), B, Y.data_ptr(), Y.stride(0),
                                                _lib.ptr(ws), wsb, s), "rsr_matmul_tc_wide")
            else:
                _lib.check(L.rsr_matmul_tc(_lib.ptr(a.keymat()), a.m, a.n, vw.bitwidth, a.k,
                                           vw.row_begin_block, vw.n_blocks, Vt.data_ptr(),
                                           _lib.RSR_BF16, Vt.stride(0), B, Y.data_ptr(),
                                           Y.stride(0), _lib.ptr(ws), wsb, s), "rsr_matmul_tc")
        return Y
    if method == "tc":
        raise ValueError("the tensor-core path needs a bf16 or int8 batch of at most 256 "
                         "vectors and k <= 16")
    if method == "auto" and B <= SINGLE_MAX_BATCH:
        for b in range(B):
            matvec_into(a, Vt[b], Y[b], view=view, stream=stream)
        return Y
    vw = a._view if view is None else view
    s = _lib.current_stream_ptr(a.device) if stream is None else stream
    L = _lib.lib()
    ref = ctypes.byref(vw)
    wsb = int(L.rsr_matmul_workspace_bytes(ref, B))
    ws, wsb = _Workspace.get(a.device, wsb, s)
    st = L.rsr_matmul(ref, Vt.data_ptr(), _dtype_code(Vt), Vt.stride(0), B, Y.data_ptr(),
                      Y.stride(0), _lib.ptr(ws), wsb, s)
    if st == _lib.RSR_ERR_INVALID:
        # no batched kernel for this stream (u32 format, > 2187 pattern keys,
        # or a tile whose 4-vector shared-memory slab exceeds 227 KiB): the
        # single-vector kernel per column (arguments were validated above)
        for b in range(B):
            matvec_into(a, Vt[b], Y[b], view=view, stream=stream)
        return Y
    _lib.check(st, "rsr_matmul")
    return Y


def rsr_matvec_batched(a: RsrArtifact, V, counter: OpCounter | None = None,
                       method: str = "auto"):
    """Y = A . V for a batch of vectors V [B, n] (not in the reference, whose
    kernels.py:196 takes one vector; the oracle is rsr_matvec per row of V).

    int8 V -> int32 [B, m] (exact); real V -> float32 [B, m].  numpy in,
    numpy out; torch in, torch (device) out.
    """
    import torch
    host = not _is_torch(V)
    if host:
        Vn = np.asarray(V)
        if Vn.ndim != 2 or Vn.shape[1] != a.n:
            raise DimensionMismatch(f"batch of shape {Vn.shape} against {a.n} columns")
        if np.issubdtype(Vn.dtype, np.integer):
            if Vn.dtype != np.int8:
                raise DimensionMismatch("integer vectors must be int8")
            Vt = torch.from_numpy(np.ascontiguousarray(Vn)).to(a.device)
        else:
            Vt = torch.from_numpy(np.ascontiguousarray(Vn.astype(np.float32, copy=False))).to(a.device)
    else:
        Vt = V
        if Vt.dim() != 2 or Vt.shape[1] != a.n:
            raise DimensionMismatch(f"batch of shape {tuple(Vt.shape)} against {a.n} columns")
        if not Vt.is_floating_point() and Vt.dtype != torch.int8:
            raise DimensionMismatch("integer vectors must be int8")
        if Vt.is_floating_point() and Vt.dtype not in (torch.float32, torch.bfloat16,
                                                       torch.float16):
            Vt = Vt.to(torch.float32)
        Vt = Vt.to(a.device).contiguous()
    B = int(Vt.shape[0])
    for _ in range(B):
        _count(a, counter)
    ydt = torch.int32 if Vt.dtype == torch.int8 else torch.float32
    Y = torch.empty(B, a.m, dtype=ydt, device=a.device)
    if B:
        matmul_into(a, Vt, Y, method=method)
    return Y.cpu().numpy() if host else Y


def batched_preprocess(mats: list, k: int, tile_width: int | None = None):
    """Stack sibling matrices sharing an input (reference kernels.py:128-160).

    Returns (artifact, offsets); the stacked artifact's weight_scale is 1.0
    and callers apply per-matrix scales after splitting at ``offsets``.
    """
    if not mats:
        raise HeterogeneousSiblings("no matrices to batch")
    n = mats[0].cols
    bw = mats[0].bitwidth
    for mm in mats[1:]:
        if mm.cols != n or mm.bitwidth != bw:
            raise HeterogeneousSiblings(
                f"expected all {bw} matrices with {n} columns, got {mm.bitwidth} with {mm.cols}")
    if any(_is_torch(mm.data) for mm in mats):
        import torch
        data = torch.cat([mm.device_data() for mm in mats], 0)
    else:
        data = np.vstack([mm.host_data() for mm in mats])
    stacked = PackedMatrix(sum(mm.rows for mm in mats), n, bw, data)
    offsets = [0]
    for mm in mats:
        offsets.append(offsets[-1] + mm.rows)
    return preprocess(stacked, k, tile_width), offsets


class Multiplier:
    """One matrix bound to one multiplication strategy (reference kernels.py:163-217).

    RSR kinds hold a GPU artifact; naive kinds hold a dense device copy.
    For real input every kind computes weight_scale * (M @ v) (NaiveF32 in
    float64, the int8 kinds through activation quantization); int8 input
    gives the raw int32 product.
    """

    def __init__(self, kind: str, matrix: PackedMatrix, k: int = 4,
                 tile_width: int | None = None):
        if kind not in KINDS:
            raise ValueError(f"unknown multiplier kind {kind!r}")
        if kind == RSR_BINARY and matrix.bitwidth != BINARY:
            raise ValueError("RsrBinary needs a binary matrix")
        if kind == RSR_TERNARY and matrix.bitwidth != TERNARY:
            raise ValueError("RsrTernary needs a ternary matrix")
        import torch
        self.kind = kind
        self.matrix = matrix
        self.artifact = None
        self._dense = None
        if kind in (RSR_BINARY, RSR_TERNARY):
            self.artifact = preprocess(matrix, k, tile_width)
        else:
            self._dense = dense_device(matrix).to(torch.float64)

    def multiply(self, v, counter: OpCounter | None = None):
        import torch
        host = not _is_torch(v)
        shape = tuple(np.asarray(v).shape) if host else tuple(v.shape)
        if len(shape) != 1 or shape[0] != self.matrix.cols:
            raise DimensionMismatch(
                f"vector of length {int(np.prod(shape))} against {self.matrix.cols} columns")
        beta = self.matrix.weight_scale
        if host:
            vn = np.asarray(v)
            is_int = np.issubdtype(vn.dtype, np.integer)
        else:
            is_int = not (v.is_floating_point() or v.is_complex())
        if self.kind in (NAIVE_F32, NAIVE_I8):
            vt = torch.from_numpy(np.ascontiguousarray(v)).cuda() if host else v
            if is_int:
                y = (self._dense @ vt.to(torch.float64)).to(torch.int32)
            elif self.kind == NAIVE_F32:
                y = beta * (self._dense @ vt.to(torch.float64))
            else:
                q = quantize_activations(vt)
                yi = self._dense @ q.values.to(torch.float64)
                y = ((beta / q.scale) * yi).to(torch.float32)
            return y.cpu().numpy() if host else y
        if is_int:
            return rsr_matvec(self.artifact, v, counter)
        if self.kind == RSR_TERNARY:
            return rsr_matvec_fused(self.artifact, v, counter)
        y = rsr_matvec(self.artifact, v, counter)
        if beta == 1.0:
            return y
        if host:
            return (beta * y.astype(np.float64)).astype(np.float32)
        return (beta * y.to(torch.float64)).to(torch.float32)


def multiplier_multiply(mul: Multiplier, v, counter: OpCounter | None = None):
    """Function form of Multiplier.multiply (reference kernels.py:220-222)."""
    return mul.multiply(v, counter)


def naive_reference(matrix: PackedMatrix, v):
    return naive_matvec(matrix, v)
