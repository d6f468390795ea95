"""ctypes binding of librsr_b200.so (the C ABI declared in include/rsr_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2603_27462_b200/csrc``).  There is no fallback: if the
library is missing, or no CUDA device is present when a kernel is called,
the call raises.  Status codes are mapped onto the reference package's
exception kinds (reference pkg/src/rsrmv/errors.py:23-74).
"""

from __future__ import annotations

import ctypes
import os

from .errors import CorruptArtifact, DimensionMismatch, KTooLarge, RsrError, TileTooWide

_HERE = os.path.dirname(os.path.abspath(__file__))
# RSR_B200_LIB selects another build of the same library (tools/ experiments
# use the knob-enabled librsr_b200_exp.so); the default is the in-tree build.
LIB_PATH = os.environ.get("RSR_B200_LIB") or os.path.join(_HERE, "librsr_b200.so")

RSR_OK = 0
RSR_ERR_TILE_TOO_WIDE = 1
RSR_ERR_K_TOO_LARGE = 2
RSR_ERR_INVALID = 3
RSR_ERR_DIMENSION = 4
RSR_ERR_CUDA = 5
RSR_ERR_WORKSPACE = 6

RSR_BINARY = 0
RSR_TERNARY = 1

RSR_F32, RSR_BF16, RSR_F16, RSR_I8, RSR_I32, RSR_F64 = 0, 1, 2, 3, 4, 5

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
SZ = ctypes.c_size_t
F64 = ctypes.c_double


class StreamView(ctypes.Structure):
    """Mirror of rsr_stream_view (include/rsr_b200.h)."""
    _fields_ = [
        ("m", I64), ("n", I64),
        ("k", I32), ("bitwidth", I32),
        ("tile_width", I64), ("block_count", I64), ("tile_count", I64),
        ("format", I32), ("chunk", I32),
        ("entries", P), ("e_off", P),
        ("row_begin_block", I64), ("n_blocks", I64),
        ("col0_key", P),
        ("device", I32),
    ]


# (name, restype, argtypes) of every exported symbol; tests check the .so
# exports exactly these and that include/rsr_b200.h declares them.
SIGNATURES = {
    "rsr_version": (ctypes.c_char_p, []),
    "rsr_last_cuda_error": (ctypes.c_char_p, []),
    "rsr_device_sm_count": (ctypes.c_int, [ctypes.c_int]),
    "rsr_group_workspace_bytes": (SZ, [I64, I64, I32, I32, I64]),
    "rsr_group_count": (I32, [P, I64, I64, I64, I32, I32, I64, P, P, P, P, P, SZ, P]),
    "rsr_group_fill": (I32, [P, I64, I64, I64, I32, I32, I64, P, P, P, P, P, SZ, P]),
    "rsr_stream_format": (I32, [I32, I32, I64]),
    "rsr_stream_count": (I32, [P, P, P, P, I64, I64, I32, I32, P, P, P]),
    "rsr_stream_build": (I32, [P, P, P, P, I64, I64, I64, I64, I32, I32, I32, P, P, P, P, P]),
    "rsr_matvec_workspace_bytes": (SZ, [ctypes.POINTER(StreamView)]),
    "rsr_matvec": (I32, [ctypes.POINTER(StreamView), P, I32, P, I32, P, SZ, P]),
    "rsr_matvec_peers": (I32, [ctypes.POINTER(StreamView), P, I32, P, I32, P, SZ, P]),
    "rsr_matvec_host": (I32, [ctypes.POINTER(StreamView), P, I32, P, P, P, P, SZ, P]),
    "rsr_fused_matvec_host": (I32, [ctypes.POINTER(StreamView), P, I32, F64, P, P, P, P, SZ, P]),
    "rsr_fused_matvec": (I32, [ctypes.POINTER(StreamView), P, I32, F64, P, P, I32, P, P, SZ, P]),
    "rsr_matmul_workspace_bytes": (SZ, [ctypes.POINTER(StreamView), I32]),
    "rsr_matmul": (I32, [ctypes.POINTER(StreamView), P, I32, I64, I32, P, I64, P, SZ, P]),
    "rsr_keymat_bytes": (SZ, [I64, I64, I32, I32]),
    "rsr_keymat_build": (I32, [P, P, P, P, I64, I64, I64, I64, I32, I32, P, P]),
    "rsr_matmul_tc_workspace_bytes": (SZ, [I64, I64, I32, I64, I64, I32]),
    "rsr_matmul_tc": (I32, [P, I64, I64, I32, I32, I64, I64, P, I32, I64, I32, P, I64, P, SZ, P]),
    "rsr_keymat_build_i8": (I32, [P, P, P, P, I64, I64, I64, I64, I32, I32, P, P]),
    "rsr_keymat_build_wide": (I32, [P, P, P, P, I64, I64, I64, I64, I32, I32, P, P]),
    "rsr_matmul_tc_wide": (I32, [P, I64, I64, I32, I32, I64, I64, P, I32, I64, I32, P, I64, P, SZ,
                                 P]),
    "rsr_matmul_tc_i8": (I32, [P, I64, I64, I32, I32, I64, I64, P, I64, I32, P, I64, P, SZ, P]),
    "rsr_matmul_tc_i8_dequant": (I32, [P, I64, I64, I32, I32, I64, I64, P, I64, I32, P, P, F64,
                                       P, I32, I64, P, SZ, P]),
    "rsr_ternarize_workspace_bytes": (SZ, []),
    "rsr_ternarize_pack": (I32, [P, I32, I64, I64, P, P, P, SZ, P]),
    "rsr_random_ternary": (I32, [I64, I64, I64, ctypes.c_uint64, F64, P, P]),
    "rsr_split_planes": (I32, [P, I64, I64, I64, P, P]),
    "rsr_rmsnorm_rows": (I32, [P, P, I64, I64, ctypes.c_float, P, P]),
    "rsr_audit": (I32, [P, P, P, P, I64, I64, I32, I32, I64, I64, I64, P, P]),
    "rsr_absmax_quantize_rows": (I32, [P, I32, I64, I64, I64, P, ctypes.c_float, P, I64, P, P]),
    "rsr_fused_matvec_norm": (I32, [ctypes.POINTER(StreamView), P, I32, P, ctypes.c_float, F64, P,
                                    P, I32, P, SZ, P]),
    "rsr_dequant_rows": (I32, [P, I64, I64, I64, P, P, F64, P, I32, I64, P]),
    "rsr_reconstruct_bytes": (SZ, [I64, I64, I32]),
    "rsr_reconstruct": (I32, [P, P, P, P, I64, I64, I32, I32, I64, I64, I64, P, P]),
    "rsr_debug_set_probe": (None, [P]),
    "rsr_count_ops": (I32, [P, I64, P, P]),
    "rsr_absmax_quantize": (I32, [P, I32, I64, P, P, P]),
}

_lib = None


def lib():
    """Load librsr_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int, what: str = "") -> None:
    """Raise the reference exception kind for a non-zero rsr_status."""
    if status == RSR_OK:
        return
    if status == RSR_ERR_TILE_TOO_WIDE:
        raise TileTooWide(
            f"{what}: a group of identical columns exceeds 65535 entries; "
            "use a tile_width of 32768 or less")
    if status == RSR_ERR_K_TOO_LARGE:
        raise KTooLarge(-1, "binary")
    if status == RSR_ERR_DIMENSION:
        raise DimensionMismatch(what)
    if status == RSR_ERR_CUDA:
        err = lib().rsr_last_cuda_error().decode()
        raise RuntimeError(f"{what}: CUDA error: {err}")
    if status == RSR_ERR_WORKSPACE:
        raise RuntimeError(f"{what}: workspace too small")
    if status == RSR_ERR_INVALID:
        raise CorruptArtifact(f"{what}: invalid argument or reserved ternary code 11")
    raise RsrError(f"{what}: rsr status {status}")


def current_stream_ptr(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())
