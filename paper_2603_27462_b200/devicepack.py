"""Device-side ternarization + packing of weights already on the GPU.

``ternarize_pack_device(w)`` is ``matcore.ternarize_weights`` for a CUDA
tensor (reference matcore.py:151-173): one reduction for beta = mean|w| in
float64 and one elementwise pass that writes the 2-bit packed codes, both in
csrc/rsr_pack.cu.  The packed matrix stays on the device, ready for
``preprocess``.
"""

from __future__ import annotations

from . import _lib
from .errors import DimensionMismatch, NonFinite
from .matcore import TERNARY, PackedMatrix, _dtype_code


def random_ternary_device(rows: int, cols: int, seed: int, density: float = 0.5, row0: int = 0,
                          device=None) -> PackedMatrix:
    """Rows [row0, row0+rows) of the counter-based synthetic ternary matrix,
    generated and packed on the device (C5-scale inputs; see
    rsr_random_ternary in include/rsr_b200.h)."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
        else torch.device(device)
    packed = torch.empty(rows, (cols + 3) // 4, dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib().rsr_random_ternary(row0, rows, cols, seed, density, packed.data_ptr(),
                                             _lib.current_stream_ptr(dev)), "random_ternary")
    return PackedMatrix(rows, cols, TERNARY, packed)


def ternarize_pack_device(w, check_finite: bool = True) -> PackedMatrix:
    import torch
    if w.dim() != 2:
        raise DimensionMismatch("ternarize_weights expects a 2-D matrix")
    if not w.is_cuda:
        raise ValueError("ternarize_pack_device needs a CUDA tensor")
    if w.dtype not in (torch.float32, torch.bfloat16, torch.float16):
        w = w.to(torch.float32)
    w = w.contiguous()
    if check_finite and not bool(torch.isfinite(w).all()):
        r, c = (int(x) for x in torch.nonzero(~torch.isfinite(w))[0])
        raise NonFinite(f"non-finite weight at ({r}, {c})", row=r, col=c)
    rows, cols = w.shape
    packed = torch.empty(rows, (cols + 3) // 4, dtype=torch.uint8, device=w.device)
    beta = torch.empty(1, dtype=torch.float64, device=w.device)
    L = _lib.lib()
    wsb = int(L.rsr_ternarize_workspace_bytes())
    ws = torch.empty(wsb, dtype=torch.uint8, device=w.device)
    _lib.check(L.rsr_ternarize_pack(w.data_ptr(), _dtype_code(w), rows, cols, packed.data_ptr(),
                                    beta.data_ptr(), ws.data_ptr(), wsb,
                                    _lib.current_stream_ptr(w.device)), "ternarize_pack")
    return PackedMatrix(rows, cols, TERNARY, packed, weight_scale=float(beta.item()))
