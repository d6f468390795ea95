"""Two-binary-plane ternary multiply (north_star (3)).

A ternary matrix M is the difference of two binary planes, M = P - N with
P = [M == +1] and N = [M == -1].  Each plane can be preprocessed as a binary
RSR artifact (reference binary grouping, pkg/src/rsrmv/_native.py:25-88)
instead of grouping M natively by base-3 patterns (_native.py:91-161).  Here
the planes are split on the device (rsr_split_planes) and stacked into ONE
binary artifact of 2m rows, so a single launch of the multiply kernel
computes [P v; N v]; y = P v - N v is one subtraction.

This is the alternative the native base-3 path is measured against
(tools/p7_planes.py, profiles/r02_p7_planes.txt): with P(0) = 1/2 the planes
cost more artifact bytes than the native patterns at every k, and the native
path is kept as the product path.
"""

from __future__ import annotations

from . import _lib
from .errors import DimensionMismatch
from .matcore import BINARY, TERNARY, PackedMatrix
from .preproc import preprocess


class TwoPlane:
    """P/N planes of a ternary matrix as one stacked binary artifact."""

    def __init__(self, m: PackedMatrix, k: int, tile_width: int | None = None, device=None):
        import torch
        if m.bitwidth != TERNARY:
            raise ValueError("two-plane decomposition needs a ternary matrix")
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        data = m.device_data(dev)
        planes = torch.empty(2 * m.rows, (m.cols + 7) // 8, dtype=torch.uint8, device=dev)
        _lib.check(_lib.lib().rsr_split_planes(data.data_ptr(), m.rows, m.cols, m.row_bytes,
                                               planes.data_ptr(), _lib.current_stream_ptr(dev)),
                   "split_planes")
        self.m, self.n, self.k = m.rows, m.cols, k
        self.weight_scale = m.weight_scale
        self.planes = PackedMatrix(2 * m.rows, m.cols, BINARY, planes)
        self.artifact = preprocess(self.planes, k, tile_width, device=dev)

    def file_bytes(self) -> int:
        return self.artifact.file_bytes()

    def matvec_into(self, vt, y_stack, view=None, stream=None):
        """y_stack[:m] = P v, y_stack[m:] = N v (one kernel launch)."""
        from .kernels import matvec_into
        return matvec_into(self.artifact, vt, y_stack, view=view, stream=stream)

    def matvec(self, v):
        """y = M v = P v - N v (int8 v -> int32, real v -> float32)."""
        import torch
        if tuple(v.shape) != (self.n,):
            raise DimensionMismatch(f"vector of length {v.numel()} against {self.n} columns")
        ydt = torch.int32 if v.dtype == torch.int8 else torch.float32
        y = torch.empty(2 * self.m, dtype=ydt, device=v.device)
        self.matvec_into(v, y)
        return y[:self.m] - y[self.m:]
