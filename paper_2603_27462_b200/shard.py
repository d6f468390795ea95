"""Row-block sharding across GPUs; the output slices are all-gathered either
by the multiply itself over peer memory (gather="peer") or by NCCL.

SURVEY.md section 8e / row K10 (not in the reference, which is one CPU
process).  Row blocks own disjoint output rows (_native.py:
246-249), so each rank preprocesses and multiplies only its contiguous range
of row blocks -- every tile of those blocks, in ascending tile order, exactly
as a single GPU would -- and the full output is one all-gather of the padded
per-rank slices.  Results are bit-equal to the 1-GPU output (integer paths)
and to its float rounding (the per-row arithmetic does not depend on the
shard).

Each rank materializes only its own strip of the matrix (``strip_fn``), so a
131072^2 matrix never exists on one device when sharded.

Gather.  gather="nccl": local multiply into a padded slice, one
all_gather_into_tensor, an index_select back to row order.  gather="peer":
the full output lives in symmetric memory (torch.distributed.
_symmetric_memory: every rank's buffer mapped into every device's address
space), and the multiply's epilogue stores each row straight into all ranks'
buffers at its global row (rsr_matvec_peers) -- the all-gather rides on the
multiply's own stores over NVLink, no separate collective and no reassembly
-- followed by one symmetric-memory barrier.  Two buffers alternate, so a
result stays valid until the call after next.

Balance.  By default the ranks get equal numbers of row blocks, which for
matrices with uniform density (the synthetic C5 matrix) is also an equal
share of artifact bytes.  Callers that know the per-block bytes -- e.g. the
``block_bytes()`` of an earlier artifact of the same matrix -- pass them as
``weights`` and the contiguous ranges are cut at equal byte shares instead.
"""

from __future__ import annotations

import numpy as np

from .preproc import make_plan, preprocess


def block_ranges(block_count: int, world: int, weights=None) -> list[tuple[int, int]]:
    """Contiguous [b0, b1) block ranges per rank, balanced by per-block
    `weights` (e.g. stream bytes) or, if None, by block count."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if weights is None:
        bounds = [block_count * r // world for r in range(world + 1)]
    else:
        w = np.asarray(weights, dtype=np.float64)
        if w.shape != (block_count,):
            raise ValueError("one weight per block expected")
        cum = np.concatenate([[0.0], np.cumsum(w)])
        bounds = [0] + [int(np.searchsorted(cum, cum[-1] * r / world, side="left"))
                        for r in range(1, world)] + [block_count]
        for i in range(1, len(bounds)):
            bounds[i] = max(bounds[i], bounds[i - 1])
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def row_ranges(m: int, k: int, world: int, weights=None) -> list[tuple[int, int]]:
    """Row ranges [r0, r1) per rank (block ranges scaled by k, clipped to m)."""
    bc = -(-m // k)
    return [(b0 * k, min(b1 * k, m)) for b0, b1 in block_ranges(bc, world, weights)]


def peer_row_addresses(base_ptrs, r0: int, elem_size: int) -> list[int]:
    """Address of global row r0 inside each rank's full output buffer."""
    return [int(b) + int(r0) * int(elem_size) for b in base_ptrs]


def gather_index(ranges: list[tuple[int, int]], pad: int):
    """Index of the full output's rows inside the flattened [world, pad]
    all-gather buffer."""
    return np.concatenate([np.arange(r0, r1) - r0 + i * pad
                           for i, (r0, r1) in enumerate(ranges)]).astype(np.int64)


class ShardedMatrix:
    """One rank's share of a row-block-sharded RSR matrix.

    strip_fn(r0, r1) -> PackedMatrix of rows [r0, r1) (on this rank's device
    or host).  `group` is a torch.distributed process group (default world).
    """

    def __init__(self, m: int, n: int, bitwidth: str, k: int, strip_fn, rank: int, world: int,
                 device=None, group=None, weight_scale: float = 1.0, weights=None,
                 tile_width: int | None = None, gather: str = "nccl"):
        import torch
        if gather not in ("nccl", "peer"):
            raise ValueError("gather must be 'nccl' or 'peer'")
        self.gather = gather
        self._peer: dict = {}
        self.m, self.n, self.k, self.bitwidth = m, n, k, bitwidth
        self.rank, self.world, self.group = rank, world, group
        self.plan = make_plan(m, n, k, bitwidth, tile_width)
        self.ranges = row_ranges(m, k, world, weights)
        self.r0, self.r1 = self.ranges[rank]
        self.pad = max(r1 - r0 for r0, r1 in self.ranges)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        self.local = None
        if self.r1 > self.r0:
            strip = strip_fn(self.r0, self.r1)
            self.local = preprocess(strip, k, self.plan.tile_width, device=self.device)
            self.local.weight_scale = weight_scale
        self.index = torch.from_numpy(gather_index(self.ranges, self.pad)).to(self.device)

    def buffers(self, dtype):
        import torch
        y_local = torch.zeros(self.pad, dtype=dtype, device=self.device)
        y_all = torch.zeros(self.pad * self.world, dtype=dtype, device=self.device)
        return y_local, y_all

    def local_matvec(self, v, y_local, fused: bool = False):
        """This rank's rows into y_local[:rows] (no communication)."""
        from .kernels import fused_into, matvec_into
        if self.local is None:
            return y_local
        rows = self.r1 - self.r0
        if fused:
            fused_into(self.local, v, y_local[:rows])
        else:
            matvec_into(self.local, v, y_local[:rows])
        return y_local

    def _peer_state(self, dtype):
        """Symmetric-memory output buffers for `dtype` (collective on first
        use: every rank must make the same calls in the same order)."""
        st = self._peer.get(dtype)
        if st is None:
            import torch
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm
            group = self.group if self.group is not None else dist.group.WORLD
            esz = torch.empty((), dtype=dtype).element_size()
            bufs = []
            for _ in range(2):
                y = symm.empty(self.m, dtype=dtype, device=self.device)
                h = symm.rendezvous(y, group)
                rows = torch.tensor(peer_row_addresses(h.buffer_ptrs, self.r0, esz),
                                    dtype=torch.int64, device=self.device)
                bufs.append((y, h, rows))
            st = self._peer[dtype] = {"bufs": bufs, "i": 0}
        return st

    def matvec(self, v, fused: bool = False, buffers=None):
        """Full y on every rank: local multiply + all-gather (peer stores in
        the multiply, or NCCL).  With gather="peer" the result is one of two
        alternating symmetric-memory buffers: valid until the call after
        next (clone it to keep it longer)."""
        import torch
        import torch.distributed as dist
        odt = torch.int32 if (v.dtype == torch.int8 and not fused) else torch.float32
        if self.gather == "peer" and not fused:
            from .kernels import matvec_peers_into
            st = self._peer_state(odt)
            y, h, rows = st["bufs"][st["i"]]
            st["i"] ^= 1
            if self.local is not None:
                matvec_peers_into(self.local, v, rows, self.world)
            h.barrier(channel=0)
            return y
        y_local, y_all = buffers if buffers is not None else self.buffers(odt)
        self.local_matvec(v, y_local, fused)
        if self.world > 1:
            dist.all_gather_into_tensor(y_all, y_local, group=self.group)
        else:
            y_all.copy_(y_local)
        return y_all.index_select(0, self.index)
