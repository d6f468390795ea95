"""Offline preprocessing on the GPU (operator API of reference preproc.py).

``preprocess(m, k, tile_width=None) -> RsrArtifact`` keeps the reference
signature, plans, caps and errors (pkg/src/rsrmv/preproc.py:26-114,
:239-289) and produces the SAME flat arrays -- ``words`` u64, ``perm`` u16
(tile-local column ids), ``group_offsets`` / ``perm_offsets`` int64 and
``sort_steps`` -- byte for byte, but computes them with the sm_100a grouping
kernels (csrc/rsr_preprocess.cu).  The artifact lives on the device; the
reference attribute names return host numpy copies on first access so code
written against the reference (validate_artifact, reconstruct, .rsra I/O)
works unchanged.

On top of the reference arrays every artifact carries the device-only chunk
stream the multiply kernels read (block-major cells of 32-byte chunks of
column / pattern-key entries, every chunk led by a key); see DESIGN.md.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import CorruptArtifact, DimensionMismatch, KTooLarge, TileTooWide
from .matcore import BINARY, TERNARY, PackedMatrix, _is_torch, encode

MAX_TILE_WIDTH = 65536          # reference preproc.py:26
DEFAULT_WIDE_TILE = 32768       # reference preproc.py:27
K_CAP = {BINARY: 16, TERNARY: 10}   # reference preproc.py:28


def pack_group(perm_start: int, perm_len: int, pos_mask: int, neg_mask: int) -> int:
    """Pack one group record: bits [0,16) perm_start, [16,32) perm_len,
    [32,48) pos_mask, [48,64) neg_mask (reference preproc.py:31-41)."""
    for name, val in (("perm_start", perm_start), ("perm_len", perm_len),
                      ("pos_mask", pos_mask), ("neg_mask", neg_mask)):
        if not 0 <= val <= 0xFFFF:
            raise ValueError(f"{name}={val} does not fit u16")
    return perm_start | (perm_len << 16) | (pos_mask << 32) | (neg_mask << 48)


def unpack_group(word: int) -> tuple[int, int, int, int]:
    """Inverse of pack_group (reference preproc.py:44-48)."""
    word = int(word)
    return (word & 0xFFFF, (word >> 16) & 0xFFFF, (word >> 32) & 0xFFFF, (word >> 48) & 0xFFFF)


@dataclass(frozen=True)
class GroupRecord:
    perm_start: int
    perm_len: int
    pos_mask: int
    neg_mask: int


@dataclass(frozen=True)
class BlockMeta:
    perm: np.ndarray
    groups: tuple


@dataclass
class StepCounter:
    steps: int = 0


@dataclass(frozen=True)
class BlockPlan:
    """Block/tile layout of one matrix (reference preproc.py:80-94)."""
    k: int
    block_count: int
    last_block_height: int
    tile_width: int
    tile_count: int

    def __post_init__(self):
        if not 1 <= self.k <= 16:
            raise ValueError(f"k={self.k} outside [1, 16]")
        if not 1 <= self.tile_width <= MAX_TILE_WIDTH:
            raise TileTooWide(f"tile_width={self.tile_width}", n_tile=self.tile_width)
        if not 1 <= self.last_block_height <= self.k:
            raise ValueError("last block height inconsistent with k")


def make_plan(m_rows: int, n_cols: int, k: int, bitwidth: str,
              tile_width: int | None = None) -> BlockPlan:
    """Validate caps and lay out blocks/tiles (reference preproc.py:97-114)."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    if k > K_CAP[bitwidth]:
        raise KTooLarge(k, bitwidth)
    if tile_width is None:
        tile_width = n_cols if n_cols <= MAX_TILE_WIDTH else DEFAULT_WIDE_TILE
    if not 1 <= tile_width <= MAX_TILE_WIDTH:
        raise TileTooWide(f"tile_width={tile_width} outside [1, {MAX_TILE_WIDTH}]",
                          n_tile=tile_width)
    bc = -(-m_rows // k)
    tc = -(-n_cols // tile_width)
    return BlockPlan(k, bc, m_rows - k * (bc - 1), tile_width, tc)


def _u64_host(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def _u16_host(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16)


class RsrArtifact:
    """Preprocessed matrix: reference flat arrays + device stream layout.

    Device tensors: ``words_d`` (int64 storage of u64 words), ``perm_d``
    (int16 storage of u16), ``go_d``/``po_d`` (int64, cells+1), and the
    chunk stream ``entries_d``/``e_off_d`` the multiply reads.  The
    reference attribute names (``words``, ``perm``, ``group_offsets``,
    ``perm_offsets``, ``sort_steps``) are host numpy views fetched lazily.
    Cells are tile-major exactly as in the reference (cell = t*bc + b).
    """

    def __init__(self, m, n, k, bitwidth, weight_scale, plan, words_d, perm_d, go_d, po_d,
                 steps_d=None, n_words=None, n_perm=None, build_stream=True):
        self.m = m
        self.n = n
        self.k = k
        self.bitwidth = bitwidth
        self.weight_scale = weight_scale
        self.plan = plan
        self.words_d = words_d
        self.perm_d = perm_d
        self.go_d = go_d
        self.po_d = po_d
        self.steps_d = steps_d
        self.n_words = int(words_d.numel()) if n_words is None else n_words
        self.n_perm = int(perm_d.numel()) if n_perm is None else n_perm
        self.device = go_d.device
        self._host = {}
        if build_stream:
            self._build_stream()

    # ---- reference attribute surface (host numpy, lazily copied) ----------
    def _h(self, key, fn):
        if key not in self._host:
            self._host[key] = fn()
        return self._host[key]

    @property
    def words(self) -> np.ndarray:
        return self._h("words", lambda: _u64_host(self.words_d))

    @property
    def perm(self) -> np.ndarray:
        return self._h("perm", lambda: _u16_host(self.perm_d))

    @property
    def group_offsets(self) -> np.ndarray:
        return self._h("go", lambda: self.go_d.cpu().numpy())

    @property
    def perm_offsets(self) -> np.ndarray:
        return self._h("po", lambda: self.po_d.cpu().numpy())

    @property
    def sort_steps(self):
        if self.steps_d is None:
            return None
        return self._h("steps", lambda: self.steps_d.cpu().numpy())

    @property
    def cells(self) -> int:
        return self.plan.tile_count * self.plan.block_count

    def cell_index(self, tile: int, block: int) -> int:
        return tile * self.plan.block_count + block

    def block_meta(self, tile: int, block: int) -> BlockMeta:
        c = self.cell_index(tile, block)
        go, po = self.group_offsets, self.perm_offsets
        groups = tuple(GroupRecord(*unpack_group(w)) for w in self.words[go[c]:go[c + 1]])
        return BlockMeta(self.perm[po[c]:po[c + 1]].copy(), groups)

    def op_totals(self) -> tuple[int, int, int]:
        """(gather adds, scatter adds, groups) of one multiply, counted on the
        GPU (reference _native.count_ops, _native.py:288-307)."""
        if "ops" not in self._host:
            import torch
            out = torch.zeros(3, dtype=torch.int64, device=self.device)
            _lib.check(_lib.lib().rsr_count_ops(
                _lib.ptr(self.words_d), self.n_words, _lib.ptr(out),
                _lib.current_stream_ptr(self.device)), "count_ops")
            self._host["ops"] = tuple(int(x) for x in out.cpu().tolist())
        return self._host["ops"]

    def file_bytes(self) -> int:
        """Serialized .rsra size (reference preproc.py:161-169)."""
        gc = np.diff(self.group_offsets)
        pl = np.diff(self.perm_offsets)
        return int(24 + np.sum(8 + 8 * gc + 2 * pl + (-(2 * pl)) % 4))

    # ---- device chunk stream ---------------------------------------------
    def _build_stream(self):
        import torch
        p = self.plan
        dev = self.device
        s = _lib.current_stream_ptr(dev)
        cells = self.cells
        L = _lib.lib()
        bw = _lib.RSR_BINARY if self.bitwidth == BINARY else _lib.RSR_TERNARY
        self.format = int(L.rsr_stream_format(bw, self.k, p.tile_width))
        self.entry_bytes = 4 if self.format == 2 else 2
        self.chunk = 32 // self.entry_bytes
        e_off = torch.zeros(cells + 1, dtype=torch.int64, device=dev)
        gslot = torch.empty(max(self.n_words, 1), dtype=torch.int32, device=dev)
        _lib.check(L.rsr_stream_count(_lib.ptr(self.words_d), _lib.ptr(self.go_d),
                                      _lib.ptr(self.perm_d), _lib.ptr(self.po_d), p.block_count,
                                      p.tile_count, self.format, self.chunk, _lib.ptr(e_off),
                                      _lib.ptr(gslot), s), "stream_count")
        ne = int(e_off[-1].item())
        edt = torch.int16 if self.entry_bytes == 2 else torch.int32
        entries = torch.empty(max(ne, self.chunk), dtype=edt, device=dev)
        # u16 formats: pattern key of each cell's column 0 (quad layout)
        col0 = torch.zeros(cells if self.format != 2 else 1, dtype=torch.int32, device=dev)
        _lib.check(L.rsr_stream_build(_lib.ptr(self.words_d), _lib.ptr(self.go_d),
                                      _lib.ptr(self.perm_d), _lib.ptr(self.po_d), p.block_count,
                                      p.tile_count, p.tile_width, self.n, bw, self.format,
                                      self.chunk,
                                      _lib.ptr(e_off), _lib.ptr(gslot), _lib.ptr(entries),
                                      _lib.ptr(col0) if self.format != 2 else None, s),
                   "stream_build")
        del gslot
        self.entries_d, self.e_off_d = entries, e_off
        self.col0_d = col0 if self.format != 2 else None
        self._view = self.view()

    def keymat(self, kind: str = "bf16"):
        """Every column's pattern key as 2-bit row codes, one row at a time
        (device u32 [ceil(n/128)][round8(bc*k)][8], 128 columns per row and
        step, in the permuted order of csrc/rsr_tc.cu for the bf16 ("bf16")
        or the int8 ("i8") tensor-core multiply: a tile's step is one
        contiguous run of rows; "wide": the bf16 order in the int8 path's
        256-column steps, for bf16 batches of at most 32 vectors), built on
        first use; None when k > 16."""
        if kind not in ("bf16", "i8", "wide"):
            raise ValueError(f"unknown code-matrix kind {kind!r}")
        attr = {"bf16": "_keymat", "i8": "_keymat_i8", "wide": "_keymat_wide"}[kind]
        if attr not in self.__dict__:
            import torch
            L = _lib.lib()
            bw = _lib.RSR_BINARY if self.bitwidth == BINARY else _lib.RSR_TERNARY
            p = self.plan
            nb = int(L.rsr_keymat_bytes(p.block_count, self.n, bw, self.k))
            km = None
            if nb:
                km = torch.empty(nb, dtype=torch.uint8, device=self.device)
                build = {"bf16": L.rsr_keymat_build, "i8": L.rsr_keymat_build_i8,
                         "wide": L.rsr_keymat_build_wide}[kind]
                _lib.check(build(
                    _lib.ptr(self.words_d), _lib.ptr(self.go_d), _lib.ptr(self.perm_d),
                    _lib.ptr(self.po_d), p.block_count, p.tile_count, p.tile_width, self.n,
                    bw, self.k, _lib.ptr(km), _lib.current_stream_ptr(self.device)),
                    "keymat_build")
            self.__dict__[attr] = km
        return self.__dict__[attr]

    def block_bytes(self) -> np.ndarray:
        """Reference-format artifact bytes of each row block (all its tiles):
        8 per cell + 8 per group + 2 per perm entry (+ padding), the weights
        for byte-balanced row-block sharding (shard.block_ranges)."""
        p = self.plan
        gc = np.diff(self.group_offsets).reshape(p.tile_count, p.block_count)
        pl = np.diff(self.perm_offsets).reshape(p.tile_count, p.block_count)
        return (8 + 8 * gc + 2 * pl + (-(2 * pl)) % 4).sum(axis=0)

    def stream_bytes(self) -> int:
        """Bytes of the device chunk stream one multiply reads."""
        return int(self.entries_d.numel() * self.entries_d.element_size()
                   + self.e_off_d.numel() * 8
                   + (0 if self.col0_d is None else self.col0_d.numel() * 4))

    def view(self, block_begin: int = 0, n_blocks: int | None = None,
             entries=None, e_off=None) -> _lib.StreamView:
        """C-ABI view over row blocks [block_begin, block_begin + n_blocks)."""
        p = self.plan
        if n_blocks is None:
            n_blocks = p.block_count - block_begin
        if block_begin < 0 or n_blocks < 0 or block_begin + n_blocks > p.block_count:
            raise ValueError(f"block range [{block_begin}, {block_begin + n_blocks}) outside "
                             f"[0, {p.block_count})")
        v = _lib.StreamView()
        v.m, v.n, v.k = self.m, self.n, self.k
        v.bitwidth = _lib.RSR_BINARY if self.bitwidth == BINARY else _lib.RSR_TERNARY
        v.tile_width, v.block_count, v.tile_count = p.tile_width, p.block_count, p.tile_count
        v.format = self.format
        v.chunk = self.chunk
        v.entries = _lib.ptr(self.entries_d if entries is None else entries)
        # a block range starts at cell block_begin*tc of the block-major order
        v.e_off = _lib.ptr(self.e_off_d if e_off is None else e_off) + 8 * block_begin * p.tile_count
        v.col0_key = (None if self.col0_d is None
                      else _lib.ptr(self.col0_d) + 4 * block_begin * p.tile_count)
        v.row_begin_block = block_begin
        v.n_blocks = n_blocks
        idx = getattr(self.device, "index", None)
        v.device = -1 if idx is None else int(idx)
        return v

    # ---- constructors ----------------------------------------------------
    @classmethod
    def from_host(cls, m, n, k, bitwidth, weight_scale, plan, words, perm, group_offsets,
                  perm_offsets, sort_steps=None, device=None, audit=False) -> "RsrArtifact":
        """Upload reference-format host arrays (e.g. a loaded .rsra file).
        audit=True runs validate_artifact on the uploaded arrays before the
        chunk stream is derived from them (CorruptArtifact otherwise)."""
        import torch
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)

        def up(a, dt, view_dt):
            a = np.ascontiguousarray(a)
            if a.size == 0:
                return torch.zeros(1, dtype=view_dt, device=dev)[:0]
            return torch.from_numpy(a.view(dt)).to(dev)

        a = cls(m, n, k, bitwidth, weight_scale, plan,
                up(np.asarray(words, np.uint64), np.int64, torch.int64),
                up(np.asarray(perm, np.uint16), np.int16, torch.int16),
                up(np.asarray(group_offsets, np.int64), np.int64, torch.int64),
                up(np.asarray(perm_offsets, np.int64), np.int64, torch.int64),
                None if sort_steps is None else
                up(np.asarray(sort_steps, np.int64), np.int64, torch.int64),
                build_stream=False)
        # reference-format host data (e.g. a file) is audited before anything
        # is derived from it; a host copy of what was uploaded is kept
        a._host.update(words=np.asarray(words, np.uint64), perm=np.asarray(perm, np.uint16))
        if audit:
            validate_artifact(a)
        a._build_stream()
        return a


def _grouping(data_d, rows, cols, row_bytes, bitwidth, k, tw, dev):
    """Run the two-phase GPU grouping; returns device arrays."""
    import torch
    bw = _lib.RSR_BINARY if bitwidth == BINARY else _lib.RSR_TERNARY
    bc = -(-rows // k)
    tc = -(-cols // tw)
    cells = bc * tc
    s = _lib.current_stream_ptr(dev)
    L = _lib.lib()
    go = torch.empty(cells + 1, dtype=torch.int64, device=dev)
    po = torch.empty(cells + 1, dtype=torch.int64, device=dev)
    steps = torch.empty(cells, dtype=torch.int64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    wsb = int(L.rsr_group_workspace_bytes(rows, cols, bw, k, tw))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    _lib.check(L.rsr_group_count(_lib.ptr(data_d), rows, cols, row_bytes, bw, k, tw,
                                 _lib.ptr(go), _lib.ptr(po), _lib.ptr(steps), _lib.ptr(status),
                                 _lib.ptr(ws), wsb, s), "preprocess")
    st, nw, npm = (int(x) for x in torch.stack(
        [status[0].to(torch.int64), go[-1], po[-1]]).cpu().tolist())
    if st == _lib.RSR_ERR_TILE_TOO_WIDE:
        raise TileTooWide(
            f"a group of identical columns exceeds {0xFFFF} entries; "
            f"use a tile_width of {DEFAULT_WIDE_TILE} or less", n_tile=min(tw, cols))
    if st != 0:
        _lib.check(st, "preprocess")
    words = torch.empty(nw, dtype=torch.int64, device=dev)
    perm = torch.empty(npm, dtype=torch.int16, device=dev)
    _lib.check(L.rsr_group_fill(_lib.ptr(data_d), rows, cols, row_bytes, bw, k, tw,
                                _lib.ptr(go), _lib.ptr(po), _lib.ptr(words), _lib.ptr(perm),
                                _lib.ptr(ws), wsb, s), "preprocess")
    return words, perm, go, po, steps


def preprocess(m: PackedMatrix, k: int, tile_width: int | None = None,
               device=None) -> RsrArtifact:
    """Preprocess a packed matrix into an RsrArtifact on the GPU.

    Deterministic and byte-identical to the reference artifact
    (preproc.py:239-289).  Raises KTooLarge / TileTooWide as the reference.
    """
    import torch
    plan = make_plan(m.rows, m.cols, k, m.bitwidth, tile_width)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
        else torch.device(device)
    data_d = m.device_data(dev)
    words, perm, go, po, steps = _grouping(data_d, m.rows, m.cols, m.row_bytes, m.bitwidth, k,
                                           plan.tile_width, dev)
    return RsrArtifact(m.rows, m.cols, k, m.bitwidth, m.weight_scale, plan, words, perm, go,
                       po, steps)


def pattern_key(m: PackedMatrix, block_rows: range, col: int) -> int:
    """The reference's pattern key of column `col` over `block_rows`
    (preproc.py:183-197): row i of the block contributes its packed code
    (binary bit / ternary 2-bit code) at bit position i (binary) or 2i
    (ternary) -- host helper, used by tests and tools."""
    if not 0 <= col < m.cols:
        raise DimensionMismatch(f"column {col} outside 0..{m.cols - 1}")
    rows = np.asarray(list(block_rows), dtype=np.int64)
    data = m.host_data()
    per_byte, width = (8, 1) if m.bitwidth == BINARY else (4, 2)
    codes = (data[rows, col // per_byte].astype(np.int64) >> (width * (col % per_byte))) \
        & ((1 << width) - 1)
    return int(np.sum(codes << (width * np.arange(rows.size, dtype=np.int64))))


def preprocess_block(m: PackedMatrix, block_rows: range, tile_cols: range,
                     counter: StepCounter | None = None) -> BlockMeta:
    """Group one (block, tile) cell on the GPU (reference preproc.py:200-236)."""
    from .matcore import decode
    h = len(block_rows)
    if h < 1:
        raise ValueError("empty block")
    if h > K_CAP[m.bitwidth]:
        raise KTooLarge(h, m.bitwidth)
    tn = len(tile_cols)
    if not 1 <= tn <= MAX_TILE_WIDTH:
        raise TileTooWide(f"tile of {tn} columns", n_tile=tn)
    dense = decode(m)[block_rows.start:block_rows.stop, tile_cols.start:tile_cols.stop]
    sub = encode(dense, h, tn, m.bitwidth)
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    words, perm, go, po, steps = _grouping(sub.device_data(dev), h, tn, sub.row_bytes,
                                           m.bitwidth, h, tn, dev)
    if counter is not None:
        counter.steps += int(steps[0].item())
    groups = tuple(GroupRecord(*unpack_group(w)) for w in _u64_host(words))
    return BlockMeta(_u16_host(perm).copy(), groups)


# messages of the device audit's per-cell checks (csrc/rsr_audit.cu AuditCheck)
_AUDIT_MESSAGES = {
    1: "a group with no columns",
    2: "group perm ranges are not back to back from 0",
    3: "group perm ranges do not end at the cell's perm length",
    4: "pos and neg masks share a row",
    5: "a group with the all-zero pattern",
    6: "mask bits at or above the block height",
    7: "a neg mask in a binary artifact",
    8: "group keys not strictly ascending",
    9: "a column id at or beyond the tile width",
    10: "a column listed twice",
    11: "columns not ascending inside a group",
    12: "perm entries but no groups",
}


def _offsets_host(x) -> np.ndarray:
    return x.cpu().numpy() if _is_torch(x) else np.asarray(x, dtype=np.int64)


def validate_artifact(a: RsrArtifact) -> None:
    """Structural audit (the reference's invariants, preproc.py:305-372);
    raises CorruptArtifact naming the first bad cell.

    Scalar and offset-array checks run on the host; the per-cell group and
    permutation checks run on the device (rsr_audit, csrc/rsr_audit.cu) over
    the artifact's device arrays, only after the offsets are known to be in
    bounds."""
    import torch
    bad = lambda msg: CorruptArtifact(f"invalid artifact: {msg}")  # noqa: E731
    if a.bitwidth not in (BINARY, TERNARY):
        raise bad(f"bitwidth {a.bitwidth!r}")
    if a.m < 1 or a.n < 1:
        raise bad(f"shape {a.m} x {a.n}")
    if not 1 <= a.k <= K_CAP[a.bitwidth]:
        raise bad(f"k={a.k} outside 1..{K_CAP[a.bitwidth]} for {a.bitwidth}")
    p = a.plan
    if (p.block_count, p.tile_count) != (-(-a.m // a.k), -(-a.n // p.tile_width)):
        raise bad("plan grid does not match the shape")
    cells = p.block_count * p.tile_count
    go, po = _offsets_host(a.go_d), _offsets_host(a.po_d)
    n_words, n_perm = int(a.words_d.numel()), int(a.perm_d.numel())
    if go.shape != (cells + 1,) or po.shape != (cells + 1,):
        raise bad(f"offset arrays of length {go.size} / {po.size} for {cells} cells")
    if go[0] != 0 or po[0] != 0 or go[-1] != n_words or po[-1] != n_perm:
        raise bad("offset arrays do not span the word / perm arrays")
    down = np.flatnonzero((np.diff(go) < 0) | (np.diff(po) < 0))
    if down.size:
        raise bad(f"offsets decrease at cell {int(down[0])}")
    if cells == 0 or (n_words == 0 and n_perm == 0):
        return
    res = torch.empty(1, dtype=torch.int64, device=a.device)
    bw = _lib.RSR_BINARY if a.bitwidth == BINARY else _lib.RSR_TERNARY
    _lib.check(_lib.lib().rsr_audit(_lib.ptr(a.words_d), _lib.ptr(a.go_d), _lib.ptr(a.perm_d),
                                    _lib.ptr(a.po_d), a.m, a.n, a.k, bw, p.tile_width,
                                    p.block_count, p.tile_count, _lib.ptr(res),
                                    _lib.current_stream_ptr(a.device)), "validate_artifact")
    code = int(res.item()) & ((1 << 64) - 1)
    if code != (1 << 64) - 1:
        cell, check = code >> 8, code & 0xFF
        t, b = divmod(cell, p.block_count)
        raise bad(f"cell {cell} (tile {t}, block {b}): "
                  f"{_AUDIT_MESSAGES.get(check, f'check {check}')}")


def reconstruct(a: RsrArtifact) -> PackedMatrix:
    """The matrix an artifact encodes (reference preproc.py:375-400), rebuilt
    on the device after the audit: every group scatters its sign pattern to
    its columns (rsr_reconstruct)."""
    import torch
    validate_artifact(a)
    bw = _lib.RSR_BINARY if a.bitwidth == BINARY else _lib.RSR_TERNARY
    L = _lib.lib()
    nbytes = int(L.rsr_reconstruct_bytes(a.m, a.n, bw))
    buf = torch.empty(nbytes, dtype=torch.uint8, device=a.device)
    p = a.plan
    _lib.check(L.rsr_reconstruct(_lib.ptr(a.words_d), _lib.ptr(a.go_d), _lib.ptr(a.perm_d),
                                 _lib.ptr(a.po_d), a.m, a.n, a.k, bw, p.tile_width,
                                 p.block_count, p.tile_count, _lib.ptr(buf),
                                 _lib.current_stream_ptr(a.device)), "reconstruct")
    row_bytes = (a.n + 7) // 8 if a.bitwidth == BINARY else (a.n + 3) // 4
    data = buf[:a.m * row_bytes].view(a.m, row_bytes)
    return PackedMatrix(a.m, a.n, a.bitwidth, data, weight_scale=a.weight_scale)
