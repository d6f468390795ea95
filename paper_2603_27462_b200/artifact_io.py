"""`.rsra` artifact files: save a GPU-built
artifact byte-identically to the reference writer and load a file straight
into device buffers, so a model's preprocessing is paid once.

Format (reference pkg/src/rsrmv/artifact_io.py:1-21), little-endian:

    "RSRA" | u8 version=1 | u8 bitwidth (0 binary, 1 ternary) | u8 k | u8 0
    u32 m | u32 n | u32 tile_width | f32 weight_scale                (24 B)
    per cell, tile-major (t * block_count + b):
        u32 group_count | u32 perm_len | u64 words[group_count]
        | u16 perm[perm_len] | zero pad to 4 bytes

The writer assembles the whole file with vectorized scatters (no per-cell
loop); the reader walks the cell headers once, gathers words and
permutations with vectorized reads, audits the result with the reference's
structural invariants (validate_artifact, reference preproc.py:305-372) and
uploads it -- a corrupt file raises CorruptArtifact and never yields an
artifact.
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import CorruptArtifact, RsrError
from .matcore import BINARY, TERNARY
from .preproc import RsrArtifact, make_plan, validate_artifact

MAGIC = b"RSRA"
VERSION = 1
_HEADER = struct.Struct("<4sBBBBIIIf")


def serialize(m: int, n: int, k: int, bitwidth: str, tile_width: int, weight_scale: float,
              words, perm, group_offsets, perm_offsets) -> bytes:
    """Reference-format bytes of host artifact arrays (reference artifact_io.py:39-55)."""
    words = np.ascontiguousarray(words, dtype=np.uint64)
    perm = np.ascontiguousarray(perm, dtype=np.uint16)
    go = np.asarray(group_offsets, dtype=np.int64)
    po = np.asarray(perm_offsets, dtype=np.int64)
    gc, pl = np.diff(go), np.diff(po)
    cell_bytes = 8 + 8 * gc + 2 * pl + (-2 * pl) % 4          # every cell is 4-byte aligned
    off = _HEADER.size + np.concatenate(([0], np.cumsum(cell_bytes)))
    total = int(off[-1])
    buf = np.zeros(total, dtype=np.uint8)
    buf[:_HEADER.size] = np.frombuffer(_HEADER.pack(
        MAGIC, VERSION, 0 if bitwidth == BINARY else 1, k, 0, m, n, tile_width,
        weight_scale), dtype=np.uint8)
    u32 = buf.view(np.uint32)
    cells = gc.size
    c0 = off[:-1] // 4
    u32[c0] = gc.astype(np.uint32)
    u32[c0 + 1] = pl.astype(np.uint32)
    if words.size:  # words start 8 bytes into their cell (4-byte aligned: two u32 each)
        wc = np.repeat(np.arange(cells), gc)
        pos = c0[wc] + 2 + 2 * (np.arange(words.size) - go[wc])
        u32[pos] = (words & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        u32[pos + 1] = (words >> np.uint64(32)).astype(np.uint32)
    if perm.size:
        u16 = buf.view(np.uint16)
        pc = np.repeat(np.arange(cells), pl)
        ppos = (off[:-1] + 8 + 8 * gc)[pc] // 2 + (np.arange(perm.size) - po[pc])
        u16[ppos] = perm
    return buf.tobytes()


def to_bytes(a: RsrArtifact) -> bytes:
    """Reference-format bytes of a (GPU) artifact."""
    return serialize(a.m, a.n, a.k, a.bitwidth, a.plan.tile_width, a.weight_scale,
                     a.words, a.perm, a.group_offsets, a.perm_offsets)


def save(a: RsrArtifact, path) -> None:
    """Write an artifact; the bytes equal the reference writer's for the same
    matrix and k (reference artifact_io.py:39-55).  Like the reference, the
    artifact is audited first: a malformed one raises CorruptArtifact and
    no file is written."""
    validate_artifact(a)
    blob = to_bytes(a)
    with open(path, "wb") as f:
        f.write(blob)


def parse(blob: bytes, name: str = "<bytes>") -> dict:
    """Host arrays of an `.rsra` byte string (reference artifact_io.py:58-121).

    Raises CorruptArtifact on a malformed header, truncation, nonzero
    padding or trailing bytes.
    """
    if len(blob) < _HEADER.size or blob[:4] != MAGIC:
        raise CorruptArtifact(f"{name}: not an .rsra file")
    _, version, bw, k, _reserved, m, n, tw, scale = _HEADER.unpack_from(blob, 0)
    if version != VERSION:
        raise CorruptArtifact(f"{name}: unsupported version {version}")
    if bw not in (0, 1):
        raise CorruptArtifact(f"{name}: bad bitwidth byte {bw}")
    bitwidth = BINARY if bw == 0 else TERNARY
    try:
        plan = make_plan(m, n, k, bitwidth, tw)
    except (RsrError, ValueError) as e:
        raise CorruptArtifact(f"{name}: invalid header: {e}") from e
    cells = plan.tile_count * plan.block_count
    total = len(blob)
    gc = np.zeros(cells, np.int64)
    pl = np.zeros(cells, np.int64)
    starts = np.zeros(cells, np.int64)
    off = _HEADER.size
    for c in range(cells):  # cell sizes chain: one pass over the 8-byte headers
        if off + 8 > total:
            raise CorruptArtifact(f"{name}: truncated at cell {c}")
        g, p = struct.unpack_from("<II", blob, off)
        starts[c] = off
        need = 8 + 8 * g + 2 * p + (-2 * p) % 4
        if off + need > total:
            raise CorruptArtifact(f"{name}: truncated at cell {c}")
        gc[c], pl[c] = g, p
        off += need
    if off != total:
        raise CorruptArtifact(f"{name}: {total - off} trailing bytes")
    go = np.concatenate(([0], np.cumsum(gc)))
    po = np.concatenate(([0], np.cumsum(pl)))
    raw = np.frombuffer(blob, dtype=np.uint8)
    if go[-1]:
        wc = np.repeat(np.arange(cells), gc)
        byte0 = starts[wc] + 8 + 8 * (np.arange(go[-1]) - go[wc])
        words = raw[byte0[:, None] + np.arange(8)].copy().view("<u8").reshape(-1).astype(np.uint64)
    else:
        words = np.zeros(0, np.uint64)
    if po[-1]:
        pc = np.repeat(np.arange(cells), pl)
        byte0 = starts[pc] + 8 + 8 * gc[pc] + 2 * (np.arange(po[-1]) - po[pc])
        perm = raw[byte0[:, None] + np.arange(2)].copy().view("<u2").reshape(-1).astype(np.uint16)
    else:
        perm = np.zeros(0, np.uint16)
    pad = (-2 * pl) % 4
    padded = np.nonzero(pad)[0]
    if padded.size:
        pstart = starts[padded] + 8 + 8 * gc[padded] + 2 * pl[padded]
        if raw[pstart].any() or raw[pstart + 1].any():
            raise CorruptArtifact(f"{name}: nonzero padding at cell {int(padded[0])}")
    return dict(m=m, n=n, k=k, bitwidth=bitwidth, weight_scale=float(scale), plan=plan,
                words=words, perm=perm, group_offsets=go, perm_offsets=po)


def from_bytes(blob: bytes, device=None, name: str = "<bytes>") -> RsrArtifact:
    """Parse, upload, audit (device) and return an `.rsra` byte string as a
    device artifact; a malformed file raises CorruptArtifact before the
    multiply stream is derived from it."""
    d = parse(blob, name)
    return RsrArtifact.from_host(d["m"], d["n"], d["k"], d["bitwidth"], d["weight_scale"],
                                 d["plan"], d["words"], d["perm"], d["group_offsets"],
                                 d["perm_offsets"], None, device, audit=True)


def load(path, device=None) -> RsrArtifact:
    """Read, audit and upload an `.rsra` file (reference artifact_io.py:58-121)."""
    with open(path, "rb") as f:
        blob = f.read()
    return from_bytes(blob, device, str(path))
