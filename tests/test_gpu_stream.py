"""Structure of the device chunk stream (include/rsr_b200.h).

The stream is ours (the reference has no device format), so these tests pin
its invariants by decoding it on the host: every cell holds exactly the
reference groups (key -> column set, paper's Step 1/2 output in
pkg/src/rsrmv/preproc.py:239-289) and the layout rules hold -- u16 formats
(quad layout): every chunk pair starts with a key, keys only at slots = 0 mod
4, inside a pair each key starts a new group; formats 0/1: column 0 is
padding and the cell's real column 0 is in col0_key; format 3 (the hot
format): every column is in the stream and padding names one of 32 zero words
(one per shared-memory bank); u32 (even layout): every chunk starts with a
key, keys at even slots, padding key 0 / column 0.  The bank-aware column
order keeps the shared-memory gathers near conflict-free.
"""
import numpy as np
import pytest

from oracle import rsr_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rsr():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_27462_b200 as rsr
    return rsr


def phys_slots(nent, CH):
    """numpy restatement of phys_slot() (csrc/rsr_preprocess.cu): u32 format,
    rounds of 64 chunks, lane L owns chunk pair L of the round."""
    p = np.arange(nent, dtype=np.int64)
    nch = nent // CH
    c, js = p // CH, p % CH
    pair, cin = c >> 1, c & 1
    r, lanep = pair >> 5, pair & 31
    np_ = np.minimum(32, (nch >> 1) - (r << 5))
    qe = CH >> 1
    q = cin * 2 + js // qe
    return r * 64 * CH + q * np_ * qe + lanep * qe + js % qe


def run_slots(nent):
    """numpy restatement of run_slot() (csrc/rsr_preprocess.cu): u16 formats,
    lane L owns the contiguous run of pairs [L*P, L*P + len_L)."""
    p = np.arange(nent, dtype=np.int64)
    N = nent // 32
    P = (N + 31) // 32
    Lf = N // P if P else 0
    rem = N - Lf * P
    j, slot = p >> 5, p & 31
    L, r = j // P, j % P
    npr = Lf + (r < rem)
    R = r * Lf + np.minimum(r, rem)
    return R * 32 + (slot >> 3) * npr * 8 + L * 8 + (slot & 7)


def dense_key(w, bitwidth_binary):
    pos, neg = (w >> 32) & 0xFFFF, w >> 48
    if bitwidth_binary:
        return int(pos)
    key, p3 = 0, 1
    for i in range(16):
        key += (((pos >> i) & 1) + 2 * ((neg >> i) & 1)) * p3
        p3 *= 3
    return int(key)


def zero_b(tn):
    """format 3: byte offset of the zero words after a tn-column image"""
    return 2 * (-(-tn // 64) * 64)


def decode_cell(ent, fmt, tn=16384):
    """-> list of (is_key, value) in logical order; format 3 padding decodes
    to (False, -1 - bank)."""
    out = []
    zb = zero_b(tn)
    for x in ent:
        x = int(x)
        if fmt == 3:
            if x & 1:
                out.append((True, x >> 2))
            elif x >= zb:
                assert (x - zb) % 4 == 0 and x < zb + 128, x
                out.append((False, -1 - (x - zb) // 4))
            else:
                out.append((False, x >> 1))
        elif fmt == 1:
            out.append((True, x >> 2) if x & 1 else (False, x >> 2))
        elif fmt == 0:
            out.append((True, x & 0x7FFF) if x & 0x8000 else (False, x))
        else:
            out.append((True, x & 0x7FFFFFFF) if x & 0x80000000 else (False, x))
    return out


def wavefronts(seq, keys_read=False, fmt=1):
    """Mean shared-memory wavefronts per gather instruction of one u16 cell:
    at round r, slot j, the active lanes L read sequence position
    (L*P + r)*32 + j; cost = max over banks of the distinct words read.
    Formats 0/1 stage 4-byte elements (bank = column % 32); format 3 stages
    bf16 halfwords (bank = (column >> 1) % 32, columns 2i and 2i+1 share a
    word) and its padding reads the zero word of bank b (value -1 - b).
    keys_read: the scaled format's kernel also reads v[key] at key slots."""
    N = len(seq) // 32
    P = (N + 31) // 32
    tot = n = 0
    for r in range(P):
        for j in range(32):
            banks = {}
            for L in range(32):
                pair = L * P + r
                if pair >= N or (pair // P) != L:
                    continue
                isk, val = seq[pair * 32 + j]
                if isk and not keys_read:
                    continue
                if fmt == 3:
                    if val < 0:
                        banks.setdefault(-1 - val, set()).add(("z", -1 - val))
                    else:
                        banks.setdefault((val >> 1) % 32, set()).add(val >> 1)
                else:
                    banks.setdefault(val % 32, set()).add(val)
            tot += max([1] + [len(v) for v in banks.values()])
            n += 1
    return tot / max(n, 1)


def check_stream(a, binary):
    fmt, CH = a.format, a.chunk
    quad = fmt != 2
    ent = a.entries_d.cpu().numpy().view(np.uint16 if a.entry_bytes == 2 else np.uint32)
    e_off = a.e_off_d.cpu().numpy()
    col0 = a.col0_d.cpu().numpy() if quad else None
    go, po = a.group_offsets, a.perm_offsets
    words, perm = a.words, a.perm
    bc, tc = a.plan.block_count, a.plan.tile_count
    wfs = []
    for dc in range(bc * tc):
        b, t = divmod(dc, tc)
        src = t * bc + b
        e0, e1 = int(e_off[dc]), int(e_off[dc + 1])
        assert (e1 - e0) % (2 * CH) == 0
        cell = ent[e0:e1]
        tn = min(a.plan.tile_width, a.n - t * a.plan.tile_width)
        seq = decode_cell(cell[run_slots(e1 - e0) if quad else phys_slots(e1 - e0, CH)], fmt, tn)
        exp, key0 = {}, 0
        for g in range(go[src], go[src + 1]):
            w = int(words[g])
            ps, L = w & 0xFFFF, (w >> 16) & 0xFFFF
            cols = sorted(int(c) for c in perm[po[src] + ps: po[src] + ps + L])
            key = dense_key(w, binary)
            if quad and fmt != 3 and cols[0] == 0:
                key0, cols = key, cols[1:]
            if cols:
                exp[key] = cols
        got, seen = {}, set()
        cur = None
        for i, (isk, val) in enumerate(seq):
            if i % (2 * CH if quad else CH) == 0:
                assert isk, f"cell {dc}: slot {i} must hold a key"
            if isk:
                assert i % (4 if quad else 2) == 0, f"cell {dc}: key at slot {i}"
                if quad and i % 32:
                    assert val not in seen, f"cell {dc}: repeated key inside a pair at {i}"
                cur = val
                seen.add(val)
                continue
            if fmt == 3:
                if val < 0:
                    continue  # padding: a zero word
                assert cur != 0, f"cell {dc}: a column after the sink key"
            elif (quad and val == 0) or cur == 0:
                assert val == 0, "padding must be column 0"
                continue
            got.setdefault(cur, []).append(val)
        got = {k: sorted(v) for k, v in got.items()}
        assert got == exp, f"cell {dc}: groups differ"
        if quad:
            assert int(col0[dc]) == key0, f"cell {dc}: col0_key"
        if quad and len(seq) >= 2048:
            wfs.append(wavefronts(seq, fmt=fmt))
    return wfs


@pytest.mark.parametrize("m,n,k,bw,tw", [
    (96, 3000, 6, "ternary", None),
    (64, 4096, 8, "binary", None),
    (40, 20000, 5, "ternary", 20000),   # format 3, tile > 16384
    (20, 65408, 6, "ternary", 32704),   # format 3, widest tile, two tiles
    (24, 33000, 4, "ternary", 32768),   # format 0 (tile > 32704)
    (30, 5000, 12, "binary", None),      # format 0 (keys > 2187)
    (24, 40000, 4, "ternary", 40000),    # format 2 (tile > 32768)
])
def test_stream_structure(rsr, m, n, k, bw, tw):
    p = orc.random_matrix(m, n, bw, m * 7 + n)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, bw, p.data), k, tw)
    check_stream(a, bw == "binary")


def test_bank_aware_order(rsr):
    """Random ternary 16384-wide cells (format 3): the per-instruction bank
    matching keeps gathers near one wavefront (tools/banksim.c models ~1.2;
    a key-sorted order costs ~3.3 and round 1's builder 1.86)."""
    p = orc.random_matrix(12, 16384, "ternary", 5)
    a = rsr.preprocess(rsr.PackedMatrix(12, 16384, "ternary", p.data), 6)
    assert a.format == 3
    wfs = check_stream(a, False)
    print("format 3 wavefronts per gather", float(np.mean(wfs)))
    assert wfs and float(np.mean(wfs)) < 1.35, wfs
