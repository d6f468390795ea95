"""Shared-memory bank-conflict simulator for the chunk-stream gather.

Lays out one ternary k-row cell (random pattern per column, P(0)=1/2) in the
device chunk order (rounds of 32 lanes x 32 slots; lane L owns sequence
positions 32L..32L+31 of the round) and reports the mean wavefronts per gather
instruction (max over banks of distinct columns at one slot across lanes)
for different placement heuristics.

usage: python tools/bank_sim.py [n] [k] [cells]
"""
import sys
import numpy as np

CH = 16


def random_cell(n, k, rng):
    d = rng.choice(3, size=(k, n), p=[0.5, 0.25, 0.25])
    key = np.zeros(n, dtype=np.int64)
    p3 = 1
    for i in range(k):
        key += d[i] * p3
        p3 *= 3
    groups = {}
    for c in range(n):
        if key[c]:
            groups.setdefault(int(key[c]), []).append(c)
    return [(kk, groups[kk]) for kk in sorted(groups)]


def place(groups):
    """Sequence of entries: ('k', key) or ('c', col), same rules as place_group."""
    seq = []
    for key, cols in groups:
        seq.append(("k", key))
        R = len(cols)
        j = 0
        while True:
            room = CH - len(seq) % CH
            if R >= room:
                for _ in range(room):
                    seq.append(("c", cols[j])); j += 1
                R -= room
                if R == 0:
                    break
                seq.append(("k", key))
                continue
            if R & 1:
                for _ in range(R):
                    seq.append(("c", cols[j])); j += 1
                break
            for _ in range(R - 1):
                seq.append(("c", cols[j])); j += 1
            seq.append(("k", key))
            seq.append(("c", cols[j])); j += 1
            break
    while len(seq) % (2 * CH):
        seq.append(("k", 0) if len(seq) % 2 == 0 else ("c", 0))
    return seq


def wavefronts(seq, nb=32):
    tot = 0
    ninst = 0
    for r0 in range(0, len(seq), 1024):
        rnd = seq[r0:r0 + 1024]
        nl = len(rnd) // 32
        for j in range(32):
            cnt = np.zeros(nb, dtype=np.int64)
            for L in range(nl):
                e = rnd[32 * L + j]
                if e[0] == "c":
                    cnt[e[1] % nb] += 1
            tot += max(1, cnt.max())
            ninst += 1
    return tot / ninst


def greedy_within_group(groups, nb=32):
    """Same key positions; within each group choose columns bank-aware."""
    seq = place(groups)
    # slot ranges per group are fixed; recollect the column multiset per group
    out = list(seq)
    used = {}  # (round, slot) -> bank counts
    # walk groups in sequence order
    i = 0
    pos_by_group = []
    cur = None
    for p, e in enumerate(seq):
        if e[0] == "k":
            if cur is None or e[1] != cur[0]:
                cur = [e[1], []]
                pos_by_group.append(cur)
        else:
            cur[1].append(p)
    gcols = {k: list(c) for k, c in groups}
    gcols[0] = [0] * 64
    for key, poss in pos_by_group:
        rem = list(gcols[key]) if key else None
        for p in poss:
            r, L, j = p // 1024, (p % 1024) // 32, p % 32
            cnt = used.setdefault((r, j), np.zeros(nb, dtype=np.int64))
            if rem is None:
                c = 0
            else:
                best = min(range(len(rem)), key=lambda t: cnt[rem[t] % nb])
                c = rem.pop(best)
            cnt[c % nb] += 1
            out[p] = ("c", c)
    return out


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    cells = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    rng = np.random.default_rng(0)
    for _ in range(cells):
        g = random_cell(n, k, rng)
        s0 = place(g)
        print("groups", len(g), "entries", len(s0),
              "base %.3f" % wavefronts(s0),
              "greedy-in-group %.3f" % wavefronts(greedy_within_group(g)))


def local_search(seq, passes=3, nb=32, rng=None):
    """Swap columns of the same segment key within a cell when that lowers
    sum(cnt^2) over the (round, slot) conflict sets."""
    seq = list(seq)
    cnt = {}
    def cs(p):
        return (p // 1024, p % 32)
    for p, e in enumerate(seq):
        if e[0] == "c":
            cnt.setdefault(cs(p), np.zeros(nb, dtype=np.int64))[e[1] % nb] += 1
    # positions per key
    bykey = {}
    cur = None
    for p, e in enumerate(seq):
        if e[0] == "k":
            cur = e[1]
        elif cur:
            bykey.setdefault(cur, []).append(p)
    for _ in range(passes):
        for key, poss in bykey.items():
            for a in range(len(poss)):
                for b in range(a + 1, len(poss)):
                    p1, p2 = poss[a], poss[b]
                    c1, c2 = seq[p1][1], seq[p2][1]
                    b1, b2 = c1 % nb, c2 % nb
                    if b1 == b2:
                        continue
                    s1, s2 = cnt[cs(p1)], cnt[cs(p2)]
                    if cs(p1) == cs(p2):
                        continue
                    # delta of sum cnt^2: move b1 out of s1, b2 in; b2 out of s2, b1 in
                    d = (-2 * s1[b1] + 2 + 2 * s1[b2] + 2 - 2 * s2[b2] + 2 + 2 * s2[b1] + 2) - 4
                    if d < 0:
                        s1[b1] -= 1; s1[b2] += 1; s2[b2] -= 1; s2[b1] += 1
                        seq[p1], seq[p2] = ("c", c2), ("c", c1)
    return seq


def greedy_two_choice(groups, nb=32, shift=16):
    """Greedy within group where each column may also be read from a second
    copy of v whose banks are rotated by `shift`; returns (seq, bank list)."""
    seq = place(groups)
    banks = [None] * len(seq)
    used = {}
    pos_by_group = []
    cur = None
    for p, e in enumerate(seq):
        if e[0] == "k":
            if cur is None or e[1] != cur[0]:
                cur = [e[1], []]
                pos_by_group.append(cur)
        else:
            cur[1].append(p)
    gcols = {k: list(c) for k, c in groups}
    for key, poss in pos_by_group:
        rem = list(gcols[key]) if key else None
        for p in poss:
            r, j = p // 1024, p % 32
            cnt = used.setdefault((r, j), np.zeros(nb, dtype=np.int64))
            if rem is None:
                c, bk = 0, 0
            else:
                best, bb, bc = None, None, 1 << 30
                for t, c in enumerate(rem):
                    for cp in (0, 1):
                        b = (c + cp * shift) % nb
                        if cnt[b] < bc:
                            best, bb, bc = t, b, cnt[b]
                c = rem.pop(best)
                bk = bb
            cnt[bk] += 1
            banks[p] = bk
    return banks


def wavefronts_banks(banks):
    tot = ninst = 0
    for r0 in range(0, len(banks), 1024):
        rnd = banks[r0:r0 + 1024]
        nl = len(rnd) // 32
        for j in range(32):
            cnt = np.zeros(32, dtype=np.int64)
            for L in range(nl):
                b = rnd[32 * L + j]
                if b is not None:
                    cnt[b] += 1
            tot += max(1, cnt.max()); ninst += 1
    return tot / ninst


def greedy_window(groups, W=32, nb=32):
    """Device-builder heuristic: a window of the next W unplaced columns of the
    group (one per lane); each position takes the window column whose bank is
    least used at that (round, slot), ties to the lowest window index; the
    freed window entry is refilled with the group's next column."""
    seq = place(groups)
    out = list(seq)
    gcols = {k: list(c) for k, c in groups}
    cur = None
    win = []
    nxt = 0
    cnt = {}
    for p, e in enumerate(seq):
        if e[0] == "k":
            if e[1] != cur:
                cur = e[1]
                cols = gcols.get(cur, [])
                win = cols[:W]
                nxt = len(win)
            continue
        r, j = p // 1024, p % 32
        c_ = cnt.setdefault((r, j), np.zeros(nb, dtype=np.int64))
        if cur == 0:
            c = 0
        else:
            best = min(range(len(win)), key=lambda t: (c_[win[t] % nb], t))
            c = win[best]
            if nxt < len(cols):
                win[best] = cols[nxt]; nxt += 1
            else:
                win.pop(best)
        c_[c % nb] += 1
        out[p] = ("c", c)
    return out
