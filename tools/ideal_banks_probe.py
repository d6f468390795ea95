"""Timing experiment (wrong results by design): how fast is the C2 multiply
when every gather instruction is conflict-free?  Column entries of the
scaled-u16 stream are rewritten so that lane L reads bank L (keys and the
group structure untouched); variant 'pads0' keeps the zero padding on
column 0 (bank 0), variant 'ideal' moves pads to the lane's bank too.

usage: python tools/ideal_banks_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn

data = bench.random_packed(16384, 16384, "ternary", 0)
a = rsr.preprocess(rsr.PackedMatrix(16384, 16384, "ternary", data), 6)
assert a.format == 1
ent = a.entries_d.cpu().numpy().view(np.uint16).copy()
e_off = a.e_off_d.cpu().numpy()


def lanes_of_cell(n):
    npairs = n // 32
    P = (npairs + 31) // 32
    Lf = npairs // P
    rem = npairs - Lf * P
    lane = np.empty(n, np.int64)
    for r in range(P):
        np_ = Lf + (1 if r < rem else 0)
        R = r * Lf + min(r, rem)
        o = np.arange(np_ * 32)
        lane[R * 32:(R + np_) * 32] = (o % (np_ * 8)) // 8
    return lane


def rewrite(keep_pads):
    out = ent.copy()
    for dc in range(len(e_off) - 1):
        e0, e1 = int(e_off[dc]), int(e_off[dc + 1])
        seg = out[e0:e1]
        lane = lanes_of_cell(e1 - e0).astype(np.uint16)
        col = (seg & 1) == 0
        if keep_pads:
            col &= seg != 0
        seg[col] = ((((seg[col] >> 2) & ~np.uint16(31)) | lane[col]) << 2).astype(np.uint16)
    return out


v = torch.from_numpy(bench.random_vector(16384, 0)).cuda().to(torch.bfloat16)
y = torch.empty(16384, dtype=torch.float32, device="cuda")


def timed(entries_np, label):
    base = torch.from_numpy(entries_np.view(np.int16)).cuda()
    copies = [base] + [base.clone() for _ in range(3)]
    views = [a.view(entries=e, e_off=a.e_off_d) for e in copies]
    f = lambda i: kn.matvec_into(a, v, y, view=views[i % 4])
    us = [bench.graph_time_us(f, copies=4, iters=200) for _ in range(3)]
    print(f"{label:28s} {np.median(us):7.2f} us/matvec", flush=True)


timed(ent, "as built (bank-aware)")
timed(rewrite(True), "conflict-free, pads bank 0")
timed(rewrite(False), "conflict-free incl. pads")
