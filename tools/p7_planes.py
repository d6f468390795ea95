"""P7 (north_star (3)): native base-3 ternary patterns vs two
binary planes (M = P - N, one stacked binary artifact) at C2 (ternary
16384^2, bf16 vector).  For each k: artifact bytes (reference file_bytes of
what the kernel streams), stream bytes, device time per matvec (CUDA-graph
replays over 4 rotated stream copies), achieved GB/s and fraction of the
measured HBM peak, and an int8 cross-check (two-plane == native, exact).

usage: python tools/p7_planes.py [--json out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn
from paper_2603_27462_b200.twoplane import TwoPlane

m = n = 16384
hbm, _ = bench.peaks()
data = bench.random_packed(m, n, "ternary", 0)
pm = rsr.PackedMatrix(m, n, "ternary", data)
v = torch.from_numpy(bench.random_vector(n, 0)).cuda().to(torch.bfloat16)
vi = torch.from_numpy(np.random.default_rng(0).integers(-128, 128, n).astype(np.int8)).cuda()
rows = []


def time_artifact(a, ylen):
    copies = [(a.entries_d, a.e_off_d)] + [(a.entries_d.clone(), a.e_off_d.clone())
                                           for _ in range(3)]
    views = [a.view(entries=e, e_off=o) for e, o in copies]
    y = torch.empty(ylen, dtype=torch.float32, device="cuda")
    us = [bench.graph_time_us(lambda i: kn.matvec_into(a, v, y, view=views[i % 4]), iters=200)
          for _ in range(3)]
    del copies, views
    return float(np.median(us))


yref = None
for k in (4, 5, 6, 7, 8):
    torch.cuda.synchronize()
    a = rsr.preprocess(pm, k)
    us = time_artifact(a, m)
    alg = (a.file_bytes() - 24) + n * 2 + m * 4
    yi = rsr.rsr_matvec(a, vi)
    if k == 6:
        yref = yi.clone()
    rows.append({"variant": "native base-3", "k": k, "format": a.format,
                 "file_bytes": a.file_bytes(), "stream_bytes": a.stream_bytes(),
                 "us": us, "alg_gbs": alg / us / 1e3, "frac_hbm": alg / us / 1e3 / hbm})
    print(json.dumps(rows[-1]), flush=True)
    del a
    torch.cuda.empty_cache()
for k in (6, 7, 8, 9, 10, 11, 12):
    tp = TwoPlane(pm, k)
    a = tp.artifact
    us = time_artifact(a, 2 * m)
    alg = (a.file_bytes() - 24) + n * 2 + m * 4
    same = bool(torch.equal(tp.matvec(vi), yref))
    rows.append({"variant": "two binary planes", "k": k, "format": a.format,
                 "file_bytes": a.file_bytes(), "stream_bytes": a.stream_bytes(),
                 "us": us, "alg_gbs": alg / us / 1e3, "frac_hbm": alg / us / 1e3 / hbm,
                 "int8_equals_native": same})
    print(json.dumps(rows[-1]), flush=True)
    assert same, f"two-plane k={k} int8 result differs from native"
    del tp, a
    torch.cuda.empty_cache()
best = {}
for r in rows:
    b = best.get(r["variant"])
    if b is None or r["us"] < b["us"]:
        best[r["variant"]] = r
print("best:", json.dumps(best))
if "--json" in sys.argv:
    with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
        json.dump({"rows": rows, "best": best, "hbm_gbs_peak": hbm}, f, indent=1)
