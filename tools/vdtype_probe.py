"""C2 device time per matvec by vector dtype (bf16 / f32 / f16), CUDA-graph
replays over rotated stream copies, plus one isolated launch + sync each.
usage: python tools/vdtype_probe.py"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn

data = bench.random_packed(16384, 16384, "ternary", 0)
a = rsr.preprocess(rsr.PackedMatrix(16384, 16384, "ternary", data), 6)
vf = torch.from_numpy(bench.random_vector(16384, 0)).cuda()
y = torch.empty(16384, dtype=torch.float32, device="cuda")
copies = [(a.entries_d, a.e_off_d)] + [(a.entries_d.clone(), a.e_off_d.clone()) for _ in range(3)]
views = [a.view(0, None, entries=e, e_off=o) for e, o in copies]
for name, v in (("bf16", vf.to(torch.bfloat16)), ("f32", vf), ("f16", vf.to(torch.float16))):
    us = [bench.graph_time_us(lambda i: kn.matvec_into(a, v, y, view=views[i % 4]), copies=4, iters=400)
          for _ in range(3)]
    for _ in range(10):
        kn.matvec_into(a, v, y)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        kn.matvec_into(a, v, y)
        torch.cuda.synchronize()
    iso = (time.perf_counter() - t0) / 200 * 1e6
    print(f"{name:5s} {np.median(us):7.2f} us/matvec (graph)   launch+sync {iso:6.1f} us", flush=True)
