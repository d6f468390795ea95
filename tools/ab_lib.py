"""A/B of two builds of librsr_b200.so on the C2 float multiply (device time
per matvec from CUDA-graph replays over rotated stream copies).  Run once per
library: RSR_B200_LIB=<path> python tools/ab_lib.py [n_blocks ...]
(n_blocks limits the row-block view, e.g. to one cell per warp)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn

k = int(os.environ.get("AB_K", "6"))
data = bench.random_packed(16384, 16384, "ternary", 0)
a = rsr.preprocess(rsr.PackedMatrix(16384, 16384, "ternary", data), k)
v = torch.from_numpy(bench.random_vector(16384, 0)).cuda().to(torch.bfloat16)
y = torch.empty(16384, dtype=torch.float32, device="cuda")
copies = [(a.entries_d, a.e_off_d)] + [(a.entries_d.clone(), a.e_off_d.clone()) for _ in range(3)]
lib = os.path.basename(os.environ.get("RSR_B200_LIB", "librsr_b200.so"))
yref = None
for nb in [None] + [int(x) for x in sys.argv[1:]]:
    views = [a.view(0, nb, entries=e, e_off=o) for e, o in copies]
    f = lambda i: kn.matvec_into(a, v, y, view=views[i % 4])
    us = [bench.graph_time_us(f, copies=4, iters=400) for _ in range(3)]
    if nb is None:
        kn.matvec_into(a, v, y)
        torch.cuda.synchronize()
        yref = y.clone()
    print(f"{lib:28s} k={k} blocks={nb or a.plan.block_count:5d} {np.median(us):7.2f} us/matvec "
          f"(runs {', '.join(f'{u:.2f}' for u in us)})", flush=True)
np.save(f"gpurun_out/ab_y_{lib}.npy", yref.cpu().numpy())
