"""Wall time of preprocess (GPU grouping + stream build) for a bench config.
usage: python tools/time_preprocess.py [c2] [k] [reps]"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2603_27462_b200 as rsr

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
k = int(sys.argv[2]) if len(sys.argv) > 2 else cfg["k"]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
data = bench.random_packed(cfg["m"], cfg["n"], cfg["bitwidth"], 0)
pm = rsr.PackedMatrix(cfg["m"], cfg["n"], cfg["bitwidth"], data)
torch.zeros(1, device="cuda")
for i in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a = rsr.preprocess(pm, k)
    torch.cuda.synchronize()
    print(f"preprocess #{i}: {1e3 * (time.perf_counter() - t0):.1f} ms")
