"""Where does the per-step time of the C2 multiply go under different
launch disciplines?  (20 steps after an idle gap, 20 steps queued behind a
device spin, 200 steps, a CUDA graph of 20 steps.)

usage: python tools/c2_timing_probe.py [k]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn

k = int(sys.argv[1]) if len(sys.argv) > 1 else 6
data = bench.random_packed(16384, 16384, "ternary", 0)
a = rsr.preprocess(rsr.PackedMatrix(16384, 16384, "ternary", data), k)
v = torch.from_numpy(bench.random_vector(16384, 0)).cuda().to(torch.bfloat16)
y = torch.empty(16384, dtype=torch.float32, device="cuda")
nc = 4
copies = [(a.entries_d, a.e_off_d)] + [(a.entries_d.clone(), a.e_off_d.clone()) for _ in range(nc - 1)]
views = [a.view(entries=e, e_off=o) for e, o in copies]
s = torch.cuda.current_stream()
sp = s.cuda_stream


def run(n, spin_us=0, sleep=0.0):
    for i in range(5):
        kn.matvec_into(a, v, y, view=views[i % nc], stream=sp)
    torch.cuda.synchronize()
    if sleep:
        time.sleep(sleep)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if spin_us:
        torch.cuda._sleep(int(spin_us * 1965))
    e0.record(s)
    t0 = time.perf_counter()
    for i in range(n):
        kn.matvec_into(a, v, y, view=views[i % nc], stream=sp)
    t1 = time.perf_counter()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n, (t1 - t0) * 1e6 / n


for label, kw in [("20 after 0.3s idle", dict(n=20, sleep=0.3)),
                  ("20 no idle", dict(n=20)),
                  ("20 queued behind 2ms spin", dict(n=20, spin_us=2000)),
                  ("20 queued behind 2ms spin after idle", dict(n=20, spin_us=2000, sleep=0.3)),
                  ("200 no idle", dict(n=200)),
                  ("200 queued behind 5ms spin", dict(n=200, spin_us=5000))]:
    r = [run(**kw) for _ in range(5)]
    dev = [x[0] for x in r]
    cpu = [x[1] for x in r]
    print(f"{label:40s} device us/step {np.median(dev):7.2f} (min {min(dev):.2f} max {max(dev):.2f})"
          f"  host launch us/step {np.median(cpu):6.2f}")
print("stream bytes", a.stream_bytes(), "file bytes", a.file_bytes())
