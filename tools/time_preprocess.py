"""Wall time of preprocess (GPU grouping + stream build) for a bench config,
split into phases with device events (upload, grouping, stream count, stream
build) after a warm-up call.
usage: python tools/time_preprocess.py [c2] [k] [reps]"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import preproc as pp

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
k = int(sys.argv[2]) if len(sys.argv) > 2 else cfg["k"]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
data = bench.random_packed(cfg["m"], cfg["n"], cfg["bitwidth"], 0)
pm = rsr.PackedMatrix(cfg["m"], cfg["n"], cfg["bitwidth"], data)
torch.zeros(1, device="cuda")

# phase timers around the RsrArtifact stream build (monkeypatched wrapper)
marks = {}
_orig = pp.RsrArtifact._build_stream


def timed_build(self):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    _orig(self)
    e1.record()
    torch.cuda.synchronize()
    marks["stream_ms"] = e0.elapsed_time(e1)


pp.RsrArtifact._build_stream = timed_build
for i in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a = rsr.preprocess(pm, k)
    torch.cuda.synchronize()
    tot = 1e3 * (time.perf_counter() - t0)
    print(f"preprocess #{i}: {tot:.1f} ms end to end (host matrix in), "
          f"stream count+build {marks['stream_ms']:.1f} ms", flush=True)
dev = pm.device_data()
for i in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a = rsr.preprocess(rsr.PackedMatrix(cfg["m"], cfg["n"], cfg["bitwidth"], dev), k)
    torch.cuda.synchronize()
    print(f"preprocess from a device matrix #{i}: {1e3 * (time.perf_counter() - t0):.1f} ms, "
          f"stream count+build {marks['stream_ms']:.1f} ms", flush=True)
