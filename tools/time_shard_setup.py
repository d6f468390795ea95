"""Where the bench's preprocess_ms goes (C2, one rank): strip construction,
upload, grouping, stream build, shard bookkeeping."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import preproc as pp
from paper_2603_27462_b200 import shard

m = n = 16384
full = bench.random_packed(m, n, "ternary", 0)
torch.zeros(1, device="cuda")
rsr.preprocess(rsr.PackedMatrix(24, n, "ternary", full[:24]), 6)
torch.cuda.synchronize()
T = {}


def timed(name, fn):
    def wrap(*a, **kw):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*a, **kw)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + 1e3 * (time.perf_counter() - t0)
        return out
    return wrap


pp._grouping = timed("grouping (incl. upload)", pp._grouping)
pp.RsrArtifact._build_stream = timed("stream count+build", pp.RsrArtifact._build_stream)
strip = timed("strip_fn", lambda r0, r1: rsr.PackedMatrix(r1 - r0, n, "ternary", full[r0:r1]))
orig_dd = rsr.PackedMatrix.device_data
rsr.PackedMatrix.device_data = timed("device_data (H2D)", orig_dd)
for rep in range(2):
    T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sm = shard.ShardedMatrix(m, n, "ternary", 6, strip, 0, 1)
    torch.cuda.synchronize()
    tot = 1e3 * (time.perf_counter() - t0)
    print(f"rep {rep}: total {tot:.1f} ms;", "; ".join(f"{k} {v:.1f}" for k, v in T.items()), flush=True)
