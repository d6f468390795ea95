"""Pieces of the host-in/host-out C2 multiply, timed separately (host clock,
300 calls each after warm-up): the raw C call, the numpy result copy, a bare
torch DMA copy each way, and device-only launch + sync."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import _lib, kernels as kn
cfg = dict(bench.CONFIGS["c2"])
data = bench.random_packed(cfg["m"], cfg["n"], cfg["bitwidth"], 0)
a = rsr.preprocess(rsr.PackedMatrix(cfg["m"], cfg["n"], cfg["bitwidth"], data), cfg["k"])
vf = bench.random_vector(cfg["n"], 0)
vh = torch.from_numpy(vf.copy()).pin_memory().numpy()


def t(fn, n=300):
    for _ in range(30):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


kn._matvec_host(a, vh)
_, fn, ref, code, hy, hyp, dvp, dyp, ws, wsb, _cs, _di, (dv, dy) = a.__dict__["_host_call_f32"]
sp = _lib.current_stream_ptr(a.device)
args = (ref, vh.ctypes.data, code, hyp, dvp, dyp, ws, wsb, sp)
print(f"public API rsr_matvec(numpy pinned)  {t(lambda: rsr.rsr_matvec(a, vh)):7.1f} us")
print(f"raw C rsr_matvec_host                {t(lambda: fn(*args)):7.1f} us")
print(f"numpy copy of the 64 KB result       {t(lambda: hy.copy()):7.1f} us")
vt = torch.from_numpy(vh)
ht = torch.from_numpy(hy)
def h2d():
    dv.copy_(vt, non_blocking=True); torch.cuda.synchronize()
def d2h():
    ht.copy_(dy, non_blocking=True); torch.cuda.synchronize()
print(f"torch H2D 64 KB pinned + sync        {t(h2d):7.1f} us")
print(f"torch D2H 64 KB pinned + sync        {t(d2h):7.1f} us")
print(f"empty sync                           {t(torch.cuda.synchronize):7.1f} us")
def dev_sync():
    kn.matvec_into(a, dv, dy); torch.cuda.synchronize()
print(f"device-only launch + sync            {t(dev_sync):7.1f} us")
print(f"launch only (back to back)           {t(lambda: kn.matvec_into(a, dv, dy)):7.1f} us")
print(f"public API rsr_matvec_fused(numpy pinned) {t(lambda: rsr.rsr_matvec_fused(a, vh)):7.1f} us")
