"""Where the e2e (host in, host out) C2 multiply spends its time: the public
numpy API vs the bare C call vs device-only launch + sync."""
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
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


print(f"public API rsr_matvec(numpy pinned)   {t(lambda: rsr.rsr_matvec(a, vh)):7.1f} us")
print(f"_matvec_host (numpy in/out)          {t(lambda: kn._matvec_host(a, vh)):7.1f} us")
dv = torch.from_numpy(vf).cuda()
y = torch.empty(a.m, device="cuda")
def dev_sync():
    kn.matvec_into(a, dv, y)
    torch.cuda.synchronize()
print(f"device-only launch + sync            {t(dev_sync):7.1f} us")
print(f"launch only (back to back)           {t(lambda: kn.matvec_into(a, dv, y)):7.1f} us")

# round-trip latency floor: an empty kernel + stream sync, and the same with
# an event polled in a loop (no blocking wait)
x = torch.zeros(1, device="cuda")
s = torch.cuda.current_stream()
def empty_sync():
    x.add_(1)
    s.synchronize()
print(f"empty kernel + stream sync           {t(empty_sync):7.1f} us")
ev = torch.cuda.Event()
def empty_poll():
    x.add_(1)
    ev.record(s)
    while not ev.query():
        pass
print(f"empty kernel + event poll            {t(empty_poll):7.1f} us")
def dev_poll():
    kn.matvec_into(a, dv, y)
    ev.record(s)
    while not ev.query():
        pass
print(f"device-only launch + event poll      {t(dev_poll):7.1f} us")
