"""Per-CTA timeline of one multiply launch (rsr_debug_set_probe).

usage: python tools/timeline.py [cfg] [k] [float|int|fused]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn, _lib

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
if cfgname.startswith("mn"):
    mm, nn = (int(x) for x in cfgname[2:].split("x"))
    cfg = dict(m=mm, n=nn, bitwidth="ternary", k=5, vdtype="bf16")
else:
    cfg = dict(bench.CONFIGS[cfgname])
if len(sys.argv) > 2:
    cfg["k"] = int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "float"
warm = len(sys.argv) > 4 and sys.argv[4] == "warm"  # keep L2 / i-cache warm
data = bench.random_packed(cfg["m"], cfg["n"], cfg["bitwidth"], 0)
a = rsr.preprocess(rsr.PackedMatrix(cfg["m"], cfg["n"], cfg["bitwidth"], data), cfg["k"])
v = torch.from_numpy(bench.random_vector(cfg["n"], 0)).cuda().to(torch.bfloat16)
y = torch.empty(cfg["m"], dtype=torch.float32, device="cuda")
f = (lambda: kn.fused_into(a, v, y)) if mode == "fused" else (lambda: kn.matvec_into(a, v, y))
copies = [a.entries_d.clone() for _ in range(3)]
for _ in range(10): f()
torch.cuda.synchronize()
probe = torch.zeros(4096 * 4, dtype=torch.int64, device="cuda")
pv = probe.view(-1, 4)
pv[:, 2] = torch.iinfo(torch.int64).max
_lib.lib().rsr_debug_set_probe(probe.data_ptr())
# evict: touch the copies (cold) or run the multiply right before (warm)
if warm:
    f()
else:
    for c in copies: c.add_(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); f(); e1.record()
torch.cuda.synchronize()
_lib.lib().rsr_debug_set_probe(None)
t = pv.cpu().numpy().astype(np.float64)
used = t[:, 0] > 0
t = t[used]
t0 = t[:, 0].min()
r = (t - t0) / 1e3
print(f"{cfgname} {mode}: event {e0.elapsed_time(e1)*1e3:.1f} us, ctas {used.sum()}")
for name, col in (("start", 0), ("prologue done", 1), ("first warp done", 2), ("last warp done", 3)):
    c = r[:, col]
    print(f"  {name:16s} min {c.min():6.2f}  median {np.median(c):6.2f}  max {c.max():6.2f} us")
print(f"  prologue duration median {np.median(r[:,1]-r[:,0]):.2f} us; main loop (prologue->last) "
      f"median {np.median(r[:,3]-r[:,1]):.2f} max {np.max(r[:,3]-r[:,1]):.2f} us")
