"""Per-step timeline of CTA (0,0) of the tcgen05 batched kernel (debug build
with -DRSR_TC_DBG: librsr_b200_tcdbg.so).  usage: python tools/tc_timeline.py [B] [i8]"""
import ctypes
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["RSR_B200_LIB"] = os.path.join(ROOT, "paper_2603_27462_b200", "librsr_b200_tcdbg.so")
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import _lib
from paper_2603_27462_b200 import kernels as kn
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
I8 = len(sys.argv) > 2 and sys.argv[2] == "i8"
m = n = 8192
data = bench.random_packed(m, n, "ternary", 0)
a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", data), 5)
if I8:
    V = torch.randint(-128, 128, (B, n), dtype=torch.int8, device="cuda")
    Y = torch.empty(B, m, dtype=torch.int32, device="cuda")
else:
    V = torch.randn(B, n, device="cuda").to(torch.bfloat16)
    Y = torch.empty(B, m, device="cuda")
for _ in range(3):
    kn.matmul_into(a, V, Y, method="tc")
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (64 * 8 + 4))()
L = _lib.lib()
L.rsr_tc_debug.argtypes = [ctypes.c_void_p]
print("rc", L.rsr_tc_debug(ctypes.addressof(buf)))
t = np.array(buf[:], dtype=np.int64)
t0 = t[512]
print(f"end of loop {(t[513]-t0)/1e3:.2f} us, exit {(t[514]-t0)/1e3:.2f} us")
print(" it   prod_issue  exp_full  expanded  aempty_ok  st_done  exp_done  mma_ready   (us from start)")
for it in range(64):
    row = t[it * 8: it * 8 + 8]
    if not row.any():
        break
    print(f"{it:3d} " + " ".join(f"{(x - t0)/1e3:9.2f}" if x else "        -" for x in (row[2], row[0], row[4], row[5], row[6], row[1], row[3])))
# every CTA: entry / setup done / expander loop done / epilogue done / after
# the CTA barrier / exit, relative to the earliest entry; slot 6 = last-arriver flags
cb = (ctypes.c_ulonglong * 8192)()
L.rsr_tc_debug_ctas.argtypes = [ctypes.c_void_p]
L.rsr_tc_debug_ctas(ctypes.addressof(cb))
c = np.array(cb[:], dtype=np.int64).reshape(1024, 8)
c = c[c[:, 0] > 0]
flags = np.zeros(len(c), np.int64)
if (c[:, 6] > 0).all():
    last = np.where(c[:, 7] > 0, c[:, 7], c[:, 6])
    print(f"cluster reduction: sums+stores median {np.median(c[:,6]-c[:,5])/1e3:.2f} us, "
          f"then to exit {np.median(c[:,3]-last)/1e3:.2f} us")
base = c[:, 0].min()
c = (c[:, [0, 1, 2, 4, 5, 3]] - base) / 1e3
print(f"CTAs {len(c)}: entry max {c[:,0].max():.2f} us; setup {np.median(c[:,1]-c[:,0]):.2f}; loop median {np.median(c[:,2]-c[:,1]):.2f} max {np.max(c[:,2]-c[:,1]):.2f}; "
      f"epilogue median {np.median(c[:,3]-c[:,2]):.2f}; barrier median {np.median(c[:,4]-c[:,3]):.2f}; reduce median {np.median(c[:,5]-c[:,4]):.2f}; last exit {c[:,5].max():.2f} us")
for name, sel in (("last arrivers", flags > 0), ("others", flags == 0)):
    if sel.any():
        x = c[sel]
        print(f"  {name} ({sel.sum()}): epilogue {np.median(x[:,3]-x[:,2]):.2f}, barrier {np.median(x[:,4]-x[:,3]):.2f}, reduce {np.median(x[:,5]-x[:,4]):.2f} (max {np.max(x[:,5]-x[:,4]):.2f}), exit median {np.median(x[:,5]):.2f} max {x[:,5].max():.2f}")
# MMA thread of CTA 0: cycles per step in the full wait, the A-ready wait, issue + commits
mb = (ctypes.c_longlong * 192)()
L.rsr_tc_debug_mma.argtypes = [ctypes.c_void_p]
L.rsr_tc_debug_mma(ctypes.addressof(mb))
m3 = np.array(mb[:], dtype=np.int64).reshape(64, 3)
m3 = m3[: max(1, int((m3.sum(1) > 0).sum()))]
print("MMA thread cycles/step (median): step period %d, aready wait %d, issue+commit %d" % tuple(np.median(m3, 0)))
print("  per step:", " ".join(f"{a}/{b}/{c}" for a, b, c in m3[:24]))
