"""Per-step timeline of CTA (0,0) of the tcgen05 batched kernel (debug build
with -DRSR_TC_DBG: librsr_b200_tcdbg.so).  usage: python tools/tc_timeline.py [B]"""
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
m = n = 8192
data = bench.random_packed(m, n, "ternary", 0)
a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", data), 5)
V = torch.randn(B, n, device="cuda").to(torch.bfloat16)
Y = torch.empty(B, m, device="cuda")
for _ in range(3):
    kn.matmul_into(a, V, Y, method="tc")
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 260)()
L = _lib.lib()
L.rsr_tc_debug.argtypes = [ctypes.c_void_p]
print("rc", L.rsr_tc_debug(ctypes.addressof(buf)))
t = np.array(buf[:], dtype=np.int64)
t0 = t[256]
print(f"end of loop {(t[257]-t0)/1e3:.2f} us, exit {(t[258]-t0)/1e3:.2f} us")
print(" it   prod_issue  exp_full  exp_done  mma_ready   (us from start)")
for it in range(64):
    row = t[it * 4: it * 4 + 4]
    if not row.any():
        break
    print(f"{it:3d} " + " ".join(f"{(x - t0)/1e3:9.2f}" if x else "        -" for x in (row[2], row[0], row[1], row[3])))
