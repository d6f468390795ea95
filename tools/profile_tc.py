"""Small driver for ncu: the tensor-core batched multiply at C4 (k=5), bf16
or int8 batch.  usage: python tools/profile_tc.py [B] [reps] [bf16|i8]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kind = sys.argv[3] if len(sys.argv) > 3 else "bf16"
m = n = 8192
data = bench.random_packed(m, n, "ternary", 0)
a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", data), 5)
if kind == "i8":
    V = torch.randint(-128, 128, (B, n), dtype=torch.int8, device="cuda")
    Y = torch.empty(B, m, dtype=torch.int32, device="cuda")
else:
    V = torch.stack([torch.from_numpy(bench.random_vector(n, b)) for b in range(B)]).to(
        torch.bfloat16).cuda()
    Y = torch.empty(B, m, dtype=torch.float32, device="cuda")
for _ in range(reps):
    kn.matmul_into(a, V, Y, method="tc")
torch.cuda.synchronize()
print("ok")
