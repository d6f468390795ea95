import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn, _lib
from oracle import rsr_oracle as orc
m, n, k, B = 96, 3000, 5, 5
p = orc.random_matrix(m, n, "ternary", m + 3 * n)
a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", p.data), k)
torch.cuda.synchronize(); print("preprocess ok", flush=True)
km = a.keymat(); torch.cuda.synchronize(); print("keymat ok", km.numel(), flush=True)
kmh = km.cpu().numpy().reshape(-1, (n + 15) // 16 * 16)
print("keymat rows", kmh.shape, "max key", kmh.max(), flush=True)
V = torch.randn(B, n).to(torch.bfloat16).cuda()
Y = torch.zeros(B, m, dtype=torch.float32, device="cuda")
kn.matmul_into(a, V, Y, method="tc")
torch.cuda.synchronize(); print("tc ok", flush=True)
