"""ncu child for P7: preprocess C2 natively or as two planes at k, then run
the multiply 3 times.  usage: python tools/p7_ncu_child.py native|planes k"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn
from paper_2603_27462_b200.twoplane import TwoPlane

kind, k = sys.argv[1], int(sys.argv[2])
pm = rsr.PackedMatrix(16384, 16384, "ternary", bench.random_packed(16384, 16384, "ternary", 0))
a = rsr.preprocess(pm, k) if kind == "native" else TwoPlane(pm, k).artifact
v = torch.from_numpy(bench.random_vector(16384, 0)).cuda().to(torch.bfloat16)
y = torch.empty(a.m, dtype=torch.float32, device="cuda")
for _ in range(3):
    kn.matvec_into(a, v, y)
torch.cuda.synchronize()
print(kind, k, "file_bytes", a.file_bytes(), "stream_bytes", a.stream_bytes())
