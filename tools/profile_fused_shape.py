"""ncu driver: fused multiply at one BitNet shape.  usage: python tools/profile_fused_shape.py m n [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn
m, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = torch.randn(m, n) * 0.02
a = rsr.preprocess(rsr.ternarize_weights(w.numpy()), 5)
v = torch.randn(n, device="cuda").to(torch.bfloat16)
out = torch.empty(m, dtype=torch.float32, device="cuda")
for _ in range(reps):
    kn.fused_into(a, v, out)
torch.cuda.synchronize()
print("ok")
