"""Time the fused multiply on the BitNet-2B linear shapes (k=5) with CUDA
events over many back-to-back launches (device time per call)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn

k = int(os.environ.get("K", "5"))
shapes = [("qkv", 3840, 2560), ("o", 2560, 2560), ("gate_up", 13824, 2560), ("down", 2560, 6912)]
for name, m, n in shapes:
    w = torch.randn(m, n, device="cuda") * 0.02
    mat = rsr.ternarize_weights(w.cpu().numpy())
    a = rsr.preprocess(mat, k)
    v = torch.randn(n, device="cuda").to(torch.bfloat16)
    out = torch.empty(m, dtype=torch.float32, device="cuda")
    for _ in range(20):
        kn.fused_into(a, v, out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(50):
            kn.fused_into(a, v, out)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 50
    mb = a.stream_bytes() / 1e6
    print(f"{name:8s} {m}x{n} k={k} stream {mb:6.2f} MB  {us:7.2f} us/call  {mb/us*1e-3*1e3:7.0f} GB/s")
