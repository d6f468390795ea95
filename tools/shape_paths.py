"""Per-call device time (CUDA graph of 50 back-to-back calls, L2-warm) of the
fused, float and int8 single-vector multiplies at the BitNet-2B linear shapes
(k=5), plus an empty-kernel floor.  usage: python tools/shape_paths.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn


def per_call_us(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


x = torch.zeros(1, device="cuda")
print(f"empty elementwise kernel: {per_call_us(lambda: x.add_(1)):.2f} us/call")
shapes = [("qkv", 3840, 2560), ("o", 2560, 2560), ("gate_up", 13824, 2560), ("down", 2560, 6912)]
for name, m, n in shapes:
    w = torch.randn(m, n, device="cuda") * 0.02
    a = rsr.preprocess(rsr.ternarize_weights(w.cpu().numpy()), 5)
    vb = torch.randn(n, device="cuda").to(torch.bfloat16)
    vi = torch.randint(-128, 128, (n,), dtype=torch.int8, device="cuda")
    yf = torch.empty(m, dtype=torch.float32, device="cuda")
    yi = torch.empty(m, dtype=torch.int32, device="cuda")
    f = per_call_us(lambda: kn.fused_into(a, vb, yf))
    fl = per_call_us(lambda: kn.matvec_into(a, vb, yf))
    it = per_call_us(lambda: kn.matvec_into(a, vi, yi))
    print(f"{name:8s} {m}x{n} stream {a.stream_bytes()/1e6:6.2f} MB  fused {f:6.2f}  float {fl:6.2f}  "
          f"int8 {it:6.2f} us/call", flush=True)
