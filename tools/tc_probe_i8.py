"""Device time of the int8 tensor-core batched multiply (kind::i8) at C4
(ternary 8192^2, k=5) vs the bf16 one, and of the batched fused prefill
(quantize rows -> int8 multiply -> dequantize).  usage: python
tools/tc_probe_i8.py B [B ...]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn


def graph_us(fn, reps=12):
    """Device time per call: 4 calls captured in one CUDA graph, replayed."""
    for i in range(4):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(4):
                fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * 4)


m = n = 8192
data = bench.random_packed(m, n, "ternary", 0)
a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", data), 5)
a.keymat("i8")
for B in [int(x) for x in sys.argv[1:]]:
    Vi = torch.randint(-128, 128, (B, n), dtype=torch.int8, device="cuda")
    Yi = torch.empty(B, m, dtype=torch.int32, device="cuda")
    us_tc = graph_us(lambda i: kn.matmul_into(a, Vi, Yi, method="tc"))
    us_st = graph_us(lambda i: kn.matmul_into(a, Vi, Yi, method="stream"))
    X = torch.randn(B, n, device="cuda").to(torch.bfloat16)
    out = torch.empty(B, m, dtype=torch.bfloat16, device="cuda")
    us_pf = graph_us(lambda i: kn.fused_rows_into(a, X, out))
    print(f"B={B:4d} int8 tc {us_tc:8.2f} us  int8 stream {us_st:8.2f} us  fused prefill {us_pf:8.2f} us",
          flush=True)
