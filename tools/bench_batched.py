"""C4: ternary 8192^2 (k=5) batched multiply vs cuBLAS bf16 GEMM, B in 1..64.

Device time per call with CUDA events over CUDA-graph replays of back-to-back
calls (host launch overhead excluded); L2 is
flushed between iterations by rotating 4 copies of the stream (and of the
dense weight for cuBLAS).  usage: python tools/bench_batched.py [k] [Bs...]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn
from oracle import rsr_oracle as orc

k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
Bs = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8, 16, 32, 64]
m = n = 8192
data = bench.random_packed(m, n, "ternary", 0)
a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", data), k)
copies = [(a.entries_d.clone(), a.e_off_d.clone()) for _ in range(4)]
views = [a.view(entries=e, e_off=o) for e, o in copies]
dense = torch.from_numpy(orc.decode(orc.random_matrix(m, n, "ternary", 0))).cuda()
Wb = [dense.to(torch.bfloat16) for _ in range(2)]  # 2 x 134 MB > L2
print(f"C4 ternary {m}x{n} k={k}: key matrix {a.keymat().numel()/1e6:.1f} MB, RSR stream {a.stream_bytes()/1e6:.1f} MB, "
      f"file_bytes {a.file_bytes()/1e6:.1f} MB, dense bf16 {m*n*2/1e6:.0f} MB")


def timeit(fn, iters=48):
    """Device time per call: 4 calls (one per rotated copy) captured in a CUDA
    graph and replayed, so host launch overhead does not hide the kernels."""
    for i in range(4):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(4):
            fn(i)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in range(4):
                fn(i)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters // 4):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (iters // 4 * 4)


for B in Bs:
    V = torch.stack([torch.from_numpy(bench.random_vector(n, b)) for b in range(B)]).to(
        torch.bfloat16).cuda()
    Y = torch.empty(B, m, dtype=torch.float32, device="cuda")
    us_rsr = timeit(lambda i: kn.matmul_into(a, V, Y, view=views[i % 4], method="stream"))
    def single(i):
        for b in range(B):
            kn.matvec_into(a, V[b], Y[b], view=views[i % 4])
    us_single = timeit(single, iters=8 if B > 8 else 48)
    a.keymat()
    kms = [a.keymat()] + [a.keymat().clone() for _ in range(3)]
    def tc(i):
        a.__dict__["_keymat"] = kms[i % 4]
        kn.matmul_into(a, V, Y, method="tc")
    us_tc = timeit(tc)
    a.__dict__["_keymat"] = kms[0]
    Yd = torch.empty(B, m, dtype=torch.bfloat16, device="cuda")
    us_cub = timeit(lambda i: torch.matmul(V, Wb[i % 2].t(), out=Yd))
    print(f"B={B:3d}  single-vector x B {us_single:8.2f} us   stream {us_rsr:8.2f} us   tcgen05 {us_tc:8.2f} us ({B/us_tc*1e6:10.0f} vec/s)   "
          f"cuBLAS bf16 {us_cub:8.2f} us ({B/us_cub*1e6:10.0f} vec/s)   tc/cuBLAS {us_cub/us_tc:5.2f}x",
          flush=True)
