"""Device time of the tcgen05 batched multiply at C4 (ternary 8192^2, k=5)
for a list of batch sizes: CUDA-graph replays of 4 calls over rotated copies
of the code matrix.  RSR_B200_LIB selects a library build (e.g. an
experiment variant).  usage: python tools/tc_probe.py B [B ...]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn

m = n = 8192
data = bench.random_packed(m, n, "ternary", 0)
a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", data), 5)
kms = [a.keymat()] + [a.keymat().clone() for _ in range(3)]
kmw = [a.keymat("wide")] + [a.keymat("wide").clone() for _ in range(3)]
tag = os.path.basename(os.environ.get("RSR_B200_LIB", "librsr_b200.so"))


def graph_us(fn, reps=12):
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


for B in [int(x) for x in sys.argv[1:]]:
    V = torch.randn(B, n, device="cuda").to(torch.bfloat16)
    Y = torch.empty(B, m, device="cuda")

    def tc(i):
        a.__dict__["_keymat"] = kms[i % 4]
        a.__dict__["_keymat_wide"] = kmw[i % 4]  # (B <= 32: the 256-column-step kernel)
        kn.matmul_into(a, V, Y, method="tc")
    print(f"{tag} B={B:4d} tc {graph_us(tc):8.2f} us", flush=True)
