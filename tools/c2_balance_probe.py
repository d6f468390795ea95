"""Does the SM-level cell imbalance of C2 (2731 cells = 67 SMs x 19 + 81 x
18) cost time?  C2-shaped ternary matrices (n = 16384, k = 6) with row
counts giving 2664 cells (18 per SM), 2731 (C2) and 2812 (19 per SM):
device time per matvec and GB/s over the stream."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn

n, k = 16384, 6
for cells in (2664, 2731, 2812):
    m = cells * k
    a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", bench.random_packed(m, n, "ternary", 0)), k)
    copies = [(a.entries_d, a.e_off_d)] + [(a.entries_d.clone(), a.e_off_d.clone()) for _ in range(3)]
    views = [a.view(entries=e, e_off=o) for e, o in copies]
    v = torch.from_numpy(bench.random_vector(n, 0)).cuda().to(torch.bfloat16)
    y = torch.empty(m, device="cuda")
    us = bench.graph_time_us(lambda i: kn.matvec_into(a, v, y, view=views[i % 4]))
    sb = a.stream_bytes()
    print(f"cells {cells}: {us:6.2f} us, stream {sb/1e6:6.1f} MB, {sb/us/1e3:6.0f} GB/s", flush=True)
    del copies, views, a
    torch.cuda.empty_cache()
