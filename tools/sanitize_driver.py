"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every multiply kernel family once on shapes that exercise the shared-memory
bucket paths (teams, multi-tile, register flush, u32 stream, batched).

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2603_27462_b200 as rsr
from oracle import rsr_oracle as orc

torch.cuda.set_device(0)
cases = [("ternary", 6, 600, 4096, None), ("ternary", 5, 96, 2560, None),
         ("binary", 8, 256, 4096, None), ("ternary", 6, 120, 20000, None),
         ("ternary", 4, 64, 3000, 1000), ("ternary", 9, 40, 3000, None),
         ("binary", 12, 48, 1000, None), ("ternary", 5, 40, 40000, None)]
for bw, k, m, n, tw in cases:
    p = orc.random_matrix(m, n, bw, k)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, bw, p.data, 0.5), k, tw)
    ref = orc.preprocess(p, k, tw)
    vi = np.random.default_rng(1).integers(-128, 128, n).astype(np.int8)
    assert np.array_equal(rsr.rsr_matvec(a, vi), orc.matvec_i8(ref, vi)), (bw, k, m, n)
    vf = orc.random_vector(n, 2)
    y = rsr.rsr_matvec(a, vf)
    vb = torch.from_numpy(vf).cuda().to(torch.bfloat16)
    yb = rsr.rsr_matvec(a, vb)
    if bw == "ternary":
        ref.weight_scale = 0.5
        assert np.array_equal(rsr.rsr_matvec_fused(a, vf), orc.fused_matvec(ref, vf))
        if k <= 8:
            V = torch.from_numpy(np.random.default_rng(3).standard_normal((8, n)).astype(
                np.float32)).to(torch.bfloat16).cuda()
            rsr.rsr_matvec_batched(a, V, method="tc")
            rsr.rsr_matvec_batched(a, V, method="stream")
    torch.cuda.synchronize()
    print("ok", bw, k, m, n, tw, flush=True)
print("sanitize driver done")
