import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn, _lib
for (m, n) in [(2560, 6912), (2560, 4096), (2560, 5000), (512, 6912), (2560, 8192)]:
    w = torch.randn(m, n) * 0.02
    mat = rsr.ternarize_weights(w.numpy())
    a = rsr.preprocess(mat, 5)
    torch.cuda.synchronize()
    print(m, n, "fmt", a.format, "plan", a.plan, "err before:", _lib.lib().rsr_last_cuda_error(), flush=True)
    v = torch.randn(n, device="cuda").to(torch.bfloat16)
    for mode in ("float", "int", "fused"):
        try:
            if mode == "fused":
                out = torch.empty(m, dtype=torch.float32, device="cuda"); kn.fused_into(a, v, out)
            elif mode == "int":
                vi = torch.randint(-5, 5, (n,), dtype=torch.int8, device="cuda"); out = torch.empty(m, dtype=torch.int32, device="cuda"); kn.matvec_into(a, vi, out)
            else:
                out = torch.empty(m, dtype=torch.float32, device="cuda"); kn.matvec_into(a, v, out)
            torch.cuda.synchronize()
            print("  ", mode, "ok", flush=True)
        except Exception as e:
            print("  ", mode, "FAIL", e, flush=True)
