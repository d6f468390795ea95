"""Small driver for ncu: build one artifact, run a few multiplies.

usage: python tools/profile_matvec.py [c2|c1|c4] [k] [float|int|fused] [reps]
"""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
if cfgname.startswith("mn"):  # e.g. mn2560x2560 -> ternary m x n, bf16 v
    mm, nn = (int(x) for x in cfgname[2:].split("x"))
    cfg = dict(workload="custom", m=mm, n=nn, bitwidth="ternary", k=5, vdtype="bf16")
else:
    cfg = dict(bench.CONFIGS[cfgname])
if len(sys.argv) > 2:
    cfg["k"] = int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "float"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
if cfg.get("gen") == "hash":  # C5: the device generator (the numpy one needs 137 GB)
    from paper_2603_27462_b200.devicepack import random_ternary_device
    pm = random_ternary_device(cfg["m"], cfg["n"], 0, 0.5)
else:
    pm = rsr.PackedMatrix(cfg["m"], cfg["n"], cfg["bitwidth"],
                          bench.random_packed(cfg["m"], cfg["n"], cfg["bitwidth"], 0))
a = rsr.preprocess(pm, cfg["k"], cfg.get("tile_width"))
v = torch.from_numpy(bench.random_vector(cfg["n"], 0)).cuda()
if cfg["vdtype"] == "bf16":
    v = v.to(torch.bfloat16)
y = torch.empty(cfg["m"], dtype=torch.float32, device="cuda")
if mode == "int":
    v = torch.randint(-128, 128, (cfg["n"],), dtype=torch.int8, device="cuda")
    y = torch.empty(cfg["m"], dtype=torch.int32, device="cuda")
for _ in range(reps):
    if mode == "fused":
        kn.fused_into(a, v, y)
    else:
        kn.matvec_into(a, v, y)
torch.cuda.synchronize()
print("ok", a.stream_bytes(), a.file_bytes())
