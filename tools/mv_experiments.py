"""Time the C2 multiply under the RSR_MV_DEBUG experiment knobs (results are
wrong by design for non-zero knobs; timing only).

usage: python tools/mv_experiments.py  (runs each knob in a subprocess)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, os, torch, numpy as np
sys.path.insert(0, ROOTDIR)
import bench, paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn
cfg = bench.CONFIGS["c2"]
data = bench.random_packed(cfg["m"], cfg["n"], cfg["bitwidth"], 0)
a = rsr.preprocess(rsr.PackedMatrix(cfg["m"], cfg["n"], cfg["bitwidth"], data), cfg["k"])
mode = sys.argv[1]
v = torch.from_numpy(bench.random_vector(cfg["n"], 0)).cuda().to(torch.bfloat16)
y = torch.empty(cfg["m"], dtype=torch.float32, device="cuda")
if mode == "int":
    v = torch.randint(-128, 128, (cfg["n"],), dtype=torch.int8, device="cuda")
    y = torch.empty(cfg["m"], dtype=torch.int32, device="cuda")
copies = [(a.entries_d.clone(), a.e_off_d.clone()) for _ in range(4)]
views = [a.view(entries=e, e_off=o) for e, o in copies]
f = (lambda i: kn.fused_into(a, v, y, view=views[i % 4])) if mode == "fused" else (lambda i: kn.matvec_into(a, v, y, view=views[i % 4]))
for i in range(20): f(i)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(100)]
for i, (e0, e1) in enumerate(ev):
    e0.record(); f(i); e1.record()
torch.cuda.synchronize()
ts = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev)
print("%s dbg=%s pf=%s median_us=%.2f min_us=%.2f" % (mode, os.environ.get("RSR_MV_DEBUG", "0"), os.environ.get("RSR_MV_PF"), ts[50], ts[0]))
'''.replace('ROOTDIR', repr(ROOT))

knobs = os.environ.get("KNOBS", "0,1,2,3,4,7,8,15").split(",")
pfs = os.environ.get("PFS", "4").split(",")
for mode in (sys.argv[1:] or ["float"]):
    for dbg in knobs:
      for pf in pfs:
        env = dict(os.environ, RSR_MV_DEBUG=dbg, RSR_MV_PF=pf)
        r = subprocess.run([sys.executable, "-c", CHILD, mode], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-500:], flush=True)
