"""Bank-aware builder A/B: mean gather wavefronts of C2 cells and back-to-back
multiply time for the library named by RSR_B200_LIB."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn
from test_gpu_stream import run_slots, decode_cell, wavefronts
cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
data = bench.random_packed(cfg["m"], cfg["n"], cfg["bitwidth"], 0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
a = rsr.preprocess(rsr.PackedMatrix(cfg["m"], cfg["n"], cfg["bitwidth"], data), cfg["k"])
e1.record()
torch.cuda.synchronize()
pre_ms = e0.elapsed_time(e1)
ent = a.entries_d.cpu().numpy().view(np.uint16)
e_off = a.e_off_d.cpu().numpy()
wfs = []
for dc in range(0, len(e_off) - 1, max(1, (len(e_off) - 1) // 40)):
    e0_, e1_ = int(e_off[dc]), int(e_off[dc + 1])
    seq = decode_cell(ent[e0_:e1_][run_slots(e1_ - e0_)], a.format)
    wfs.append((wavefronts(seq), wavefronts(seq, keys_read=a.format == 1)))
copies = [(a.entries_d.clone(), a.e_off_d.clone()) for _ in range(4)]
views = [a.view(entries=e, e_off=o) for e, o in copies]
v = torch.from_numpy(bench.random_vector(cfg["n"], 0)).cuda().to(torch.bfloat16)
y = torch.empty(cfg["m"], dtype=torch.float32, device="cuda")
for i in range(20):
    kn.matvec_into(a, v, y, view=views[i % 4])
torch.cuda.synchronize()
ts = []
for rep in range(5):
    e0.record()
    for i in range(400):
        kn.matvec_into(a, v, y, view=views[i % 4])
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3 / 400)
w = np.mean(np.array(wfs), axis=0)
print(f"{os.path.basename(os.environ.get('RSR_B200_LIB', 'default'))}: wavefronts {w[0]:.3f} (with key reads {w[1]:.3f}) "
      f"preprocess {pre_ms:.1f} ms  multiply {np.median(ts):.2f} us (min {min(ts):.2f})")
