"""Back-to-back C2 multiplies: time per call with / without PDL (RSR_MV_PDL)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_27462_b200 as rsr
from paper_2603_27462_b200 import kernels as kn
cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
data = bench.random_packed(cfg["m"], cfg["n"], cfg["bitwidth"], 0)
a = rsr.preprocess(rsr.PackedMatrix(cfg["m"], cfg["n"], cfg["bitwidth"], data), cfg["k"])
copies = [(a.entries_d.clone(), a.e_off_d.clone()) for _ in range(4)]
views = [a.view(entries=e, e_off=o) for e, o in copies]
v = torch.from_numpy(bench.random_vector(cfg["n"], 0)).cuda().to(torch.bfloat16)
y = torch.empty(cfg["m"], dtype=torch.float32, device="cuda")
for i in range(20):
    kn.matvec_into(a, v, y, view=views[i % 4])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(400):
    kn.matvec_into(a, v, y, view=views[i % 4])
e1.record()
torch.cuda.synchronize()
print(f"PDL={os.environ.get('RSR_MV_PDL', '1')}: {e0.elapsed_time(e1) * 1e3 / 400:.2f} us per call")
