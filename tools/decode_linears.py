"""Linear-layer time per decode token of BitNetForCausalLM(BitNetConfig())
(random init) for the RSR replacement vs dense bf16 (cuBLAS), all linears of
all layers in model order in one CUDA graph (weights stream from HBM, as in
decode).  usage: python tools/decode_linears.py [k] [layers]"""
import copy
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from transformers import BitNetConfig, BitNetForCausalLM

from paper_2603_27462_b200.decode import linear_time_per_token
from paper_2603_27462_b200.hf import replace_linear_with_rsr

k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = BitNetConfig()
if len(sys.argv) > 2:
    cfg.num_hidden_layers = int(sys.argv[2])
torch.manual_seed(0)
with torch.device("cuda"):
    model = BitNetForCausalLM(cfg).to(torch.bfloat16).eval()
rsr_model = copy.deepcopy(model)
replace_linear_with_rsr(rsr_model, k=k)
for name, mdl in (("dense_bf16", model), ("rsr", rsr_model)):
    r = linear_time_per_token(mdl, reps=50)
    print(f"{name:10s} {r['us']:8.1f} us/token  {r['launches']} launches  "
          f"{r['bytes'] / 1e9:.3f} GB  {r['gbs']:.0f} GB/s", flush=True)
