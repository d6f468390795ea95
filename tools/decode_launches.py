"""One graph-replayed decode step of BitNet-2B (RSR linears) for an ncu launch
list: python tools/decode_launches.py [rsr|dense]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from transformers import BitNetConfig, BitNetForCausalLM
from paper_2603_27462_b200.hf import replace_linear_with_rsr
from paper_2603_27462_b200.decode import GraphDecoder
torch.manual_seed(0)
cfg = BitNetConfig()
cfg._attn_implementation = "sdpa"
with torch.device("cuda"):
    model = BitNetForCausalLM(cfg).to(torch.bfloat16).eval()
if (sys.argv[1] if len(sys.argv) > 1 else "rsr") == "rsr":
    replace_linear_with_rsr(model, k=5)
prompt = torch.randint(0, cfg.vocab_size, (1, 16), device="cuda")
dec = GraphDecoder(model, max_len=64)
dec.prefill(prompt)
dec.capture()
dec.reset(); dec.prefill(prompt)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
dec.tok.copy_(dec.next_tok)
dec.graph.replay()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
