"""Small-config check of the decode path (dense vs RSR), graph capture included."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from transformers import BitNetConfig, BitNetForCausalLM
from paper_2603_27462_b200.hf import replace_linear_with_rsr
from paper_2603_27462_b200.decode import GraphDecoder

torch.manual_seed(0)
full = len(sys.argv) > 1 and sys.argv[1] == "full"
if full:
    cfg = BitNetConfig()
else:
    cfg = BitNetConfig(hidden_size=256, intermediate_size=512, num_hidden_layers=2,
                       num_attention_heads=4, num_key_value_heads=2, vocab_size=1000)
cfg._attn_implementation = "sdpa"
with torch.device("cuda"):
    model = BitNetForCausalLM(cfg).to(torch.bfloat16).eval()
prompt = torch.randint(0, cfg.vocab_size, (1, 16), device="cuda")
steps = int(os.environ.get("STEPS", "64"))
for name in ("dense", "rsr"):
    if name == "rsr":
        t0 = time.time(); replace_linear_with_rsr(model, k=5); torch.cuda.synchronize()
        print("convert s", time.time() - t0, "converted", model._rsr_converted, flush=True)
    dec = GraphDecoder(model, max_len=16 + steps + 8)
    dec.prefill(prompt)
    dec.capture()
    toks, dt = dec.generate(prompt, steps)
    t = dec.time_steps(prompt, steps)
    print(name, "tokens", toks[:8], "tok/s (events)", steps / t, "wall", steps / dt, flush=True)
