"""Greedy decode with a static KV cache and one CUDA graph per step.

Used identically for the RSR model (linears replaced by RSRLinear) and the
dense bf16 baseline (cuBLAS nn.Linear), so tokens/s compare the linear layers
and nothing else: same HF modules, same attention, same cache, same graph.
"""

from __future__ import annotations

import time

import torch


class GraphDecoder:
    def __init__(self, model, max_len: int, use_graph: bool = True):
        from transformers import StaticCache
        self.model = model
        self.max_len = max_len
        self.use_graph = use_graph
        dev = next(model.parameters()).device
        self.cache = StaticCache(config=model.config, max_cache_len=max_len)
        self.tok = torch.zeros(1, 1, dtype=torch.long, device=dev)
        self.pos = torch.zeros(1, 1, dtype=torch.long, device=dev)
        self.next_tok = torch.zeros(1, 1, dtype=torch.long, device=dev)
        self.graph = None

    def _forward(self, ids, pos):
        out = self.model(input_ids=ids, position_ids=pos, past_key_values=self.cache,
                         use_cache=True)
        return out.logits[:, -1, :]

    def _step(self):
        logits = self._forward(self.tok, self.pos)
        self.next_tok.copy_(torch.argmax(logits, dim=-1, keepdim=True))
        self.pos.add_(1)

    def reset(self):
        self.cache.reset()

    @torch.no_grad()
    def prefill(self, prompt_ids: torch.Tensor):
        """Run the prompt eagerly; leaves next_tok = greedy token after it."""
        P = prompt_ids.shape[-1]
        pos = torch.arange(P, device=self.tok.device).unsqueeze(0)
        logits = self._forward(prompt_ids.view(1, -1), pos)
        self.next_tok.copy_(torch.argmax(logits, dim=-1, keepdim=True))
        self.pos.fill_(P)

    @torch.no_grad()
    def capture(self):
        """Capture one decode step (warms up on a side stream first)."""
        if not self.use_graph:
            return
        # capturing mutates the cache; callers re-prefill afterwards
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                self.tok.copy_(self.next_tok)
                self._step()
        torch.cuda.current_stream().wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._step()

    @torch.no_grad()
    def generate(self, prompt_ids: torch.Tensor, steps: int):
        """Greedy tokens after the prompt; returns (tokens list, seconds of decode)."""
        self.reset()
        self.prefill(prompt_ids)
        out = torch.empty(steps, dtype=torch.long, device=self.tok.device)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(steps):
            self.tok.copy_(self.next_tok)
            out[i].copy_(self.tok[0, 0])  # this step's input token (device copy)
            if self.graph is not None:
                self.graph.replay()
            else:
                self._step()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        return out.tolist(), dt

    @torch.no_grad()
    def time_steps(self, prompt_ids: torch.Tensor, steps: int) -> float:
        """Device-timed seconds for `steps` graph replays (CUDA events)."""
        self.reset()
        self.prefill(prompt_ids)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            self.tok.copy_(self.next_tok)
            self.graph.replay() if self.graph is not None else self._step()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3


@torch.no_grad()
def linear_time_per_token(model, reps: int = 20) -> dict:
    """Device time of one token's worth of the model's linear layers alone
    (batch 1), lm_head excluded (dense bf16 in both arms).

    Every linear of every layer runs once, in model order, on a (1, in)
    bf16 input, all captured in one CUDA graph (so the host launch rate is
    not measured) and replayed `reps` times; weights stream from HBM as in
    decode (the whole set exceeds L2).  RSR linears are timed per stacked
    sibling group (one fused launch computes q|k|v or gate|up)."""
    from torch import nn

    from .hf import RSRLinear
    dev = next(model.parameters()).device if any(True for _ in model.parameters()) \
        else torch.device("cuda")
    calls, seen = [], set()
    for name, mod in model.named_modules():
        if name.endswith("lm_head"):
            continue
        if isinstance(mod, RSRLinear):
            g = mod.group
            if id(g) in seen:
                continue
            seen.add(id(g))
            x = torch.randn(1, g.in_features, device=dev, dtype=torch.bfloat16)
            calls.append((lambda g=g, x=x: g.compute(x), g.artifact.stream_bytes()))
        elif isinstance(mod, nn.Linear):
            x = torch.randn(1, mod.in_features, device=dev, dtype=mod.weight.dtype)
            calls.append((lambda mod=mod, x=x: mod(x),
                          mod.weight.numel() * mod.weight.element_size()))
    if not calls:
        return {"us": 0.0, "launches": 0, "bytes": 0}
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for fn, _ in calls:
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for fn, _ in calls:
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    nbytes = int(sum(b for _, b in calls))
    return {"us": us, "launches": len(calls), "bytes": nbytes, "gbs": nbytes / us / 1e3}
