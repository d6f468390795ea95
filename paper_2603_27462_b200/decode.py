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
        toks = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            self.tok.copy_(self.next_tok)
            if self.graph is not None:
                self.graph.replay()
            else:
                self._step()
            toks.append(self.tok)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        return [int(t.item()) for t in toks], dt

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
