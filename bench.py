"""Benchmark of the RSR hot path on B200 (driver contract: one JSON line).

Workloads (BASELINE.json configs):
  c2  (default at N=1) ternary 16384x16384 single-vector RSR matvec, bf16
      vector, k=6 (fewest artifact bytes); matrix = reference generator
      (rsrmv bench.py:102-113), seed 0.  A step is one matvec.
  c5  (default at N>1) ternary 131072x131072, k=6, row-block sharded across
      the ranks (each rank generates and preprocesses only its strip with the
      device generator); the output slices are all-gathered by the multiply
      itself, storing its rows into every rank's symmetric-memory output
      (--gather peer, then one barrier), or by NCCL + reassembly in row order
      (--gather nccl).  Strong scaling: every step is one
      full 131072^2 matvec for the whole job.  The N > 1 line also carries
      the same matrix on rank 0's GPU alone, timed in the same run
      (`c5_1gpu`, `scaling_vs_1gpu_same_run`): the N = 1 bench line is the
      C2 headline, not this matrix.
  c1, c4 (binary 4096^2 k=8 f32 vector; ternary 8192^2 k=5) on request.

`value` = matvec/s with the stream resident in HBM; L2 is defeated by
rotating >= 3 copies of the stream (inputs larger than L2 per step).  The K
timed launches are queued behind a short device spin, so the region measures
the device back to back (not the host's launch rate or a cold first launch
after an idle gap); --graph (one GPU) replays them as one CUDA graph instead.  `e2e` = the same metric through the public API with a
host (numpy float32) vector and a host result (rank 0, unsharded configs).

Sub-objects (N=1): `cublas_bf16` (the dense bf16 GEMV of the same matrix,
north_star's context number), `c4` (ternary 8192^2 batched multiply, B =
1..64, vs the cuBLAS bf16 GEMM), `decode` (greedy decode tok/s of
BitNetForCausalLM(BitNetConfig()) with the HF linear replacement vs dense
bf16 nn.Linear, identical graph-captured loop, plus linear-only time per
token), and `roofline.traffic` measured by an ncu child process on one
launch of the same kernel.  --impl reference times the CPU restatement of the
reference float path (oracle/, all host cores) on the same config.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

CONFIGS = {
    "c2": dict(workload="ternary 16384x16384 RSR matvec, bf16 vector, single vector",
               m=16384, n=16384, bitwidth="ternary", k=6, vdtype="bf16", gen="numpy"),
    "c1": dict(workload="binary 4096x4096 RSR matvec, fp32 vector, k=8",
               m=4096, n=4096, bitwidth="binary", k=8, vdtype="f32", gen="numpy"),
    "c4": dict(workload="ternary 8192x8192 RSR matvec, bf16 vector, single vector",
               m=8192, n=8192, bitwidth="ternary", k=5, vdtype="bf16", gen="numpy"),
    "c5": dict(workload="ternary 131072x131072 RSR matvec, bf16 vector, row-block sharded "
                        "+ all-gather of outputs",
               m=131072, n=131072, bitwidth="ternary", k=6, vdtype="bf16", gen="hash",
               # 8 tiles of 16384 columns (measured on one GPU, tools/c5_tile_width.py:
               # 1.084 ms vs 1.186 at 21846, 1.361 at 32704 -- wide tiles' 64 KB v images
               # leave fewer warps per SM -- and 1.475 at 13108; 7.7% more artifact
               # bytes than at 32704)
               tile_width=16384),
}
METRIC = "ternary matvec/s & %HBM roofline at 16384^2; BitNet-2B-shape decode tok/s"
UNIT = "matvec/s"
L2_DEFEAT = "rotating >= 3 copies of the chunk stream (each step's inputs exceed L2)"
L2_LARGE = "none needed: each step streams > 3x the 126 MB L2 (C5: 6.4 GB, 0.8 GB per rank at 8)"


def make_config(cname: str, cfg: dict, world: int) -> dict:
    """The workload description, identical for both arms."""
    return {"workload": cfg["workload"], "name": cname, "m": cfg["m"], "n": cfg["n"],
            "k": cfg["k"], "bitwidth": cfg["bitwidth"], "vector_dtype": cfg["vdtype"],
            "tile_width": cfg.get("tile_width") or (cfg["n"] if cfg["n"] <= 65536 else 32768),
            "seed": 0, "density": 0.5,
            "generator": "rsrmv random_matrix (numpy)" if cfg["gen"] == "numpy"
            else "counter-based splitmix64 (device; CPU restatement in oracle/)",
            "l2_defeat": L2_LARGE if cname == "c5" else L2_DEFEAT,
            "parallelism": f"rowblock{world}" if world > 1 else "single"}


def random_packed(m, n, bitwidth, seed, density=0.5):
    """Reference generator (rsrmv bench.py:102-113) + packing (matcore.py:114-125)."""
    rng = np.random.default_rng(seed)
    u = rng.random((m, n))
    if bitwidth == "binary":
        ent = (u < density).astype(np.uint8)
        return np.packbits(ent, axis=1, bitorder="little")
    codes = (u < density / 2).astype(np.uint8) | ((u > 1 - density / 2).astype(np.uint8) << 1)
    del u
    pad = (-n) % 4
    if pad:
        codes = np.concatenate([codes, np.zeros((m, pad), np.uint8)], axis=1)
    c4 = codes.reshape(m, -1, 4)
    return np.ascontiguousarray(c4[:, :, 0] | (c4[:, :, 1] << 2) | (c4[:, :, 2] << 4)
                                | (c4[:, :, 3] << 6))


def random_vector(n, seed):
    """rsrmv bench.py:116-117."""
    return np.random.default_rng(seed ^ 0x5EED).standard_normal(n).astype(np.float32)


def bf16_round(v):
    b = v.view(np.uint32).astype(np.uint64)
    return ((((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16).astype(np.uint32)).view(np.float32)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except (ValueError, IndexError):
                continue
            for nm, val in zip(names, f[2:]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": mx or None, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference arm (oracle/ = C restatement of the reference float path)

def cpu_reference_run(cfg, steps, warmup, seconds=None):
    """Matvec/s of the reference float path (float64 accumulation, exactly
    rsrmv matvec_f32) on all host threads.  For c5 the sample is one row
    strip (the whole matrix does not fit the host); the rate is scaled to the
    full matrix by rows."""
    from oracle import rsr_oracle as orc
    rows = cfg["m"]
    if cfg["gen"] == "hash":
        rows = 1200
        p = orc.random_ternary_rows(0, rows, cfg["n"], 0, 0.5)
    else:
        p = orc.Packed(cfg["m"], cfg["n"], cfg["bitwidth"],
                       random_packed(cfg["m"], cfg["n"], cfg["bitwidth"], 0))
    a = orc.preprocess(p, cfg["k"], cfg.get("tile_width"))
    v = random_vector(cfg["n"], 0)
    if cfg["vdtype"] == "bf16":
        v = bf16_round(v)
    threads = orc.max_threads()
    for _ in range(max(warmup, 1)):
        orc.matvec_f32(a, v, threads=threads)
    n = 0
    t0 = time.perf_counter()
    while True:
        orc.matvec_f32(a, v, threads=threads)
        n += 1
        el = time.perf_counter() - t0
        if (seconds is None and n >= steps) or (seconds is not None and el >= seconds):
            break
    frac = rows / cfg["m"]
    rate = n / el * frac
    sample = (f"{n} {'strip (' + str(rows) + ' rows) ' if frac < 1 else ''}"
              f"{rows}x{cfg['n']} float-path matvecs in {el:.1f}s on {threads} threads "
              f"(C restatement of rsrmv matvec_f32, block-parallel, float64 accumulation)"
              + (f"; rate scaled by rows to the full {cfg['m']}x{cfg['n']}" if frac < 1 else ""))
    return rate, threads, n, el, sample


# ---------------------------------------------------------------------------
# device timing helpers

def spin_cycles(steps: int) -> int:
    """Device spin long enough for the host to enqueue `steps` launches
    behind it (~15 us of host time per launch, generous), >= 2 ms."""
    return int(max(2000.0, 40.0 * steps) * 1965)


def graph_time_us(fn, copies: int = 4, iters: int = 48) -> float:
    """Device time per call: `copies` calls (fn(i), one per rotated input
    copy) captured in one CUDA graph and replayed back to back."""
    import torch
    for i in range(copies):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(copies):
            fn(i)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in range(copies):
                fn(i)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(1, iters // copies)
    torch.cuda._sleep(spin_cycles(reps))
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * copies)


# ---------------------------------------------------------------------------
# cuBLAS bf16 dense GEMV of the same matrix (north_star: "reported for context")

def cublas_bf16_bench(packed, m, n, v_bf16, hbm, rsr_value):
    import torch
    from paper_2603_27462_b200.matcore import dense_device
    W = dense_device(packed).to(torch.bfloat16)  # [m, n] bf16, 2*m*n bytes (> L2)
    y = torch.empty(m, dtype=torch.bfloat16, device=W.device)
    for _ in range(5):
        torch.mv(W, v_bf16, out=y)
    torch.cuda.synchronize()
    reps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(spin_cycles(reps))
    e0.record()
    for _ in range(reps):
        torch.mv(W, v_bf16, out=y)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    nbytes = 2 * m * n + 2 * n + 2 * m
    del W
    torch.cuda.empty_cache()
    return {"op": f"torch.mv(W bf16 [{m}x{n}], v bf16) -> cuBLAS GEMV, same matrix decoded",
            "us": us, "matvec_s": 1e6 / us, "bytes": nbytes, "gbs": nbytes / us / 1e3,
            "frac_hbm": nbytes / us / 1e3 / hbm, "rsr_speedup": rsr_value / (1e6 / us)}


# ---------------------------------------------------------------------------
# single-vector side configs: C1 (binary 4096^2, f32 vector, k=8) and C5 on
# one GPU (ternary 131072^2, 32704-wide tiles, device generator)

def side_config_bench(cname: str, hbm: float):
    import torch
    import paper_2603_27462_b200 as rsr
    from paper_2603_27462_b200 import kernels as kn
    from paper_2603_27462_b200.devicepack import random_ternary_device
    cfg = CONFIGS[cname]
    m, n, k = cfg["m"], cfg["n"], cfg["k"]
    if cfg["gen"] == "hash":
        pm = random_ternary_device(m, n, 0, 0.5)
    else:
        pm = rsr.PackedMatrix(m, n, cfg["bitwidth"], random_packed(m, n, cfg["bitwidth"], 0))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a = rsr.preprocess(pm, k, cfg.get("tile_width"))
    torch.cuda.synchronize()
    pre_ms = 1e3 * (time.perf_counter() - t0)
    del pm
    v = torch.from_numpy(random_vector(n, 0)).cuda()
    if cfg["vdtype"] == "bf16":
        v = v.to(torch.bfloat16)
    y = torch.empty(m, dtype=torch.float32, device="cuda")
    sb = a.stream_bytes()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    nc = int(max(1, min(4, -(-3 * l2 // max(sb, 1)))))
    copies = [(a.entries_d, a.e_off_d)] + [(a.entries_d.clone(), a.e_off_d.clone())
                                           for _ in range(nc - 1)]
    views = [a.view(entries=e, e_off=o) for e, o in copies]
    us = graph_time_us(lambda i: kn.matvec_into(a, v, y, view=views[i % nc]), copies=nc,
                       iters=max(nc, 40 if sb < 1e9 else 8))
    alg = (a.file_bytes() - 24) + n * (2 if cfg["vdtype"] == "bf16" else 4) + m * 4
    wl = cfg["workload"].split(", row-block sharded")[0]
    out = {"workload": wl + (", one GPU, unsharded" if wl != cfg["workload"] else ""),
           "k": k, "tile_width": a.plan.tile_width,
           "format": a.format, "us": us, "matvec_s": 1e6 / us, "alg_bytes": int(alg),
           "alg_gbs": alg / us / 1e3, "frac_hbm": alg / us / 1e3 / hbm,
           "preprocess_ms": pre_ms,
           "l2": f"{nc} rotated stream copies" if nc > 1 else "stream larger than L2"}
    del copies, views, a
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# C4: batched multiply vs cuBLAS bf16 GEMM

def c4_bench(Bs=(1, 2, 4, 8, 16, 32, 64)):
    import torch
    import paper_2603_27462_b200 as rsr
    from paper_2603_27462_b200 import kernels as kn
    from paper_2603_27462_b200.matcore import dense_device
    m = n = 8192
    k = 5
    pm = rsr.PackedMatrix(m, n, "ternary", random_packed(m, n, "ternary", 0))
    a = rsr.preprocess(pm, k)
    copies = [(a.entries_d, a.e_off_d)] + [(a.entries_d.clone(), a.e_off_d.clone())
                                           for _ in range(3)]
    views = [a.view(entries=e, e_off=o) for e, o in copies]
    km = a.keymat()
    kms = [km] + ([km.clone() for _ in range(3)] if km is not None else [])
    kw = a.keymat("wide")  # B <= 32: the 256-column-step kernel's code matrix
    kmw = [kw] + ([kw.clone() for _ in range(3)] if kw is not None else [])
    dense = dense_device(pm).to(torch.bfloat16)
    Wb = [dense, dense.clone()]  # 2 x 134 MB > L2
    Wi = [dense.to(torch.int8), dense.to(torch.int8)]  # 2 x 67 MB
    rows = []
    for B in Bs:
        V = torch.stack([torch.from_numpy(random_vector(n, b)) for b in range(B)]).to(
            torch.bfloat16).cuda()
        Y = torch.empty(B, m, dtype=torch.float32, device="cuda")

        def ours(i):
            if kms:
                a.__dict__["_keymat"] = kms[i % 4]
                a.__dict__["_keymat_wide"] = kmw[i % 4]
            kn.matmul_into(a, V, Y, view=views[i % 4])
        us = graph_time_us(ours)
        Yd = torch.empty(B, m, dtype=torch.bfloat16, device="cuda")
        us_cub = graph_time_us(lambda i: torch.matmul(V, Wb[i % 2].t(), out=Yd))
        alg = (a.file_bytes() - 24) + B * (n * 2 + m * 4)
        row = {"B": B, "us": us, "vectors_s": B / us * 1e6, "cublas_us": us_cub,
               "vs_cublas": us_cub / us, "alg_bytes": int(alg), "alg_gbs": alg / us / 1e3}
        if B >= 2:
            # the exact integer path on the int8 tensor cores (int8 batch ->
            # int32), beside cuBLASLt's dense int8 GEMM of the same matrix
            Vi = torch.randint(-128, 128, (B, n), dtype=torch.int8, device="cuda")
            Yi = torch.empty(B, m, dtype=torch.int32, device="cuda")
            kmi = [a.keymat("i8")] + [a.keymat("i8").clone() for _ in range(3)]

            def ours_i8(i):
                a.__dict__["_keymat_i8"] = kmi[i % 4]
                kn.matmul_into(a, Vi, Yi)
            row["int8_us"] = graph_time_us(ours_i8)
            a.__dict__["_keymat_i8"] = kmi[0]
            if B > 16 and Wi is not None:
                try:
                    row["cublas_int8_us"] = graph_time_us(
                        lambda i: torch._int_mm(Vi, Wi[i % 2].t()))
                    row["int8_vs_cublas_int8"] = row["cublas_int8_us"] / row["int8_us"]
                except RuntimeError:
                    pass
        rows.append(row)
    if kms:
        a.__dict__["_keymat"] = kms[0]
        a.__dict__["_keymat_wide"] = kmw[0]
    del Wb, Wi, dense
    torch.cuda.empty_cache()
    return {"workload": "ternary 8192x8192, k=5, bf16 vectors [B, 8192] -> f32 [B, 8192]",
            "api": "rsr_matvec_batched / kernels.matmul_into(method='auto')",
            "timing": "CUDA-graph replays of 4 back-to-back calls over rotated stream copies",
            "cublas": "torch.matmul(V bf16 [B, 8192], W bf16 [8192, 8192]^T)",
            "int8": "int8_us: int8 batch -> exact int32 on tcgen05 kind::i8 (matmul_into auto); "
                    "cublas_int8_us: torch._int_mm(V int8, W int8^T) (cuBLASLt, B > 16)",
            "rows": rows}


# ---------------------------------------------------------------------------
# decode sub-benchmark (C3)

def decode_bench(steps=64, k=5):
    import torch
    from transformers import BitNetConfig, BitNetForCausalLM
    from paper_2603_27462_b200.decode import GraphDecoder, linear_time_per_token
    from paper_2603_27462_b200.hf import fuse_rms_norms, replace_linear_with_rsr
    torch.manual_seed(0)
    cfg = BitNetConfig()
    cfg._attn_implementation = "sdpa"
    with torch.device("cuda"):
        model = BitNetForCausalLM(cfg).to(torch.bfloat16).eval()
    prompt = torch.randint(0, cfg.vocab_size, (1, 16), device="cuda")
    import copy
    rsr_model = copy.deepcopy(model)
    replace_linear_with_rsr(rsr_model, k=k)
    bl_model = copy.deepcopy(model)
    replace_linear_with_rsr(bl_model, k=k, fuse_norms=True)
    dn_model = copy.deepcopy(model)
    fuse_rms_norms(dn_model)
    decs = {}
    for name, mdl in (("dense_bf16_cublas", model), ("rsr", rsr_model), ("rsr_bitlinear", bl_model),
                      ("dense_fused_norm", dn_model)):
        dec = GraphDecoder(mdl, max_len=16 + steps + 8)
        dec.prefill(prompt)
        dec.capture()
        dec.time_steps(prompt, 8)
        decs[name] = dec
    # interleaved repetitions (clock / thermal drift hits both arms alike)
    samples = {name: [] for name in decs}
    for _ in range(5):
        for name, dec in decs.items():
            samples[name].append(steps / dec.time_steps(prompt, steps))
    res = {name: float(np.median(v)) for name, v in samples.items()}
    del decs
    torch.cuda.empty_cache()
    lin = {"dense_bf16_cublas": linear_time_per_token(model),
           "rsr": linear_time_per_token(rsr_model)}
    del bl_model, dn_model
    return {"model": "BitNetForCausalLM(BitNetConfig()) random init, bf16, 30 layers, "
                     "hidden 2560, FFN 6912",
            "loop": "greedy, HF StaticCache, one CUDA graph per step, batch 1",
            "k": k, "steps": steps, "reps": "median of 5 interleaved runs per arm",
            "rsr_tok_s": res["rsr"],
            "dense_tok_s": res["dense_bf16_cublas"],
            "speedup": res["rsr"] / res["dense_bf16_cublas"],
            "rsr_bitlinear_tok_s": res["rsr_bitlinear"],
            "bitlinear_speedup": res["rsr_bitlinear"] / res["dense_bf16_cublas"],
            "bitlinear": "replace_linear_with_rsr(fuse_norms=True): the four RMSNorms of each "
                         "layer run inside the following RSR launches (BitLinear); the dense "
                         "arm keeps HF's unfused norms",
            "dense_fused_norm_tok_s": res["dense_fused_norm"],
            "bitlinear_vs_dense_fused_norm": res["rsr_bitlinear"] / res["dense_fused_norm"],
            "dense_fused_norm": "dense bf16 linears with each RMSNorm as one launch "
                                "(hf.fuse_rms_norms, same arithmetic as the BitLinear prologue): "
                                "the like-for-like comparison for rsr_bitlinear",
            "linear_us_per_token": {name: v["us"] for name, v in lin.items()},
            "linear_speedup": lin["dense_bf16_cublas"]["us"] / lin["rsr"]["us"],
            "linear_detail": lin}


# ---------------------------------------------------------------------------
# roofline.traffic: DRAM bytes of one launch, measured by an ncu child

def traffic_child(cname: str, k: int):
    """Run under ncu by measure_traffic(): preprocess + 3 launches."""
    import torch
    import paper_2603_27462_b200 as rsr
    from paper_2603_27462_b200 import kernels as kn
    cfg = CONFIGS[cname]
    m, n = cfg["m"], cfg["n"]
    a = rsr.preprocess(rsr.PackedMatrix(m, n, cfg["bitwidth"],
                                        random_packed(m, n, cfg["bitwidth"], 0)), k,
                       cfg.get("tile_width"))
    v = torch.from_numpy(random_vector(n, 0)).cuda()
    if cfg["vdtype"] == "bf16":
        v = v.to(torch.bfloat16)
    y = torch.empty(m, dtype=torch.float32, device="cuda")
    for _ in range(3):
        kn.matvec_into(a, v, y)
    torch.cuda.synchronize()


def measure_traffic(cname: str, k: int, timeout: int = 300):
    """dram__bytes_read.sum + dram__bytes_write.sum of the third launch of the
    multiply kernel (ncu flushes caches before the replay: cold HBM bytes)."""
    ncu = "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "-k", "regex:rsr_mv_kernel", "--launch-skip", "2", "-c", "1", "--csv",
           sys.executable, os.path.abspath(__file__), "--traffic-child", "--config", cname,
           "--k", str(k)]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout).stdout
    except Exception as e:
        return None, f"ncu child failed: {e!r}"[:200]
    vals = {}
    for line in out.splitlines():
        f = [x.strip('"') for x in line.split('","')]
        if len(f) >= 3 and f[-3] in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                                     "gpu__time_duration.sum"):
            unit, val = f[-2], float(f[-1].replace(",", "").strip('"'))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                     "KB": 1e3, "MB": 1e6, "GB": 1e9, "nsecond": 1e-3, "usecond": 1.0,
                     "msecond": 1e3}.get(unit, 1.0)
            vals[f[-3]] = val * scale
    if "dram__bytes_read.sum" not in vals:
        return None, "ncu output not parsed"
    rd, wr = vals["dram__bytes_read.sum"], vals.get("dram__bytes_write.sum", 0.0)
    return {"bytes": int(rd + wr), "read": int(rd), "write": int(wr),
            "ncu_us": vals.get("gpu__time_duration.sum")}, None


# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS))
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="one GPU: time the K steps as one CUDA-graph replay (pays the graph "
                         "launch once: slower than queued launches at K = 20, faster at 200)")
    ap.add_argument("--gather", choices=["peer", "nccl"], default="peer",
                    help="N > 1: all-gather of the output slices by the multiply's own peer "
                         "stores into symmetric memory (default) or by NCCL")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip cublas_bf16 / c4 / traffic sub-measurements")
    ap.add_argument("--traffic-child", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cname = args.config or ("c2" if world == 1 else "c5")
    cfg = dict(CONFIGS[cname])
    if args.k:
        cfg["k"] = args.k
    if args.traffic_child:
        traffic_child(cname, cfg["k"])
        return
    warmup = max(args.warmup, 3)
    config = make_config(cname, cfg, world)

    if args.impl == "reference":
        if rank != 0:
            return
        val, threads, n, el, sample = cpu_reference_run(cfg, args.steps, warmup)
        line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
                "steps": n, "warmup": warmup, "ms_per_step": 1e3 / val,
                "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config, "impl": "reference",
                "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "port",
                                 "sample": sample},
                "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_2603_27462_b200 as rsr
    from paper_2603_27462_b200 import kernels as kn
    from paper_2603_27462_b200 import shard
    from paper_2603_27462_b200.devicepack import random_ternary_device

    # functional check of the N > 1 code path on a one-GPU box (never a
    # measurement): RSR_BENCH_ONE_DEVICE=1 puts every rank on cuda:0 and
    # RSR_BENCH_DIST_BACKEND=gloo carries the collective
    if os.environ.get("RSR_BENCH_ONE_DEVICE"):
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("RSR_BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    m, n, k = cfg["m"], cfg["n"], cfg["k"]
    full_packed = None
    if cfg["gen"] == "numpy":
        full = random_packed(m, n, cfg["bitwidth"], 0)
        full_packed = rsr.PackedMatrix(m, n, cfg["bitwidth"], full)
        strip = lambda r0, r1: rsr.PackedMatrix(r1 - r0, n, cfg["bitwidth"], full[r0:r1])
    else:
        strip = lambda r0, r1: random_ternary_device(r1 - r0, n, 0, 0.5, row0=r0, device=dev)
    # warm-up preprocess of a few rows (same width and k: the same kernels),
    # so preprocess_ms times the preprocessing, not CUDA's lazy module loading
    tw = cfg.get("tile_width")
    rsr.preprocess(strip(0, min(m, 4 * k)), k,
                   shard.make_plan(m, n, k, cfg["bitwidth"], tw).tile_width, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sm = shard.ShardedMatrix(m, n, cfg["bitwidth"], k, strip, rank, world, device=dev,
                             tile_width=tw)
    torch.cuda.synchronize()
    preprocess_cold_ms = 1e3 * (time.perf_counter() - t0)
    # and again with the allocator and host paths warm (a serving process
    # preprocessing its next matrix): the artifact used below is this one
    del sm
    t0 = time.perf_counter()
    sm = shard.ShardedMatrix(m, n, cfg["bitwidth"], k, strip, rank, world, device=dev,
                             tile_width=tw)
    torch.cuda.synchronize()
    preprocess_ms = 1e3 * (time.perf_counter() - t0)
    a = sm.local
    tc = a.plan.tile_count

    # L2 defeat: rotate copies of the local stream
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    sb = a.stream_bytes()
    # a stream far larger than L2 needs no rotation (rotating three 6.4 GB
    # copies only adds TLB pressure a single artifact does not have)
    ncopies = 1 if sb > 3 * l2 else int(max(3, min(16, -(-3 * l2 // max(sb, 1)))))
    copies = [(a.entries_d, a.e_off_d)] + [(a.entries_d.clone(), a.e_off_d.clone())
                                           for _ in range(ncopies - 1)]
    views = [a.view(entries=e, e_off=o) for e, o in copies]

    vf = random_vector(n, 0)
    vt = torch.from_numpy(vf).to(dev)
    if cfg["vdtype"] == "bf16":
        vt = vt.to(torch.bfloat16)
    y_local, y_all = sm.buffers(torch.float32)
    rows = sm.r1 - sm.r0
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    y_full = torch.empty(m, dtype=torch.float32, device=dev)

    # N > 1: the all-gather rides on the multiply's own stores into every
    # rank's symmetric-memory output (--gather peer, rsr_matvec_peers) plus
    # one barrier; NCCL all-gather + reassembly if that is unavailable
    gather = "none"
    if world > 1:
        gather = args.gather
        if os.environ.get("RSR_BENCH_ONE_DEVICE"):
            gather = "nccl"  # ranks sharing one GPU must not spin on each other's barrier
        if gather == "peer":
            ok = 1
            try:
                sm.gather = "peer"
                pst = sm._peer_state(torch.float32)
            except Exception as e:  # all ranks fall back together
                print(f"[bench] symmetric-memory gather unavailable: {e}", file=sys.stderr)
                ok = 0
            okt = torch.tensor([ok], dtype=torch.int32, device=dev)
            dist.all_reduce(okt, op=dist.ReduceOp.MIN)
            if not int(okt.item()):
                gather, sm.gather = "nccl", "nccl"
    if gather == "peer":
        def step(i, sp=None):
            y, h, prow = pst["bufs"][i & 1]
            kn.matvec_peers_into(a, vt, prow, world, view=views[i % ncopies],
                                 stream=sptr if sp is None else sp)
            h.barrier(channel=0)  # every rank's rows are in y (row order)
    else:
        def step(i, sp=None):
            kn.matvec_into(a, vt, y_local[:rows], view=views[i % ncopies],
                           stream=sptr if sp is None else sp)
            if world > 1:
                dist.all_gather_into_tensor(y_all, y_local)
                torch.index_select(y_all, 0, sm.index, out=y_full)  # full y in row order

    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    if gather == "peer":
        # one-time check against the NCCL gather; every rank falls back
        # together if any rank's peer-gathered output differs
        y_peer = pst["bufs"][(warmup - 1) & 1][0].clone()
        kn.matvec_into(a, vt, y_local[:rows], view=views[0], stream=sptr)
        dist.all_gather_into_tensor(y_all, y_local)
        torch.index_select(y_all, 0, sm.index, out=y_full)
        okt = torch.tensor([int(torch.equal(y_peer, y_full))], dtype=torch.int32, device=dev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        if not int(okt.item()):
            print("[bench] peer gather differs from NCCL: using NCCL", file=sys.stderr)
            gather, sm.gather = "nccl_fallback", "nccl"

            def step(i, sp=None):
                kn.matvec_into(a, vt, y_local[:rows], view=views[i % ncopies],
                               stream=sptr if sp is None else sp)
                dist.all_gather_into_tensor(y_all, y_local)
                torch.index_select(y_all, 0, sm.index, out=y_full)
        torch.cuda.synchronize()

    # per-launch kernel durations (CUDA events on the launching stream)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(min(args.steps, 100))]
    for i, (e0, e1) in enumerate(kev):
        e0.record(stream)
        kn.matvec_into(a, vt, y_local[:rows], view=views[i % ncopies], stream=sptr)
        e1.record(stream)
    torch.cuda.synchronize()
    kernel_ms = float(np.median([e0.elapsed_time(e1) for e0, e1 in kev]))

    # ---- timed region: exactly K steps, queued behind a device spin (or, with
    # --graph on one GPU, captured as one CUDA graph and replayed once)
    use_graph = world == 1 and args.graph
    graph = None
    if use_graph:
        gstream = torch.cuda.Stream(dev)
        gstream.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(gstream):
            for i in range(args.steps):  # warm the capture stream's path
                step(i, gstream.cuda_stream)
            gstream.synchronize()
            with torch.cuda.graph(graph, stream=gstream):
                for i in range(args.steps):
                    step(i, gstream.cuda_stream)
        stream.wait_stream(gstream)
        for _ in range(max(1, warmup // max(1, args.steps))):
            graph.replay()
        torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t_load = time.perf_counter()  # untimed load while the sampler starts
        while time.perf_counter() - t_load < 0.3:
            for i in range(20):
                step(i)
            torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        if use_graph:
            start.record(stream)
            graph.replay()
            end.record(stream)
        else:
            torch.cuda._sleep(spin_cycles(args.steps))
            start.record(stream)
            for i in range(args.steps):
                step(i)
            end.record(stream)
        torch.cuda.synchronize()
        t_hold = time.perf_counter()  # keep the GPU loaded for the sampler (untimed)
        while time.perf_counter() - t_hold < 0.5:
            for i in range(50):
                step(i)
            torch.cuda.synchronize()
    if dist:
        dist.barrier()
    total_ms = start.elapsed_time(end)
    if dist:
        tt = torch.tensor([total_ms, kernel_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms, kernel_ms = (float(x) for x in tt.tolist())
    ms_per_step = total_ms / args.steps
    value = 1e3 / ms_per_step  # whole-job matvecs/s (each step = one full matvec)

    # ---- e2e through the public API with host buffers (rank 0, 1 GPU)
    e2e = None
    if rank == 0 and world == 1:
        def host_rate(vh):
            for _ in range(5):
                rsr.rsr_matvec(a, vh)
            torch.cuda.synchronize()
            ne = max(20, min(args.steps, 200))
            t0 = time.perf_counter()
            for _ in range(ne):
                yh = rsr.rsr_matvec(a, vh)
            return ne / (time.perf_counter() - t0), yh
        # the step's input in pinned host memory, in the workload's vector
        # dtype: a bf16 tensor for bf16 configs (numpy has no bf16), numpy
        # float32 otherwise -- the reference's own call, timed beside it
        vh32 = torch.from_numpy(vf.copy()).pin_memory().numpy()
        rate32, yh = host_rate(vh32)
        if cfg["vdtype"] == "bf16":
            vhb = torch.from_numpy(vf.copy()).to(torch.bfloat16).pin_memory()
            rate, yh = host_rate(vhb)
            vin_bytes = vhb.numel() * 2
            api = ("paper_2603_27462_b200.rsr_matvec(artifact, bf16 vector in pinned host "
                   "memory) -> numpy float32")
        else:
            rate, vin_bytes = rate32, vh32.nbytes
            api = ("paper_2603_27462_b200.rsr_matvec(artifact, numpy float32 vector in "
                   "pinned memory) -> numpy float32")
        e2e = {"value": rate, "unit": UNIT, "h2d_bytes_per_step": int(vin_bytes),
               "d2h_bytes_per_step": int(yh.nbytes), "api": api,
               "numpy_f32": {"value": rate32, "h2d_bytes_per_step": int(vh32.nbytes),
                             "api": "rsr_matvec(artifact, numpy float32 vector, pinned): "
                                    "the float32 kernel"}}
    elif world > 1:
        # sharded: every rank takes the host vector (pinned) to its GPU, runs
        # ShardedMatrix.matvec (local multiply + all-gather + reassembly) and
        # reads the full result back to the host; max over ranks
        vh = torch.from_numpy(vf.copy()).pin_memory()
        if cfg["vdtype"] == "bf16":
            vh = vh.to(torch.bfloat16).pin_memory()
        vd = torch.empty_like(vh, device=dev)
        yh = torch.empty(m, dtype=torch.float32).pin_memory()
        bufs = sm.buffers(torch.float32)

        def e2e_step():
            vd.copy_(vh, non_blocking=True)
            yh.copy_(sm.matvec(vd, buffers=bufs), non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
        for _ in range(5):
            e2e_step()
        dist.barrier()
        ne = max(10, min(args.steps, 50))
        t0 = time.perf_counter()
        for _ in range(ne):
            e2e_step()
        tt = torch.tensor([(time.perf_counter() - t0) / ne], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
        e2e = {"value": 1.0 / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(vh.numel() * vh.element_size()),
               "d2h_bytes_per_step": int(yh.numel() * 4),
               "api": "shard.ShardedMatrix.matvec on every rank: pinned host vector -> device, "
                      + ("multiply storing into every rank's symmetric-memory output + barrier"
                         if gather == "peer" else "local multiply + NCCL all-gather + reassembly")
                      + ", full y -> pinned host; "
                      "max over ranks"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    hbm, peak_kind = peaks()
    vbytes = 2 if cfg["vdtype"] == "bf16" else 4
    local_alg = (a.file_bytes() - 24) + n * vbytes + rows * 4
    # average launch duration over the timed region: one multiply per step at
    # N=1 (back-to-back launches overlap prologue and tail via PDL); with a
    # collective in the step, the separately timed per-launch duration
    launch_ms = ms_per_step if world == 1 else kernel_ms
    achieved = local_alg / (launch_ms * 1e-3) / 1e9
    own = sb + n * vbytes + rows * 4
    traffic, traffic_note = None, "skipped (--no-extras)"
    if world == 1 and not args.no_extras:
        tr, err = measure_traffic(cname, k)
        if tr is not None:
            traffic = tr["bytes"]
            traffic_note = (f"ncu child process (dram__bytes_read.sum {tr['read']} + "
                            f"dram__bytes_write.sum {tr['write']}) on the 3rd launch of "
                            f"rsr_mv_kernel, caches flushed; ncu duration {tr['ncu_us']} us")
        else:
            traffic_note = err
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_note,
            "peak_kind": peak_kind,
            "algorithmic_bytes": int(local_alg), "stream_bytes": int(own),
            "achieved_own_bytes_gbs": own / (launch_ms * 1e-3) / 1e9,
            "launch_us": launch_ms * 1e3,
            "isolated_kernel_us": kernel_ms * 1e3, "frac_of_8TBs_nominal": achieved / 8000.0,
            "note": "per rank (rank 0's shard) when sharded"}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        val, threads, nn_, el, sample = cpu_reference_run(cfg, 0, 1, seconds=args.cpu_seconds)
        cpu = {"value": val, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample}

    extras = {}
    if world == 1 and not args.no_extras:
        for name, fn in (("cublas_bf16", lambda: cublas_bf16_bench(full_packed, m, n, vt, hbm,
                                                                     value)
                          if full_packed is not None and cfg["vdtype"] == "bf16" else None),
                         ("c4", c4_bench),
                         ("c1", lambda: side_config_bench("c1", hbm)),
                         ("c5_1gpu", lambda: side_config_bench("c5", hbm))):
            try:
                extras[name] = fn()
            except Exception as e:  # reported, never silently replaced
                extras[name] = {"error": repr(e)[:300]}
    if world > 1 and not args.no_extras:
        # the same matrix on rank 0's GPU alone, in this run: the N = 1 point
        # of this strong-scaling line (the N = 1 bench line is C2, the headline)
        try:
            c5 = side_config_bench(cname, hbm)
            extras["c5_1gpu"] = c5
            extras["scaling_vs_1gpu_same_run"] = {
                "one_gpu_matvec_s": c5["matvec_s"], "n_gpus": world,
                "speedup": value / c5["matvec_s"],
                "efficiency": value / c5["matvec_s"] / world,
                "note": "whole-job matvec/s of this sharded run over rank 0's GPU alone on the "
                        "unsharded matrix (same process, same box)"}
        except Exception as e:  # reported, never silently replaced
            extras["c5_1gpu"] = {"error": repr(e)[:300]}

    decode = None
    if world == 1 and not args.no_decode:
        try:
            decode = decode_bench()
        except Exception as e:  # reported, never silently replaced
            decode = {"error": repr(e)[:300]}

    launches_per_step = 1 + (1 if tc > 1 else 0)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config,
            "l2_copies": f"{ncopies} stream copies ({sb / 1e6:.1f} MB each, L2 {l2 / 1e6:.0f} MB)",
            "timing": ("the K steps as one CUDA-graph replay (captured launches, PDL edges kept)"
                       if use_graph else "K launches queued behind a device spin")
                      + "; CUDA events on the launch stream; max over ranks",
            "preprocess_ms": preprocess_ms, "preprocess_cold_ms": preprocess_cold_ms,
            "preprocess_note": "host matrix in -> device artifact + chunk stream, wall clock; "
                               "cold = first full-size call of the process, preprocess_ms = "
                               "the same call again (warm allocator)",
            "gpu_launches": args.steps * launches_per_step,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e}
    if world > 1:
        line["gather"] = gather
    line.update(extras)
    line["decode"] = decode
    line["clocks"] = clk.summary()
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
