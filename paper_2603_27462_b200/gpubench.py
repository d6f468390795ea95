"""GPU benchmark harness, k sweep and bytes-based autotuner (SURVEY.md
section 8f, rank 2).

Mirrors the reference harness (pkg/src/rsrmv/bench.py:32-34, 142-274): the
same BenchReport JSON/CSV schema (ROW_FIELDS) so the reference dashboard can
render GPU runs, the same seeded generators, and an autotuner that prunes
candidate k with a cost model and then picks by measured latency.  Two
things change on the GPU:

* time is device time (CUDA events around each launch) -- ``ns_*`` fields
  are kernel nanoseconds, not host wall clock;
* the cost model counts BYTES, not adds: the multiply streams its artifact
  from HBM once, so the model is the expected reference artifact size
  2*retained + 8*groups + 8*cells (= file_bytes - 24), and candidates are the
  k within 25% of the cheapest.
"""

from __future__ import annotations

import csv
import io
import json
import math
import time
from dataclasses import dataclass, field

import numpy as np

from .errors import RsrError
from .matcore import BINARY, TERNARY, PackedMatrix, encode
from .preproc import K_CAP, preprocess

ROW_FIELDS = ("kind", "m", "n", "bitwidth", "k", "ns_median", "ns_p10",
              "ns_p90", "gather_adds", "scatter_adds", "preprocess_ms",
              "artifact_bytes", "best_k", "env")
DEFAULT_DENSITY = 0.5
CUBLAS_BF16 = "cublas_bf16"   # dense bf16 GEMV baseline (torch.mv -> cuBLAS)


@dataclass
class BenchConfig:
    m: int
    n: int
    bitwidth: str
    k_list: list[int] = field(default_factory=lambda: [4, 5, 6, 7, 8])
    reps: int = 50
    warmup: int = 5
    seed: int = 0
    density: float = DEFAULT_DENSITY
    tile_width: int | None = None
    vector_dtype: str = "bfloat16"   # float32 | bfloat16 | int8
    baselines: tuple[str, ...] = (CUBLAS_BF16,)

    def __post_init__(self):
        if self.reps < 1:
            raise ValueError("reps must be at least 1")
        if self.warmup < 0:
            raise ValueError("warmup cannot be negative")
        if not 0.0 <= self.density <= 1.0:
            raise ValueError("density must lie in [0, 1]")
        if self.bitwidth not in (BINARY, TERNARY):
            raise ValueError(f"bitwidth must be {BINARY!r} or {TERNARY!r}")
        if self.vector_dtype not in ("float32", "bfloat16", "int8"):
            raise ValueError("vector_dtype must be float32, bfloat16 or int8")
        bad = set(self.baselines) - {CUBLAS_BF16}
        if bad:
            raise ValueError(f"unknown baselines {sorted(bad)}")


@dataclass
class BenchReport:
    rows: list[dict]
    errors: list[dict]
    best_k: int | None
    env: dict

    def to_json(self, indent: int | None = 2) -> str:
        return json.dumps({"env": self.env, "best_k": self.best_k,
                           "rows": self.rows, "errors": self.errors}, indent=indent)

    def to_csv(self) -> str:
        buf = io.StringIO()
        w = csv.DictWriter(buf, fieldnames=ROW_FIELDS)
        w.writeheader()
        for r in self.rows:
            flat = dict(r)
            flat["best_k"] = self.best_k
            flat["env"] = json.dumps(self.env)
            w.writerow(flat)
        return buf.getvalue()


def random_matrix(m: int, n: int, bitwidth: str, seed: int,
                  density: float = DEFAULT_DENSITY) -> PackedMatrix:
    """The reference generator (bench.py:102-113): i.i.d. entries, density =
    nonzero probability (ternary +1 and -1 equally likely)."""
    rng = np.random.default_rng(seed)
    if bitwidth == BINARY:
        ent = (rng.random((m, n)) < density).astype(np.int8)
    else:
        u = rng.random((m, n))
        ent = np.zeros((m, n), np.int8)
        ent[u < density / 2] = 1
        ent[u > 1 - density / 2] = -1
    return encode(ent, m, n, bitwidth)


def random_vector(n: int, seed: int) -> np.ndarray:
    """The reference generator (bench.py:116-117)."""
    return np.random.default_rng(seed ^ 0x5EED).standard_normal(n).astype(np.float32)


def gpu_env() -> dict:
    import torch
    p = torch.cuda.get_device_properties(torch.cuda.current_device())
    return {"gpu": p.name, "sm_count": p.multi_processor_count,
            "hbm_gb": round(p.total_memory / 2**30, 1), "timer": "cuda_events"}


def bytes_model(m: int, n: int, k: int, bitwidth: str,
                density: float = DEFAULT_DENSITY, tile_width: int | None = None) -> float:
    """Expected bytes one multiply streams: the reference artifact body
    2*retained + 8*groups + 8*cells (+ pad), under i.i.d. entries and
    uniformly occupied patterns (same occupancy argument as the reference
    cost_model, bench.py:205-229, but weighted in bytes)."""
    if not 0.0 <= density <= 1.0:
        raise ValueError("density must lie in [0, 1]")
    tw = tile_width or (n if n <= 65536 else 32768)
    blocks = math.ceil(m / k)
    tiles = math.ceil(n / tw)
    z = 1.0 - density
    u = 1.0 - z ** k
    total = 0.0
    for t in range(tiles):
        tn = min(tw, n - t * tw)
        retained = tn * u
        buckets_nz = (2 ** k if bitwidth == BINARY else 3 ** k) - 1
        groups = buckets_nz * (1.0 - (1.0 - 1.0 / buckets_nz) ** retained) if buckets_nz else 0.0
        total += blocks * (8 + 8 * groups + 2 * retained + 1)  # +1: mean pad
    return total


def _vector(n, seed, dtype, device):
    import torch
    if dtype == "int8":
        return torch.from_numpy(np.random.default_rng(seed).integers(-128, 128, n).astype(
            np.int8)).to(device)
    v = torch.from_numpy(random_vector(n, seed)).to(device)
    return v.to(torch.bfloat16) if dtype == "bfloat16" else v


def _time_device(fn, reps: int, warmup: int) -> tuple[float, float, float]:
    """Median / p10 / p90 device nanoseconds of fn() (one CUDA event pair each)."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for e0, e1 in ev:
        e0.record()
        fn()
        e1.record()
    torch.cuda.synchronize()
    s = np.array([e0.elapsed_time(e1) * 1e6 for e0, e1 in ev])
    return float(np.median(s)), float(np.percentile(s, 10)), float(np.percentile(s, 90))


def run_bench(cfg: BenchConfig) -> BenchReport:
    """Sweep k over one seeded matrix on the GPU and time the baselines on the
    same inputs (reference bench.py:142-202).  A k that fails produces an
    entry in report.errors; the rest still run."""
    import torch
    from .kernels import matvec_into
    dev = torch.device("cuda", torch.cuda.current_device())
    env = gpu_env()
    env["vector_dtype"] = cfg.vector_dtype
    matrix = random_matrix(cfg.m, cfg.n, cfg.bitwidth, cfg.seed, cfg.density)
    v = _vector(cfg.n, cfg.seed, cfg.vector_dtype, dev)
    ydt = torch.int32 if cfg.vector_dtype == "int8" else torch.float32
    y = torch.empty(cfg.m, dtype=ydt, device=dev)
    rows, errors = [], []
    for k in cfg.k_list:
        try:
            torch.cuda.synchronize()
            t0 = time.perf_counter_ns()
            a = preprocess(matrix, k, cfg.tile_width, device=dev)
            torch.cuda.synchronize()
            pre_ms = (time.perf_counter_ns() - t0) / 1e6
            med, p10, p90 = _time_device(lambda: matvec_into(a, v, y), cfg.reps, cfg.warmup)
            g, sc, _ = a.op_totals()
            rows.append({"kind": "rsr", "m": cfg.m, "n": cfg.n, "bitwidth": cfg.bitwidth,
                         "k": k, "ns_median": med, "ns_p10": p10, "ns_p90": p90,
                         "gather_adds": g, "scatter_adds": sc, "preprocess_ms": pre_ms,
                         "artifact_bytes": a.file_bytes()})
            del a
        except RsrError as e:
            errors.append({"k": k, "error": e.kind, "message": str(e)})
    for kind in cfg.baselines:
        from .matcore import dense_device
        t0 = time.perf_counter_ns()
        W = dense_device(matrix, dev).to(torch.bfloat16)
        torch.cuda.synchronize()
        pre_ms = (time.perf_counter_ns() - t0) / 1e6
        vb = v.to(torch.bfloat16)
        med, p10, p90 = _time_device(lambda: torch.mv(W, vb), cfg.reps, cfg.warmup)
        rows.append({"kind": kind, "m": cfg.m, "n": cfg.n, "bitwidth": cfg.bitwidth,
                     "k": None, "ns_median": med, "ns_p10": p10, "ns_p90": p90,
                     "gather_adds": cfg.m * cfg.n, "scatter_adds": 0, "preprocess_ms": pre_ms,
                     "artifact_bytes": cfg.m * cfg.n * 2})
        del W
    rsr_rows = [r for r in rows if r["kind"] == "rsr"]
    best_k = min(rsr_rows, key=lambda r: (r["ns_median"], r["k"]))["k"] if rsr_rows else None
    for r in rows:
        r["best_k"] = best_k
        r["env"] = env
    return BenchReport(rows, errors, best_k, env)


def feasible_k(bitwidth: str) -> range:
    return range(1, K_CAP[bitwidth] + 1)


def autotune_k(m: int, n: int, bitwidth: str, budget_ms: float = 2000.0, seed: int = 0,
               density: float = DEFAULT_DENSITY, matrix: PackedMatrix | None = None,
               vector_dtype: str = "bfloat16") -> int:
    """Pick the block height with the lowest measured GPU multiply time
    (reference bench.py:236-274 with a bytes model): candidates are the
    feasible k whose modelled bytes are within 25% of the minimum; each is
    preprocessed on the device and timed round-robin until the budget runs
    out (at least one timed batch each).  Ties break toward smaller k."""
    import torch
    from .kernels import matvec_into
    costs = {k: bytes_model(m, n, k, bitwidth, density) for k in feasible_k(bitwidth)}
    floor = min(costs.values())
    candidates = [k for k, c in costs.items() if c <= 1.25 * floor]
    dev = torch.device("cuda", torch.cuda.current_device())
    if matrix is None:
        matrix = random_matrix(m, n, bitwidth, seed, density)
    v = _vector(n, seed, vector_dtype, dev)
    y = torch.empty(m, dtype=torch.int32 if vector_dtype == "int8" else torch.float32, device=dev)
    arts = {k: preprocess(matrix, k, device=dev) for k in candidates}
    samples = {k: [] for k in candidates}
    deadline = time.perf_counter_ns() + budget_ms * 1e6
    for _ in range(20):
        for k in candidates:
            med, _, _ = _time_device(lambda: matvec_into(arts[k], v, y), 10, 2)
            samples[k].append(med)
        if time.perf_counter_ns() >= deadline:
            break
    medians = {k: float(np.median(s)) for k, s in samples.items()}
    return min(candidates, key=lambda k: (medians[k], k))
