"""Loader for the committed golden vectors (tests/golden/)."""

from __future__ import annotations

import hashlib
import json
import os
from functools import lru_cache

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@lru_cache(maxsize=None)
def meta() -> dict:
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        return json.load(f)


@lru_cache(maxsize=None)
def _small():
    return dict(np.load(os.path.join(GOLDEN_DIR, "small_cases.npz")))


@lru_cache(maxsize=None)
def _large():
    return dict(np.load(os.path.join(GOLDEN_DIR, "large_outputs.npz")))


def small_case(i: int) -> dict:
    s = _small()
    pre = f"c{i}_"
    d = {k[len(pre):]: v for k, v in s.items() if k.startswith(pre)}
    d["meta"] = meta()["small"][i]
    return d


def n_small() -> int:
    return len(meta()["small"])


def large_output(name: str) -> np.ndarray:
    return _large()[name]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bf16_round(v: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 (round to nearest even) -> float32."""
    b = np.asarray(v, np.float32).view(np.uint32).astype(np.uint64)
    lsb = (b >> 16) & 1
    b = ((b + 0x7FFF + lsb) >> 16) << 16
    return b.astype(np.uint32).view(np.float32)


def int_vector(n, seed):
    return np.random.default_rng(seed).integers(-128, 128, n).astype(np.int8)
