"""Generate golden vectors by importing the REFERENCE package (rsrmv).

Run in the build container only (the reference lives at /root/reference and
does not travel to the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes, next to this script:
  * small_cases.npz   -- full artifacts + multiply outputs for small seeded
                         shapes (both bitwidths, ragged blocks, multi-tile,
                         all-zero, known-answer matrices);
  * golden.json       -- per-case metadata, known-answer values (2x4
                         oracle, GOLDEN .rsra bytes, fused known values) and
                         sha256 digests of artifacts/outputs for the BASELINE
                         configs (C1 binary 4096^2 k=8, C2 ternary 16384^2
                         k=4..6, C4 ternary 8192^2 k=5), op totals, file_bytes;
  * large_outputs.npz -- the reference's multiply outputs at those sizes.
Inputs are regenerated bit-identically by oracle.rsr_oracle.random_matrix /
random_vector (same numpy generators as reference bench.py:102-117).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from rsrmv import _native, bench, kernels, matcore, preproc  # noqa: E402
from rsrmv import artifact_io  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def int_vector(n, seed):
    return np.random.default_rng(seed).integers(-128, 128, n).astype(np.int8)


def bf16_round(v: np.ndarray) -> np.ndarray:
    """Round float32 to bfloat16 (RNE) and back, as torch does on device."""
    b = v.astype(np.float32).view(np.uint32).astype(np.uint64)
    lsb = (b >> 16) & 1
    b = ((b + 0x7FFF + lsb) >> 16) << 16
    return b.astype(np.uint32).view(np.float32)


SMALL = [
    # (m, n, bitwidth, k, tile_width, seed, density, weight_scale)
    (1, 1, "binary", 1, None, 1, 0.5, 1.0),
    (1, 1, "ternary", 1, None, 2, 0.5, 1.0),
    (2, 4, "binary", 2, None, 0, 0.5, 1.0),
    (7, 33, "binary", 3, None, 3, 0.5, 1.0),
    (13, 100, "ternary", 4, None, 4, 0.5, 0.37),
    (57, 301, "ternary", 5, 100, 5, 0.5, 1.0),
    (60, 200, "binary", 9, 48, 6, 0.5, 1.0),
    (64, 256, "binary", 8, None, 7, 0.3, 0.25),
    (40, 130, "ternary", 6, 48, 8, 0.5, 0.5),
    (33, 517, "ternary", 7, None, 9, 0.8, 1.0),
    (16, 64, "binary", 16, None, 10, 0.5, 1.0),
    (20, 90, "ternary", 10, None, 11, 0.5, 1.0),
    (12, 40, "ternary", 3, None, 12, 0.0, 1.0),      # all-zero matrix
    (9, 70, "binary", 4, None, 13, 1.0, 1.0),        # all-ones
    (512, 2048, "ternary", 6, None, 14, 0.5, 0.8),
    (256, 1024, "binary", 8, None, 15, 0.5, 1.0),
    (16, 70000, "binary", 8, None, 16, 0.5, 1.0),    # 3 tiles of 32768
    (10, 40000, "ternary", 5, None, 17, 0.5, 1.0),   # one 40000-wide tile
    (128, 1000, "ternary", 2, 256, 18, 0.69, 0.02),
]


def packed_for(m, n, bw, seed, density, ws):
    p = bench.random_matrix(m, n, bw, seed, density)
    if ws != 1.0:
        p = matcore.PackedMatrix(p.rows, p.cols, p.bitwidth, p.data, ws)
    return p


def small_cases():
    out = {}
    meta = []
    for i, (m, n, bw, k, tw, seed, dens, ws) in enumerate(SMALL):
        p = packed_for(m, n, bw, seed, dens, ws)
        a = preproc.preprocess(p, k, tile_width=tw)
        vi = int_vector(n, seed)
        vf = bench.random_vector(n, seed)
        pre = f"c{i}_"
        out[pre + "data"] = p.data
        out[pre + "words"] = a.words
        out[pre + "perm"] = a.perm
        out[pre + "go"] = a.group_offsets
        out[pre + "po"] = a.perm_offsets
        out[pre + "steps"] = a.sort_steps
        out[pre + "vi"] = vi
        out[pre + "vf"] = vf
        out[pre + "y_i8"] = kernels.rsr_matvec(a, vi)
        out[pre + "y_f32"] = kernels.rsr_matvec(a, vf)
        out[pre + "naive_f64"] = matcore.naive_matvec(p, vf)
        out[pre + "naive_i32"] = matcore.naive_matvec(p, vi)
        if bw == "ternary":
            out[pre + "fused"] = kernels.rsr_matvec_fused(a, vf)
            out[pre + "fused_mul"] = kernels.Multiplier(kernels.RSR_TERNARY, p, k=k,
                                                        tile_width=tw).multiply(vf)
        q = matcore.quantize_activations(vf)
        out[pre + "q"] = q.values
        meta.append(dict(idx=i, m=m, n=n, bitwidth=bw, k=k, tile_width=tw, seed=seed,
                         density=dens, weight_scale=ws, file_bytes=a.file_bytes(),
                         op_totals=list(a.op_totals()), q_scale=q.scale,
                         plan=[a.plan.block_count, a.plan.tile_count, a.plan.tile_width,
                               a.plan.last_block_height]))
    # known-answer matrices from the reference tests
    ka = {}
    m2x4 = matcore.encode(np.array([[1, 0, 1, 0], [1, 1, 0, 0]], np.int8), 2, 4, "binary")
    a = preproc.preprocess(m2x4, 2)
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        fp = os.path.join(td, "g.rsra")
        artifact_io.save(a, fp)
        ka["golden_rsra_hex"] = open(fp, "rb").read().hex()
    ka["perm_2x4"] = [int(x) for x in a.perm]
    ka["words_2x4"] = [int(x) for x in a.words]
    ka["ops_2x4"] = list(a.op_totals())
    mt = matcore.PackedMatrix(2, 3, "ternary", matcore.encode(
        np.array([[1, -1, 0], [0, 1, 1]], np.int8), 2, 3, "ternary").data, 0.5)
    at = preproc.preprocess(mt, 2)
    fused = kernels.rsr_matvec_fused(at, np.array([2.0, 3.0, 5.0], np.float32))
    ka["fused_known"] = [float(x) for x in fused]
    ka["fused_known_bits"] = [int(x) for x in fused.view(np.uint32)]
    return out, meta, ka


LARGE = [
    # (name, m, n, bitwidth, k, seed)
    ("C1_binary_4096_k8", 4096, 4096, "binary", 8, 0),
    ("C2_ternary_16384_k4", 16384, 16384, "ternary", 4, 0),
    ("C2_ternary_16384_k5", 16384, 16384, "ternary", 5, 0),
    ("C2_ternary_16384_k6", 16384, 16384, "ternary", 6, 0),
    ("C4_ternary_8192_k5", 8192, 8192, "ternary", 5, 0),
]


def large_cases():
    meta = {}
    outs = {}
    for name, m, n, bw, k, seed in LARGE:
        p = bench.random_matrix(m, n, bw, seed)
        a = preproc.preprocess(p, k)
        vf = bench.random_vector(n, seed)
        vb = bf16_round(vf)
        vi = int_vector(n, seed)
        y_f = kernels.rsr_matvec(a, vb)
        y_i = kernels.rsr_matvec(a, vi)
        rec = dict(m=m, n=n, bitwidth=bw, k=k, seed=seed,
                   data_sha=sha(p.data), words_sha=sha(a.words), perm_sha=sha(a.perm),
                   go_sha=sha(a.group_offsets), po_sha=sha(a.perm_offsets),
                   steps_sha=sha(a.sort_steps),
                   n_words=int(a.words.size), n_perm=int(a.perm.size),
                   file_bytes=a.file_bytes(), op_totals=list(a.op_totals()),
                   y_i8_sha=sha(y_i))
        outs[name + "_y_bf16v"] = y_f
        outs[name + "_y_i8"] = y_i
        if bw == "ternary":
            y_fused = kernels.rsr_matvec_fused(a, vb)
            outs[name + "_fused_bf16v"] = y_fused
            rec["fused_sha"] = sha(y_fused)
        meta[name] = rec
        print(name, rec["file_bytes"], rec["op_totals"], flush=True)
    return meta, outs


def main():
    _native.warmup()
    out, meta, ka = small_cases()
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **out)
    lmeta, louts = large_cases()
    np.savez_compressed(os.path.join(HERE, "large_outputs.npz"), **louts)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump({"small": meta, "known_answer": ka, "large": lmeta,
                   "reference": "rsrmv @ /root/reference/pkg (numba)"}, f, indent=1)


if __name__ == "__main__":
    main()
