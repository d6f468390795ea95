"""Golden vectors for float64 activations, made by importing the REFERENCE
package (rsrmv) in the build container (quantize_activations and
the NaiveI8 multiplier on float64 input must keep the float64 values):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_quantize_golden.py

Writes quantize_f64.npz next to this script: for each case i, v{i} (float64
input), q{i} / scale{i} (rsrmv.matcore.quantize_activations), and for the
ternary matrix of random_matrix(40, n, ternary, i) with k=4 and weight_scale
0.37: naive{i} = Multiplier(NaiveI8).multiply(v) and fused{i} =
Multiplier(RsrTernary).multiply(v) (the fused path casts v to float32 first,
reference kernels.py:119).
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from rsrmv import bench, kernels, matcore  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
out = {}
for i, n in enumerate([1, 7, 100, 1000, 4096]):
    rng = np.random.default_rng(1000 + i)
    v = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4)
    v[rng.integers(0, n)] = 0.5 * (1 + 2 * rng.integers(0, 50)) / 127.0 * np.max(np.abs(v))
    qv = matcore.quantize_activations(v)
    out[f"v{i}"] = v
    out[f"q{i}"] = qv.values
    out[f"scale{i}"] = np.float64(qv.scale)
    mat = bench.random_matrix(40, n, matcore.TERNARY, i)
    mat = matcore.PackedMatrix(mat.rows, mat.cols, mat.bitwidth, mat.data, 0.37)
    out[f"data{i}"] = mat.data
    out[f"naive{i}"] = kernels.Multiplier(kernels.NAIVE_I8, mat).multiply(v)
    out[f"fused{i}"] = kernels.Multiplier(kernels.RSR_TERNARY, mat, k=4).multiply(v)
np.savez_compressed(os.path.join(HERE, "quantize_f64.npz"), **out)
print("wrote", len(out), "arrays")
