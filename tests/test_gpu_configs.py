"""GPU parity at the BASELINE configs and edge inputs (VERDICT r1 "pin every
config"):

* C1 binary 4096^2, k=8, full size: the int path equals the reference's
  committed output bit for bit; the float path (bf16-valued and float32
  vectors) meets the stated tolerance against the reference float path.
* C4 ternary 8192^2, k=5, full size: int / fused bit-exact vs the reference
  outputs, float within tolerance.
* C5 ternary 131072 columns: sampled row strips of the device generator
  (the full matrix does not fit the host) preprocessed and multiplied on the
  GPU against the CPU oracle on the same strips (its C restatement of the
  generator), bit-exact artifacts and int/fused outputs.
* Non-finite activations: NaN / +-Inf in the vector give exactly the
  reference's NaN / Inf pattern (y += sgn * s, so 0 * NaN poisons the block).
* float64 activations: quantize_activations and the NaiveI8 / RsrTernary
  multipliers equal the reference on float64 input (golden vectors made by
  the reference, tests/golden/make_quantize_golden.py).
"""

import os

import numpy as np
import pytest

from oracle import rsr_oracle as orc
from tests import golden_data as gd

pytestmark = pytest.mark.gpu

RTOL = 1e-6


@pytest.fixture(scope="module")
def rsr():
    import torch
    import paper_2603_27462_b200 as pkg
    torch.cuda.set_device(0)
    return pkg


def float_ok(y, ref, dense_abs, v):
    cond = dense_abs @ np.abs(np.asarray(v, np.float64))
    return np.abs(y.astype(np.float64) - ref) <= RTOL * cond + RTOL * np.abs(ref)


def test_c1_binary_4096_k8_full_size(rsr):
    import torch
    name = "C1_binary_4096_k8"
    rec = gd.meta()["large"][name]
    p = orc.random_matrix(4096, 4096, "binary", 0)
    assert gd.sha(p.data) == rec["data_sha"]
    a = rsr.preprocess(rsr.PackedMatrix(4096, 4096, "binary", p.data), 8)
    assert gd.sha(a.words) == rec["words_sha"] and gd.sha(a.perm) == rec["perm_sha"]
    assert a.file_bytes() == rec["file_bytes"]
    vi = gd.int_vector(4096, 0)
    yi = rsr.rsr_matvec(a, vi)
    assert np.array_equal(yi, gd.large_output(name + "_y_i8"))
    dense_abs = np.abs(orc.decode(p)).astype(np.float64)
    ref_a = orc.preprocess(p, 8)
    # bf16-valued vector on the device (the committed reference output)
    vf = orc.random_vector(4096, 0)
    vb = torch.from_numpy(vf).cuda().to(torch.bfloat16)
    y = rsr.rsr_matvec(a, vb).cpu().numpy()
    vr = gd.bf16_round(vf)
    yr = orc.matvec_f64(ref_a, vr, threads=8)
    assert float_ok(y, yr, dense_abs, vr).all()
    # the reference's own float32 output agrees with the f64 sums to 1 ulp
    assert np.allclose(gd.large_output(name + "_y_bf16v"), yr.astype(np.float32), rtol=1e-6,
                       atol=1e-6)
    # the C1 workload's float32 vector through the numpy API
    y32 = rsr.rsr_matvec(a, vf)
    assert y32.dtype == np.float32
    assert float_ok(y32, orc.matvec_f64(ref_a, vf, threads=8), dense_abs, vf).all()


def test_c4_ternary_8192_k5_full_size(rsr):
    import torch
    name = "C4_ternary_8192_k5"
    rec = gd.meta()["large"][name]
    p = orc.random_matrix(8192, 8192, "ternary", 0)
    a = rsr.preprocess(rsr.PackedMatrix(8192, 8192, "ternary", p.data), 5)
    assert gd.sha(a.words) == rec["words_sha"] and gd.sha(a.perm) == rec["perm_sha"]
    assert np.array_equal(rsr.rsr_matvec(a, gd.int_vector(8192, 0)),
                          gd.large_output(name + "_y_i8"))
    vf = orc.random_vector(8192, 0)
    vb = torch.from_numpy(vf).cuda().to(torch.bfloat16)
    assert np.array_equal(rsr.rsr_matvec_fused(a, vb).cpu().numpy(),
                          gd.large_output(name + "_fused_bf16v"))
    vr = gd.bf16_round(vf)
    y = rsr.rsr_matvec(a, vb).cpu().numpy()
    yr = orc.matvec_f64(orc.preprocess(p, 5), vr, threads=8)
    assert float_ok(y, yr, np.abs(orc.decode(p)).astype(np.float64), vr).all()


@pytest.mark.parametrize("strip,tw", [(0, None), (1, None), (2, 32704), (3, 32704), (4, 16384)])
def test_c5_sampled_strips_vs_oracle(rsr, strip, tw):
    """C5 (ternary 131072 columns, k=6): random row strips of the device
    generator vs the oracle's restatement of it, at the reference's default
    tiles (4 x 32768, format 0), the widest halfword-format tiles (32704: 5
    tiles, the last 256 columns) and the bench's 8 x 16384."""
    import torch
    from paper_2603_27462_b200.devicepack import random_ternary_device
    n, k, rows = 131072, 6, 36
    rng = np.random.default_rng(500 + strip)
    row0 = int(rng.integers(0, 131072 // k - rows // k)) * k
    dev = random_ternary_device(rows, n, 0, 0.5, row0=row0, device="cuda")
    host = orc.random_ternary_rows(row0, rows, n, 0, 0.5)
    assert np.array_equal(dev.device_data().cpu().numpy(), host.data)
    a = rsr.preprocess(dev, k, tw)
    assert a.plan.tile_count == {None: 4, 32704: 5, 16384: 8}[tw]
    assert a.format == (0 if tw is None else 3)
    ref = orc.preprocess(host, k, tw)
    assert np.array_equal(a.words, ref.words) and np.array_equal(a.perm, ref.perm)
    assert np.array_equal(a.group_offsets, ref.group_offsets)
    vi = rng.integers(-128, 128, n).astype(np.int8)
    assert np.array_equal(rsr.rsr_matvec(a, vi), orc.matvec_i8(ref, vi, threads=8))
    vf = orc.random_vector(n, 0)
    vb = torch.from_numpy(vf).cuda().to(torch.bfloat16)
    vr = gd.bf16_round(vf)
    y = rsr.rsr_matvec(a, vb).cpu().numpy()
    yr = orc.matvec_f64(ref, vr, threads=8)
    assert float_ok(y, yr, np.abs(orc.decode(host)).astype(np.float64), vr).all()
    ref.weight_scale = 1.0
    assert np.array_equal(rsr.rsr_matvec_fused(a, vb).cpu().numpy(),
                          orc.fused_matvec(ref, vr, threads=8))


@pytest.mark.parametrize("bw,k,n", [("ternary", 6, 3000), ("binary", 8, 2000),
                                    ("ternary", 5, 40000), ("ternary", 9, 500)])
def test_non_finite_vector_matches_reference_pattern(rsr, bw, k, n):
    """NaN / +-Inf activations: the reference adds sgn * s for every row of
    the block (0 * NaN = NaN), so the NaN/Inf pattern of y is fixed by the
    artifact; the kernel reproduces it exactly (every stream format)."""
    m_ = 4 * k + 3
    p = orc.random_matrix(m_, n, bw, 11)
    a = rsr.preprocess(rsr.PackedMatrix(m_, n, bw, p.data), k)
    ref = orc.preprocess(p, k)
    rng = np.random.default_rng(3)
    v = rng.standard_normal(n).astype(np.float32)
    v[rng.integers(0, n, 2)] = np.nan
    v[rng.integers(0, n)] = np.inf
    v[rng.integers(0, n)] = -np.inf
    v[0] = np.inf  # the tile's column 0 takes the epilogue path
    y = rsr.rsr_matvec(a, v).astype(np.float64)
    yr = orc.matvec_f64(ref, v)
    assert np.array_equal(np.isnan(y), np.isnan(yr))
    assert np.array_equal(np.isposinf(y), np.isposinf(yr))
    assert np.array_equal(np.isneginf(y), np.isneginf(yr))
    fin = np.isfinite(yr)
    vz = np.where(np.isfinite(v), v, 0).astype(np.float64)
    assert float_ok(y[fin], yr[fin], np.abs(orc.decode(p)).astype(np.float64)[fin], vz).all()


def test_float64_activations_match_reference(rsr):
    d = np.load(os.path.join(gd.GOLDEN_DIR, "quantize_f64.npz"))
    for i, n in enumerate([1, 7, 100, 1000, 4096]):
        v = d[f"v{i}"]
        assert v.dtype == np.float64
        qv = rsr.quantize_activations(v)
        assert qv.scale == float(d[f"scale{i}"])
        assert np.array_equal(qv.values, d[f"q{i}"])
        mat = rsr.PackedMatrix(40, n, "ternary", d[f"data{i}"], 0.37)
        assert np.array_equal(rsr.Multiplier("NaiveI8", mat).multiply(v), d[f"naive{i}"])
        assert np.array_equal(rsr.Multiplier("RsrTernary", mat, k=4).multiply(v), d[f"fused{i}"])


def test_threads_share_one_artifact(rsr):
    """Eight threads multiplying one artifact through the numpy API (the C
    call releases the GIL) stay bit-exact."""
    from concurrent.futures import ThreadPoolExecutor
    p = orc.random_matrix(300, 3000, "ternary", 21)
    a = rsr.preprocess(rsr.PackedMatrix(300, 3000, "ternary", p.data, 0.5), 5)
    ref = orc.preprocess(p, 5)
    ref.weight_scale = 0.5
    rng = np.random.default_rng(9)
    vis = [rng.integers(-128, 128, 3000).astype(np.int8) for _ in range(8)]
    vfs = [rng.standard_normal(3000).astype(np.float32) for _ in range(8)]
    want_i = [orc.matvec_i8(ref, v) for v in vis]
    want_f = [orc.fused_matvec(ref, v) for v in vfs]

    def work(t):
        bad = 0
        for _ in range(50):
            bad += not np.array_equal(rsr.rsr_matvec(a, vis[t]), want_i[t])
            bad += not np.array_equal(rsr.rsr_matvec_fused(a, vfs[t]), want_f[t])
        return bad

    with ThreadPoolExecutor(8) as ex:
        assert sum(ex.map(work, range(8))) == 0
