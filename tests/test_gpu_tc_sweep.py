"""Randomized acceptance sweeps for the batched tensor-core multiply (SURVEY
8a K9), in the style of the reference's gate (pkg/tests/test_acceptance.py
:25-78) -- the batched path has no reference implementation, so every column
is held to the single-vector reference semantics:

* int8 batches (tcgen05 kind::i8): 150 randomized cases (both bitwidths,
  k = 1..16 within the reference caps, B = 2..256, ragged shapes, some all-zero
  matrices and column ranges past a 128-column step), every column equal to
  the dense integer product exactly;
* bf16 batches (kind::f16): 100 randomized cases over five decades of
  magnitude, every column within the stated per-row tolerance
  |y - ref| <= 1e-6 * sum_j |M_ij v_j| + 1e-6 * |ref| of the exact product;
* the batched fused path (per-row quantization -> int8 tensor cores with the
  dequantization in the epilogue): 40 cases, each row bit-identical to the
  single-vector fused multiply.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

K_CAP = {"binary": 16, "ternary": 10}


def random_entries(rng, m, n, bitwidth, density=0.5):
    if bitwidth == "binary":
        return (rng.random((m, n)) < density).astype(np.int8)
    u = rng.random((m, n))
    ent = np.zeros((m, n), np.int8)
    ent[u < density / 2] = 1
    ent[u > 1 - density / 2] = -1
    return ent


@pytest.fixture(scope="module")
def rsr():
    import torch
    import paper_2603_27462_b200 as pkg
    torch.cuda.set_device(0)
    return pkg


def _case(rng, i):
    m_ = int(rng.integers(1, 700))
    n_ = int(rng.integers(1, 1500))
    bw = "binary" if i % 2 == 0 else "ternary"
    k = int(rng.integers(1, K_CAP[bw] + 1))
    B = int(rng.choice([2, 3, 5, 8, 16, 17, 31, 64, 100, 256]))
    return m_, n_, k, bw, B


def test_int8_batches_bit_exact_150_cases(rsr):
    import torch
    from paper_2603_27462_b200 import kernels as kn
    rng = np.random.default_rng(0x7C18)
    bad = []
    for i in range(150):
        m_, n_, k, bw, B = _case(rng, i)
        ent = random_entries(rng, m_, n_, bw, float(rng.choice([0.1, 0.5, 0.9])))
        if i % 37 == 5:
            ent[:] = 0
        a = rsr.preprocess(rsr.encode(ent, m_, n_, bw), k)
        V = rng.integers(-128, 128, (B, n_)).astype(np.int8)
        Y = torch.empty(B, m_, dtype=torch.int32, device="cuda")
        kn.matmul_into(a, torch.from_numpy(V).cuda(), Y, method="tc")
        ref = V.astype(np.int64) @ ent.astype(np.int64).T
        if not np.array_equal(Y.cpu().numpy().astype(np.int64), ref):
            bad.append((i, m_, n_, k, bw, B))
    assert not bad, bad[:10]


def test_bf16_batches_within_tolerance_100_cases(rsr):
    import torch
    from paper_2603_27462_b200 import kernels as kn
    rng = np.random.default_rng(0x7CBF)
    bad, worst = [], 0.0
    for i in range(100):
        m_, n_, k, bw, B = _case(rng, i)
        ent = random_entries(rng, m_, n_, bw)
        a = rsr.preprocess(rsr.encode(ent, m_, n_, bw), k)
        Vf = (rng.standard_normal((B, n_)) * 10.0 ** rng.integers(-2, 3)).astype(np.float32)
        Vb = torch.from_numpy(Vf).cuda().to(torch.bfloat16)
        Y = torch.empty(B, m_, dtype=torch.float32, device="cuda")
        kn.matmul_into(a, Vb, Y, method="tc")
        Vr = Vb.float().cpu().numpy().astype(np.float64)
        ref = Vr @ ent.astype(np.float64).T
        cond = np.abs(Vr) @ np.abs(ent).astype(np.float64).T
        err = np.abs(Y.cpu().numpy().astype(np.float64) - ref)
        bound = 1e-6 * cond + 1e-6 * np.abs(ref)
        worst = max(worst, float((err / np.maximum(bound, 1e-300)).max()))
        if not (err <= bound).all():
            bad.append((i, m_, n_, k, bw, B))
    print(f"[bf16 tc sweep] worst error = {worst:.3f} of the stated bound")
    assert not bad, bad[:10]


def test_fused_batches_equal_single_vector_fused_40_cases(rsr):
    import torch
    from paper_2603_27462_b200 import kernels as kn
    rng = np.random.default_rng(0x7CF5)
    bad = []
    for i in range(40):
        m_ = int(rng.integers(1, 400))
        n_ = int(rng.integers(1, 1200))
        k = int(rng.integers(1, 11))
        T = int(rng.choice([2, 3, 7, 16, 40]))
        ent = random_entries(rng, m_, n_, "ternary")
        pm = rsr.encode(ent, m_, n_, "ternary")
        pm = rsr.PackedMatrix(pm.rows, pm.cols, "ternary", pm.data, float(rng.choice([1.0, 0.37])))
        a = rsr.preprocess(pm, k)
        X = torch.from_numpy(rng.standard_normal((T, n_)).astype(np.float32)).cuda()
        out = torch.empty(T, m_, dtype=torch.float32, device="cuda")
        kn.fused_rows_into(a, X, out)
        one = torch.empty(m_, dtype=torch.float32, device="cuda")
        for t in range(T):
            kn.fused_into(a, X[t], one)
            if not torch.equal(out[t], one):
                bad.append((i, m_, n_, k, T, t))
                break
    assert not bad, bad[:10]
