"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle and
the reference golden vectors.  Integer/byte work is bit-exact; the float path
is held to |y - ref| <= 1e-6 * sum_j |M_ij v_j| + 1e-6 * |ref| per row
(ref = the reference's float64 accumulation)."""

import numpy as np
import pytest

from oracle import rsr_oracle as orc
from tests import golden_data as gd

pytestmark = pytest.mark.gpu

FLOAT_RTOL = 1e-6


@pytest.fixture(scope="module")
def rsr():
    import torch
    import paper_2603_27462_b200 as pkg
    torch.cuda.set_device(0)
    return pkg


def float_ok(y, ref_f64, dense, v):
    cond = np.abs(dense.astype(np.float64)) @ np.abs(np.asarray(v, np.float64))
    return np.abs(y.astype(np.float64) - ref_f64) <= FLOAT_RTOL * cond + FLOAT_RTOL * np.abs(ref_f64)




@pytest.mark.parametrize("i", range(19))
def test_preprocess_bit_exact_vs_reference(rsr, i):
    case = gd.small_case(i)
    md = case["meta"]
    m = rsr.PackedMatrix(md["m"], md["n"], md["bitwidth"], case["data"], md["weight_scale"])
    a = rsr.preprocess(m, md["k"], md["tile_width"])
    assert np.array_equal(a.words, case["words"])
    assert np.array_equal(a.perm, case["perm"])
    assert np.array_equal(a.group_offsets, case["go"])
    assert np.array_equal(a.perm_offsets, case["po"])
    assert np.array_equal(a.sort_steps, case["steps"])
    assert a.file_bytes() == md["file_bytes"]
    assert list(a.op_totals()) == md["op_totals"]
    rsr.validate_artifact(a)


@pytest.mark.parametrize("i", range(19))
def test_multiply_vs_reference(rsr, i):
    case = gd.small_case(i)
    md = case["meta"]
    m = rsr.PackedMatrix(md["m"], md["n"], md["bitwidth"], case["data"], md["weight_scale"])
    a = rsr.preprocess(m, md["k"], md["tile_width"])
    y = rsr.rsr_matvec(a, case["vi"])
    assert y.dtype == np.int32
    assert np.array_equal(y, case["y_i8"])
    yf = rsr.rsr_matvec(a, case["vf"])
    assert yf.dtype == np.float32
    dense = orc.decode(orc.Packed(md["m"], md["n"], md["bitwidth"], case["data"]))
    assert float_ok(yf, case["naive_f64"], dense, case["vf"]).all()
    if md["bitwidth"] == "ternary":
        assert np.array_equal(rsr.rsr_matvec_fused(a, case["vf"]), case["fused"])


def test_known_answers(rsr):
    m = rsr.encode(np.array([[1, 0, 1, 0], [1, 1, 0, 0]], np.int8), 2, 4, "binary")
    a = rsr.preprocess(m, 2)
    assert list(a.perm) == [2, 1, 0]
    assert [(g.perm_start, g.perm_len, g.pos_mask, g.neg_mask)
            for g in a.block_meta(0, 0).groups] == [(0, 1, 1, 0), (1, 1, 2, 0), (2, 1, 3, 0)]
    assert a.op_totals() == (3, 4, 3)
    assert list(rsr.rsr_matvec(a, np.array([1, 2, 3, 4], np.int8))) == [4, 3]
    mt = rsr.PackedMatrix(2, 3, "ternary", rsr.encode(
        np.array([[1, -1, 0], [0, 1, 1]], np.int8), 2, 3, "ternary").data, 0.5)
    at = rsr.preprocess(mt, 2)
    y = rsr.rsr_matvec_fused(at, np.array([2.0, 3.0, 5.0], np.float32))
    exp = (np.array([-25, 203], np.float64) * (0.5 / 25.4)).astype(np.float32)
    assert np.array_equal(y, exp)
    assert list(rsr.rsr_matvec(at, np.array([2, 3, 5], np.int8))) == [-1, 8]


def test_saturating_inputs(rsr):
    n = 4096
    a = rsr.preprocess(rsr.encode(np.ones((3, n), np.int8), 3, n, "binary"), 3)
    assert list(rsr.rsr_matvec(a, np.full(n, -128, np.int8))) == [-128 * n] * 3


def test_zero_matrix(rsr):
    a = rsr.preprocess(rsr.encode(np.zeros((4, 8), np.int8), 4, 8, "ternary"), 3)
    assert a.words.size == 0 and a.perm.size == 0
    assert a.op_totals() == (0, 0, 0)
    assert list(rsr.rsr_matvec(a, np.ones(8, np.int8))) == [0, 0, 0, 0]
    assert list(rsr.rsr_matvec_fused(a, np.ones(8, np.float32))) == [0.0] * 4


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("bw", ["binary", "ternary"])
def test_random_shapes_vs_oracle(rsr, seed, bw):
    """Random shapes/k/tile widths: every stream format (scaled u16, u16,
    u32) and both flush variants (pattern buckets, register flush)."""
    rng = np.random.default_rng(100 + seed)
    m_, n_ = int(rng.integers(1, 300)), int(rng.integers(1, 3000))
    k = int(rng.integers(1, (16 if bw == "binary" else 10) + 1))
    tw = [None, 48, 1000, 777][seed % 4]
    dens = [0.5, 0.1, 0.9, 0.69][seed % 4]
    p = orc.random_matrix(m_, n_, bw, seed, dens)
    ref = orc.preprocess(p, k, tw)
    a = rsr.preprocess(rsr.PackedMatrix(m_, n_, bw, p.data, 0.37), k, tw)
    assert np.array_equal(a.words, ref.words)
    assert np.array_equal(a.perm, ref.perm)
    assert np.array_equal(a.group_offsets, ref.group_offsets)
    assert np.array_equal(a.sort_steps, ref.sort_steps)
    vi = rng.integers(-128, 128, n_).astype(np.int8)
    assert np.array_equal(rsr.rsr_matvec(a, vi), orc.matvec_i8(ref, vi))
    vf = (rng.standard_normal(n_) * 3).astype(np.float32)
    assert float_ok(rsr.rsr_matvec(a, vf), orc.matvec_f64(ref, vf), orc.decode(p), vf).all()
    if bw == "ternary":
        ref.weight_scale = 0.37
        assert np.array_equal(rsr.rsr_matvec_fused(a, vf), orc.fused_matvec(ref, vf))


@pytest.mark.parametrize("n_,off", [(2999, 0), (3000, 1), (16, 3), (1, 0)])
def test_pinned_host_vectors_take_the_mapped_copy(rsr, n_, off):
    """numpy vectors in page-locked memory go through the host-link copy
    kernels (rsr_matvec_host); odd lengths and misaligned starts take the
    byte loop.  Results equal the pageable (DMA) path and the oracle."""
    import torch
    m_ = 97
    p = orc.random_matrix(m_, n_, "ternary", 5)
    ref = orc.preprocess(p, 4)
    a = rsr.preprocess(rsr.PackedMatrix(m_, n_, "ternary", p.data), 4)
    rng = np.random.default_rng(7)
    vi = rng.integers(-128, 128, n_).astype(np.int8)
    hi = torch.empty(n_ + off, dtype=torch.int8, pin_memory=True).numpy()[off:]
    hi[:] = vi
    assert np.array_equal(rsr.rsr_matvec(a, hi), orc.matvec_i8(ref, vi))
    vf = (rng.standard_normal(n_) * 3).astype(np.float32)
    hf = torch.empty(n_ + off, dtype=torch.float32, pin_memory=True).numpy()[off:]
    hf[:] = vf
    yp = rsr.rsr_matvec(a, hf)
    assert np.array_equal(yp, rsr.rsr_matvec(a, vf))
    assert float_ok(yp, orc.matvec_f64(ref, vf), orc.decode(p), vf).all()
    a.weight_scale = ref.weight_scale = 0.37
    assert np.array_equal(rsr.rsr_matvec_fused(a, hf), orc.fused_matvec(ref, vf))
    assert np.array_equal(rsr.rsr_matvec_fused(a, vf), orc.fused_matvec(ref, vf))
    mul = rsr.Multiplier("RsrTernary", rsr.PackedMatrix(m_, n_, "ternary", p.data, 0.37), k=4)
    assert np.array_equal(mul.multiply(hf), orc.fused_matvec(ref, vf))


def test_torch_inputs_stay_on_device(rsr):
    import torch
    p = orc.random_matrix(64, 512, "ternary", 3)
    a = rsr.preprocess(rsr.PackedMatrix(64, 512, "ternary", p.data), 4)
    ref = orc.preprocess(p, 4)
    v = orc.random_vector(512, 3)
    vb = torch.from_numpy(v).cuda().to(torch.bfloat16)
    y = rsr.rsr_matvec(a, vb)
    assert y.is_cuda and y.dtype == torch.float32
    vr = vb.float().cpu().numpy()
    assert float_ok(y.cpu().numpy(), orc.matvec_f64(ref, vr), orc.decode(p), vr).all()
    yq = rsr.rsr_matvec_fused(a, vb)
    assert np.array_equal(yq.cpu().numpy(), orc.fused_matvec(ref, vr))
    vi = torch.randint(-128, 128, (512,), dtype=torch.int8, device="cuda")
    assert np.array_equal(rsr.rsr_matvec(a, vi).cpu().numpy(),
                          orc.matvec_i8(ref, vi.cpu().numpy()))


def test_c2_full_size_bit_exact_vs_reference(rsr):
    """Ternary 16384^2 (BASELINE config 1) at k=6: GPU artifact digests equal
    the reference's; the int path equals the reference output; the float
    path meets the stated tolerance; fused equals the reference exactly."""
    import torch
    name = "C2_ternary_16384_k6"
    rec = gd.meta()["large"][name]
    p = orc.random_matrix(16384, 16384, "ternary", 0)
    assert gd.sha(p.data) == rec["data_sha"]
    a = rsr.preprocess(rsr.PackedMatrix(16384, 16384, "ternary", p.data), 6)
    assert gd.sha(a.words) == rec["words_sha"]
    assert gd.sha(a.perm) == rec["perm_sha"]
    assert gd.sha(a.group_offsets) == rec["go_sha"]
    assert gd.sha(a.perm_offsets) == rec["po_sha"]
    assert gd.sha(a.sort_steps) == rec["steps_sha"]
    assert a.file_bytes() == rec["file_bytes"]
    assert list(a.op_totals()) == rec["op_totals"]
    vi = gd.int_vector(16384, 0)
    assert np.array_equal(rsr.rsr_matvec(a, vi), gd.large_output(name + "_y_i8"))
    vf = orc.random_vector(16384, 0)
    vb = torch.from_numpy(vf).cuda().to(torch.bfloat16)
    y = rsr.rsr_matvec(a, vb).cpu().numpy()
    vr = gd.bf16_round(vf)
    ref = orc.preprocess(p, 6)
    yr = orc.matvec_f64(ref, vr, threads=8)
    assert float_ok(y, yr, orc.decode(p), vr).all()
    assert np.array_equal(rsr.rsr_matvec_fused(a, vb).cpu().numpy(),
                          gd.large_output(name + "_fused_bf16v"))


@pytest.mark.parametrize("seed", [1, 2])
def test_c2_full_size_other_seeds_vs_oracle(rsr, seed):
    """C2 at seeds 1 and 2 as well -- the GPU artifact equals the
    oracle's preprocess array for array, the int path is exact, the float
    path meets the tolerance and the fused path equals the oracle's."""
    import torch
    p = orc.random_matrix(16384, 16384, "ternary", seed)
    a = rsr.preprocess(rsr.PackedMatrix(16384, 16384, "ternary", p.data), 6)
    ref = orc.preprocess(p, 6)
    for name in ("words", "perm", "group_offsets", "perm_offsets"):
        assert np.array_equal(getattr(a, name), getattr(ref, name)), name
    vi = gd.int_vector(16384, seed)
    assert np.array_equal(rsr.rsr_matvec(a, vi), orc.matvec_i8(ref, vi, threads=8))
    vf = orc.random_vector(16384, seed)
    vb = torch.from_numpy(vf).cuda().to(torch.bfloat16)
    vr = gd.bf16_round(vf)
    y = rsr.rsr_matvec(a, vb).cpu().numpy()
    assert float_ok(y, orc.matvec_f64(ref, vr, threads=8), orc.decode(p), vr).all()
    assert np.array_equal(rsr.rsr_matvec_fused(a, vb).cpu().numpy(), orc.fused_matvec(ref, vr))


@pytest.mark.parametrize("n,tw,k,bw", [(40000, None, 5, "ternary"), (65536, None, 4, "binary"),
                                       (70000, None, 6, "ternary"), (30000, 20000, 7, "ternary"),
                                       (3000, None, 9, "ternary"), (2000, None, 13, "binary"),
                                       (5000, 2500, 10, "ternary"), (1000, None, 16, "binary")])
def test_wide_tiles_and_large_k(rsr, n, tw, k, bw):
    """Tiles wider than 32768 columns (u32 stream) and pattern spaces too big
    for shared-memory buckets (register flush), bit-exact on the int paths."""
    rng = np.random.default_rng(n + k)
    m_ = 3 * k + 1
    p = orc.random_matrix(m_, n, bw, k)
    ref = orc.preprocess(p, k, tw)
    a = rsr.preprocess(rsr.PackedMatrix(m_, n, bw, p.data, 0.7), k, tw)
    assert np.array_equal(a.words, ref.words) and np.array_equal(a.perm, ref.perm)
    vi = rng.integers(-128, 128, n).astype(np.int8)
    assert np.array_equal(rsr.rsr_matvec(a, vi), orc.matvec_i8(ref, vi))
    vf = rng.standard_normal(n).astype(np.float32)
    assert float_ok(rsr.rsr_matvec(a, vf), orc.matvec_f64(ref, vf), orc.decode(p), vf).all()
    if bw == "ternary":
        ref.weight_scale = 0.7
        assert np.array_equal(rsr.rsr_matvec_fused(a, vf), orc.fused_matvec(ref, vf))


def test_fused_smem_just_under_48k(rsr):
    """BitNet down_proj shape (2560 x 6912, k=5): the team launch needs ~48 KiB
    of dynamic shared memory, just above the default cap left by the fused
    kernel's static reduction scratch -- the launch must raise the cap."""
    m_, n_ = 2560, 6912
    p = orc.random_matrix(m_, n_, "ternary", 7)
    ref = orc.preprocess(p, 5)
    ref.weight_scale = 0.5
    a = rsr.preprocess(rsr.PackedMatrix(m_, n_, "ternary", p.data, 0.5), 5)
    vf = np.random.default_rng(3).standard_normal(n_).astype(np.float32)
    assert np.array_equal(rsr.rsr_matvec_fused(a, vf), orc.fused_matvec(ref, vf))


@pytest.mark.parametrize("n", [2560, 1000, 3072, 6912, 8])
def test_fused_bf16_vector_bit_exact(rsr, n):
    """bf16 activations (the decode case; register-resident staging when the
    vector fits two 16-byte loads per thread) against the reference fused path
    on the same (bf16-valued) vector, bit for bit."""
    import torch
    m_ = 50
    p = orc.random_matrix(m_, n, "ternary", n)
    ref = orc.preprocess(p, 5)
    ref.weight_scale = 0.37
    a = rsr.preprocess(rsr.PackedMatrix(m_, n, "ternary", p.data, 0.37), 5)
    vb = torch.from_numpy(np.random.default_rng(n).standard_normal(n).astype(np.float32)).to(
        torch.bfloat16)
    y = rsr.rsr_matvec_fused(a, vb.cuda()).cpu().numpy()
    assert np.array_equal(y, orc.fused_matvec(ref, vb.float().numpy()))


def test_bf16_host_vector_round_trip(rsr):
    """A CPU bf16 tensor (pinned or pageable) goes host in / host out through
    the bf16 kernel: bit-identical to the same vector on the device."""
    import torch
    p = orc.random_matrix(300, 1000, "ternary", 5)
    a = rsr.preprocess(rsr.PackedMatrix(300, 1000, "ternary", p.data), 5)
    vb = torch.from_numpy(orc.random_vector(1000, 5) * 3).to(torch.bfloat16)
    yd = rsr.rsr_matvec(a, vb.cuda()).cpu().numpy()
    for vh in (vb, vb.pin_memory()):
        y = rsr.rsr_matvec(a, vh)
        assert isinstance(y, np.ndarray) and y.dtype == np.float32
        assert np.array_equal(y, yd)
    ref = orc.preprocess(p, 5)
    vr = vb.float().numpy()
    assert float_ok(y, orc.matvec_f64(ref, vr), orc.decode(p), vr).all()
