"""Batched multi-vector multiply.

Not in the reference (kernels.py:196 takes one vector); the oracle is the
single-vector path per column: int8 batches are bit-exact against the
reference integer core, real batches are held to the float tolerance of
test_gpu_parity.py per row, against the reference float64 path.
"""
import numpy as np
import pytest

from oracle import rsr_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rsr():
    import torch
    import paper_2603_27462_b200 as pkg
    torch.cuda.set_device(0)
    return pkg


def float_ok(y, ref, dense, v):
    bound = 1e-6 * (np.abs(dense.astype(np.float64)) @ np.abs(v.astype(np.float64)))
    return np.abs(y.astype(np.float64) - ref) <= bound + 1e-6 * np.abs(ref)


@pytest.mark.parametrize("m,n,k,bw,tw,B", [
    (96, 3000, 5, "ternary", None, 5),
    (64, 4096, 6, "ternary", None, 8),
    (40, 2000, 8, "binary", None, 3),
    (30, 20000, 4, "ternary", 20000, 7),   # u16 unscaled format
    (33, 5000, 5, "ternary", 2048, 9),     # multi-tile (partials)
    (50, 3000, 12, "binary", None, 4),     # > 2187 keys: column-by-column path
    (24, 40000, 4, "ternary", 40000, 3),   # u32 format: column-by-column path
])
def test_batched_vs_single_vector_oracle(rsr, m, n, k, bw, tw, B):
    rng = np.random.default_rng(m * 31 + B)
    p = orc.random_matrix(m, n, bw, m + n)
    ref = orc.preprocess(p, k, tw)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, bw, p.data), k, tw)
    dense = orc.decode(p)
    Vi = rng.integers(-128, 128, (B, n)).astype(np.int8)
    Yi = rsr.rsr_matvec_batched(a, Vi)
    assert Yi.shape == (B, m) and Yi.dtype == np.int32
    for b in range(B):
        assert np.array_equal(Yi[b], orc.matvec_i8(ref, Vi[b])), b
    Vf = rng.standard_normal((B, n)).astype(np.float32)
    Yf = rsr.rsr_matvec_batched(a, Vf)
    assert Yf.shape == (B, m) and Yf.dtype == np.float32
    for b in range(B):
        assert float_ok(Yf[b], orc.matvec_f64(ref, Vf[b]), dense, Vf[b]).all(), b


def test_batched_bf16_c4_shape(rsr):
    """C4 (ternary 8192^2, k=5) with a bf16 batch of 16: every column against
    the single-vector kernel's float tolerance vs the reference float path."""
    import torch
    m = n = 8192
    p = orc.random_matrix(m, n, "ternary", 0)
    ref = orc.preprocess(p, 5)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", p.data), 5)
    V = torch.stack([torch.from_numpy(orc.random_vector(n, b)) for b in range(16)]).to(
        torch.bfloat16).cuda()
    Y = rsr.rsr_matvec_batched(a, V).cpu().numpy()
    Vh = V.float().cpu().numpy()
    dense = orc.decode(p)
    for b in (0, 7, 15):
        assert float_ok(Y[b], orc.matvec_f64(ref, Vh[b]), dense, Vh[b]).all(), b


def test_batched_errors(rsr):
    from paper_2603_27462_b200.errors import DimensionMismatch
    p = orc.random_matrix(10, 100, "ternary", 1)
    a = rsr.preprocess(rsr.PackedMatrix(10, 100, "ternary", p.data), 4)
    with pytest.raises(DimensionMismatch):
        rsr.rsr_matvec_batched(a, np.zeros((2, 99), np.float32))
    with pytest.raises(DimensionMismatch):
        rsr.rsr_matvec_batched(a, np.zeros((2, 100), np.int16))
    assert rsr.rsr_matvec_batched(a, np.zeros((0, 100), np.float32)).shape == (0, 10)


@pytest.mark.parametrize("m,n,k,bw,B", [
    (96, 3000, 5, "ternary", 5),     # u8 keys, K tail, partial row tile
    (200, 4096, 6, "ternary", 16),   # u16 keys
    (64, 2048, 8, "binary", 33),     # N padded to 48
    (2000, 1000, 4, "ternary", 2),   # several row tiles, split-K
    (120, 1500, 8, "ternary", 8),    # 6561 keys: pair-table expansion
    (48, 70000, 4, "ternary", 3),    # multi-tile artifact (tw 32768)
    (64, 640, 5, "ternary", 256),    # N = 256
    (300, 3000, 12, "binary", 4),    # k > 8 (rows straddle 128-row tiles)
    (130, 1000, 16, "binary", 20),   # k = 16
    (1000, 9000, 5, "ternary", 130), # N = 256 with a K tail, several tiles
])
def test_tensor_core_batched(rsr, m, n, k, bw, B):
    """bf16 batches on tcgen05 (key matrix -> sign expansion -> MMA): each
    column within the float tolerance of the reference float path."""
    import torch
    p = orc.random_matrix(m, n, bw, m + 3 * n)
    ref = orc.preprocess(p, k)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, bw, p.data), k)
    rng = np.random.default_rng(B)
    V = torch.from_numpy(rng.standard_normal((B, n)).astype(np.float32)).to(torch.bfloat16).cuda()
    Y = rsr.rsr_matvec_batched(a, V, method="tc").cpu().numpy()
    Vh = V.float().cpu().numpy()
    dense = orc.decode(p)
    for b in range(B):
        assert float_ok(Y[b], orc.matvec_f64(ref, Vh[b]), dense, Vh[b]).all(), b


def test_tensor_core_batched_shards(rsr):
    """Row-block views (shards starting at any block) through the tcgen05
    path match the rows of the whole multiply (the split-K partition may
    differ, so fp32 rounding may too)."""
    import torch
    from paper_2603_27462_b200 import kernels as kn
    m, n, k, B = 999, 2000, 5, 12
    p = orc.random_matrix(m, n, "ternary", 17)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", p.data), k)
    V = torch.randn(B, n, device="cuda").to(torch.bfloat16)
    Yall = torch.empty(B, m, device="cuda")
    kn.matmul_into(a, V, Yall, method="tc")
    bc = a.plan.block_count
    for b0, nb in [(0, 17), (17, 40), (57, bc - 57), (199, 1)]:
        rows = min(nb * k, m - b0 * k)
        Y = torch.full((B, rows), float("nan"), device="cuda")
        kn.matmul_into(a, V, Y, view=a.view(b0, nb), method="tc")
        torch.testing.assert_close(Y, Yall[:, b0 * k:b0 * k + rows], rtol=1e-5, atol=1e-3)


@pytest.mark.parametrize("m,n,k,bw,tw", [
    (101, 300, 5, "ternary", None),    # partial last block, K tail
    (64, 200, 8, "binary", None),
    (37, 5000, 3, "ternary", 2048),    # several tiles
    (50, 333, 12, "binary", 100),      # k > 8, tiles not a multiple of 16 columns
])
def test_code_matrix_layout(rsr, m, n, k, bw, tw):
    """The tensor-core code matrix equals the dense matrix's 2-bit codes
    (+1 -> 01, -1 -> 10; reference pattern_key code form, preproc.py:183-197)
    at u32 [col // 128][row][(col % 128) // 16], column pair j = (col % 16) // 2
    at bit 8 (2 (j // 4) + col % 2) + 2 (j % 4) (csrc/rsr_tc.cu)."""
    p = orc.random_matrix(m, n, bw, 7 * m + n)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, bw, p.data), k, tw)
    km = a.keymat().cpu().numpy().view(np.uint32)
    dense = orc.decode(p).astype(np.int64)
    code = np.where(dense == 1, 1, np.where(dense == -1, 2, 0))
    steps, rows_pad = (n + 127) // 128, (a.plan.block_count * k + 7) // 8 * 8
    assert km.size >= steps * rows_pad * 8  # (sized for the int8 layout)
    km = km[:steps * rows_pad * 8]
    exp = np.zeros((steps, rows_pad, 8), np.int64)
    for c in range(n):
        j = (c % 16) // 2
        bit = 8 * (2 * (j // 4) + c % 2) + 2 * (j % 4)
        exp[c // 128, :m, (c % 128) // 16] |= code[:, c] << bit
    assert np.array_equal(km.reshape(steps, rows_pad, 8).astype(np.int64), exp)


@pytest.mark.parametrize("offset,pad", [(1, 3), (0, 5), (8, 8)])
def test_tensor_core_strided_vectors(rsr, offset, pad):
    """bf16 rows that start off a 16-byte boundary or have an odd pitch are
    re-laid into aligned rows before the TMA loads (the C entry point rejects
    them); aligned strided rows are loaded in place: both equal the
    contiguous batch bit for bit."""
    import torch
    from paper_2603_27462_b200 import kernels as kn
    m, n, k, B = 300, 1000, 5, 6
    p = orc.random_matrix(m, n, "ternary", 41)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", p.data), k)
    big = torch.randn(B, offset + n + pad, device="cuda").to(torch.bfloat16)
    V = big[:, offset:offset + n]
    Yc = torch.empty(B, m, device="cuda")
    kn.matmul_into(a, V.contiguous(), Yc, method="tc")
    Ys = torch.empty(B, m, device="cuda")
    kn.matmul_into(a, V, Ys, method="tc")
    assert torch.equal(Yc, Ys)
    if offset % 8 or (offset + n + pad) % 8:
        from paper_2603_27462_b200 import _lib
        L = _lib.lib()
        ws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
        rc = L.rsr_matmul_tc(_lib.ptr(a.keymat()), m, n, 1, k, 0, a.plan.block_count,
                             V.data_ptr(), _lib.RSR_BF16, V.stride(0), B, Ys.data_ptr(), m,
                             _lib.ptr(ws), ws.numel(), 0)
        assert rc == _lib.RSR_ERR_INVALID


def test_tensor_core_split_k_is_deterministic(rsr):
    """Tiles split across the CTAs of a cluster are summed in rank order:
    repeated calls (with other batch sizes in between) give bit-identical
    results."""
    import torch
    from paper_2603_27462_b200 import kernels as kn
    m, n, k = 2000, 6000, 5
    p = orc.random_matrix(m, n, "ternary", 77)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", p.data), k)
    V = torch.randn(16, n, device="cuda").to(torch.bfloat16)
    first = torch.empty(16, m, device="cuda")
    kn.matmul_into(a, V, first, method="tc")
    for rep in range(20):
        Vb = torch.randn(1 + rep % 7, n, device="cuda").to(torch.bfloat16)
        kn.matmul_into(a, Vb, torch.empty(Vb.shape[0], m, device="cuda"), method="tc")
        Y = torch.empty(16, m, device="cuda")
        kn.matmul_into(a, V, Y, method="tc")
        assert torch.equal(Y, first), rep


@pytest.mark.parametrize("m,n,k,bw,B", [
    (96, 3000, 5, "ternary", 5),
    (200, 4096, 6, "ternary", 16),
    (64, 2048, 8, "binary", 33),
    (2000, 1000, 4, "ternary", 2),
    (300, 3000, 12, "binary", 4),
    (130, 1000, 16, "binary", 20),
    (1000, 9000, 5, "ternary", 130),
    (64, 640, 5, "ternary", 256),
])
def test_tensor_core_int8_batched_is_exact(rsr, m, n, k, bw, B):
    """int8 batches on tcgen05 kind::i8: every column equals the reference
    integer core bit for bit (int32, saturating-free exact sums)."""
    import torch
    from paper_2603_27462_b200 import kernels as kn
    p = orc.random_matrix(m, n, bw, m + 5 * n)
    ref = orc.preprocess(p, k)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, bw, p.data), k)
    rng = np.random.default_rng(B + 1)
    Vi = rng.integers(-128, 128, (B, n)).astype(np.int8)
    Vi[0, :7] = -128  # extremes
    Y = torch.empty(B, m, dtype=torch.int32, device="cuda")
    kn.matmul_into(a, torch.from_numpy(Vi).cuda(), Y, method="tc")
    Yh = Y.cpu().numpy()
    for b in range(B):
        assert np.array_equal(Yh[b], orc.matvec_i8(ref, Vi[b])), b
    # numpy through the public batched API (auto policy -> tensor cores)
    assert np.array_equal(rsr.rsr_matvec_batched(a, Vi), Yh)


@pytest.mark.parametrize("m,n,k,bw,tw", [
    (101, 300, 5, "ternary", None),
    (50, 333, 12, "binary", 100),
])
def test_code_matrix_layout_i8(rsr, m, n, k, bw, tw):
    """The int8 path's code matrix: 256-column steps, u32 [col // 256][row]
    [(col % 256) // 16]; column 4w + i of a 16-column word in nibble
    i + 4 (w // 2) at bit offset 2 (w % 2) (csrc/rsr_tc.cu)."""
    p = orc.random_matrix(m, n, bw, 3 * m + n)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, bw, p.data), k, tw)
    km = a.keymat("i8").cpu().numpy().view(np.uint32)
    dense = orc.decode(p).astype(np.int64)
    code = np.where(dense == 1, 1, np.where(dense == -1, 2, 0))
    steps, rows_pad = (n + 255) // 256, (a.plan.block_count * k + 7) // 8 * 8
    assert km.size == steps * rows_pad * 16
    exp = np.zeros((steps, rows_pad, 16), np.int64)
    for c in range(n):
        w, i = (c % 16) // 4, c % 4
        bit = 4 * (i + 4 * (w // 2)) + 2 * (w % 2)
        exp[c // 256, :m, (c % 256) // 16] |= code[:, c] << bit
    assert np.array_equal(km.reshape(steps, rows_pad, 16).astype(np.int64), exp)


@pytest.mark.parametrize("m,n,k,bw,tw", [
    (101, 300, 5, "ternary", None),
    (50, 333, 12, "binary", 100),
    (37, 5000, 3, "ternary", 2048),
])
def test_code_matrix_layout_wide(rsr, m, n, k, bw, tw):
    """The wide bf16 code matrix (B <= 32): the int8 layout's 256-column
    steps, u32 [col // 256][row][(col % 256) // 16], with the bf16 bit order
    of test_code_matrix_layout inside each 16-column word."""
    p = orc.random_matrix(m, n, bw, 5 * m + n)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, bw, p.data), k, tw)
    km = a.keymat("wide").cpu().numpy().view(np.uint32)
    dense = orc.decode(p).astype(np.int64)
    code = np.where(dense == 1, 1, np.where(dense == -1, 2, 0))
    steps, rows_pad = (n + 255) // 256, (a.plan.block_count * k + 7) // 8 * 8
    assert km.size == steps * rows_pad * 16
    exp = np.zeros((steps, rows_pad, 16), np.int64)
    for c in range(n):
        j = (c % 16) // 2
        bit = 8 * (2 * (j // 4) + c % 2) + 2 * (j % 4)
        exp[c // 256, :m, (c % 256) // 16] |= code[:, c] << bit
    assert np.array_equal(km.reshape(steps, rows_pad, 16).astype(np.int64), exp)


@pytest.mark.parametrize("m,n,B", [(300, 1000, 16), (1000, 9000, 3), (130, 264, 1), (64, 4096, 9),
                                   (500, 2000, 32), (257, 1024, 17)])
def test_tensor_core_wide_steps_match_narrow(rsr, m, n, B):
    """bf16 batches of B <= 32 take 256-column steps (rsr_matmul_tc_wide):
    each column within the float tolerance of the exact product, and within
    a few fp32 ulps of the 128-column-step kernel (same products, the step
    boundaries move the partial sums)."""
    import torch
    from paper_2603_27462_b200 import _lib
    p = orc.random_matrix(m, n, "ternary", m + 3 * n)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", p.data), 5)
    V = torch.randn(B, n, device="cuda").to(torch.bfloat16)
    L = _lib.lib()
    Yw = torch.empty(B, m, device="cuda")
    Yn = torch.empty(B, m, device="cuda")
    ws = torch.empty(256, dtype=torch.uint8, device="cuda")
    s = _lib.current_stream_ptr(a.device)
    for fn, km, Y in ((L.rsr_matmul_tc_wide, a.keymat("wide"), Yw), (L.rsr_matmul_tc, a.keymat(), Yn)):
        assert fn(_lib.ptr(km), m, n, 1, 5, 0, a.plan.block_count, V.data_ptr(), _lib.RSR_BF16,
                  V.stride(0), B, Y.data_ptr(), Y.stride(0), ws.data_ptr(), 256, s) == 0
    torch.cuda.synchronize()
    dense = orc.decode(p).astype(np.float64)
    Vh = V.float().cpu().numpy().astype(np.float64)
    ref = Vh @ dense.T
    cond = np.abs(Vh) @ np.abs(dense).T
    for Y in (Yw, Yn):
        err = np.abs(Y.cpu().numpy() - ref)
        assert (err <= 1e-6 * cond + 1e-6 * np.abs(ref)).all()
    assert L.rsr_matmul_tc_wide(_lib.ptr(a.keymat("wide")), m, n, 1, 5, 0, a.plan.block_count,
                                V.data_ptr(), _lib.RSR_BF16, V.stride(0), 33, Yw.data_ptr(),
                                Yw.stride(0), ws.data_ptr(), 256, s) == _lib.RSR_ERR_INVALID


@pytest.mark.parametrize("offset,pad", [(1, 3), (16, 16), (0, 7)])
def test_tensor_core_int8_strided_vectors(rsr, offset, pad):
    """int8 rows off a 16-byte boundary or with a pitch not a multiple of 16
    are re-laid before the TMA loads; every column stays exact."""
    import torch
    from paper_2603_27462_b200 import kernels as kn
    m, n, k, B = 300, 1000, 5, 6
    p = orc.random_matrix(m, n, "ternary", 43)
    ref = orc.preprocess(p, k)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", p.data), k)
    rng = np.random.default_rng(offset + pad)
    big = torch.from_numpy(rng.integers(-128, 128, (B, offset + n + pad)).astype(np.int8)).cuda()
    V = big[:, offset:offset + n]
    Y = torch.empty(B, m, dtype=torch.int32, device="cuda")
    kn.matmul_into(a, V, Y, method="tc")
    Vh = V.cpu().numpy()
    for b in range(B):
        assert np.array_equal(Y[b].cpu().numpy(), orc.matvec_i8(ref, Vh[b])), b
