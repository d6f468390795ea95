"""Two-binary-plane ternary multiply: M = P - N as one stacked
binary artifact; integer results equal the oracle exactly, float results
meet the stated tolerance (|y - ref| <= 1e-6 sum|M v| + 1e-6 |ref|)."""
import numpy as np
import pytest

from oracle import rsr_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,k", [(37, 300, 6), (64, 4096, 10), (9, 5000, 12), (300, 100, 3)])
def test_two_plane_matches_oracle(m, n, k):
    import torch
    import paper_2603_27462_b200 as rsr
    from paper_2603_27462_b200.twoplane import TwoPlane
    p = orc.random_matrix(m, n, "ternary", m + n)
    tp = TwoPlane(rsr.PackedMatrix(m, n, "ternary", p.data), k)
    ent = orc.decode(p)
    P, N = (ent == 1).astype(np.int8), (ent == -1).astype(np.int8)
    planes = tp.planes.device_data().cpu().numpy()
    assert np.array_equal(planes[:m], orc.encode(P, m, n, "binary").data)
    assert np.array_equal(planes[m:], orc.encode(N, m, n, "binary").data)
    rng = np.random.default_rng(k)
    vi = rng.integers(-128, 128, n).astype(np.int8)
    yi = tp.matvec(torch.from_numpy(vi).cuda()).cpu().numpy()
    assert np.array_equal(yi, orc.matvec_i8(orc.preprocess(p, 4), vi))
    vf = rng.standard_normal(n).astype(np.float32)
    y = tp.matvec(torch.from_numpy(vf).cuda()).cpu().numpy().astype(np.float64)
    ref = ent.astype(np.float64) @ vf.astype(np.float64)
    cond = np.abs(ent).astype(np.float64) @ np.abs(vf.astype(np.float64))
    assert (np.abs(y - ref) <= 1e-6 * cond + 1e-6 * np.abs(ref)).all()
