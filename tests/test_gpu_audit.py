"""Device audit (rsr_audit) and inverse (rsr_reconstruct) of artifacts.

* Lossless: reconstruct(preprocess(M)) == M for randomized shapes, both
  bitwidths, and a save/load round trip is byte-identical (reference
  test_acceptance.py criterion 3, :81-112).
* Every invariant of the reference's validate_artifact (preproc.py:305-372)
  rejects a hand-corrupted artifact with CorruptArtifact, before any chunk
  stream is derived from it.
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


def test_reconstruct_is_lossless_and_files_round_trip(rsr, tmp_path):
    from paper_2603_27462_b200 import artifact_io
    rng = np.random.default_rng(0xACC3)
    path = tmp_path / "case.rsra"
    for i in range(200):
        m_, n_ = int(rng.integers(1, 65)), int(rng.integers(1, 257))
        k = int(rng.integers(1, 11))
        bw = "binary" if i % 2 == 0 else "ternary"
        scale = float(rng.choice([1.0, 0.25, 3.5]))
        p = orc.random_matrix(m_, n_, bw, 1000 + i, float(rng.choice([0.0, 0.3, 0.5, 1.0])))
        a = rsr.preprocess(rsr.PackedMatrix(m_, n_, bw, p.data, scale), k)
        r = rsr.reconstruct(a)
        assert np.array_equal(r.device_data().cpu().numpy(), p.data), f"case {i}"
        assert r.weight_scale == scale
        artifact_io.save(a, path)
        first = path.read_bytes()
        artifact_io.save(artifact_io.load(path), path)
        assert path.read_bytes() == first, f"case {i}: round trip drifted"


def _host_arrays(rsr):
    p = orc.random_matrix(12, 300, "ternary", 5)
    a = rsr.preprocess(rsr.PackedMatrix(12, 300, "ternary", p.data), 4, 128)
    return a, dict(words=a.words.copy(), perm=a.perm.copy(), go=a.group_offsets.copy(),
                   po=a.perm_offsets.copy())


def _rebuild(rsr, a, arrs, bitwidth=None):
    from paper_2603_27462_b200.preproc import RsrArtifact
    return RsrArtifact.from_host(a.m, a.n, a.k, bitwidth or a.bitwidth, 1.0, a.plan,
                                 arrs["words"], arrs["perm"], arrs["go"], arrs["po"],
                                 audit=True)


def _w(ps, pl, pos, neg):
    return np.uint64(ps | (pl << 16) | (pos << 32) | (neg << 48))


CORRUPTIONS = {
    "empty group": lambda d: d["words"].__setitem__(0, d["words"][0] & ~np.uint64(0xFFFF << 16)),
    "keys out of order": lambda d: d["words"].__setitem__(
        slice(0, 2), d["words"][[1, 0]] - np.uint64(0)),
    "overlapping masks": lambda d: d["words"].__setitem__(
        0, d["words"][0] | (((d["words"][0] >> np.uint64(32)) & np.uint64(0xFFFF)) << np.uint64(48))),
    "bits above height": lambda d: d["words"].__setitem__(0, d["words"][0] | (np.uint64(1 << 10) << np.uint64(32))),
    "duplicate column": lambda d: d["perm"].__setitem__(1, d["perm"][0]),
    "column beyond tile": lambda d: d["perm"].__setitem__(0, np.uint16(200)),
    "columns descending": lambda d: d["perm"].__setitem__(slice(0, 2), d["perm"][[1, 0]]),
    "offsets beyond arrays": lambda d: d["go"].__setitem__(-1, d["go"][-1] + 5),
}


@pytest.mark.parametrize("what", sorted(CORRUPTIONS))
def test_each_invariant_rejects_a_corrupt_artifact(rsr, what):
    a, arrs = _host_arrays(rsr)
    _rebuild(rsr, a, {k: v.copy() for k, v in arrs.items()})  # the sound one passes
    bad = {k: v.copy() for k, v in arrs.items()}
    if what == "duplicate column" or what == "columns descending":
        # make sure the first group has at least two columns
        pl = int((bad["words"][0] >> np.uint64(16)) & np.uint64(0xFFFF))
        assert pl >= 2
    CORRUPTIONS[what](bad)
    with pytest.raises(rsr.CorruptArtifact):
        _rebuild(rsr, a, bad)


def test_negative_mask_in_binary_artifact(rsr):
    p = orc.random_matrix(8, 100, "binary", 3)
    a = rsr.preprocess(rsr.PackedMatrix(8, 100, "binary", p.data), 4)
    words = a.words.copy()
    words[0] |= np.uint64(1) << np.uint64(48)
    from paper_2603_27462_b200.preproc import RsrArtifact
    with pytest.raises(rsr.CorruptArtifact):
        RsrArtifact.from_host(a.m, a.n, a.k, a.bitwidth, 1.0, a.plan, words, a.perm,
                              a.group_offsets, a.perm_offsets, audit=True)
