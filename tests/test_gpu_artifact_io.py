"""`.rsra` I/O of GPU artifacts: artifacts
preprocessed on the B200 save to exactly the bytes the reference writer
produces (sha256 of reference-written files), and loading a file gives a
device artifact whose multiplies are bit-identical."""
import hashlib

import numpy as np
import pytest

from oracle import rsr_oracle as orc
from tests import golden_data as gd

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rsr():
    import torch
    import paper_2603_27462_b200 as pkg
    torch.cuda.set_device(0)
    return pkg


@pytest.mark.parametrize("name", ["C1_binary_4096_k8", "C4_ternary_8192_k5",
                                  "C2_ternary_16384_k6"])
def test_save_matches_reference_file(rsr, name, tmp_path):
    from paper_2603_27462_b200 import artifact_io as aio
    meta = gd.meta()["large"][name]
    p = orc.random_matrix(meta["m"], meta["n"], meta["bitwidth"], meta["seed"])
    a = rsr.preprocess(rsr.PackedMatrix(meta["m"], meta["n"], meta["bitwidth"], p.data),
                       meta["k"])
    path = tmp_path / "a.rsra"
    aio.save(a, path)
    blob = path.read_bytes()
    ref = gd.meta()["rsra"]["large"][name]
    assert len(blob) == ref["bytes"] == a.file_bytes()
    assert hashlib.sha256(blob).hexdigest() == ref["sha"]
    # load it back: same arrays, bit-identical integer multiply
    b = aio.load(path)
    assert np.array_equal(b.words, a.words) and np.array_equal(b.perm, a.perm)
    vi = gd.int_vector(meta["n"], 1)
    assert np.array_equal(rsr.rsr_matvec(b, vi), rsr.rsr_matvec(a, vi))


def test_golden_file_loads_and_multiplies(rsr, tmp_path):
    from paper_2603_27462_b200 import artifact_io as aio
    path = tmp_path / "g.rsra"
    path.write_bytes(bytes.fromhex(gd.meta()["known_answer"]["golden_rsra_hex"]))
    a = aio.load(path)
    assert (a.m, a.n, a.k) == (2, 4, 2)
    # [[1,0,1,0],[1,1,0,0]] . [1,2,3,4] = [4, 3] (reference test_matcore.py:134-143)
    y = rsr.rsr_matvec(a, np.array([1, 2, 3, 4], np.int8))
    assert list(y) == [4, 3]


def test_corrupt_file_never_uploads(rsr, tmp_path):
    from paper_2603_27462_b200 import artifact_io as aio
    from paper_2603_27462_b200.errors import CorruptArtifact
    p = orc.random_matrix(20, 50, "ternary", 3)
    a = rsr.preprocess(rsr.PackedMatrix(20, 50, "ternary", p.data), 4)
    blob = bytearray(aio.to_bytes(a))
    # duplicate a column inside the first cell's permutation: structurally
    # well-formed bytes that fail the audit
    gc = int.from_bytes(blob[24:28], "little")
    perm0 = 24 + 8 + 8 * gc
    blob[perm0 + 2:perm0 + 4] = blob[perm0:perm0 + 2]
    with pytest.raises(CorruptArtifact):
        aio.from_bytes(bytes(blob))
