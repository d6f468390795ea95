"""`.rsra` files on the host (no GPU): the writer reproduces the reference
writer's bytes (sha256 of reference-written files, tests/golden/
make_rsra_golden.py) and the GOLDEN 64-byte file (reference
test_artifact_io.py:18-25); the reader round-trips and rejects corrupt files
like reference artifact_io.py:58-121."""
import hashlib
import struct

import numpy as np
import pytest

from paper_2603_27462_b200 import artifact_io as aio
from paper_2603_27462_b200.errors import CorruptArtifact
from tests import golden_data as gd


def small_args(i):
    c = gd.small_case(i)
    meta = c["meta"]
    tw = meta["plan"][2]
    return (meta["m"], meta["n"], meta["k"], meta["bitwidth"], tw, meta["weight_scale"],
            c["words"], c["perm"], c["go"], c["po"])


@pytest.mark.parametrize("i", range(gd.n_small()))
def test_writer_matches_reference_bytes(i):
    blob = aio.serialize(*small_args(i))
    ref = gd.meta()["rsra"]["small"][str(i)]
    assert len(blob) == ref["bytes"] == gd.meta()["small"][i]["file_bytes"]
    assert hashlib.sha256(blob).hexdigest() == ref["sha"]


@pytest.mark.parametrize("i", range(gd.n_small()))
def test_round_trip(i):
    args = small_args(i)
    d = aio.parse(aio.serialize(*args))
    for key, want in zip(("words", "perm", "group_offsets", "perm_offsets"), args[6:]):
        assert np.array_equal(d[key], want), key
    assert (d["m"], d["n"], d["k"], d["bitwidth"]) == args[:4]


def golden_blob():
    return bytes.fromhex(gd.meta()["known_answer"]["golden_rsra_hex"])


def test_golden_file():
    blob = golden_blob()
    assert len(blob) == 64
    d = aio.parse(blob)
    assert (d["m"], d["n"], d["k"], d["bitwidth"]) == (2, 4, 2, "binary")
    assert list(d["perm"]) == [2, 1, 0]
    assert [int(w) for w in d["words"]] == gd.meta()["known_answer"]["words_2x4"]
    assert aio.serialize(2, 4, 2, "binary", 4, 1.0, d["words"], d["perm"], d["group_offsets"],
                         d["perm_offsets"]) == blob


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XXXX" + b[4:], "not an .rsra"),
    (lambda b: b[:4] + bytes([2]) + b[5:], "version"),
    (lambda b: b[:5] + bytes([7]) + b[6:], "bitwidth"),
    (lambda b: b[:-3], "truncated"),
    (lambda b: b + b"\x00\x00\x00\x00", "trailing"),
    (lambda b: b[:-1] + b"\x01", "padding"),
    (lambda b: b[:6] + bytes([0]) + b[7:], "invalid header"),  # k = 0
])
def test_corrupt_files(mutate, msg):
    with pytest.raises(CorruptArtifact, match=msg):
        aio.parse(mutate(golden_blob()))


def test_empty_cells_and_header_only_shapes():
    # an all-zero 3x5 binary matrix at k=2: two cells, no groups, no padding
    blob = aio.serialize(3, 5, 2, "binary", 5, 1.0, np.zeros(0, np.uint64),
                         np.zeros(0, np.uint16), [0, 0, 0], [0, 0, 0])
    assert len(blob) == 24 + 2 * 8
    assert struct.unpack_from("<II", blob, 24) == (0, 0)
    d = aio.parse(blob)
    assert d["words"].size == 0 and d["perm"].size == 0
