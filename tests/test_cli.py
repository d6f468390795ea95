"""CLI helpers and `.rsrm` files on the host (reference cli.py:36-71,
matcore.py:217-258).  The GPU commands are exercised in test_gpu_cli.py."""
import json

import numpy as np
import pytest

from paper_2603_27462_b200 import cli
from paper_2603_27462_b200 import matcore as mc
from paper_2603_27462_b200.errors import CorruptArtifact


def test_parse_ks():
    assert cli.k_list("2,4,8") == [2, 4, 8]
    assert cli.k_list(" 3..6 ") == [3, 4, 5, 6]


def test_load_vector_auto_dtype(tmp_path):
    assert cli.read_vector("[1, -2, 3]", "auto").dtype == np.int8
    assert cli.read_vector("[1.5, 2]", "auto").dtype == np.float32
    assert cli.read_vector("[300, 2]", "auto").dtype == np.float32
    assert cli.read_vector("[1, 2]", "float32").dtype == np.float32
    p = tmp_path / "v.txt"
    p.write_text("1 2\n3")
    assert list(cli.read_vector(str(p), "auto")) == [1, 2, 3]
    np.save(tmp_path / "v.npy", np.array([0.5, 1.0], np.float32))
    assert cli.read_vector(str(tmp_path / "v.npy"), "auto").dtype == np.float32
    with pytest.raises(FileNotFoundError):
        cli.read_vector(str(tmp_path / "missing.npy"), "auto")


def test_bench_config_validation():
    cfg = cli.bench_config({"m": 8, "n": 8, "bitwidth": "binary", "k_list": [2, 4]})
    assert cfg.k_list == [2, 4]
    with pytest.raises(ValueError):
        cli.bench_config({"m": 8, "n": 8})
    with pytest.raises(ValueError):
        cli.bench_config({"m": 8, "n": 8, "bitwidth": "binary", "colour": 1})
    with pytest.raises(ValueError):
        cli.bench_config([1, 2])


def test_rsrm_round_trip_and_errors(tmp_path):
    e = np.array([[1, -1, 0, 1], [0, 1, 1, -1], [1, 1, 1, 0]], np.int8)
    m = mc.PackedMatrix(3, 4, "ternary", mc.encode(e, 3, 4, "ternary").data, 0.25)
    path = tmp_path / "m.rsrm"
    mc.save_rsrm(m, path)
    blob = path.read_bytes()
    assert len(blob) == 18 + 12
    q = mc.load_rsrm(path)
    assert np.array_equal(mc.decode(q), e) and q.weight_scale == 0.25
    for bad in (b"XXXX" + blob[4:], blob[:-1], blob[:18] + bytes([5]) + blob[19:],
                blob[:4] + bytes([9]) + blob[5:]):
        path.write_bytes(bad)
        with pytest.raises(CorruptArtifact):
            mc.load_rsrm(path)


def test_errors_are_single_json_objects(capsys, tmp_path):
    rc = cli.main(["bench", "--config", str(tmp_path / "missing.json")])
    assert rc == 1
    assert json.loads(capsys.readouterr().out)["error"] == "FileNotFound"
    rc = cli.main(["bench", "--config", '{"m": 4}'])
    assert rc == 1
    assert json.loads(capsys.readouterr().out)["error"] == "InvalidConfig"
