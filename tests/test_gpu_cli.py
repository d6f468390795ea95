"""The CLI end to end on the GPU, plus the toy
runtime's GPU backend (rank 3): JSON on stdout, `.rsra` output byte-identical
to the reference writer, toy decode token-identical to the reference's."""
import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from tests import golden_data as gd

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_cli(*args, whole=False):
    r = subprocess.run([sys.executable, "-m", "paper_2603_27462_b200.cli", *args],
                       capture_output=True, text=True, cwd=ROOT, timeout=600)
    if whole:  # one (indented) JSON document
        return r.returncode, [json.loads(r.stdout)]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.strip()]
    return r.returncode, lines


@pytest.mark.parametrize("i", [4, 5, 8])
def test_preprocess_then_multiply(i, tmp_path):
    from paper_2603_27462_b200 import matcore as mc
    c = gd.small_case(i)
    meta = c["meta"]
    m = mc.PackedMatrix(meta["m"], meta["n"], meta["bitwidth"], c["data"], meta["weight_scale"])
    src = tmp_path / "m.rsrm"
    mc.save_rsrm(m, src)
    out = tmp_path / "m.rsra"
    args = ["preprocess", "--in", str(src), "--k", str(meta["k"]), "--out", str(out)]
    if meta["tile_width"]:
        args += ["--tile-width", str(meta["tile_width"])]
    rc, lines = run_cli(*args)
    assert rc == 0 and lines[0]["artifact_bytes"] == meta["file_bytes"]
    assert hashlib.sha256(out.read_bytes()).hexdigest() == gd.meta()["rsra"]["small"][str(i)]["sha"]
    vi = c["vi"]
    rc, lines = run_cli("multiply", "--artifact", str(out), "--vec",
                        json.dumps([int(x) for x in vi]), "--dtype", "int8")
    assert rc == 0 and lines[0]["y"] == [int(x) for x in c["y_i8"]]


def test_decode_matches_reference_tokens():
    for t in gd.meta()["toyrt"]:
        rc, lines = run_cli("decode", "--seed", str(t["seed"]), "--d", str(t["d"]),
                            "--V", str(t["V"]), "--depth", str(t["depth"]), "--k", str(t["k"]),
                            "--steps", str(t["steps"]),
                            "--prompt", ",".join(str(x) for x in t["prompt"]),
                            "--backend", "both")
        assert rc == 0 and lines[0]["sequences_equal"]
        assert lines[0]["tokens"] == t["tokens"]


def test_toy_model_digest_matches_reference():
    from paper_2603_27462_b200 import toyrt
    t = gd.meta()["toyrt"][0]
    model = toyrt.build_toy_model(t["seed"], t["d"], t["V"], t["depth"], k=t["k"])
    assert model.digest() == t["digest"]


def test_sweep_bench_autotune():
    rc, lines = run_cli("sweep", "--m", "512", "--n", "1024", "--bitwidth", "ternary",
                        "--ks", "4..6", "--reps", "5")
    assert rc == 0 and [r["k"] for r in lines] == [4, 5, 6]
    assert all(r["ns_median"] > 0 and r["kind"] == "rsr" for r in lines)
    rc, lines = run_cli("bench", "--config",
                        json.dumps({"m": 256, "n": 512, "bitwidth": "binary", "k_list": [4, 8],
                                    "reps": 5}), whole=True)
    rep = lines[0]
    assert rc == 0 and rep["best_k"] in (4, 8)
    assert {r["kind"] for r in rep["rows"]} == {"rsr", "cublas_bf16"}
    rc, lines = run_cli("autotune", "--m", "1024", "--n", "1024", "--bitwidth", "ternary",
                        "--budget-ms", "200")
    assert rc == 0 and 1 <= lines[0]["best_k"] <= 10
    rc, lines = run_cli("bench", "--config", '{"m": 4}')
    assert rc == 1 and lines[0]["error"] == "InvalidConfig"
