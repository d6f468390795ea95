"""GPU bench harness / bytes-based autotuner:
host-side parts.  The bytes model is checked against the reference's
file_bytes for the BASELINE configs (tests/golden), the report schema against
the reference's ROW_FIELDS (pkg/src/rsrmv/bench.py:32-34)."""
import json

import pytest

from paper_2603_27462_b200 import gpubench as gb
from tests import golden_data as gd


@pytest.mark.parametrize("name", ["C1_binary_4096_k8", "C2_ternary_16384_k4",
                                  "C2_ternary_16384_k5", "C2_ternary_16384_k6",
                                  "C4_ternary_8192_k5"])
def test_bytes_model_tracks_reference_file_bytes(name):
    m = gd.meta()["large"][name]
    est = gb.bytes_model(m["m"], m["n"], m["k"], m["bitwidth"])
    assert abs(est - (m["file_bytes"] - 24)) / m["file_bytes"] < 0.02


def test_bytes_model_picks_the_reference_sweep_minimum():
    # C2 ternary bytes are minimal at k=6 (104.0 MB)
    costs = {k: gb.bytes_model(16384, 16384, k, "ternary") for k in range(2, 11)}
    assert min(costs, key=costs.get) == 6


def test_report_schema():
    r = gb.BenchReport([{"kind": "rsr", "m": 1, "n": 2, "bitwidth": "binary", "k": 2,
                         "ns_median": 1.0, "ns_p10": 1.0, "ns_p90": 1.0, "gather_adds": 3,
                         "scatter_adds": 4, "preprocess_ms": 0.1, "artifact_bytes": 64}],
                       [], 2, {"gpu": "x"})
    d = json.loads(r.to_json())
    assert set(d) == {"env", "best_k", "rows", "errors"}
    hdr = r.to_csv().splitlines()[0].split(",")
    assert tuple(hdr) == gb.ROW_FIELDS


@pytest.mark.parametrize("kw", [dict(reps=0), dict(warmup=-1), dict(density=1.5),
                                dict(bitwidth="int4"), dict(vector_dtype="f16"),
                                dict(baselines=("naive",))])
def test_config_validation(kw):
    base = dict(m=4, n=4, bitwidth="binary")
    base.update(kw)
    with pytest.raises(ValueError):
        gb.BenchConfig(**base)


def test_generators_match_reference_bench():
    from oracle import rsr_oracle as orc
    import numpy as np
    p = gb.random_matrix(33, 70, "ternary", 4)
    assert np.array_equal(p.data, orc.random_matrix(33, 70, "ternary", 4).data)
    assert np.array_equal(gb.random_vector(70, 3), orc.random_vector(70, 3))
