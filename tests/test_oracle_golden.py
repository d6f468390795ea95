"""Pin the CPU oracle (oracle/) against golden vectors made by importing the
reference package (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import rsr_oracle as orc
from tests import golden_data as gd


def _packed(case):
    m = case["meta"]
    return orc.Packed(m["m"], m["n"], m["bitwidth"], case["data"], m["weight_scale"])


@pytest.mark.parametrize("i", range(19))
def test_oracle_preprocess_matches_reference(i):
    case = gd.small_case(i)
    md = case["meta"]
    regen = orc.random_matrix(md["m"], md["n"], md["bitwidth"], md["seed"], md["density"])
    assert np.array_equal(regen.data, case["data"])
    a = orc.preprocess(_packed(case), md["k"], md["tile_width"])
    assert np.array_equal(a.words, case["words"])
    assert np.array_equal(a.perm, case["perm"])
    assert np.array_equal(a.group_offsets, case["go"])
    assert np.array_equal(a.perm_offsets, case["po"])
    assert np.array_equal(a.sort_steps, case["steps"])
    assert a.file_bytes() == md["file_bytes"]
    assert list(a.op_totals()) == md["op_totals"]
    assert [a.block_count, a.tile_count, a.tile_width] == md["plan"][:3]


@pytest.mark.parametrize("i", range(19))
def test_oracle_multiply_matches_reference(i):
    case = gd.small_case(i)
    md = case["meta"]
    a = orc.preprocess(_packed(case), md["k"], md["tile_width"])
    assert np.array_equal(orc.matvec_i8(a, case["vi"]), case["y_i8"])
    assert np.array_equal(orc.matvec_i8(a, case["vi"], threads=4), case["y_i8"])
    assert np.array_equal(orc.matvec_f32(a, case["vf"]), case["y_f32"])
    assert np.array_equal(orc.matvec_f32(a, case["vf"], threads=4), case["y_f32"])
    q, s = orc.absmax_quantize(case["vf"])
    assert np.array_equal(q, case["q"]) and s == md["q_scale"]
    q2, s2 = orc.quantize(case["vf"])
    assert np.array_equal(q2, case["q"]) and s2 == md["q_scale"]
    if md["bitwidth"] == "ternary":
        assert np.array_equal(orc.fused_matvec(a, case["vf"]), case["fused"])
        assert np.array_equal(orc.fused_matvec(a, case["vf"]), case["fused_mul"])
    assert np.array_equal(orc.naive_matvec(_packed(case), case["vi"]), case["naive_i32"])
    assert np.array_equal(orc.naive_matvec(_packed(case), case["vf"]), case["naive_f64"])


def test_known_answers():
    ka = gd.meta()["known_answer"]
    m = orc.encode(np.array([[1, 0, 1, 0], [1, 1, 0, 0]], np.int8), 2, 4, "binary")
    a = orc.preprocess(m, 2)
    assert list(a.perm) == ka["perm_2x4"] == [2, 1, 0]
    assert [int(w) for w in a.words] == ka["words_2x4"]
    assert list(a.op_totals()) == ka["ops_2x4"] == [3, 4, 3]
    assert a.file_bytes() == 64 == len(bytes.fromhex(ka["golden_rsra_hex"]))
    mt = orc.encode(np.array([[1, -1, 0], [0, 1, 1]], np.int8), 2, 3, "ternary")
    at = orc.preprocess(orc.Packed(2, 3, "ternary", mt.data, 0.5), 2)
    y = orc.fused_matvec(at, np.array([2.0, 3.0, 5.0], np.float32))
    assert [int(x) for x in y.view(np.uint32)] == ka["fused_known_bits"]
    exp = (np.array([-25, 203], np.float64) * (0.5 / 25.4)).astype(np.float32)
    assert np.array_equal(y, exp)


def test_oracle_large_c1_matches_reference_digests():
    rec = gd.meta()["large"]["C1_binary_4096_k8"]
    p = orc.random_matrix(4096, 4096, "binary", 0)
    assert gd.sha(p.data) == rec["data_sha"]
    a = orc.preprocess(p, 8)
    assert gd.sha(a.words) == rec["words_sha"]
    assert gd.sha(a.perm) == rec["perm_sha"]
    assert gd.sha(a.group_offsets) == rec["go_sha"]
    assert gd.sha(a.perm_offsets) == rec["po_sha"]
    assert gd.sha(a.sort_steps) == rec["steps_sha"]
    assert a.file_bytes() == rec["file_bytes"]
    vi = gd.int_vector(4096, 0)
    assert np.array_equal(orc.matvec_i8(a, vi, threads=4),
                          gd.large_output("C1_binary_4096_k8_y_i8"))
    vb = gd.bf16_round(orc.random_vector(4096, 0))
    assert np.array_equal(orc.matvec_f32(a, vb), gd.large_output("C1_binary_4096_k8_y_bf16v"))


def test_oracle_large_c4_matches_reference_digests():
    name = "C4_ternary_8192_k5"
    rec = gd.meta()["large"][name]
    p = orc.random_matrix(8192, 8192, "ternary", 0)
    a = orc.preprocess(p, 5)
    assert gd.sha(a.words) == rec["words_sha"]
    assert gd.sha(a.perm) == rec["perm_sha"]
    vb = gd.bf16_round(orc.random_vector(8192, 0))
    assert np.array_equal(orc.matvec_f32(a, vb, threads=4), gd.large_output(name + "_y_bf16v"))
    assert np.array_equal(orc.fused_matvec(a, vb, threads=4),
                          gd.large_output(name + "_fused_bf16v"))
