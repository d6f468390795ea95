"""The C-ABI library loads on CPU and exports exactly what include/rsr_b200.h
declares; host-side logic of the operator API (no kernel launches)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rsr_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rsr_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_header_symbols():
    from paper_2603_27462_b200 import _lib
    L = _lib.lib()
    declared = header_functions()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(L, name), f"{name} declared in rsr_b200.h but not exported"
    assert set(declared) == set(_lib.SIGNATURES), "ctypes signatures out of sync with header"
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (rsr_[a-z0-9_]+)$", out, flags=re.M))
    assert exported == set(declared)
    assert L.rsr_version().decode().startswith("rsr_b200")


def test_library_is_sm100a():
    from paper_2603_27462_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_queries_need_no_gpu():
    from paper_2603_27462_b200 import _lib
    L = _lib.lib()
    # small pattern spaces use shared-memory tables: no workspace
    assert L.rsr_group_workspace_bytes(16384, 16384, 1, 6, 16384) == 0
    assert L.rsr_group_workspace_bytes(64, 64, 0, 16, 64) > 0
    v = _lib.StreamView()
    v.tile_count = 1
    assert L.rsr_matvec_workspace_bytes(ctypes.byref(v)) == 0
    # argument validation happens before any launch
    assert L.rsr_group_count(None, 4, 4, 1, 0, 2, 4, None, None, None, None, None, 0,
                             None) == _lib.RSR_ERR_INVALID
    assert L.rsr_group_count(None, 4, 4, 1, 1, 11, 4, None, None, None, None, None, 0,
                             None) == _lib.RSR_ERR_K_TOO_LARGE
    assert L.rsr_matvec(ctypes.byref(v), None, 0, None, 0, None, 0, None) == _lib.RSR_ERR_INVALID
    # the peer-store form needs a peer table and at least one peer
    assert L.rsr_matvec_peers(ctypes.byref(v), None, 0, None, 2, None, 0, None) == \
        _lib.RSR_ERR_INVALID
    fake = (ctypes.c_void_p * 1)(1)
    assert L.rsr_matvec_peers(ctypes.byref(v), None, 0, fake, 0, None, 0, None) == \
        _lib.RSR_ERR_INVALID
    # tensor-core code matrix: u16 per (8-row group, column), columns padded to 64
    assert L.rsr_keymat_bytes(1639, 8192, 1, 5) == 128 * 1025 * 64 * 2   # C4: 16.8 MB
    assert L.rsr_keymat_bytes(3, 65, 0, 8) == 24 * 64                      # one 256-column step, 24 rows
    assert L.rsr_keymat_bytes(10, 100, 1, 9) == 96 * 64                    # k = 9: rows padded to 8
    assert L.rsr_keymat_bytes(10, 100, 1, 17) == 0                         # k > 16: no tc path
    assert L.rsr_matmul_tc(None, 8, 8, 1, 2, 0, 4, None, 1, 8, 1, None, 8, None, 0,
                           None) == _lib.RSR_ERR_INVALID


def test_status_mapping():
    from paper_2603_27462_b200 import _lib, errors
    _lib.check(0)
    with pytest.raises(errors.TileTooWide):
        _lib.check(_lib.RSR_ERR_TILE_TOO_WIDE)
    with pytest.raises(errors.CorruptArtifact):
        _lib.check(_lib.RSR_ERR_INVALID)
    with pytest.raises(errors.DimensionMismatch):
        _lib.check(_lib.RSR_ERR_DIMENSION)


def test_plan_and_caps():
    import paper_2603_27462_b200 as rsr
    p = rsr.make_plan(10, 7, 4, "binary")
    assert (p.block_count, p.last_block_height, p.tile_width, p.tile_count) == (3, 2, 7, 1)
    wide = rsr.make_plan(4, 100_000, 2, "binary")
    assert wide.tile_width == 32768 and wide.tile_count == 4
    with pytest.raises(rsr.KTooLarge):
        rsr.make_plan(4, 4, 17, "binary")
    with pytest.raises(rsr.KTooLarge):
        rsr.make_plan(4, 4, 11, "ternary")
    with pytest.raises(ValueError):
        rsr.make_plan(4, 4, 0, "binary")
    with pytest.raises(rsr.TileTooWide):
        rsr.make_plan(4, 4, 2, "binary", tile_width=65537)
    c2 = rsr.make_plan(16384, 16384, 6, "ternary")
    assert (c2.block_count, c2.last_block_height, c2.tile_count) == (2731, 4, 1)


def test_pack_group_layout():
    import paper_2603_27462_b200 as rsr
    assert rsr.pack_group(2, 1, 3, 0) == 0x0000000300010002
    assert rsr.pack_group(0, 5, 1, 0) == 0x0000000100050000
    assert rsr.pack_group(1, 1, 0, 2) == 0x0002000000010001
    for tup in [(0, 1, 1, 0), (65535, 65535, 65535, 0), (7, 9, 0b101, 0b010)]:
        assert rsr.unpack_group(rsr.pack_group(*tup)) == tup
    with pytest.raises(ValueError):
        rsr.pack_group(65536, 1, 0, 0)


def test_encode_decode_matches_oracle():
    import paper_2603_27462_b200 as rsr
    from oracle import rsr_oracle as orc
    rng = np.random.default_rng(0)
    for bw in ("binary", "ternary"):
        for (m, n) in [(1, 1), (3, 7), (17, 33), (8, 64)]:
            p = orc.random_matrix(m, n, bw, int(rng.integers(1 << 30)))
            ent = orc.decode(p)
            q = rsr.encode(ent, m, n, bw)
            assert np.array_equal(q.data, p.data)
            assert np.array_equal(rsr.decode(q), ent)
    with pytest.raises(rsr.OutOfAlphabet) as ei:
        rsr.encode(np.array([[0, 1], [2, 0]]), 2, 2, "binary")
    assert ei.value.to_json()["row"] == 1
    with pytest.raises(rsr.DimensionMismatch):
        rsr.encode(np.zeros(5), 2, 3, "ternary")


def test_error_json():
    import paper_2603_27462_b200 as rsr
    e = rsr.KTooLarge(11, "ternary")
    assert e.to_json() == {"error": "KTooLarge", "message": "k=11 exceeds the ternary cap of 10",
                           "k": 11, "bitwidth": "ternary"}


def test_ternarize_host_matches_oracle():
    import paper_2603_27462_b200 as rsr
    from oracle import rsr_oracle as orc
    w = np.random.default_rng(3).standard_normal((20, 30)) * 0.02
    a = rsr.ternarize_weights(w)
    b = orc.ternarize(w)
    assert np.array_equal(a.data, b.data) and a.weight_scale == b.weight_scale
    with pytest.raises(rsr.NonFinite):
        rsr.ternarize_weights(np.array([[1.0, np.nan]]))


def test_hostcall_binding_passes_through_without_a_gpu():
    """The CPython fast-call binding (csrc/hostcall.c) is built in-tree and
    reaches the C entry points: a null view returns RSR_ERR_INVALID before
    any CUDA call; bad arguments raise TypeError."""
    import ctypes
    import numpy as np
    from paper_2603_27462_b200 import _hostcall, _lib
    L = _lib.lib()
    f1 = ctypes.cast(L.rsr_matvec_host, ctypes.c_void_p).value
    f2 = ctypes.cast(L.rsr_fused_matvec_host, ctypes.c_void_p).value
    v = np.zeros(8, np.float32)
    assert _hostcall.matvec_host(f1, 0, v, _lib.RSR_F32, 1, 1, 1, 0, 0, 0) == _lib.RSR_ERR_INVALID
    assert _hostcall.fused_host(f2, 0, v, _lib.RSR_F32, 1.0, 1, 1, 1, 0, 0, 0) == \
        _lib.RSR_ERR_INVALID
    with pytest.raises(TypeError):
        _hostcall.matvec_host(f1, 0, v)
    with pytest.raises((TypeError, ValueError, BufferError)):
        _hostcall.matvec_host(f1, 0, np.zeros((4, 4), np.float32)[:, 0], 0, 1, 1, 1, 0, 0, 0)
