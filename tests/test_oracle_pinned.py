"""The C restatement (oracle/hull_oracle.c) pinned against the reference:
golden outputs of the unmodified reference and the reference test suite's
known-answer examples.  CPU only."""

from __future__ import annotations

import numpy as np
import pytest


def test_oracle_matches_reference_outputs(small, oracle_mod):
    for name in small.names:
        c = small.case(name)
        got = oracle_mod.convex_hull_3d(c["pts"])
        assert np.array_equal(got.faces, c["faces"]), name
        assert np.array_equal(got.vertices, c["vertices"]), name
        assert (got.lower_events, got.upper_events) == (c["lower"], c["upper"]), name
        assert got.perturbed == c["perturbed"], name


def test_oracle_level_logs_and_links(levels_npz, oracle_mod):
    names = [str(s) for s in levels_npz["__names__"]]
    for name in names:
        P = levels_npz[f"{name}__pts"]
        for lv, _, buf, links in oracle_mod.level_logs(P):
            assert np.array_equal(buf, levels_npz[f"{name}__slots{lv}"]), (name, lv)
            assert np.array_equal(links, levels_npz[f"{name}__links{lv}"]), (name, lv)


def test_event_time_kats(oracle_mod):
    # tests/test_geometry.py:33-44 in the reference
    P = np.array([[0, 0, 0], [1, 0, 1], [2, 1, 0]], dtype=np.float64)
    assert oracle_mod.evtime(P, 0, 1, 2) == -2.0
    Q = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], dtype=np.float64)
    assert oracle_mod.evtime(Q, 0, 1, 2) == np.inf
    assert oracle_mod.evtime(Q, -1, 1, 2) == np.inf


def test_act_kats(oracle_mod):
    # tests/test_store.py:29-51 in the reference
    import ctypes

    L = oracle_mod.lib()
    K = np.array([[-1, 1], [0, 2], [1, -1]], dtype=np.int32)
    p = K.ctypes.data_as(ctypes.c_void_p)
    assert L.orc_act(p, 1) == 0
    assert K[0, 1] == 2 and K[2, 0] == 0 and K[1, 0] == 0 and K[1, 1] == 2
    assert L.orc_act(p, 1) == 0
    assert K[0, 1] == 1 and K[2, 0] == 1
    assert L.orc_act(p, 0) == -1


def test_bridge_kats(oracle_mod):
    # tests/test_merge.py:38-49 in the reference
    import ctypes

    L = oracle_mod.lib()
    P = np.array([[0.0, 0, 0], [1, 0, -1], [2, 0, -1], [3, 0, 0]])
    # level-1 merges link the pairs (0,1) and (2,3)
    K = np.full((4, 2), -1, dtype=np.int32)
    A = np.full(8, -1, dtype=np.int32)
    B = np.full(8, -1, dtype=np.int32)
    vp = ctypes.c_void_p
    assert L.orc_merge(P.ctypes.data_as(vp), K.ctypes.data_as(vp), A.ctypes.data_as(vp),
                       B.ctypes.data_as(vp), 0, 1, 2) == 0
    assert L.orc_merge(P.ctypes.data_as(vp), K.ctypes.data_as(vp), A.ctypes.data_as(vp),
                       B.ctypes.data_as(vp), 2, 3, 4) == 0
    u, v = ctypes.c_int64(1), ctypes.c_int64(2)
    assert L.orc_find_bridge(P.ctypes.data_as(vp), K.ctypes.data_as(vp), ctypes.byref(u),
                             ctypes.byref(v), 4) == 0
    assert (u.value, v.value) == (1, 2)


def test_perturb_exact_values(oracle_mod):
    # tests/test_api.py:96-105 in the reference
    eps16 = 16 * np.finfo(np.float64).eps
    pts = np.array([[1.0, 0, 0], [1.0, 1, 1], [2.0, 0, 0]])
    out, order, pert = oracle_mod.sort_and_perturb(pts)
    assert pert
    assert out[0, 0] == 1.0 and out[1, 0] == 1.0 + eps16 and out[2, 0] == 2.0
    assert order.tolist() == [0, 1, 2]


def test_reference_itself_when_present(oracle_mod):
    ref = oracle_mod.reference()
    if ref is None:
        pytest.skip("reference not built here (oracle/build_ref.sh)")
    for dist in ("ball", "cube"):
        pts = ref.generate(3000, dist, 11)
        r = ref.convex_hull_3d(pts)
        o = oracle_mod.convex_hull_3d(pts)
        assert np.array_equal(r.faces, o.faces)
