"""Host-side logic that needs no GPU: generators, error mapping, level
arithmetic, the host perturb_ties helper."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1205_1171_b200 import errors as E
from paper_1205_1171_b200.engine import level_count
from paper_1205_1171_b200.generators import generate, integer_cloud


def test_level_count_examples():
    # tests/test_serial_parallel.py:41-47 in the reference
    assert level_count(1) == 0
    assert level_count(2) == 1
    assert level_count(3) == 2
    assert level_count(2**23) == 23
    with pytest.raises(ValueError):
        level_count(0)


def test_generator_digests_match_reference(large_json):
    import hashlib

    if not large_json:
        pytest.skip("large.json not generated")
    for name, gen in (("C2_ball_2^20", lambda: generate(2**20, "ball", 0)),
                      ("C3_sphere_2^20", lambda: generate(2**20, "sphere", 0)),
                      ("int_2^20_R2^31", lambda: integer_cloud(2**20, 0))):
        if name in large_json:
            pts = gen()
            assert hashlib.sha256(pts.tobytes()).hexdigest() == large_json[name]["points_sha256"]


def test_generator_small_cases_match_golden(small):
    for dist in ("ball", "sphere", "cube", "gauss"):
        for n in (4, 100, 1000):
            assert np.array_equal(generate(n, dist, n), small.case(f"{dist}_{n}")["pts"])


def test_mixed_definition():
    pts = generate(1024, "mixed", 0)
    assert pts.shape == (1024, 3)
    r = np.linalg.norm(pts, axis=1)
    assert (r[-8:] > 1.99).all() and (r[:-8] <= 1.0).all()


def test_error_mapping_matches_reference_classes():
    with pytest.raises(E.MergeOverflowError):
        E.check_merge(E.E_OVERFLOW)
    with pytest.raises(E.BridgeWalkError, match="bridge walk"):
        E.check_merge(E.E_BRIDGE)
    with pytest.raises(E.BridgeWalkError, match="chain state corrupt"):
        E.check_merge(E.E_CHAIN)
    with pytest.raises(E.ChainError):
        E.check_store(E.E_CHAIN)
    with pytest.raises(E.LogError):
        E.check_store(E.E_COUNT)
    with pytest.raises(E.LogError):
        E.check_store(E.E_UNTERMINATED)
    with pytest.raises(ValueError, match="finite"):
        E.check_api(E.E_NONFINITE)
    for code, msg in ((E.E_COINCIDENT, "coincide"), (E.E_COLLINEAR, "collinear"),
                      (E.E_COPLANAR, "coplanar"), (E.E_TIES, "survived"),
                      (E.E_NOFACETS, "no facets")):
        with pytest.raises(E.DegenerateInputError, match=msg):
            E.check_api(code)
    assert issubclass(E.DegenerateInputError, ValueError)
    assert E.check_merge(5) == 5


def test_perturb_ties_host_helper():
    # tests/test_api.py:91-105 in the reference
    from paper_1205_1171_b200 import perturb_ties

    pts = np.array([[0.0, 1, 2], [1.0, 0, 0], [2.0, -1, 3]])
    assert np.array_equal(perturb_ties(pts), pts)
    eps16 = 16 * np.finfo(np.float64).eps
    pts = np.array([[1.0, 0, 0], [1.0, 1, 1], [2.0, 0, 0]])
    out = perturb_ties(pts)
    assert out[1, 0] == 1.0 + eps16 and pts[1, 0] == 1.0


def test_integer_cloud_takes_tie_path(oracle_mod):
    pts = integer_cloud(5000, 3, half_range=2**12)
    _, _, pert = oracle_mod.sort_and_perturb(pts)
    assert pert


def test_snapshot_check_on_the_oracle_movie(oracle_mod):
    """movie.snapshot_check (host replay) accepts the pinned oracle's final
    movie at random probe times and rejects a chain it does not match."""
    import numpy as np

    from paper_1205_1171_b200 import movie
    from paper_1205_1171_b200.generators import generate

    pts = generate(200, "ball", 11)
    coords = pts[np.lexsort((pts[:, 2], pts[:, 1], pts[:, 0]))]
    final = None
    for _lv, _k, buf, links in oracle_mod.level_logs(coords):
        final = (buf, links)
    buf, links = final
    rng = np.random.default_rng(0)
    checked = 0
    while checked < 20:
        try:
            assert movie.snapshot_check(coords, links.astype(np.int64), buf, movie.random_probe_time(rng))
            checked += 1
        except movie.EventTimeCollision:
            pass
    # an empty log leaves the t = -inf chain: wrong at a late time
    assert not movie.snapshot_check(coords, links.astype(np.int64), np.array([-1]), 1e6)
    assert movie.lower_hull_2d([(0.0, 0.0), (1.0, -1.0), (2.0, 0.0), (3.0, 5.0)]) == [0, 1, 2, 3]
