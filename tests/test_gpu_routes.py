"""Every kernel route of the fused fast path, forced on its own through the
routing knobs (csrc/fast.cu h3d_tune), reproduces the C oracle's faces bit
for bit with no exact-engine fallback:

* leaf kernel depth 0 / 3 / 4 (levels 1..B fused in shared memory);
* the time-split pipeline (big.cu) on almost every level (big_kin=16);
* lane-per-job on every level (tpj_min_jobs=1, pipeline off), on k_fast_tpj
  (its default and its 128-register build) and on lane.cu (coordinates / merged events staged in shared memory or not);
* warp-per-job on every level (tpj_min_jobs huge, pipeline off);
* each mini variant (one CTA per job in shared memory) wherever its jobs fit
  (tiny, small, medium, large2, large), and the huge one (one CTA per job, its arrays in global memory).
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_1205_1171_b200 as H
from paper_1205_1171_b200 import fast
from paper_1205_1171_b200.generators import generate, integer_cloud

pytestmark = pytest.mark.gpu

BIG_OFF = 1 << 40
ROUTES = {
    "default": {},
    "no_leaf_no_big": {"leaf_b": 0, "big_kin": BIG_OFF},
    "leaf4": {"leaf_b": 4},
    "leaf_b2_is_off": {"leaf_b": 2},
    "mini_spec_off": {"mini_spec": 0},  # top levels measured one by one
    "mini_seg16": {"mini_seg": 16},
    "big_everywhere": {"big_kin": 16, "mini": 0},
    "big_everywhere_no_leaf": {"big_kin": 2, "leaf_b": 0, "mini": 0},
    "tpj_everywhere": {"tpj_min_jobs": 1, "big_kin": BIG_OFF, "mini_tiny_ctas": 0, "lane": 0},
    "tpj_r128_everywhere": {"tpj_min_jobs": 1, "big_kin": BIG_OFF, "mini_tiny_ctas": 0, "lane": 0,
                            "tpj_cap_level": 40},
    # every lane-per-job level split at its median CTA: half the CTAs on the
    # small-pool launch, the rest through the overflow list
    "tpj_split_everywhere": {"tpj_min_jobs": 1, "big_kin": BIG_OFF, "mini_tiny_ctas": 0, "lane": 0,
                             "tpj_split": 2, "tpj_xyz_kb": 0, "tpj_xyz_ctas": 0},
    # lane per job + the large CTAs' jobs on a mini variant, wherever the
    # time-split pipeline would run (big_kin small)
    "hybrid_everywhere": {"big_kin": 16, "tpj_min_jobs": 1, "mini_tiny_ctas": 0, "mini_ctas": 0, "lane": 0},
    "lane_everywhere": {"tpj_min_jobs": 1, "big_kin": BIG_OFF, "mini_tiny_ctas": 0,
                        "lane_max_level": 40},
    "lane_staged_everywhere": {"tpj_min_jobs": 1, "big_kin": BIG_OFF, "mini_tiny_ctas": 0,
                               "lane_max_level": 40, "lane_xyz_kb": 200, "lane_stage": 1},
    "lane_own_everywhere": {"tpj_min_jobs": 1, "big_kin": BIG_OFF, "mini_tiny_ctas": 0,
                            "lane_max_level": 40, "lane_own": 40},
    "lane_events_staged": {"tpj_min_jobs": 1, "big_kin": BIG_OFF, "mini_tiny_ctas": 0,
                           "lane_max_level": 40, "lane_stage": 1},
    "warp_everywhere": {"tpj_min_jobs": BIG_OFF, "big_kin": BIG_OFF, "leaf_b": 0, "mini": 0},
    "mini_everywhere": {"tpj_min_jobs": BIG_OFF, "big_kin": BIG_OFF, "leaf_b": 0, "mini": 1,
                        "mini_ctas": BIG_OFF, "mini_tiny_ctas": 0},
    # every level past the one-wave limit: the medium / large2 / large
    # variants by fit (several CTAs per SM)
    "mini_multiwave_everywhere": {"tpj_min_jobs": BIG_OFF, "big_kin": BIG_OFF, "leaf_b": 0, "mini": 1,
                                  "mini_ctas": BIG_OFF, "mini_tiny_ctas": 0, "mini_one_wave": 0},
    "mini_huge_everywhere": {"tpj_min_jobs": BIG_OFF, "big_kin": BIG_OFF, "leaf_b": 0, "mini": 1,
                             "mini_ctas": 0, "mini_tiny_ctas": 0, "mini_huge_kin": 0,
                             "mini_huge_ctas": 1 << 20},
    "mini_huge_top": {"mini_huge_kin": 64},
    "mini_tiny_everywhere": {"tpj_min_jobs": BIG_OFF, "big_kin": BIG_OFF, "leaf_b": 0, "mini": 1,
                             "mini_ctas": 0, "mini_tiny_ctas": BIG_OFF},
}
CLOUDS = [("ball", 3001), ("sphere", 20000), ("cube", 65537), ("gauss", 9999), ("sphere", 4097)]


@pytest.fixture(scope="module")
def expected(oracle_mod):
    out = {}
    for dist, n in CLOUDS:
        pts = generate(n, dist, n % 13)
        out[(dist, n)] = (pts, oracle_mod.convex_hull_3d(pts))
    return out


@pytest.mark.parametrize("route", sorted(ROUTES))
def test_route_matches_oracle(route, expected):
    with fast.tuned(**ROUTES[route]):
        for (dist, n), (pts, exp) in expected.items():
            before = fast.FALLBACKS[0]
            r = H.convex_hull_3d(pts)
            assert fast.FALLBACKS[0] == before, (route, dist, n, fast.LAST_ERROR[0])
            assert np.array_equal(r.faces, exp.faces), (route, dist, n)
            assert np.array_equal(r.vertices, exp.vertices), (route, dist, n)


def test_integer_cloud_pipeline(oracle_mod):
    """Integer coordinates take the tie/perturbation path; the pipeline must
    still agree with the oracle (or hand the input to the exact engine, which
    then agrees)."""
    pts = integer_cloud(50000, 3)
    exp = oracle_mod.convex_hull_3d(pts)
    with fast.tuned(big_kin=16, mini=0):
        r = H.convex_hull_3d(pts)
    assert np.array_equal(r.faces, exp.faces)


def test_tune_roundtrip():
    old = fast.tune("big_kin", 1234)
    assert fast.tune("big_kin", old) == 1234
    with pytest.raises(KeyError):
        fast.tune("no_such_knob")


def test_presort_clustered_x_fallback(oracle_mod):
    """A tight x-cluster collapses the presort's 32-bit fixed-point keys into
    long equal runs; the presort must fall back to the exact 64-bit sort and
    still reproduce the reference."""
    rng = np.random.default_rng(11)
    pts = rng.uniform(-1.0, 1.0, (20000, 3))
    pts[:19990, 0] = rng.uniform(0.0, 1e-12, 19990)  # 19990 points within 1e-12 in x
    exp = oracle_mod.convex_hull_3d(pts)
    r = H.convex_hull_3d(pts)
    assert np.array_equal(r.faces, exp.faces)
    assert np.array_equal(r.vertices, exp.vertices)


KNOB_CHOICES = {
    "leaf_b": [0, 1, 2, 3, 4],
    "big_kin": [2, 16, 300, 1000, BIG_OFF],
    "big_total": [0, 1000, 200000],
    "big_max_jobs": [0, 1 << 18, BIG_OFF],
    "tpj_min_jobs": [1, 64, 4736, BIG_OFF],
    "tpj_xyz_kb": [0, 16, 200],
    "tpj_max_level": [2, 6, 40],
    "mini": [0, 1],
    "mini_ctas": [0, 4, 296, BIG_OFF],
    "mini_tiny_ctas": [0, 64, 8192, BIG_OFF],
    "mini_tiny_kin": [0, 160, BIG_OFF],
    "mini_seg": [1, 3, 16],
    "mini_spec": [0, 1],
    "mini_one_wave": [0, 296, BIG_OFF],
    "mini_huge_ctas": [0, 296, 4736],
    "mini_huge_kin": [0, 1000, BIG_OFF],
    "tpj_split": [0, 1, 2],
    "tpj_xyz_ctas": [0, 592],
    "tpj_cap_level": [0, 6, 40],
    "lane_own": [0, 4, 40],
    "lane_pf1": [0, 4, 40],
    "lane_pf2": [0, 5, 40],
    "lane": [0, 1],
    "interleave": [0, 1],
}


def test_random_knob_combinations(oracle_mod):
    """Any combination of routing knobs still reproduces the oracle (each
    level's route is chosen independently, so mixed routes must hand each
    other valid compact groups)."""
    rng = np.random.default_rng(2024)
    clouds = [generate(20000, "cube", 4), generate(6000, "ball", 5), generate(3000, "sphere", 6)]
    exp = [oracle_mod.convex_hull_3d(p) for p in clouds]
    for trial in range(24):
        kv = {k: int(rng.choice(v)) for k, v in KNOB_CHOICES.items()}
        with fast.tuned(**kv):
            for p, e in zip(clouds, exp):
                r = H.convex_hull_3d(p)
                assert np.array_equal(r.faces, e.faces), (trial, kv, len(p))
                assert np.array_equal(r.vertices, e.vertices), (trial, kv, len(p))


REPLAY_KNOBS = {
    "default": {},
    # every lane-per-job level split (small pool + overflow list), and the
    # hybrid route (lane per job + mini list launches) wherever the
    # pipeline would run: a replayed plan's pools and list grids must take
    # the next cloud's CTAs or resume measured
    "split": {"tpj_split": 2, "tpj_xyz_ctas": 0, "tpj_min_jobs": 1, "mini_tiny_ctas": 0, "lane": 0},
    "hybrid": {"big_kin": 16, "tpj_min_jobs": 1, "mini_tiny_ctas": 0, "mini_ctas": 0, "lane": 0},
}


@pytest.mark.parametrize("knobs", sorted(REPLAY_KNOBS))
@pytest.mark.parametrize("order", ["cube_then_sphere", "sphere_then_cube", "ball_then_int"])
def test_plan_replay_across_clouds(order, knobs, oracle_mod):
    """A call replays the level plan the previous call with the same n
    recorded (no per-level measurement); a cloud whose jobs do not fit the
    recorded launches makes the replay resume, measured, from that level --
    every result still equals the oracle, with no exact-engine fallback."""
    n = 50000
    first, second = order.split("_then_")

    def make(kind, seed):
        return integer_cloud(n, seed) if kind == "int" else generate(n, kind, seed)

    clouds = [make(first, 1), make(first, 2), make(second, 3), make(second, 4), make(first, 5)]
    with fast.tuned(plan=1, **REPLAY_KNOBS[knobs]):
        for pts in clouds:
            before = fast.FALLBACKS[0]
            r = H.convex_hull_3d(pts)
            exp = oracle_mod.convex_hull_3d(pts)
            if order != "ball_then_int":
                assert fast.FALLBACKS[0] == before
            assert np.array_equal(r.faces, exp.faces)
            assert np.array_equal(r.vertices, exp.vertices)
