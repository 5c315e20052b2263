"""Kinetic movie tools (movie.py; the reference's snapshot_check,
oracle.py:142-196): the device's final lower-pass movie -- from the fused
path and from the exact engine -- replays to the independent 2D lower hull
at random probe times, both movies are the same canonical log, and a
corrupted log is caught."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1205_1171_b200 import movie
from paper_1205_1171_b200.generators import generate

pytestmark = pytest.mark.gpu

CLOUDS = [(100, "ball", 1), (64, "sphere", 2), (128, "gauss", 3), (1000, "cube", 4),
          (5000, "ball", 5)]


@pytest.mark.parametrize("n,dist,seed", CLOUDS)
def test_fast_and_exact_movies_replay(n, dist, seed, oracle_mod):
    pts = generate(n, dist, seed)
    c_f, l_f, log_f = movie.final_movie(pts, "fast")
    c_e, l_e, log_e = movie.final_movie(pts, "exact")
    assert np.array_equal(c_f, c_e)
    # the final log is canonical: both engines and the oracle agree
    end = int(np.argmax(log_e == movie.NIL))
    assert np.array_equal(log_f[:-1], log_e[:end])
    final = None
    for _lv, _k, buf, links in oracle_mod.level_logs(c_e):
        final = (buf, links)
    assert np.array_equal(log_e[:end], oracle_mod.group_log(final[0], 0))
    rng = np.random.default_rng(seed)
    for _ in range(25):
        t = movie.random_probe_time(rng)
        try:
            assert movie.snapshot_check(c_f, l_f, log_f, t)
            assert movie.snapshot_check(c_e, l_e, log_e, t)
        except movie.EventTimeCollision:
            continue


def test_corrupted_log_is_caught():
    pts = generate(400, "ball", 7)
    coords, links, log = movie.final_movie(pts, "fast")
    bad = log.copy()
    k = len(bad) - 1
    i = k // 2
    bad[i], bad[i + 1] = bad[i + 1], bad[i]  # two events out of order
    rng = np.random.default_rng(1)
    caught = False
    for _ in range(400):
        try:
            if not movie.snapshot_check(coords, links, bad, movie.random_probe_time(rng)):
                caught = True
                break
        except (movie.EventTimeCollision, RuntimeError, IndexError):
            caught = True
            break
    assert caught


def test_final_group_snapshot_ok_both_engines():
    pts = generate(128, "ball", 9)
    for engine in ("fast", "exact"):
        assert movie.final_group_snapshot_ok(pts, 10, np.random.default_rng(3), engine)
