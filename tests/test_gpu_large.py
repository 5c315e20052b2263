"""BASELINE.json configs at full size on the B200: bit-exact against the
unmodified reference through sha256 digests of its face/vertex arrays
(tests/golden/large.json), plus size-independent hull properties."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import paper_1205_1171_b200 as H
from paper_1205_1171_b200 import fast
from paper_1205_1171_b200.generators import generate, integer_cloud

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GEN = {
    "C2_ball_2^20": lambda: generate(2**20, "ball", 0),
    "C3_sphere_2^20": lambda: generate(2**20, "sphere", 0),
    "int_2^20_R2^31": lambda: integer_cloud(2**20, 0),
    "C4_cube_2^24": lambda: generate(2**24, "cube", 0),
    "C5_mixed_2^27": lambda: generate(2**27, "mixed", 0),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(GEN))
def test_large_config_matches_reference_digest(name, large_json):
    exp = large_json[name]
    pts = GEN[name]()
    assert sha(pts) == exp["points_sha256"]
    fb = fast.FALLBACKS[0]
    r = H.convex_hull_3d(pts)
    # the fused fast path produced it (no exact-engine rerun)
    assert fast.FALLBACKS[0] == fb, f"fast path declined the input (err {fast.LAST_ERROR[0]})"
    assert len(r.faces) == exp["nfaces"] and len(r.vertices) == exp["nvertices"]
    assert (r.stats.lower_events, r.stats.upper_events) == (exp["lower_events"], exp["upper_events"])
    assert r.stats.perturbed == exp["perturbed"]
    assert sha(r.faces) == exp["faces_sha256"]
    assert sha(r.vertices) == exp["vertices_sha256"]
    # Euler: a simplicial 3-polytope has F = 2V - 4
    assert len(r.faces) == 2 * len(r.vertices) - 4
