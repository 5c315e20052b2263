"""Near-degenerate stress: every kernel route against the oracle (the C
restatement pinned to the reference) on inputs where event times nearly tie,
a bridge foot can be deleted by a child event, x values crowd, or whole
groups are (nearly) coplanar.  The fast path may hand an input to the exact
engine; either way faces, vertices and raised exceptions must equal the
reference's."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1205_1171_b200 as H
from paper_1205_1171_b200 import fast

pytestmark = pytest.mark.gpu

BIG_OFF = 1 << 40
ROUTES = {
    "default": {},
    "tpj": {"tpj_min_jobs": 1, "big_kin": BIG_OFF, "leaf_b": 0, "mini_tiny_ctas": 0},
    "warp": {"tpj_min_jobs": BIG_OFF, "big_kin": BIG_OFF, "leaf_b": 0, "mini": 0},
    "mini": {"tpj_min_jobs": BIG_OFF, "big_kin": BIG_OFF, "leaf_b": 0, "mini": 1,
             "mini_ctas": BIG_OFF, "mini_tiny_ctas": 0},
    "mini_tiny": {"tpj_min_jobs": BIG_OFF, "big_kin": BIG_OFF, "leaf_b": 0, "mini": 1,
                  "mini_ctas": 0, "mini_tiny_ctas": BIG_OFF},
    "big": {"big_kin": 2, "leaf_b": 0, "mini": 0},
    "leaf4": {"leaf_b": 4},
}


def family(name: str, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    n = 6000
    p = rng.uniform(-1.0, 1.0, (n, 3))
    if name.startswith("slab"):
        ax = "xyz".index(name[-1])
        p[: n - 8, ax] = rng.uniform(0.0, 1e-12, n - 8)
    elif name == "near_plane":
        p[:, 2] = p[:, 0] * 0.3 + p[:, 1] * 0.7 + rng.normal(0.0, 1e-11, n)
        p[:4, 2] += 1.0
    elif name == "clusters":
        c = rng.uniform(-1.0, 1.0, (6, 3))
        p = c[rng.integers(0, 6, n)] + rng.normal(0.0, 1e-9, (n, 3))
    elif name == "int_small":
        p = rng.integers(-2**8, 2**8, (n, 3)).astype(np.float64)
    elif name == "int_mid":
        p = rng.integers(-2**14, 2**14, (n, 3)).astype(np.float64)
    elif name == "sphere_tight":
        v = rng.normal(size=(n, 3))
        p = v / np.linalg.norm(v, axis=1, keepdims=True)
    return p


FAMILIES = ["slab_x", "slab_y", "slab_z", "near_plane", "clusters", "int_small", "int_mid",
            "sphere_tight"]


def outcome(fn, pts):
    try:
        r = fn(pts)
        return ("ok", r.faces.copy(), r.vertices.copy())
    except Exception as exc:  # DegenerateInputError, merge/chain errors
        kind = type(exc).__name__
        msg = str(exc) if kind == "DegenerateInputError" else ""
        return ("err", "Degenerate" if kind == "DegenerateInputError" else "kernel", msg)


@pytest.mark.parametrize("fam", FAMILIES)
def test_stress_family_all_routes(fam, oracle_mod):
    for seed in (1, 2):
        pts = family(fam, seed)
        exp = outcome(oracle_mod.convex_hull_3d, pts)
        for route, kv in ROUTES.items():
            with fast.tuned(**kv):
                got = outcome(H.convex_hull_3d, pts)
            assert got[0] == exp[0], (fam, seed, route, got[:2], exp[:2])
            if exp[0] == "err":
                assert got[1:] == exp[1:], (fam, seed, route, got, exp)
            else:
                assert np.array_equal(got[1], exp[1]), (fam, seed, route)
                assert np.array_equal(got[2], exp[2]), (fam, seed, route)
