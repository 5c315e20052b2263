"""Randomised families through the default routes (tools/robust_sweep.py at
test sizes): uniform clouds, small- and wide-range integer grids (ties,
perturbation), tight clusters, near-planar and thin-slab clouds, a shell
ball and a paraboloid (every point on the lower hull).  Faces, vertices
-- or the raised exception -- equal the C oracle's, whichever engine the
fast path hands the input to."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

import paper_1205_1171_b200 as H

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tools"))
from robust_sweep import FAMS, family, outcome  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [10_007, 65_537])
def test_families_match_oracle(n, oracle_mod):
    rng = np.random.default_rng(n)
    for fam in FAMS:
        pts = family(fam, n, rng)
        got, exp = outcome(H.convex_hull_3d, pts), outcome(oracle_mod.convex_hull_3d, pts)
        assert got[0] == exp[0], (fam, got[:2], exp[:2])
        if got[0] == "ok":
            assert np.array_equal(got[1], exp[1]) and np.array_equal(got[2], exp[2]), fam
        else:
            assert got[1:] == exp[1:], fam
