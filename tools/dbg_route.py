"""Debug: which fast route disagrees with the oracle on a given cloud."""
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1205_1171_b200 as H  # noqa: E402
from paper_1205_1171_b200 import fast  # noqa: E402
from oracle import oracle as O  # noqa: E402

rng = np.random.default_rng(11)
pts = rng.uniform(-1.0, 1.0, (20000, 3))
pts[:19990, 0] = rng.uniform(0.0, 1e-12, 19990)
exp = O.convex_hull_3d(pts)
BIG = 1 << 40
routes = {
    "default": {}, "leaf0": {"leaf_b": 0}, "leaf0_bigoff": {"leaf_b": 0, "big_kin": BIG},
    "tpj_all": {"tpj_min_jobs": 1, "big_kin": BIG, "leaf_b": 0},
    "warp_all": {"tpj_min_jobs": BIG, "big_kin": BIG, "leaf_b": 0, "mini": 0},
    "mini_all": {"tpj_min_jobs": BIG, "big_kin": BIG, "leaf_b": 0, "mini": 1},
    "big_all": {"big_kin": 2, "leaf_b": 0},
    "leaf3_warp": {"tpj_min_jobs": BIG, "big_kin": BIG},
}
for name, kv in routes.items():
    with fast.tuned(**kv):
        f0 = fast.FALLBACKS[0]
        r = H.convex_hull_3d(pts)
        print(f"{name:14s} equal={np.array_equal(r.faces, exp.faces)} nf={len(r.faces)} "
              f"fallback={fast.FALLBACKS[0]-f0} err={fast.LAST_ERROR[0]}")
# per-level logs of the oracle vs the fast engine could be compared here
