"""Every kernel route of the fast path (tests/test_gpu_routes.py ROUTES) on
small clouds, checked against the oracle -- the workload the
compute-sanitizer runs (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_routes.py [n_max]
"""
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_1205_1171_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1205_1171_b200 import fast  # noqa: E402
from paper_1205_1171_b200.generators import generate, integer_cloud  # noqa: E402
from test_gpu_routes import ROUTES  # noqa: E402

n_max = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
clouds = [("ball", 3001), ("sphere", 5000), ("cube", 20000), ("gauss", 999)]
bad = 0
for route, kv in sorted(ROUTES.items()):
    with fast.tuned(**kv):
        for dist, n in clouds:
            if n > n_max:
                continue
            pts = generate(n, dist, n % 13)
            r = H.convex_hull_3d(pts)
            e = O.convex_hull_3d(pts)
            ok = np.array_equal(r.faces, e.faces)
            r2 = H.convex_hull_3d(generate(n, dist, n % 13 + 1))  # replays the recorded level plan
            ok = ok and np.array_equal(r2.faces, O.convex_hull_3d(generate(n, dist, n % 13 + 1)).faces)
            bad += not ok
            print(f"{route:24s} {dist:7s} {n:6d} {'ok' if ok else 'MISMATCH'}", flush=True)
pts = integer_cloud(4000, 3)
ok = np.array_equal(H.convex_hull_3d(pts).faces, O.convex_hull_3d(pts).faces)
print("integer 4000", "ok" if ok else "MISMATCH")
bad += not ok
print("routes checked, mismatches:", bad)
sys.exit(1 if bad else 0)
