"""Cost of the per-level stats of solver="parallel" (device events)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1205_1171_b200 as H  # noqa: E402
from paper_1205_1171_b200 import fast  # noqa: E402
from paper_1205_1171_b200.api import presort  # noqa: E402
from paper_1205_1171_b200.generators import generate  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
n, dist, seed, _ = bench.CONFIGS[cfg]
pts = torch.from_numpy(generate(n, dist, seed)).cuda()


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


sp, _, _ = presort(pts)
print("api parallel", round(t(lambda: H.convex_hull_3d(pts, return_device=True)), 3))
print("api serial", round(t(lambda: H.convex_hull_3d(pts, solver="serial", return_device=True)), 3))
print("run_both", round(t(lambda: fast.run_both(sp)), 3))


def prof_run():
    fast.profile_enable(True)
    fast.run_both(sp)
    fast.profile_enable(False)
    fast.profile_collect()


def prof_nocollect():
    fast.profile_enable(True)
    fast.run_both(sp)
    fast.profile_enable(False)


print("run_both + profile", round(t(prof_run), 3))
print("run_both + profile (no collect)", round(t(prof_nocollect), 3))
fast.profile_collect()
