"""Wall time of convex_hull_3d variants (host/device input and result,
solver parallel/serial), repeated, plus a cProfile of the slowest."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1205_1171_b200 as H  # noqa: E402
from paper_1205_1171_b200.generators import generate  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
n, dist, seed, _ = bench.CONFIGS[cfg]
pinned = torch.from_numpy(generate(n, dist, seed)).pin_memory()
dpts = pinned.cuda()
V = {
    "host_par": lambda: H.convex_hull_3d(pinned),
    "host_ser": lambda: H.convex_hull_3d(pinned, solver="serial"),
    "host_par_dev": lambda: H.convex_hull_3d(pinned, return_device=True),
    "dev_par_dev": lambda: H.convex_hull_3d(dpts, return_device=True),
    "dev_par_host": lambda: H.convex_hull_3d(dpts),
}
for _ in range(3):
    for f in V.values():
        f()
torch.cuda.synchronize()
for name, f in V.items():
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(name, [round(t, 2) for t in ts])
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    V["host_par"]()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
