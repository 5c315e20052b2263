"""Where the end-to-end time of convex_hull_3d(host input) goes."""
import os
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1205_1171_b200 as H  # noqa: E402
from paper_1205_1171_b200 import api, fast  # noqa: E402
from paper_1205_1171_b200.generators import generate  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
n, dist, seed, _ = bench.CONFIGS[cfg]
pinned = torch.from_numpy(generate(n, dist, seed)).pin_memory()
for _ in range(3):
    H.convex_hull_3d(pinned)
torch.cuda.synchronize()
T = {}
def tick(name, t0):
    torch.cuda.synchronize()
    T[name] = T.get(name, 0) + (time.perf_counter() - t0) * 1e3
    return time.perf_counter()
for _ in range(3):
    t = time.perf_counter()
    dev = torch.device("cuda", 0)
    pts = api._to_device(pinned, dev); t = tick("h2d", t)
    sp, order, pert = api.presort(pts); t = tick("presort", t)
    res = fast.run_both(sp); t = tick("merges+extract", t)
    raw = res[0]
    verts, faces = api.orient_remap(sp, order, raw); t = tick("orient_remap", t)
    v, f = verts.cpu().numpy(), faces.cpu().numpy(); t = tick("d2h", t)
    t0 = time.perf_counter(); H.convex_hull_3d(pinned); t = tick("whole_api", t0)
    t0 = time.perf_counter(); H.convex_hull_3d(pinned, solver="serial"); t = tick("whole_api_serial", t0)
    t0 = time.perf_counter(); H.convex_hull_3d(pinned, return_device=True); t = tick("whole_api_dev", t0)
    t0 = time.perf_counter(); H.convex_hull_3d(pts, return_device=True); t = tick("whole_api_devin", t0)
print({k: round(v / 3, 2) for k, v in T.items()})
