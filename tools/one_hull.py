"""Run one hull of a bench config (for ncu captures): python tools/one_hull.py C2"""
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1205_1171_b200 as H  # noqa: E402
from paper_1205_1171_b200.generators import generate  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n, dist, seed, _ = bench.CONFIGS[cfg]
pts = torch.from_numpy(generate(n, dist, seed)).cuda()
for _ in range(reps):
    r = H.convex_hull_3d(pts, return_device=True)
torch.cuda.synchronize()
print(cfg, "faces", r.faces.shape[0])
