"""Debug helper: one fast-engine hull vs the exact engine.
    python tools/dbg_one.py N DIST [SEED]"""
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1205_1171_b200 as H  # noqa: E402
from paper_1205_1171_b200 import fast  # noqa: E402
from paper_1205_1171_b200.generators import generate  # noqa: E402

n = int(sys.argv[1])
dist = sys.argv[2]
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 3
pts = generate(n, dist, seed)
b = H.convex_hull_3d(pts)
torch.cuda.synchronize()
print("fast done; fallbacks", fast.FALLBACKS[0], "err", fast.LAST_ERROR[0])
a = H.convex_hull_3d(pts, H.CudaBackend(0, engine="exact"))
print(n, dist, "equal:", np.array_equal(a.faces, b.faces), len(a.faces), len(b.faces))
