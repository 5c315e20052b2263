"""Fast engine vs exact engine on many clouds (debug helper; set H3D_* env to route)."""
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1205_1171_b200 as H  # noqa: E402
from paper_1205_1171_b200 import fast  # noqa: E402
from paper_1205_1171_b200.generators import generate  # noqa: E402

sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "100,1000,5000,20000,100003").split(",")]
bad = 0
for dist in ("ball", "sphere", "cube", "gauss"):
    for n in sizes:
        pts = generate(n, dist, n % 97)
        f0 = fast.FALLBACKS[0]
        b = H.convex_hull_3d(pts)
        fb = fast.FALLBACKS[0] - f0
        a = H.convex_hull_3d(pts, H.CudaBackend(0, engine="exact"))
        ok = np.array_equal(a.faces, b.faces)
        bad += (not ok) or fb
        print(f"{dist:6s} {n:8d} equal={ok} fallback={fb} err={fast.LAST_ERROR[0] if fb else 0}", flush=True)
print("BAD", bad)
