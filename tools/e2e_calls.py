"""Per-call wall time of convex_hull_3d(pinned host input) -> numpy."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1205_1171_b200 as H  # noqa: E402
from paper_1205_1171_b200.generators import generate  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
n, dist, seed, _ = bench.CONFIGS[cfg]
pinned = torch.from_numpy(generate(n, dist, seed)).pin_memory()
be = H.CudaBackend(0)
r = None
ts = []
for i in range(16):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = H.convex_hull_3d(pinned, be)
    torch.cuda.synchronize()
    ts.append(round((time.perf_counter() - t0) * 1e3, 1))
print(ts)
