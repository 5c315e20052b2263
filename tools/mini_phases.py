"""Per-phase clocks of the mini merge (CTA 0 of each mini level), from a
profiling build: H3D_NVCC_EXTRA=-DH3D_MINI_PROF python -m
paper_1205_1171_b200.build --force, copied to lib/variants/miniprof.so.
Usage on the box: python tools/mini_phases.py C4 [n]"""
import ctypes
import os
import shutil
import sys

sys.path.insert(0, ".")
lib = "paper_1205_1171_b200/lib/libhull3d_b200.so"
shutil.copy("paper_1205_1171_b200/lib/variants/miniprof.so", lib)
os.utime(lib)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1205_1171_b200 as H  # noqa: E402
from paper_1205_1171_b200 import _lib  # noqa: E402
from paper_1205_1171_b200.generators import generate  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
n, dist, seed, _ = bench.CONFIGS[cfg]
if len(sys.argv) > 2:
    n = int(sys.argv[2])
pts = torch.from_numpy(generate(n, dist, seed)).cuda()
for _ in range(2):
    H.convex_hull_3d(pts, return_device=True)
torch.cuda.synchronize()
L = _lib.load()
arr = (ctypes.c_longlong * (64 * 16))()
L.h3d_mini_prof_read(arr)
names = {1: "points", 2: "mergeS", 3: "scatter", 4: "lists+links", 5: "walks", 10: "sweeps",
         6: "slabs", 7: "classify", 8: "output", 9: "rebuild"}
order = [1, 2, 3, 4, 5, 10, 6, 7, 8, 9]
for lv in range(64):
    v = arr[lv * 16:(lv + 1) * 16]
    if not v[0] or not v[9]:
        continue
    prev, parts = v[0], []
    for i in order:
        parts.append(f"{names[i]} {v[i] - prev}")
        prev = v[i]
    walks = (f" | walk moves: max {v[12]}, segment 0 {v[13]}, mean {v[14] / v[15]:.1f} over {v[15]}"
             if v[15] else "")
    print(f"level {lv}: total {v[9] - v[0]} cycles | " + ", ".join(parts) + walks)
