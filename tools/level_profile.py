"""Per-level kernel times of one hull (both passes) with CUDA events.

    python tools/level_profile.py --config C4 [--engine fast|exact] [--reps 3]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1205_1171_b200 as H  # noqa: E402
from paper_1205_1171_b200 import engine as E  # noqa: E402
from paper_1205_1171_b200.generators import generate  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--engine", default="fast")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n", type=int, default=0, help="override the config's size")
    a = ap.parse_args()
    n, dist, seed, _ = bench.CONFIGS[a.config]
    if a.n:
        n = a.n
    pts = torch.from_numpy(generate(n, dist, seed)).cuda()
    be = H.CudaBackend(0, engine=a.engine)
    for _ in range(2):
        H.convex_hull_3d(pts, be, return_device=True)
    torch.cuda.synchronize()
    acc: dict = {}
    for _ in range(a.reps):
        prof: list = []
        E.PROFILE = prof
        H.convex_hull_3d(pts, be, return_device=True)
        torch.cuda.synchronize()
        E.PROFILE = None
        for name, p, lv, t in prof:
            acc.setdefault((name, p, lv), []).append(t)
    lb = bench.level_bytes(a.config) or {}
    rows = []
    for (name, p, lv), ts in sorted(acc.items(), key=lambda kv: (kv[0][1], kv[0][2], kv[0][0])):
        ms = min(ts)
        b = lb.get((p, lv))
        rows.append({"kernel": name, "pass": p, "level": lv, "ms": round(ms, 4),
                     "B_alg": b, "GBps": round(b / ms / 1e6, 1) if b and ms > 0 else None})
    for r in rows:
        print(json.dumps(r))
    tot = sum(r["ms"] for r in rows)
    print(json.dumps({"total_ms": tot}))


if __name__ == "__main__":
    main()
