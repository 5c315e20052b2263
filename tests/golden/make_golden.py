"""Generate the golden fixtures from the UNMODIFIED reference (run here only).

    python tests/golden/make_golden.py [--large [--c4]] | --c5

Needs oracle/_ref/site (oracle/build_ref.sh).  Writes:

* small.npz   -- inputs and reference convex_hull_3d outputs (faces, vertices,
                 lower/upper counts, perturbed flag) for small/medium cases,
                 including the tie-perturbation path and C1 (10^4 cube).
* levels.npz  -- per-level output buffers and links of the reference's own
                 level loop (parallel.plan_level + merge.merge_movies +
                 kernels.copy_log) for a few n, the per-level parity gate.
* large.json  -- sha256 digests of inputs and outputs for C2/C3/C4 and an
                 integer-coordinate 2^20 cloud (outputs too big to commit).
* level_stats.json -- per-level J, E_in, E_out, D, kmax for C2/C3/C4/C5, both
                 passes (SURVEY.md 8(d) algorithmic-bytes model inputs),
                 computed with the C restatement (pinned by small.npz).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

TETRA = np.array([[0.0, 0, 0], [1, 0.1, 2], [2, 1.9, 0.3], [3, 0.2, 0.1]])


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def small_cases(ref):
    cases = {"tetra": TETRA, "dup_tetra": np.vstack([TETRA, TETRA[:2]])}
    cases["ball_64_s42"] = ref.generate(64, "ball", 42)
    cases["gauss_48_s17"] = ref.generate(48, "gauss", 17)
    for dist in ("ball", "sphere", "cube", "gauss"):
        for n in (4, 5, 8, 17, 64, 100, 257, 1000, 4096):
            cases[f"{dist}_{n}"] = ref.generate(n, dist, n)
    for s in range(3):
        cases[f"C1_cube_10000_s{s}"] = ref.generate(10_000, "cube", s)
    rng = np.random.default_rng(1)
    for R in (2**6, 2**12, 2**31):
        cases[f"int_R{R}_3000"] = rng.integers(-R, R, (3000, 3)).astype(np.float64)
    cases["int_R2e20_10000"] = (
        np.random.default_rng(7).integers(-(2**20), 2**20, (10_000, 3)).astype(np.float64)
    )
    return cases


def make_small(ref):
    out = {}
    names = []
    for name, pts in small_cases(ref).items():
        r = ref.convex_hull_3d(pts)
        s = ref.convex_hull_3d(pts, solver="serial")
        # outside general position (duplicate points, dense integer grids)
        # the reference's own solvers disagree; the level engine is the target
        general = int(np.array_equal(r.faces, s.faces))
        out[f"{name}__pts"] = pts
        out[f"{name}__faces"] = r.faces
        out[f"{name}__vertices"] = r.vertices
        out[f"{name}__meta"] = np.array(
            [r.stats.lower_events, r.stats.upper_events, int(r.stats.perturbed), general],
            dtype=np.int64
        )
        names.append(name)
    out["__names__"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    print("small.npz:", len(names), "cases")


def make_levels(ref):
    from hull3d import kernels
    from hull3d.merge import MergeJob, merge_movies
    from hull3d.parallel import level_count, plan_level
    from hull3d.store import MovieBuffer, PointStore, init_base_logs

    out = {}
    names = []
    for dist, n, seed in (("ball", 5, 0), ("gauss", 16, 1), ("gauss", 53, 13), ("ball", 100, 3),
                          ("sphere", 256, 2), ("cube", 1000, 5), ("sphere", 777, 9)):
        pts = ref.generate(n, dist, seed)
        pts = pts[np.lexsort((pts[:, 2], pts[:, 1], pts[:, 0]))]
        for which, zs in (("lower", 1.0), ("upper", -1.0)):
            P = pts * np.array([1.0, 1.0, zs])
            store = PointStore(P)
            A, B = MovieBuffer(n), MovieBuffer(n)
            init_base_logs(store, A)
            src, dst = A, B
            name = f"{dist}_{n}_{seed}_{which}"
            out[f"{name}__pts"] = P
            for lv in range(1, level_count(n) + 1):
                plan = plan_level(n, lv)
                for L, M, R in plan.jobs:
                    merge_movies(MergeJob(int(L), int(M), int(R), src, dst), store)
                for Lc in plan.carries:
                    kernels.active().copy_log(src.slots, dst.slots, 2 * Lc, 2 * n - 2 * Lc)
                out[f"{name}__slots{lv}"] = dst.slots.copy()
                out[f"{name}__links{lv}"] = store.links.copy()
                src, dst = dst, src
            names.append(name)
    out["__names__"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "levels.npz"), **out)
    print("levels.npz:", len(names), "passes")


def _valid_slots(buf, starts2, ks):
    """Concatenated events of the logs at slot offsets starts2 with lengths ks."""
    if len(ks) == 0 or ks.sum() == 0:
        return np.empty(0, dtype=np.int64)
    base = np.repeat(starts2 - np.concatenate([[0], np.cumsum(ks)[:-1]]), ks)
    return buf[base + np.arange(int(ks.sum()))]


def level_stats(pts_sorted: np.ndarray):
    """Per level: J, E_in, E_out, D (distinct indices in input or output
    logs), kmax -- SURVEY.md 8(d)."""
    n = len(pts_sorted)
    rows = []
    prev_buf = np.full(2 * n, O.NIL, dtype=np.int32)
    prev_k = np.zeros(n, dtype=np.int64)  # level-0 groups: single points, empty logs
    for lv, kout, buf, _ in O.level_logs(pts_sorted):
        size = 1 << lv
        half = size >> 1
        starts = np.arange(0, n, size, dtype=np.int64)
        ends = np.minimum(starts + size, n)
        merged = (ends - starts) > half
        g = np.flatnonzero(merged)
        kl = prev_k[2 * g]
        kr = prev_k[2 * g + 1]
        ko = kout[g]
        mark = np.zeros(n, dtype=bool)
        mark[_valid_slots(prev_buf, 2 * starts[g], kl)] = True
        mark[_valid_slots(prev_buf, 2 * (starts[g] + half), kr)] = True
        mark[_valid_slots(buf, 2 * starts[g], ko)] = True
        rows.append({"level": lv, "J": int(len(g)), "E_in": int(kl.sum() + kr.sum()),
                     "E_out": int(ko.sum()), "D": int(mark.sum()),
                     "kmax": int(ko.max()) if len(ko) else 0})
        prev_buf = buf
        prev_k = kout
    return rows


def make_large(ref, with_c4: bool, only_c5: bool = False):
    from paper_1205_1171_b200.generators import generate, integer_cloud

    configs = [("C2_ball_2^20", lambda: generate(2**20, "ball", 0)),
               ("C3_sphere_2^20", lambda: generate(2**20, "sphere", 0)),
               ("int_2^20_R2^31", lambda: integer_cloud(2**20, 0))]
    if with_c4:
        configs.append(("C4_cube_2^24", lambda: generate(2**24, "cube", 0)))
    if only_c5:  # C5 (2^27 mixed): digests only, no per-level statistics
        configs = [("C5_mixed_2^27", lambda: generate(2**27, "mixed", 0))]
    large = {}
    stats = {}
    path = os.path.join(HERE, "large.json")
    if os.path.exists(path):
        large = json.load(open(path))
    spath = os.path.join(HERE, "level_stats.json")
    if os.path.exists(spath):
        stats = json.load(open(spath))
    for name, gen in configs:
        pts = gen()
        t0 = time.time()
        with ref.ThreadBackend(os.cpu_count()) as be:
            r = ref.convex_hull_3d(pts, be)
        dt = time.time() - t0
        large[name] = {
            "n": int(len(pts)), "points_sha256": sha(pts), "faces_sha256": sha(r.faces),
            "vertices_sha256": sha(r.vertices), "nfaces": int(len(r.faces)),
            "nvertices": int(len(r.vertices)), "lower_events": int(r.stats.lower_events),
            "upper_events": int(r.stats.upper_events), "perturbed": bool(r.stats.perturbed),
            "ref_seconds_threads": round(dt, 3), "ref_threads": os.cpu_count(),
        }
        print(name, large[name])
        if not name.startswith("C5"):
            sp, _, _ = O.sort_and_perturb(pts)
            up = sp.copy()
            up[:, 2] = -up[:, 2]
            stats[name] = {"lower": level_stats(sp), "upper": level_stats(up)}
        json.dump(large, open(path, "w"), indent=1)
        json.dump(stats, open(spath, "w"), indent=1)


if __name__ == "__main__":
    ref = O.reference()
    if ref is None:
        sys.exit("build the reference first: oracle/build_ref.sh")
    if "--c5-stats" in sys.argv:  # C5 per-level statistics (C restatement, ~20 GB of RAM)
        from paper_1205_1171_b200.generators import generate
        spath = os.path.join(HERE, "level_stats.json")
        stats = json.load(open(spath)) if os.path.exists(spath) else {}
        sp, _, _ = O.sort_and_perturb(generate(2**27, "mixed", 0))
        lower = level_stats(sp)
        sp[:, 2] = -sp[:, 2]
        stats["C5_mixed_2^27"] = {"lower": lower, "upper": level_stats(sp)}
        json.dump(stats, open(spath, "w"), indent=1)
        sys.exit(0)
    if "--c5" in sys.argv:
        make_large(ref, with_c4=False, only_c5=True)
        sys.exit(0)
    make_small(ref)
    make_levels(ref)
    if "--large" in sys.argv:
        make_large(ref, with_c4="--c4" in sys.argv)
