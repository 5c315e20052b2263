"""Randomised robustness sweep (not a unit test: minutes of oracle time):
many families and sizes through the default routes, bit-compared with the
C oracle (faces, vertices, or the same exception).
Usage: python tools/robust_sweep.py [max_n]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1205_1171_b200 as H  # noqa: E402
from paper_1205_1171_b200 import fast  # noqa: E402
from paper_1205_1171_b200.generators import generate  # noqa: E402


def family(name, n, rng):
    if name in ("ball", "sphere", "cube", "gauss"):
        return generate(n, name, int(rng.integers(1 << 30)))
    p = rng.uniform(-1, 1, (n, 3))
    if name == "int_small":
        return rng.integers(-2**10, 2**10, (n, 3)).astype(np.float64)
    if name == "int_wide":
        return rng.integers(-2**30, 2**30, (n, 3)).astype(np.float64)
    if name == "clusters":
        c = rng.uniform(-1, 1, (12, 3))
        return c[rng.integers(0, 12, n)] + rng.normal(0, 1e-7, (n, 3))
    if name == "near_plane":
        p[:, 2] = 0.2 * p[:, 0] - 0.4 * p[:, 1] + rng.normal(0, 1e-10, n)
        p[:8, 2] += 1.0
        return p
    if name == "thin_slab_x":
        p[: n - 16, 0] = rng.uniform(0, 1e-11, n - 16)
        return p
    if name == "shell_ball":
        v = rng.normal(size=(n, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        r = np.where(rng.random(n) < 0.5, 1.0, rng.random(n) ** (1 / 3))
        return v * r[:, None]
    if name == "paraboloid":
        p[:, 2] = p[:, 0] ** 2 + p[:, 1] ** 2
        return p
    raise KeyError(name)


def outcome(fn, pts):
    try:
        r = fn(pts)
        return ("ok", r.faces, r.vertices)
    except Exception as exc:  # noqa: BLE001
        return ("err", type(exc).__name__, str(exc))


FAMS = ["ball", "sphere", "cube", "gauss", "int_small", "int_wide", "clusters", "near_plane",
        "thin_slab_x", "shell_ball", "paraboloid"]


def main():
    max_n = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000
    from oracle import oracle as O

    rng = np.random.default_rng(20261017)
    bad = 0
    t0 = time.time()
    for n in (10_007, 65_537, 131_072, max_n):
        for fam in FAMS:
            pts = family(fam, n, rng)
            got, exp = outcome(H.convex_hull_3d, pts), outcome(O.convex_hull_3d, pts)
            same = got[0] == exp[0] and (
                (got[0] == "ok" and np.array_equal(got[1], exp[1]) and np.array_equal(got[2], exp[2]))
                or (got[0] == "err" and got[1:] == exp[1:]))
            if not same:
                bad += 1
            print(f"n={n} {fam}: {'same' if same else 'DIFFERENT'} ({got[0]}"
                  f"{'' if got[0] == 'ok' else ' ' + got[1]}), fallbacks so far "
                  f"{fast.FALLBACKS[0]}", flush=True)
    print(f"done in {time.time() - t0:.0f}s, {bad} mismatches")


if __name__ == "__main__":
    main()
