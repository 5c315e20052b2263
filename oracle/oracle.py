"""CPU oracle for the kinetic 3D hull path -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product (paper_1205_1171_b200) never calls it.

Two oracles live here:

* ``hull_oracle.c`` (built to ``liborc.so`` by oracle/Makefile): a plain-C
  restatement of the reference kernels and level loop, wrapped below with
  ctypes.  The numpy glue restates ``convex_hull_3d``'s host steps
  (pkg/src/hull3d/api.py:113-147 degeneracy scan, :252-266 orientation,
  remap and ``np.unique``) line for line.
* ``reference()``: the unmodified reference package built into
  ``oracle/_ref/site`` by ``oracle/build_ref.sh`` (absent -> None).  It pins
  the restatement (tests/test_oracle_pinned.py) and generates the golden
  fixtures under tests/golden/.
"""

from __future__ import annotations

import ctypes
import os
import sys
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
NIL = -1
E_OVERFLOW, E_BRIDGE, E_CHAIN, E_COUNT, E_UNTERMINATED = -1, -2, -3, -4, -5
E_DEGENERATE_TIES = -6

_lib = None


def lib() -> ctypes.CDLL:
    """Load (building if needed) the C restatement."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.path.join(HERE, "liborc.so")
    src = os.path.join(HERE, "hull_oracle.c")
    if not os.path.exists(path) or (
        os.path.exists(src) and os.path.getmtime(src) > os.path.getmtime(path)
    ):
        rc = os.system(f"make -s -C {HERE} >/dev/null")
        if rc != 0 or not os.path.exists(path):
            raise RuntimeError("cannot build oracle/liborc.so")
    L = ctypes.CDLL(path)
    i64, dp, ip = ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p
    L.orc_evtime.restype = ctypes.c_double
    L.orc_evtime.argtypes = [dp, i64, i64, i64]
    L.orc_act.restype = ctypes.c_int
    L.orc_act.argtypes = [ip, i64]
    L.orc_find_bridge.restype = i64
    L.orc_find_bridge.argtypes = [dp, ip, ctypes.POINTER(i64), ctypes.POINTER(i64), i64]
    L.orc_merge.restype = i64
    L.orc_merge.argtypes = [dp, ip, ip, ip, i64, i64, i64]
    L.orc_init_base.restype = None
    L.orc_init_base.argtypes = [ip, ip, i64]
    L.orc_copy_log.restype = i64
    L.orc_copy_log.argtypes = [ip, ip, i64, i64]
    L.orc_run_level.restype = i64
    L.orc_run_level.argtypes = [dp, i64, ip, ip, ip, i64, ip]
    L.orc_build_movie.restype = i64
    L.orc_build_movie.argtypes = [dp, i64, ip, ip, ip]
    L.orc_extract_faces.restype = i64
    L.orc_extract_faces.argtypes = [ip, ip, i64, ip, i64]
    L.orc_replay.restype = i64
    L.orc_replay.argtypes = [ip, ip, i64, i64, ctypes.c_int]
    L.orc_hull_pass.restype = i64
    L.orc_hull_pass.argtypes = [dp, i64, ip, i64]
    L.orc_sort_and_perturb.restype = ctypes.c_int
    L.orc_sort_and_perturb.argtypes = [dp, i64, dp, ip]
    L.orc_level_count.restype = i64
    L.orc_level_count.argtypes = [i64]
    _lib = L
    return L


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class DegenerateInputError(ValueError):
    pass


class OracleKernelError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle kernel error code {code}")
        self.code = code


def evtime(pts: np.ndarray, a: int, b: int, c: int) -> float:
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    return float(lib().orc_evtime(_p(pts), a, b, c))


def sort_and_perturb(coords: np.ndarray):
    """(sorted coords, order int64, perturbed) -- api.py:90-110."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    n = len(coords)
    out = np.empty_like(coords)
    order = np.empty(n, dtype=np.int64)
    r = lib().orc_sort_and_perturb(_p(coords), n, _p(out), _p(order))
    if r == E_DEGENERATE_TIES:
        raise DegenerateInputError("duplicate x coordinates survived perturbation")
    return out, order, bool(r)


def scan_degenerate(coords: np.ndarray, tol: float = 1e-9) -> None:
    """Restates _scan_degenerate (api.py:113-147)."""
    n = len(coords)
    p0 = coords[0]
    scale = max(float(np.abs(coords).max()), 1e-30)

    def first_hit(mask_fn) -> int:
        for lo in range(1, n, 65536):
            hits = np.flatnonzero(mask_fn(lo, min(lo + 65536, n)))
            if len(hits):
                return lo + int(hits[0])
        return -1

    i = first_hit(lambda lo, hi: np.linalg.norm(coords[lo:hi] - p0, axis=1) > tol * scale)
    if i < 0:
        raise DegenerateInputError("all points coincide")
    di = coords[i] - p0
    j = first_hit(
        lambda lo, hi: np.linalg.norm(np.cross(di, coords[lo:hi] - p0), axis=1)
        > tol * scale * scale
    )
    if j < 0:
        raise DegenerateInputError("all points are collinear")
    normal = np.cross(di, coords[j] - p0)
    thr = tol * scale * float(np.linalg.norm(normal))
    k = first_hit(lambda lo, hi: np.abs((coords[lo:hi] - p0) @ normal) > thr)
    if k < 0:
        raise DegenerateInputError("all points are coplanar")


def hull_pass(sorted_pts: np.ndarray) -> np.ndarray:
    """Raw facet triples of one pass (sorted indices), int32 (k, 3)."""
    P = np.ascontiguousarray(sorted_pts, dtype=np.float64)
    n = len(P)
    faces = np.empty((2 * n, 3), dtype=np.int32)
    r = lib().orc_hull_pass(_p(P), n, _p(faces), 2 * n)
    if r < 0:
        raise OracleKernelError(int(r))
    return faces[:r].copy()


@dataclass
class OracleHull:
    vertices: np.ndarray
    faces: np.ndarray
    lower_events: int
    upper_events: int
    perturbed: bool
    lower_raw: np.ndarray
    upper_raw: np.ndarray
    order: np.ndarray

    def face_set(self):
        return {tuple(sorted(map(int, row))) for row in self.faces}


def orient_and_remap(sorted_pts, order, lower_raw, upper_raw):
    """api.py:252-266: concat, orient vs centroid, map to caller indices."""
    faces = np.concatenate([lower_raw, upper_raw]).astype(np.int64)
    if len(faces) == 0:
        raise DegenerateInputError("no facets produced; input is degenerate")
    a = sorted_pts[faces[:, 0]]
    normals = np.cross(sorted_pts[faces[:, 1]] - a, sorted_pts[faces[:, 2]] - a)
    centroid = sorted_pts.mean(axis=0)
    flip = np.einsum("ij,ij->i", normals, centroid - a) > 0.0
    faces[flip, 1], faces[flip, 2] = faces[flip, 2], faces[flip, 1]
    faces = order[faces]
    return np.unique(faces), faces


def convex_hull_3d(points) -> OracleHull:
    """Whole-path oracle: same outputs as the reference convex_hull_3d."""
    coords = np.asarray(points, dtype=np.float64)
    if coords.ndim != 2 or coords.shape[1] != 3:
        raise ValueError("points must have shape (n, 3)")
    n = coords.shape[0]
    if n == 0:
        raise ValueError("no points")
    if not np.isfinite(coords).all():
        raise ValueError("coordinates must be finite")
    if n <= 3:
        e = np.empty((0, 3), dtype=np.int64)
        return OracleHull(np.arange(n, dtype=np.int64), e, 0, 0, False, e, e, np.arange(n))
    sorted_pts, order, perturbed = sort_and_perturb(coords)
    scan_degenerate(sorted_pts)
    upper = sorted_pts.copy()
    upper[:, 2] = -upper[:, 2]
    lo = hull_pass(sorted_pts)
    up = hull_pass(upper)
    vertices, faces = orient_and_remap(sorted_pts, order, lo, up)
    return OracleHull(vertices, faces, len(lo), len(up), perturbed, lo, up, order)


def level_logs(sorted_pts: np.ndarray):
    """Run the level loop, yielding (level, kout per group, out buffer copy,
    links copy) after each level -- the per-level parity gate."""
    P = np.ascontiguousarray(sorted_pts, dtype=np.float64)
    n = len(P)
    L = lib()
    K = np.full((n, 2), NIL, dtype=np.int32)
    A = np.full(2 * n, NIL, dtype=np.int32)
    B = np.full(2 * n, NIL, dtype=np.int32)
    L.orc_init_base(_p(K), _p(A), n)
    src, dst = A, B
    for lv in range(1, int(L.orc_level_count(n)) + 1):
        groups = (n + (1 << lv) - 1) >> lv
        kout = np.zeros(groups, dtype=np.int64)
        r = L.orc_run_level(_p(P), n, _p(K), _p(src), _p(dst), lv, _p(kout))
        if r < 0:
            raise OracleKernelError(int(r))
        yield lv, kout, dst.copy(), K.copy()
        src, dst = dst, src


def group_log(buf: np.ndarray, L: int) -> np.ndarray:
    """Events of the group log at slot 2L (terminator excluded)."""
    s = buf[2 * L:]
    end = int(np.argmax(s == NIL))
    return s[:end].copy()


def reference():
    """The unmodified reference package from oracle/_ref/site, or None."""
    site = os.path.join(HERE, "_ref", "site")
    if not os.path.isdir(os.path.join(site, "hull3d")):
        return None
    if site not in sys.path:
        sys.path.insert(0, site)
    import hull3d  # noqa: WPS433 -- the reference itself

    return hull3d
