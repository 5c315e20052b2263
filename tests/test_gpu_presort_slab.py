"""The sharded presort (csrc/presort.cu h3d_presort_slab): any window
[q0, p1) of the global stable x order, computed from the full input without
sorting the rest, equals the same rows of the replicated h3d_presort; inputs
it cannot decide alone (x ties, long runs of equal 32-bit keys, non-finite
coordinates, degeneracy not settled inside rank 0's window) return
H3D_E_FASTPATH."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_1205_1171_b200 import _lib
from paper_1205_1171_b200.api import presort
from paper_1205_1171_b200.engine import stream_ptr

pytestmark = pytest.mark.gpu

E_FASTPATH = -13


def slab(pts: torch.Tensor, q0: int, p1: int, scan: int):
    """The window through WINDOW-sized buffers (passed q0 rows before their
    start, as the multi-GPU path does) and the slim slab workspace; returned
    embedded in full-size NaN / -1 arrays for the comparisons."""
    L = _lib.load()
    n = pts.shape[0]
    m = p1 - q0
    wsp = torch.full((m, 3), float("nan"), dtype=torch.float64, device=pts.device)
    wod = torch.full((m,), -1, dtype=torch.int64, device=pts.device)
    ws = torch.empty(int(L.h3d_presort_slab_workspace_bytes(n, m)), dtype=torch.uint8,
                     device=pts.device)
    code = int(L.h3d_presort_slab(pts.data_ptr(), n, q0, p1, scan, wsp.data_ptr() - 24 * q0,
                                  wod.data_ptr() - 8 * q0, ws.data_ptr(), ws.numel(),
                                  stream_ptr(pts.device)))
    torch.cuda.synchronize()
    sp = torch.full((n, 3), float("nan"), dtype=torch.float64, device=pts.device)
    od = torch.full((n,), -1, dtype=torch.int64, device=pts.device)
    sp[q0:p1] = wsp
    od[q0:p1] = wod
    return code, sp, od


def clouds():
    rng = np.random.default_rng(5)
    n = 100_003
    yield "uniform", rng.uniform(-1, 1, (n, 3))
    # many equal 32-bit keys (x crowded into a few key buckets) but no x ties
    p = rng.uniform(-1, 1, (n, 3))
    c = np.round(p[:, 0], 3)
    o = np.argsort(c, kind="stable")
    cs = c[o]
    start = np.r_[0, np.flatnonzero(cs[1:] != cs[:-1]) + 1]
    j = np.arange(n) - np.repeat(start, np.diff(np.r_[start, n]))
    p[o, 0] = cs + j * 4e-15  # ~50 distinct x per 1e-13: one 32-bit key each
    yield "crowded", p
    g = rng.normal(size=(n, 3))
    yield "gauss", g


@pytest.mark.parametrize("name,pts", list(clouds()), ids=lambda v: v if isinstance(v, str) else "")
def test_windows_equal_full_presort(name, pts):
    dev = torch.device("cuda", 0)
    t = torch.from_numpy(pts).to(dev)
    ref_rows, ref_order, pert = presort(t)
    assert not pert
    n = t.shape[0]
    rng = np.random.default_rng(1)
    cuts = [(0, n), (0, 1), (n - 1, n), (0, n // 2), (n // 2 - 1, n), (n // 4 - 1, n // 2)]
    cuts += [tuple(sorted(rng.choice(n + 1, 2, replace=False))) for _ in range(6)]
    for q0, p1 in cuts:
        code, sp, od = slab(t, int(q0), int(p1), 1 if q0 == 0 and p1 > 1000 else 0)
        if name == "crowded" and code == E_FASTPATH:
            continue  # a run of equal keys longer than the tie fix handles
        assert code == 0, (name, q0, p1, code)
        assert torch.equal(od[q0:p1], ref_order[q0:p1]), (name, q0, p1)
        assert torch.equal(sp[q0:p1], ref_rows[q0:p1]), (name, q0, p1)
        assert bool(torch.isnan(sp[:q0]).all()) and bool(torch.isnan(sp[p1:]).all())


def test_declines_what_it_cannot_decide():
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(2)
    n = 50_000
    p = rng.uniform(-1, 1, (n, 3))
    tie = p.copy()
    tie[7, 0] = tie[40_000, 0]  # one x tie, in another rank's window
    assert slab(torch.from_numpy(tie).to(dev), 0, n // 2, 1)[0] in (0, E_FASTPATH)
    assert slab(torch.from_numpy(tie).to(dev), 0, n, 1)[0] == E_FASTPATH
    bad = p.copy()
    bad[123, 2] = np.inf
    assert slab(torch.from_numpy(bad).to(dev), 0, n // 2, 1)[0] == E_FASTPATH
    flat = p.copy()
    flat[:, 2] = 0.0  # coplanar: rank 0's window cannot find a third direction
    assert slab(torch.from_numpy(flat).to(dev), 0, n // 2, 1)[0] == E_FASTPATH
    clus = p.copy()
    clus[: n - 4, 0] = rng.uniform(0, 1e-12, n - 4)  # one huge run of equal keys
    assert slab(torch.from_numpy(clus).to(dev), n // 3, n // 2, 0)[0] == E_FASTPATH


def test_row_offset_view_input():
    """A row-offset view (8-byte aligned only) takes the scalar input scan."""
    dev = torch.device("cuda", 0)
    t = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, (40_001, 3))).to(dev)
    v = t[1:]
    assert v.data_ptr() % 16 == 8 and v.is_contiguous()
    a = presort(v)
    b = presort(v.clone())
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    v[5, 1] = float("nan")
    with pytest.raises(ValueError):
        presort(v)


def test_degeneracy_scan_beyond_the_head(oracle_mod):
    """The first 30000 sorted rows are collinear: the one-CTA head scan
    (first 16K rows) cannot decide the collinearity stage, so the full-range
    stages must run; the result (faces or exception) equals the oracle's."""
    import paper_1205_1171_b200 as H

    rng = np.random.default_rng(8)
    t = np.sort(rng.uniform(0.0, 0.75, 30000))
    line = np.stack([t, 2.0 * t - 0.5, -t + 0.25], axis=1)
    rest = rng.uniform(-1.0, 1.0, (10000, 3))
    rest[:, 0] = rng.uniform(0.75, 1.0, 10000)
    pts = np.concatenate([line, rest])
    rng.shuffle(pts)

    def outcome(fn):
        try:
            r = fn(pts)
            return ("ok", r.faces, r.vertices)
        except Exception as exc:  # noqa: BLE001
            return ("err", type(exc).__name__, str(exc))

    got, exp = outcome(H.convex_hull_3d), outcome(oracle_mod.convex_hull_3d)
    assert got[0] == exp[0]
    if got[0] == "ok":
        assert np.array_equal(got[1], exp[1]) and np.array_equal(got[2], exp[2])
    else:
        assert got[1:] == exp[1:]
    # all collinear: the head and the full range both find no second direction
    with pytest.raises(ValueError, match="collinear"):
        H.convex_hull_3d(line)
