"""Kinetic movie tools over the device's final group:
replay the final lower-pass movie up to a probe time t and compare the
kinetic chain with an independently computed 2D lower hull of the projected
points -- the reference's `snapshot_check` (pkg/src/hull3d/oracle.py:142-196)
and `final_group_snapshot_ok` (cli.py:99-123), used by `verify --times`.

The movie comes from the device, in the reference's layout (start-of-time
links (n, 2) and the NIL-terminated log of event point ids):

* engine "exact": the step-for-step seam engine's own final buffer and links;
* engine "fast": the fused path's final compact group (group-local links,
  ids and events) mapped back to sorted indices.  Points the
  final group does not keep get NIL links: the replay never reaches them
  (each point is inserted at most once, at its recorded links).

The replay itself is host code: a verification aid for small clouds
(verify runs n <= 128), not a hot path.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .engine import ExactPass, level_count, stream_ptr

NIL = -1


class EventTimeCollision(RuntimeError):
    """The probe time essentially equals an event time; pick another t."""


def event_time(p, q, r) -> float:
    """geometry.py:46-58: turn_xz / turn_xy, +inf when turn_xy == 0."""
    den = (q[0] - p[0]) * (r[1] - p[1]) - (r[0] - p[0]) * (q[1] - p[1])
    if den == 0.0:
        return math.inf
    return ((q[0] - p[0]) * (r[2] - p[2]) - (r[0] - p[0]) * (q[2] - p[2])) / den


def lower_hull_2d(pts) -> list:
    """oracle.py:113-135: monotone-chain lower hull of (x, w) pairs sorted by
    strictly increasing x; collinear middle points excluded."""
    chain: list = []
    last_x = None
    for i, (px, pw) in enumerate(pts):
        if last_x is not None and px <= last_x:
            raise ValueError("points must be sorted by strictly increasing x")
        last_x = px
        while len(chain) >= 2:
            ax, aw = pts[chain[-2]]
            bx, bw = pts[chain[-1]]
            if (bx - ax) * (pw - aw) - (px - ax) * (bw - aw) <= 0.0:
                chain.pop()
            else:
                break
        chain.append(i)
    return chain


def _act(prev: np.ndarray, nxt: np.ndarray, e: int) -> None:
    """_ckernels.pyx:49-60: toggle e between its recorded neighbours."""
    p, q = int(prev[e]), int(nxt[e])
    if nxt[p] == e:
        nxt[p], prev[q] = q, p
    else:
        nxt[p], prev[q] = e, e


def snapshot_check(coords: np.ndarray, links: np.ndarray, log: np.ndarray, t: float,
                   collision_tol: float = 1e-12) -> bool:
    """Replay `log` (event point ids, NIL-terminated) from the start-of-time
    `links` while the replayed event time is <= t; the chain from point 0
    must equal the 2D lower hull of (x, z - t*y) over all points."""
    n = len(coords)
    prev, nxt = links[:, 0].copy(), links[:, 1].copy()
    for e in log:
        e = int(e)
        if e == NIL:
            break
        pe, ne = int(prev[e]), int(nxt[e])
        te = event_time(coords[pe], coords[e], coords[ne])
        if abs(te - t) <= collision_tol * max(1.0, abs(te)):
            raise EventTimeCollision(f"probe time {t} collides with event time {te}")
        if te > t:
            break
        _act(prev, nxt, e)
    got = []
    i = 0
    while i != NIL:
        got.append(i)
        i = int(nxt[i])
        if len(got) > n:
            raise RuntimeError("chain walk exceeded the group size")
    projected = [(float(c[0]), float(c[2] - t * c[1])) for c in coords]
    return got == lower_hull_2d(projected)


def final_movie(points, engine: str = "fast", device=None):
    """(sorted coords, start-of-time links (n,2), final lower-pass log) of
    the device's movie, in the reference's layout (numpy)."""
    from .api import presort

    dev = device or torch.device("cuda", torch.cuda.current_device())
    pts = torch.as_tensor(np.asarray(points, dtype=np.float64)).to(dev)
    sp, _, _ = presort(pts)
    n = sp.shape[0]
    coords = sp.cpu().numpy()
    if engine == "exact":
        st = ExactPass(n, dev)
        final = st.run(sp, 1.0)
        return coords, st.links.cpu().numpy().astype(np.int64), final.cpu().numpy()
    from .fast import _WS
    from .multigpu import GroupLayout

    L = _lib.load()
    wsb = int(L.h3d_fast_pass_workspace_bytes(n))
    ws = [_WS.get(dev, 0, wsb), _WS.get(dev, 1, wsb)]
    err = torch.zeros(1, dtype=torch.int64, device=dev)
    levels = level_count(n)
    r = L.h3d_fast_passes_range(sp.data_ptr(), n, 0, n, 1, levels, ws[0].data_ptr(),
                                ws[1].data_ptr(), wsb, err.data_ptr(), 0, stream_ptr(dev))
    if r < 0 or int(err.item()) != 0:
        raise RuntimeError(f"fast path declined this input (code {min(int(r), int(err.item()))})")
    lay = GroupLayout(ws[0], n)
    buf = levels & 1
    nS, k = (int(v) for v in lay.hdr_view(buf, 0).view(torch.int32).cpu().tolist())
    lnk = lay.lnk_view(buf, 0, nS).view(torch.int32).view(nS, 2).cpu().numpy().astype(np.int64)
    gid = lay.gid_view(buf, 0, nS).view(torch.int32).cpu().numpy().astype(np.int64)
    # EvP (16 B): t f64, then a | b << 21 | c << 42 | kind << 63
    w = lay.ev_view(buf, 0, k).cpu().numpy().view(np.uint64).reshape(k, 2)[:, 1]
    b = ((w >> np.uint64(21)) & np.uint64((1 << 21) - 1)).astype(np.int64)
    links = np.full((n, 2), NIL, dtype=np.int64)
    glob = np.where(lnk == NIL, NIL, gid[np.clip(lnk, 0, None)])
    links[gid] = glob
    log = np.append(gid[b], NIL) if k else np.array([NIL])
    return coords, links, log


def random_probe_time(rng) -> float:
    """cli.py:99-101: heavy-tailed, so probes land below, between and above
    all event times."""
    return math.tan(math.pi * (rng.random() - 0.5))


def final_group_snapshot_ok(points, times: int, rng, engine: str = "fast") -> bool:
    """cli.py:104-123: snapshot-check the final merged group at `times`
    random probe times."""
    try:
        coords, links, log = final_movie(points, engine)
    except RuntimeError:  # the fast path declined: the exact engine's movie
        coords, links, log = final_movie(points, "exact")
    for _ in range(times):
        for _attempt in range(100):
            try:
                ok = snapshot_check(coords, links, log, random_probe_time(rng))
                break
            except EventTimeCollision:
                continue
        else:
            raise RuntimeError("could not find a collision-free probe time")
        if not ok:
            return False
    return True


__all__ = ["snapshot_check", "final_movie", "final_group_snapshot_ok", "lower_hull_2d",
           "event_time", "EventTimeCollision", "random_probe_time"]
