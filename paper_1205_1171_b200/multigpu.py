"""Multi-GPU x-slab sharding of the hull.

One process per GPU (torch.distributed, NCCL over NVLink; gloo in the CPU
tests).  After the global sort, rank r owns the sorted ranks
[r*S, (r+1)*S) with S = 2^(L - log2 G) and L = ceil(log2 n): exactly the
level-(L - log2 G) groups of the single-GPU merge tree, so every log is the
one `plan_level` (pkg/src/hull3d/parallel.py:49-65) would produce.

* Levels 1 .. L - log2 G run on every rank's own slab with no communication
  (`h3d_fast_passes_range`).
* Each of the last log2 G levels pairs slabs: at level l a group spans
  2^(l-s) slabs; the owner of its right half sends its compact group (header,
  links, ids, events of both passes -- everything the merge reads) to the
  owner of the left half, which runs that one merge job.  A left half with no
  right half (ragged n) is a carry and needs no message.
* Rank 0 ends with the final groups and runs facet extraction and the
  orientation / remap epilogue.

Data path: only the final log2 G levels exchange anything, point-to-point,
and the messages are the compact groups (a few KB for cube/ball, ~24 MB for
a sphere-like top level).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib


@dataclass(frozen=True)
class SlabPlan:
    n: int
    world: int

    @property
    def levels(self) -> int:
        return (self.n - 1).bit_length()

    @property
    def G(self) -> int:
        """Ranks that own slabs: the largest power of two <= world whose slabs
        still hold at least two points."""
        g = 1
        while g * 2 <= self.world and (self.n + g * 2 - 1) // (g * 2) >= 2 and g * 2 <= (1 << max(self.levels - 1, 0)):
            g *= 2
        return g

    @property
    def slab_level(self) -> int:
        return self.levels - (self.G.bit_length() - 1)

    @property
    def S(self) -> int:
        return 1 << self.slab_level

    def slab(self, rank: int):
        """Point range [p0, p1) of a rank's slab, or None."""
        if rank >= self.G:
            return None
        p0 = rank * self.S
        if p0 >= self.n:
            return None
        return p0, min(self.n, p0 + self.S)

    def role(self, level: int, rank: int):
        """What a rank does at a cross level: ("merge", partner),
        ("send", partner), ("carry", None) or ("idle", None)."""
        s = self.slab_level
        if level <= s or rank >= self.G:
            return ("idle", None)
        span = 1 << (level - s)
        half = span >> 1
        if rank % span == 0:
            if rank * self.S >= self.n:
                return ("idle", None)
            right = rank + half
            if right * self.S < self.n:
                return ("merge", right)
            return ("carry", None)
        if rank % span == half and rank * self.S < self.n:
            return ("send", rank - half)
        return ("idle", None)


class GroupLayout:
    """Views of one pass workspace's compact-group arrays (see
    h3d_fast_layout in include/hull3d_b200.h)."""

    LNK = 8
    EV = 16  # EvP: t f64 + one word with the 21-bit local ids and the kind

    def __init__(self, ws: torch.Tensor, n: int):
        offs = (ctypes.c_int64 * 9)()
        _lib.load().h3d_fast_layout(n, ctypes.addressof(offs))
        self.ws = ws
        self.n = n
        self.off = list(offs)

    def _arr(self, buf: int, which: int) -> int:
        return self.off[4 * buf + which]

    def hdr_view(self, buf: int, g: int) -> torch.Tensor:
        o = self._arr(buf, 0) + 8 * g
        return self.ws[o:o + 8]

    def lnk_view(self, buf: int, L: int, nS: int) -> torch.Tensor:
        o = self._arr(buf, 1) + self.LNK * L
        return self.ws[o:o + self.LNK * nS]

    def gid_view(self, buf: int, L: int, nS: int) -> torch.Tensor:
        o = self._arr(buf, 2) + 4 * L
        return self.ws[o:o + 4 * nS]

    def ev_view(self, buf: int, L: int, k: int) -> torch.Tensor:
        o = self._arr(buf, 3) + self.EV * 2 * L
        return self.ws[o:o + self.EV * k]


def group_header(layouts, buf: int, g: int) -> torch.Tensor:
    """(nS, k) of group g in both passes as one int32 tensor [4]."""
    return torch.cat([lay.hdr_view(buf, g) for lay in layouts]).view(torch.int32).clone()


def _p2p_via_host() -> bool:
    """gloo cannot move CUDA tensors point-to-point: stage them through host
    memory (the single-GPU multi-process tests run gloo on one device)."""
    import torch.distributed as dist

    return dist.get_backend() == "gloo"


def _send(t: torch.Tensor, dst: int) -> None:
    import torch.distributed as dist

    dist.send(t.cpu() if (t.is_cuda and _p2p_via_host()) else t, dst)


def _recv(t: torch.Tensor, src: int) -> None:
    import torch.distributed as dist

    if t.is_cuda and _p2p_via_host():
        tmp = torch.empty(t.shape, dtype=t.dtype)
        dist.recv(tmp, src)
        t.copy_(tmp)
    else:
        dist.recv(t, src)


def _rows_of(gid_view: torch.Tensor, rows) -> torch.Tensor:
    """(nS, 4) int64: the sorted row (x, y, z bits) and caller index of every
    point of a group -- what the receiver of a sharded presort lacks."""
    sorted_pts, order = rows
    idx = gid_view.view(torch.int32).long()
    return torch.cat([sorted_pts.index_select(0, idx).view(torch.int64),
                      order.index_select(0, idx).unsqueeze(1)], dim=1)


def _group_views(lay, buf: int, L: int, nS: int, k: int):
    return (lay.lnk_view(buf, L, nS), lay.gid_view(buf, L, nS), lay.ev_view(buf, L, k))


def _sizes(h, p: int, level: int):
    """(nS, k) of pass p from a header, clamped to the group's slot capacity
    (2^level points, twice as many event slots): after a declined level the
    header may be stale, and both sides must still size the same views
    inside the group (the result is discarded by the error flag)."""
    cap = 1 << level
    nS = min(max(int(h[2 * p]), 0), cap)
    k = min(max(int(h[2 * p + 1]), 0), 2 * cap)
    return nS, k


def send_group(layouts, buf: int, level: int, g: int, dst: int, rows=None) -> None:
    """Ship group g of `level` (in buffer `buf`) of both passes to rank dst:
    the header, then ONE packed payload (links, ids, events of both passes;
    with rows = (sorted_pts, order) also the coordinates and caller indices
    of the group's points -- under the sharded presort the receiver never
    sorted them)."""
    hdr = group_header(layouts, buf, g)
    _send(hdr, dst)
    L = g << level
    h = hdr.cpu().tolist()
    parts = []
    for p, lay in enumerate(layouts):
        nS, k = _sizes(h, p, level)
        parts.extend(v for v in _group_views(lay, buf, L, nS, k) if v.numel())
        if rows is not None and nS:
            parts.append(_rows_of(lay.gid_view(buf, L, nS), rows).view(torch.uint8).reshape(-1))
    if parts:
        _send(torch.cat(parts), dst)


def recv_group(layouts, buf: int, level: int, g: int, src: int, rows=None) -> None:
    """Receive group g of `level` of both passes from rank src into the same
    slots of this rank's buffer `buf` (and, with rows, scatter the points'
    sorted rows and caller indices into this rank's full-size arrays)."""
    dev = layouts[0].ws.device
    hdr = torch.empty(4, dtype=torch.int32, device=dev)
    _recv(hdr, src)
    L = g << level
    h = hdr.cpu().tolist()
    total = 0
    for p, lay in enumerate(layouts):
        nS, k = _sizes(h, p, level)
        lay.hdr_view(buf, g).copy_(hdr[2 * p:2 * p + 2].view(torch.uint8))
        total += sum(v.numel() for v in _group_views(lay, buf, L, nS, k))
        if rows is not None:
            total += 32 * nS
    if total == 0:
        return
    payload = torch.empty(total, dtype=torch.uint8, device=dev)
    _recv(payload, src)
    at = 0
    for p, lay in enumerate(layouts):
        nS, k = _sizes(h, p, level)
        for view in _group_views(lay, buf, L, nS, k):
            view.copy_(payload[at:at + view.numel()])
            at += view.numel()
        if rows is not None and nS:
            sorted_pts, order = rows
            tmp = payload[at:at + 32 * nS].clone().view(torch.int64).view(nS, 4)  # 8-byte aligned
            at += 32 * nS
            idx = lay.gid_view(buf, L, nS).view(torch.int32).long()
            sorted_pts.index_copy_(0, idx, tmp[:, :3].contiguous().view(torch.float64))
            order.index_copy_(0, idx, tmp[:, 3].contiguous())


SHARD_PRESORT_MIN = 1 << 14
SHARDED_RUNS = [0]  # hulls whose presort ran sharded (tests check it is taken)


def sharded_presort(pts_dev: torch.Tensor, plan: "SlabPlan", rank: int):
    """Every rank sorts only its own slab (plus the row before it, for the
    tie test across the boundary) with h3d_presort_slab into WINDOW-sized
    buffers; rank 0 also runs the degeneracy scan.  Returns the rank's slab
    rows and caller indices (rows [p0, p1) of the global sorted order; None
    for a rank without a slab), or False on every rank when any rank's
    window cannot reproduce the replicated presort (ties, long key runs,
    non-finite input, undecided degeneracy)."""
    import os

    import torch.distributed as dist

    from .engine import stream_ptr
    from .fast import _WS

    L = _lib.load()
    n = pts_dev.shape[0]
    dev = pts_dev.device
    code = 0
    local = None
    sl = plan.slab(rank)
    if sl is not None:
        p0, p1 = sl
        q0 = max(0, p0 - 1)
        m = p1 - q0
        if os.environ.get("H3D_DIST_POISON"):  # tests: unfilled rows must never be read
            rows = torch.full((m, 3), float("nan"), dtype=torch.float64, device=dev)
            order = torch.full((m,), -1, dtype=torch.int64, device=dev)
        else:
            rows = torch.empty((m, 3), dtype=torch.float64, device=dev)
            order = torch.empty(m, dtype=torch.int64, device=dev)
        ws = _WS.get(dev, 5, int(L.h3d_presort_slab_workspace_bytes(n, m)))
        # the window buffers are passed q0 rows before their start: the
        # function only touches global rows [q0, p1)
        code = int(L.h3d_presort_slab(pts_dev.data_ptr(), n, q0, p1, 1 if rank == 0 else 0,
                                      rows.data_ptr() - 24 * q0, order.data_ptr() - 8 * q0,
                                      ws.data_ptr(), ws.numel(), stream_ptr(dev)))
        local = (rows[p0 - q0:], order[p0 - q0:])
    flag = torch.tensor([1 if code != 0 else 0], dtype=torch.int64,
                        device="cpu" if _p2p_via_host() else dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX)
    if int(flag.item()) != 0:
        return False
    SHARDED_RUNS[0] += 1
    return local


def _pow2_at_least(x: int) -> int:
    p = 1
    while p < x:
        p <<= 1
    return p


def hull_distributed(pts_dev: torch.Tensor, rank: int, world: int):
    """Both passes of the hull over x-slabs with O(n / G) state per rank.
    Every rank passes the same input (caller order, on its own device).

    * The slab levels run on the rank's slab as a problem of its own (its
      rows [p0, p1) only; the merge tree inside a slab is the global one,
      slabs being aligned level-(L - log2 G) groups).
    * The cross levels run in a small VIRTUAL space: every slab's final
      group is relocated to virtual points [r*C, r*C + C), C = a power of two
      >= twice the largest slab group (its kept points of both passes); with
      n_v = (non-empty slabs) * C the virtual tree has the real tree's
      merges and carries at the last log2 G levels, and the merged logs are
      the real ones (events carry group-local ids; a job's span only bounds
      its bridge walk and log size, both far above any group's kept points).
      Group ids of the virtual space index rows_v/order_v (the kept points'
      sorted rows and caller indices), which travel with the groups.

    Returns on rank 0 (raw faces in virtual ids, lower and upper counts,
    rows_v, order_v, perturbed, sharded, memory report); None on the other
    ranks; None on rank 0 too when the exact engine must take over."""
    import torch.distributed as dist

    from .api import presort
    from .engine import stream_ptr
    from .fast import _WS

    L = _lib.load()
    n = pts_dev.shape[0]
    dev = pts_dev.device
    s = stream_ptr(dev)
    plan = SlabPlan(n, world)
    marks = []  # (name, event) phase boundaries, only when PHASES is set
    mem: dict = {}

    def mark(name):
        if PHASES is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(torch.cuda.current_stream(dev))
            marks.append((name, e))

    mark("start")
    sl = plan.slab(rank)
    sh = sharded_presort(pts_dev, plan, rank) if n >= SHARD_PRESORT_MIN else False
    perturbed = False
    if sh is not False:
        local = sh
    else:  # the replicated presort (ties, long key runs, small n): O(n), rare
        full_rows, full_order, perturbed = presort(pts_dev)
        local = (full_rows[sl[0]:sl[1]], full_order[sl[0]:sl[1]]) if sl is not None else None
    mark("presort")
    state = torch.zeros(4, dtype=torch.int64, device=dev)
    err = state[0:1]
    # ---- slab levels: the slab as a cloud of its own
    U = None
    if sl is not None:
        rows_loc, order_loc = local
        n_r = sl[1] - sl[0]
        if n_r >= 2:
            wsb = int(L.h3d_fast_pass_workspace_bytes(n_r))
            ws_s = [_WS.get(dev, 0, wsb), _WS.get(dev, 1, int(L.h3d_fast_upper_workspace_bytes(n_r)))]
            mem["slab_passes"] = wsb + int(L.h3d_fast_upper_workspace_bytes(n_r))
            r = L.h3d_fast_passes_range(rows_loc.data_ptr(), n_r, 0, n_r, 1, plan.slab_level,
                                        ws_s[0].data_ptr(), ws_s[1].data_ptr(), wsb,
                                        err.data_ptr(), 0, s)
            if r < 0:
                err.fill_(int(r))
                r = 0
            lays_s = [GroupLayout(ws_s[0], n_r), GroupLayout(ws_s[1], n_r)]
            buf_s = int(r)
            hdr = group_header(lays_s, buf_s, 0).cpu().tolist()
            if int(err.item()) != 0:
                # a declined slab level wrote nothing valid: relocate an empty
                # group (the error flag sends the hull to the exact engine)
                parts = [(0, 0, torch.zeros(0, dtype=torch.int32, device=dev))] * 2
            else:
                parts = []
                for p, lay in enumerate(lays_s):
                    nS, k = _sizes(hdr, p, plan.slab_level)
                    parts.append((nS, k, lay.gid_view(buf_s, 0, nS).view(torch.int32)))
            U = torch.unique(torch.cat([g for _, _, g in parts]).long())  # sorted = x order
        else:  # a one-point slab: its group is the point itself
            parts = [(1, 0, torch.zeros(1, dtype=torch.int32, device=dev))] * 2
            U = torch.zeros(1, dtype=torch.int64, device=dev)
            lays_s, buf_s = None, 0
    mark("slab_levels")
    # ---- the virtual space of the cross levels
    u_cnt = torch.tensor([0 if U is None else int(U.numel())], dtype=torch.int64,
                         device="cpu" if _p2p_via_host() else dev)
    dist.all_reduce(u_cnt, op=dist.ReduceOp.MAX)
    C = _pow2_at_least(max(2, 2 * int(u_cnt.item())))
    G_eff = (n + plan.S - 1) // plan.S  # non-empty slabs
    n_v = G_eff * C
    lev_c = C.bit_length() - 1
    levels_v = (n_v - 1).bit_length()
    wsb_v = int(L.h3d_fast_pass_workspace_bytes(n_v))
    ws_v = [_WS.get(dev, 6, wsb_v), _WS.get(dev, 7, int(L.h3d_fast_upper_workspace_bytes(n_v)))]
    mem["cross_passes"] = wsb_v + int(L.h3d_fast_upper_workspace_bytes(n_v))
    lays_v = [GroupLayout(ws_v[0], n_v), GroupLayout(ws_v[1], n_v)]
    rows_v = torch.full((n_v, 3), float("nan"), dtype=torch.float64, device=dev)
    order_v = torch.full((n_v,), -1, dtype=torch.int64, device=dev)
    mem["cross_rows"] = 32 * n_v
    buf_v = lev_c & 1
    if sl is not None:
        base = rank * C
        u = int(U.numel())
        rows_v[base:base + u] = rows_loc.index_select(0, U)
        order_v[base:base + u] = order_loc.index_select(0, U)
        for p, lay in enumerate(lays_v):
            nS, k, gid = parts[p]
            vid = (base + torch.searchsorted(U, gid.long())).to(torch.int32)
            lay.gid_view(buf_v, base, nS).copy_(vid.view(torch.uint8))
            if lays_s is not None:
                if nS:
                    lay.lnk_view(buf_v, base, nS).copy_(lays_s[p].lnk_view(buf_s, 0, nS))
                if k:
                    lay.ev_view(buf_v, base, k).copy_(lays_s[p].ev_view(buf_s, 0, k))
            else:
                lay.lnk_view(buf_v, base, 1).copy_(
                    torch.tensor([-1, -1], dtype=torch.int32, device=dev).view(torch.uint8))
            lay.hdr_view(buf_v, rank).copy_(torch.tensor([nS, k], dtype=torch.int32,
                                                         device=dev).view(torch.uint8))
    rows = (rows_v, order_v)
    for t in range(1, levels_v - lev_c + 1):
        lv_v = lev_c + t
        role, peer = plan.role(plan.slab_level + t, rank)
        prev_buf = (lv_v - 1) & 1
        if role == "send":
            send_group(lays_v, prev_buf, lv_v - 1, (rank * C) >> (lv_v - 1), peer, rows)
        elif role in ("merge", "carry"):
            if role == "merge":
                recv_group(lays_v, prev_buf, lv_v - 1, (peer * C) >> (lv_v - 1), peer, rows)
            p0 = rank * C
            p1 = min(n_v, p0 + (1 << lv_v))
            r = L.h3d_fast_passes_range(rows_v.data_ptr(), n_v, p0, p1, lv_v, lv_v,
                                        ws_v[0].data_ptr(), ws_v[1].data_ptr(), wsb_v,
                                        err.data_ptr(), 0, s)
            if r < 0:
                err.fill_(int(r))
    mark("cross_levels")
    if PHASES is not None:
        torch.cuda.synchronize(dev)
        PHASES.append({b[0]: round(a[1].elapsed_time(b[1]), 4) for a, b in zip(marks, marks[1:])})
    # any error anywhere sends the whole hull to the exact engine on rank 0
    flag = (err != 0).to(torch.int64)
    if _p2p_via_host():
        flag = flag.cpu()
    dist.all_reduce(flag, op=dist.ReduceOp.MAX)
    if rank != 0:
        return None
    if int(flag.item()) != 0:
        return None
    final = levels_v & 1
    cap = max(2 * n_v, 8)
    faces = torch.empty((cap, 3), dtype=torch.int32, device=dev)
    counts = state[1:3]
    L.h3d_fast_extract(ws_v[0].data_ptr(), ws_v[1].data_ptr(), n_v, final, final, faces.data_ptr(),
                       cap, counts.data_ptr(), err.data_ptr(), s)
    h = state.cpu()
    if int(h[0]) != 0:
        return None
    k_lo, k_up = int(h[1]), int(h[2])
    mem["virtual"] = {"C": C, "n_v": n_v}
    return faces[: k_lo + k_up], k_lo, k_up, rows_v, order_v, perturbed, sh is not False, mem


def rank_memory_bytes(n: int, world: int, kept_max: int | None = None) -> dict:
    """Device bytes one rank holds for an n-point hull on `world` GPUs
    (host arithmetic from the library's sizing functions): the replicated
    input and presort keys are O(n); everything else O(n / G) plus the
    virtual cross-level space (C per slab, C >= 2 * the largest slab group;
    kept_max defaults to a tenth of a slab)."""
    L = _lib.load()
    plan = SlabPlan(n, world)
    S = plan.S
    m = min(S + 1, n)
    kept = kept_max if kept_max is not None else max(2, S // 10)
    C = _pow2_at_least(2 * kept)
    n_v = ((n + S - 1) // S) * C
    out = {
        "input_replica": 24 * n,
        "slab_presort_ws": int(L.h3d_presort_slab_workspace_bytes(n, m)),
        "slab_rows": 32 * m,
        "slab_passes": int(L.h3d_fast_pass_workspace_bytes(S) + L.h3d_fast_upper_workspace_bytes(S)),
        "cross_passes": int(L.h3d_fast_pass_workspace_bytes(n_v) + L.h3d_fast_upper_workspace_bytes(n_v)),
        "cross_rows": 32 * n_v,
        "epilogue_rank0": int(L.h3d_epilogue_workspace_bytes(n)) + 12 * n + 48 * n_v,
    }
    out["total"] = sum(out.values())
    return out


GATHER_INPUT_MIN = 1 << 16
PHASES: list | None = None  # set to a list to get this rank's phase times (ms)


def gather_input(points, dev: torch.device, rank: int, world: int) -> torch.Tensor:
    """Every rank's device copy of the whole cloud.  A host input is not
    copied whole by every rank over PCIe: rank r copies only its 1/world row
    chunk and an all-gather (NVLink under NCCL) assembles the rest."""
    import numpy as np
    import torch.distributed as dist

    from .api import _to_device

    if (isinstance(points, torch.Tensor) and points.is_cuda) or world == 1:
        return _to_device(points, dev)
    host = points if isinstance(points, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(points, dtype=np.float64)))
    if host.ndim != 2 or host.shape[1] != 3:
        raise ValueError("points must have shape (n, 3)")
    host = host.to(dtype=torch.float64).contiguous()
    n = host.shape[0]
    if n < GATHER_INPUT_MIN:
        return _to_device(host, dev)
    C = (n + world - 1) // world
    lo, hi = min(n, rank * C), min(n, (rank + 1) * C)
    if _p2p_via_host():
        mine = torch.zeros((C, 3), dtype=torch.float64)
        mine[:hi - lo] = host[lo:hi]
        parts = [torch.empty((C, 3), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, mine)
        return torch.cat(parts)[:n].to(dev)
    full = torch.empty((world * C, 3), dtype=torch.float64, device=dev)
    mine = full[rank * C:(rank + 1) * C]
    if hi > lo:
        mine[:hi - lo].copy_(host[lo:hi], non_blocking=host.is_pinned())
    dist.all_gather_into_tensor(full, mine)  # in place: mine is rank r's slice
    return full[:n]


def convex_hull_3d_distributed(points, device=None, return_device: bool = False):
    """Distributed drop-in: every rank calls it with the same points; rank 0
    gets the HullResult (identical to the single-GPU one), the others None."""
    import time

    import numpy as np
    import torch.distributed as dist

    from .api import HullResult, HullStats, convex_hull_3d, orient_remap, to_host
    from .engine import level_count

    rank, world = dist.get_rank(), dist.get_world_size()
    dev = device or torch.device("cuda", torch.cuda.current_device())
    t0 = time.perf_counter()
    pts = gather_input(points, dev, rank, world)
    n = pts.shape[0]
    if world == 1 or n <= 3 or SlabPlan(n, world).G == 1:
        return convex_hull_3d(pts, return_device=return_device) if rank == 0 else None
    from .api import _device_lock

    # the per-device workspaces (presort, both passes) are shared with
    # convex_hull_3d: hold the device's lock while they are in use, and
    # launch on `dev` whatever the caller's current device is
    with _device_lock(dev), torch.cuda.device(dev):
        res = hull_distributed(pts, rank, world)
        if rank == 0 and res is not None:
            raw, k_lo, k_up, rows_v, order_v, perturbed, sharded, _mem = res
            # faces index the virtual rows; the centroid is taken over the
            # caller-order input (the same points) and the vertex marks over
            # the caller indices
            verts, faces = orient_remap(rows_v, order_v, raw, pts, n_callers=n)
    if rank != 0:
        return None
    if res is None:  # exact engine, single GPU, reference semantics (takes the lock itself)
        return convex_hull_3d(pts, _exact_backend(dev), return_device=return_device)
    total_ms = (time.perf_counter() - t0) * 1e3
    stats = HullStats(n=n, levels=level_count(n), lower_events=k_lo, upper_events=k_up,
                      sort_ms=0.0, lower_ms=0.0, upper_ms=0.0, total_ms=total_ms,
                      perturbed=perturbed, solver="parallel", workers=world)
    if not return_device:
        verts, faces = to_host(verts), to_host(faces)
    return HullResult(vertices=verts, faces=faces, stats=stats)


def _exact_backend(dev):
    from .api import CudaBackend

    return CudaBackend(dev, engine="exact")


__all__ = ["SlabPlan", "GroupLayout", "send_group", "recv_group", "hull_distributed",
           "convex_hull_3d_distributed"]
