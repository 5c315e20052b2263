"""Public entry point -- drop-in for ``hull3d.convex_hull_3d``.

Same signature, result types, orientation, vertex order, stats semantics
and exceptions as pkg/src/hull3d/api.py:162-284.  Every step after the
host->device copy runs on the B200: presort + tie perturbation + degeneracy
scan (csrc/presort.cu), both hull passes (engine.py), facet extraction and
the orientation/remap/unique epilogue.  There is no CPU fallback: without a
CUDA device or the built library this raises.
"""

from __future__ import annotations

import os
import threading
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .engine import level_count, run_pass_exact, stream_ptr
from .errors import DegenerateInputError, check_api


@dataclass
class HullStats:
    """Run metadata (api.py:28-44).  As in the reference, ``*_level_ms``
    hold per-level SECONDS and are empty for the serial
    solver."""

    n: int
    levels: int
    lower_events: int
    upper_events: int
    sort_ms: float
    lower_ms: float
    upper_ms: float
    total_ms: float
    perturbed: bool
    solver: str
    workers: int
    lower_level_ms: list[float] = field(default_factory=list)
    upper_level_ms: list[float] = field(default_factory=list)


@dataclass
class HullResult:
    """Hull vertices (sorted ascending) and outward-oriented facets, both in
    the caller's input indexing (api.py:47-58).  With ``return_device=True``
    the arrays are CUDA int64 tensors instead of numpy arrays."""

    vertices: np.ndarray
    faces: np.ndarray
    stats: HullStats

    def face_set(self) -> set[tuple[int, int, int]]:
        faces = self.faces.cpu().numpy() if isinstance(self.faces, torch.Tensor) else self.faces
        return {tuple(sorted(map(int, row))) for row in faces}


class CudaBackend:
    """Backend object selecting the B200 engine (passed in the reference's
    ``backend`` slot).  ``workers`` is reported in HullStats like the
    reference's ThreadBackend.workers."""

    def __init__(self, device: int | str | torch.device | None = None, engine: str = "fast"):
        if not torch.cuda.is_available():
            raise RuntimeError("CudaBackend needs a CUDA device")
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        if engine not in ("fast", "exact"):
            raise ValueError(f"unknown engine {engine!r}")
        self.engine = engine
        self.workers = 1

    def __repr__(self):
        return f"CudaBackend(device={self.device}, engine={self.engine!r})"


_LOCKS: dict = {}
_LOCKS_GUARD = threading.Lock()


def _device_lock(dev: torch.device) -> threading.Lock:
    with _LOCKS_GUARD:
        return _LOCKS.setdefault(str(dev), threading.Lock())


def _device_of(points, backend) -> torch.device:
    if isinstance(backend, CudaBackend):
        return backend.device
    if isinstance(points, torch.Tensor) and points.is_cuda:
        return points.device
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1205_1171_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


class _Workspace:
    """Grow-only device scratch per (device) for presort/epilogue."""

    _cache: dict = {}

    @classmethod
    def get(cls, device: torch.device, nbytes: int) -> torch.Tensor:
        buf = cls._cache.get(device)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
            cls._cache[device] = buf
        return buf


def presort(pts_dev: torch.Tensor):
    """Device _sort_and_perturb + _scan_degenerate -> (sorted, order, perturbed)."""
    L = _lib.load()
    n = pts_dev.shape[0]
    dev = pts_dev.device
    ws_bytes = int(L.h3d_presort_workspace_bytes(n))
    ws = _Workspace.get(dev, ws_bytes)
    sorted_pts = torch.empty((n, 3), dtype=torch.float64, device=dev)
    order = torch.empty(n, dtype=torch.int64, device=dev)
    import ctypes

    pert = ctypes.c_int32(0)
    code = L.h3d_presort(pts_dev.data_ptr(), n, sorted_pts.data_ptr(), order.data_ptr(),
                         ws.data_ptr(), ws.numel(), ctypes.addressof(pert), stream_ptr(dev))
    check_api(code)
    return sorted_pts, order, bool(pert.value)


def orient_remap(sorted_pts: torch.Tensor, order: torch.Tensor, raw: torch.Tensor,
                 centroid_pts: torch.Tensor | None = None, n_callers: int | None = None):
    """Device api.py:252-266 -> (vertices i64, faces i64) on device.
    centroid_pts: rows the centroid is taken over (default sorted_pts; the
    multi-GPU path passes the caller-order input, with n_callers = the
    number of caller points when sorted_pts holds only the rows the faces
    index)."""
    L = _lib.load()
    n = n_callers if n_callers is not None else sorted_pts.shape[0]
    dev = sorted_pts.device
    F = raw.shape[0]
    if F == 0:
        raise DegenerateInputError("no facets produced; input is degenerate")
    ws_bytes = int(L.h3d_epilogue_workspace_bytes(n))
    ws = _Workspace.get(dev, ws_bytes)
    faces = torch.empty((F, 3), dtype=torch.int64, device=dev)
    mark = torch.empty(n, dtype=torch.int32, device=dev)
    verts = torch.empty(n, dtype=torch.int64, device=dev)
    raw = raw.contiguous()
    cen = centroid_pts.contiguous().data_ptr() if centroid_pts is not None else None
    h = check_api(L.h3d_orient_remap_ex(sorted_pts.data_ptr(), n, order.data_ptr(), raw.data_ptr(),
                                        F, faces.data_ptr(), mark.data_ptr(), verts.data_ptr(),
                                        cen, ws.data_ptr(), ws.numel(), stream_ptr(dev)))
    return verts[:h], faces


def to_host(t: torch.Tensor) -> np.ndarray:
    """Device result -> numpy.  Large results go through a fresh pinned
    buffer (the returned array owns it): a pageable copy of a sphere's 2M
    faces costs ~2x more (tools/d2h_probe.py)."""
    if t.numel() * t.element_size() < (1 << 20):
        return t.cpu().numpy()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


def _to_device(points, dev: torch.device) -> torch.Tensor:
    if isinstance(points, torch.Tensor):
        t = points.to(dtype=torch.float64)
        if t.ndim != 2 or t.shape[1] != 3:
            raise ValueError("points must have shape (n, 3)")
        if not t.is_cuda:
            t = t.to(dev, non_blocking=t.is_pinned())
        elif t.device != dev:
            t = t.to(dev)
        return t.contiguous()
    coords = np.asarray(points, dtype=np.float64)
    if coords.ndim != 2 or coords.shape[1] != 3:
        raise ValueError("points must have shape (n, 3)")
    return torch.from_numpy(np.ascontiguousarray(coords)).to(dev)


def _level_rows_to_stats(rows, n, level_lists):
    """Profile rows -> per-level seconds per pass (F12) and the two passes'
    shares of the kernel time."""
    from . import engine as E
    from . import fast

    ms = [0.0, 0.0]
    nlev = level_count(n)
    per = [[0.0] * nlev, [0.0] * nlev]
    for lv, p, t in rows:
        name, lv = fast.kernel_of(lv)
        # pass 2 = one launch covering both passes: split evenly
        shares = ((0, t / 2), (1, t / 2)) if p == 2 else ((p, t),)
        for pp, tt in shares:
            ms[pp] += tt
            # a negative level is a fused kernel (levels 1..|lv|); its time
            # is reported at its last level, 0.0 below it
            per[pp][abs(lv) - 1] += tt / 1e3
        if E.PROFILE is not None:
            E.PROFILE.append((name, p, lv, t))
    if level_lists is not None:
        level_lists[0].extend(per[0])
        level_lists[1].extend(per[1])
    return ms


def _run_passes(sorted_pts, engine, solver, level_lists):
    """Both passes; returns (raw faces int32 (F,3) on device, lower count,
    upper count, finish).  Per-level times (solver="parallel") come from
    device time stamps written by the level kernels themselves and read back
    with the facet counts (no event records, no extra synchronisation);
    ``finish()`` turns them into per-level seconds (like the reference's
    perf_counter deltas) and the two passes' shares.  Tools
    that set engine.PROFILE get per-level CUDA events instead; bench.py's
    engine.KERNEL_EVENTS brackets only the lane-per-job kernel launches."""
    from . import engine as E
    from . import fast

    want_levels = solver == "parallel"
    if engine == "fast":
        t0 = time.perf_counter()
        ev_mode = 1 if E.PROFILE is not None else (2 if E.KERNEL_EVENTS else 0)
        if ev_mode:
            fast.profile_enable(ev_mode)
        try:
            res = fast.run_both(sorted_pts, stamps=want_levels and ev_mode != 1)
        finally:
            if ev_mode:
                fast.profile_enable(0)
        if res is not None:
            dt = (time.perf_counter() - t0) * 1e3
            raw, k_lo, k_up = res
            split = [dt / 2, dt / 2]
            rows = list(fast.LAST_LEVEL_ROWS) if want_levels and ev_mode != 1 else None

            def finish():
                if ev_mode == 1:
                    if E.PROFILE_DEFER:
                        # deferred: the records stay with this thread until the
                        # caller collects a whole timed loop at once
                        return split
                    lrows = fast.profile_collect()
                else:
                    lrows = rows
                if not lrows:
                    return split
                ms = _level_rows_to_stats(lrows, sorted_pts.shape[0],
                                          level_lists if want_levels else None)
                tot = ms[0] + ms[1]
                lo = dt * ms[0] / tot if tot > 0 else dt / 2
                return [lo, dt - lo]

            return raw, k_lo, k_up, finish
        if ev_mode:
            fast.profile_collect()  # drop the declined run's records
    out = []
    ms = []
    for which, zsign in ((0, 1.0), (1, -1.0)):
        t0 = time.perf_counter()
        lv = level_lists[which] if want_levels else None
        raw = run_pass_exact(sorted_pts, zsign, lv)
        torch.cuda.current_stream(sorted_pts.device).synchronize()
        ms.append((time.perf_counter() - t0) * 1e3)
        out.append(raw)
    return torch.cat(out), out[0].shape[0], out[1].shape[0], (lambda: ms)


def convex_hull_3d(points, backend=None, *, solver: str = "parallel",
                   concurrent_passes: bool | None = None,
                   return_device: bool = False) -> HullResult:
    """Convex hull of 3D points on the B200 (drop-in for api.py:162-284).

    ``points`` may be any (n,3) array-like, a CPU tensor (pinned tensors are
    copied asynchronously) or a CUDA tensor (device-resident input).
    ``solver`` is accepted for signature compatibility: both values run the
    device engine, whose final logs equal the serial solver's (the final
    movie is canonical, tests/test_serial_parallel.py:106-116 in the
    reference); as in the reference, the serial solver reports no per-level
    times.  ``concurrent_passes`` is accepted and ignored (both passes are
    stream-ordered on one device).
    """
    if solver not in ("parallel", "serial"):
        raise ValueError(f"unknown solver {solver!r}")
    total_t0 = time.perf_counter()
    dev = _device_of(points, backend)
    pts = _to_device(points, dev)
    n = pts.shape[0]
    if n == 0:
        raise ValueError("no points")
    workers = getattr(backend, "workers", 1)
    engine = getattr(backend, "engine", "fast")
    if n <= 3:
        if not bool(torch.isfinite(pts).all()):
            raise ValueError("coordinates must be finite")
        total_ms = (time.perf_counter() - total_t0) * 1e3
        stats = HullStats(n=n, levels=0, lower_events=0, upper_events=0, sort_ms=0.0,
                          lower_ms=0.0, upper_ms=0.0, total_ms=total_ms, perturbed=False,
                          solver=solver, workers=workers)
        verts = torch.arange(n, dtype=torch.int64, device=dev)
        faces = torch.empty((0, 3), dtype=torch.int64, device=dev)
        if not return_device:
            verts, faces = verts.cpu().numpy(), faces.cpu().numpy()
        return HullResult(vertices=verts, faces=faces, stats=stats)

    # the per-device workspaces are shared: one hull at a time per device
    # (calls from several threads are serialised, not interleaved); every
    # launch goes to `dev` whatever the caller's current device is
    from . import engine as E

    with _device_lock(dev), torch.cuda.device(dev):
        if engine == "fast" and E.PROFILE is None:
            # the whole device pipeline in one native call (csrc/hull.cu)
            from . import fast

            if E.KERNEL_EVENTS:  # bench.py: events around the lane-per-job launches
                fast.profile_enable(2)
            try:
                h = fast.hull(pts, stamps=True)
            finally:
                if E.KERNEL_EVENTS:
                    fast.profile_enable(0)
            if not h.declined:
                lower_levels: list[float] = []
                upper_levels: list[float] = []
                if solver == "parallel" and h.level_rows:
                    _level_rows_to_stats(h.level_rows, n, (lower_levels, upper_levels))
                verts, faces = h.vertices, h.faces
                if return_device:  # own the result (the buffers are reused)
                    verts, faces = verts.clone(), faces.clone()
                else:
                    verts, faces = to_host(verts), to_host(faces)
                total_ms = (time.perf_counter() - total_t0) * 1e3
                pass_ms = h.passes_ms if h.passes_ms is not None else 0.0
                stats = HullStats(n=n, levels=level_count(n), lower_events=h.k_lo,
                                  upper_events=h.k_up,
                                  sort_ms=h.sort_ms if h.sort_ms is not None else 0.0,
                                  lower_ms=pass_ms / 2, upper_ms=pass_ms / 2, total_ms=total_ms,
                                  perturbed=h.perturbed, solver=solver, workers=workers,
                                  lower_level_ms=lower_levels, upper_level_ms=upper_levels)
                return HullResult(vertices=verts, faces=faces, stats=stats)
            # declined: the exact engine on the rows the call presorted
            sorted_pts, order, perturbed = h.sorted_pts.clone(), h.order.clone(), h.perturbed
            sort_ms = h.sort_ms or 0.0
            engine = "exact"
        else:
            sort_t0 = time.perf_counter()
            sorted_pts, order, perturbed = presort(pts)
            sort_ms = (time.perf_counter() - sort_t0) * 1e3

        lower_levels: list[float] = []
        upper_levels: list[float] = []
        raw, k_lo, k_up, finish = _run_passes(sorted_pts, engine, solver,
                                              (lower_levels, upper_levels))
        verts, faces = orient_remap(sorted_pts, order, raw)
        if not return_device:
            verts, faces = to_host(verts), to_host(faces)
        lo_ms, up_ms = finish()
    total_ms = (time.perf_counter() - total_t0) * 1e3
    stats = HullStats(n=n, levels=level_count(n), lower_events=int(k_lo),
                      upper_events=int(k_up), sort_ms=sort_ms, lower_ms=lo_ms,
                      upper_ms=up_ms, total_ms=total_ms, perturbed=perturbed, solver=solver,
                      workers=workers, lower_level_ms=lower_levels, upper_level_ms=upper_levels)
    return HullResult(vertices=verts, faces=faces, stats=stats)


def convex_hull_3d_stream(clouds, backend=None, *, solver: str = "parallel", return_device: bool = False):
    """Throughput form of convex_hull_3d for a sequence of clouds (an
    extension, not a reference interface): yields one HullResult per cloud,
    in order, each identical to ``convex_hull_3d(cloud, backend, ...)``.
    While cloud i's hull runs, the host->device copy of cloud i+1 already
    runs on a second CUDA stream (pinned CPU tensors copy asynchronously by
    DMA), so the PCIe transfer hides behind the previous hull's kernels.
    Every cloud is still copied in full; nothing is cached between clouds."""
    it = iter(clouds)
    dev = _device_of(None, backend)
    copy_stream = torch.cuda.Stream(device=dev)
    bufs: list = [None, None]

    def stage(cloud, slot):
        host = cloud if isinstance(cloud, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(np.asarray(cloud, dtype=np.float64)))
        if host.is_cuda:
            return host, None
        host = host.to(dtype=torch.float64)
        if host.ndim != 2 or host.shape[1] != 3:
            raise ValueError("points must have shape (n, 3)")
        b = bufs[slot]
        if b is None or b.shape != host.shape:
            b = bufs[slot] = torch.empty(host.shape, dtype=torch.float64, device=dev)
        with torch.cuda.stream(copy_stream):
            b.copy_(host, non_blocking=host.is_pinned())
            ev = torch.cuda.Event()
            ev.record(copy_stream)
        return b, ev

    try:
        nxt = stage(next(it), 0)
    except StopIteration:
        return
    slot = 0
    while nxt is not None:
        cur, ev = nxt
        try:  # the next cloud's copy starts before this hull runs
            nxt = stage(next(it), slot ^ 1)
        except StopIteration:
            nxt = None
        if ev is not None:
            torch.cuda.current_stream(dev).wait_event(ev)
        yield convex_hull_3d(cur, backend, solver=solver, return_device=return_device)
        slot ^= 1


def perturb_ties(points) -> np.ndarray:
    """api.py:61-83, exposed for API parity (host helper, not on the hot path:
    the device presort performs the same perturbation in csrc/presort.cu)."""
    pts = np.array(points, dtype=np.float64, copy=True)
    x = pts[:, 0]
    n = len(x)
    eps16 = 16 * np.finfo(np.float64).eps
    i = 0
    while i < n:
        j = i + 1
        while j < n and x[j] == x[i]:
            j += 1
        if j - i > 1:
            base = x[i]
            step = eps16 * max(1.0, abs(base))
            for rank in range(1, j - i):
                x[i + rank] = base + rank * step
        i = j
    return pts
