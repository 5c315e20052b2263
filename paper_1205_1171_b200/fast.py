"""Fused fast engine: both hull passes over compact groups (csrc/fast.cu).

The final logs equal the reference's (tests/test_gpu_fast.py checks every
level's log against the reference's per-level buffers).  If the device
reports that the fast path cannot reproduce the reference semantics for an
input (degenerate inputs: an exact tie between event times, a child event
whose stored facet or kind disagrees with the current links, a
compact-capacity overflow, a dangling link), or any merge
error, the pass is rerun on the exact seam engine, which reproduces the
reference's behaviour (and its exceptions) step for step.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .engine import stream_ptr

E_FASTPATH = -13
E_VERIFY = -14

# verify mode (tests): every level's groups are checked on the device
# (csrc/fast.cu k_verify_level); a violation raises VerifyError
VERIFY = [0]


class VerifyError(AssertionError):
    """A level of the fast path wrote a group that fails the device checks."""


class verifying:
    """Context manager: run the fast path in verify mode."""

    def __enter__(self):
        self.old = VERIFY[0]
        VERIFY[0] = 1
        return self

    def __exit__(self, *exc):
        VERIFY[0] = self.old
        return False

# how many pass pairs the exact engine had to redo (tests assert 0 on
# general-position inputs: the fast path must be the one that runs)
FALLBACKS = [0]
LAST_ERROR = [0]


class _WS:
    """Grow-only per-device workspaces for the two passes."""

    cache: dict = {}

    @classmethod
    def get(cls, device, which: int, nbytes: int) -> torch.Tensor:
        key = (device, which)
        buf = cls.cache.get(key)
        if buf is None or buf.numel() < nbytes:
            cls.cache.pop(key, None)
            buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
            cls.cache[key] = buf
        return buf


def tune(name: str, value: int = -1) -> int:
    """Set (value >= 0) or query a routing knob of the fast path; returns the
    previous value (csrc/fast.cu h3d_tune)."""
    r = int(_lib.load().h3d_tune(name.encode(), int(value)))
    if r < 0:
        raise KeyError(name)
    return r


class tuned:
    """Context manager: temporarily set routing knobs, e.g.
    ``with fast.tuned(big_kin=16): ...``"""

    def __init__(self, **kv):
        self.kv = kv
        self.old: dict = {}

    def __enter__(self):
        for k, v in self.kv.items():
            self.old[k] = tune(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.old.items():
            tune(k, v)
        return False


def profile_enable(on: int) -> None:
    """0 off; 1 (True): every level bracketed by CUDA events; 2: only the
    lane-per-job kernel launches (bench.py's roofline)."""
    _lib.load().h3d_profile_enable(int(on))


def kernel_of(tag: int):
    """Decode a profile row's level tag -> (kernel name, level)."""
    if tag >= 5000:
        return "k_mini", tag - 5000
    if tag >= 4000:
        return "k_big_level", tag - 4000
    if tag >= 3000:
        return "k_fast_leaf", -(tag - 3000)
    if tag >= 2000:
        return "k_fast_init1", tag - 2000
    if tag >= 1000:
        return "k_fast_tpj", tag - 1000
    if tag < 0:
        return "k_fast_leaf", tag
    return "k_fast_warp", tag


def profile_collect(max_rows: int = 4096):
    """[(level, pass, ms)] recorded since the last collect."""
    L = _lib.load()
    lv = np.zeros(max_rows, dtype=np.int32)
    ps = np.zeros(max_rows, dtype=np.int32)
    ms = np.zeros(max_rows, dtype=np.float32)
    m = L.h3d_profile_collect(lv.ctypes.data, ps.ctypes.data, ms.ctypes.data, max_rows)
    return [(int(lv[i]), int(ps[i]), float(ms[i])) for i in range(m)]


STAMP_SLOTS = 64
STAMP_END = 40
# the level rows (tag, pass, ms) of the last run_both(stamps=True) of this
# thread's caller: device time stamps, no event records (csrc/common.cu)
LAST_LEVEL_ROWS: list = []
LAST_SORT_MS: list = [None]  # the last stamped hull's presort (device ms)


def stamp_rows(stamps, routes) -> list:
    """Device level stamps (ns) + host route tags -> [(tag, 2, ms)]: each
    stamped level lasts until the next stamped one (the last until the end
    stamp); 2 = one launch covering both passes."""
    slots = [lv for lv in range(1, STAMP_END) if routes[lv] >= 0 and stamps[lv] > 0]
    rows = []
    for i, lv in enumerate(slots):
        t1 = stamps[slots[i + 1]] if i + 1 < len(slots) else stamps[STAMP_END]
        rows.append((int(routes[lv]), 2, max(0.0, (int(t1) - int(stamps[lv])) / 1e6)))
    return rows


def run_both(sorted_pts: torch.Tensor, stamps: bool = False):
    """Both passes + facet extraction.  Returns (raw faces int32 (F,3) on
    device, lower count, upper count) or None when the exact engine must
    take over.  stamps: record per-level device time stamps (read back with
    the counts in the one synchronisation) into LAST_LEVEL_ROWS."""
    L = _lib.load()
    n = sorted_pts.shape[0]
    dev = sorted_pts.device
    s = stream_ptr(dev)
    wsb = int(L.h3d_fast_pass_workspace_bytes(n))
    ws_lo = _WS.get(dev, 0, wsb)
    ws_up = _WS.get(dev, 1, int(L.h3d_fast_upper_workspace_bytes(n)))
    # err, kLo, kUp, verify diagnostics, then the level stamps
    state = torch.zeros(4 + (STAMP_SLOTS if stamps else 0), dtype=torch.int64, device=dev)
    err = state[0:1]
    counts = state[1:3]
    fin = (ctypes.c_int64 * 2)()
    if stamps:
        L.h3d_profile_stamps(state[4:].data_ptr())
    try:
        r = L.h3d_fast_passes(sorted_pts.data_ptr(), n, ws_lo.data_ptr(), ws_up.data_ptr(), wsb,
                              err.data_ptr(), 2 if VERIFY[0] else 0, ctypes.addressof(fin), s)
    finally:
        if stamps:
            routes = np.zeros(STAMP_SLOTS, dtype=np.int32)
            L.h3d_profile_routes(routes.ctypes.data, STAMP_SLOTS)
            L.h3d_profile_stamps(None)
    if r < 0:
        from .errors import check_merge

        check_merge(int(r))
    fin = [int(fin[0]), int(fin[1])]
    cap = max(2 * n, 8)
    faces = torch.empty((cap, 3), dtype=torch.int32, device=dev)
    r = L.h3d_fast_extract(ws_lo.data_ptr(), ws_up.data_ptr(), n, fin[0], fin[1],
                           faces.data_ptr(), cap, counts.data_ptr(), err.data_ptr(), s)
    if r < 0:
        from .errors import check_merge

        check_merge(int(r))
    h = state.cpu()  # the one host sync of the pass pair
    if int(h[0]) == E_VERIFY:
        d = int(h[3]) & ((1 << 64) - 1)
        raise VerifyError("fast path: a level wrote a group that fails the device checks "
                          f"(check {d >> 60}, level {(d >> 54) & 63}, pass {(d >> 53) & 1}, "
                          f"group {(d >> 20) & 0xffffffff}, item {d & 0xfffff})")
    if int(h[0]) != 0:
        FALLBACKS[0] += 1
        LAST_ERROR[0] = int(h[0])
        return None
    k_lo, k_up = int(h[1]), int(h[2])
    if stamps:
        LAST_LEVEL_ROWS[:] = stamp_rows(h[4:].numpy(), routes)
    return faces[: k_lo + k_up], k_lo, k_up


HULL_STATE = 96
HULL_INFO = 128
_STAMP_AT = HULL_INFO - HULL_STATE + 8  # info index of stamp slot 0


class HullOut:
    """Result of one h3d_hull call (csrc/hull.cu)."""

    __slots__ = ("faces", "vertices", "k_lo", "k_up", "perturbed", "declined", "sorted_pts",
                 "order", "level_rows", "sort_ms", "passes_ms")


def hull(pts: torch.Tensor, stamps: bool = True) -> HullOut:
    """The whole device pipeline in one C-ABI call: presort, both passes,
    extraction, orientation/remap/vertex compaction, one read-back.  faces
    and vertices are views of per-device cached buffers (copy before the
    next call).  declined != 0: the fast path declined the input, run the
    exact engine on sorted_pts/order.  Raises the API's exceptions."""
    from .errors import check_api

    L = _lib.load()
    n = pts.shape[0]
    dev = pts.device
    s = stream_ptr(dev)
    wsb = int(L.h3d_fast_pass_workspace_bytes(n))
    pwsb = int(L.h3d_presort_workspace_bytes(n))
    ws_lo = _WS.get(dev, 0, wsb)
    ws_up = _WS.get(dev, 1, int(L.h3d_fast_upper_workspace_bytes(n)))
    pws = _WS.get(dev, 2, pwsb)
    cap = 2 * n
    # outputs and scratch, carved from one cached buffer per device
    o_sorted, o_order, o_raw = 0, 24 * n, 32 * n
    o_faces = o_raw + 12 * cap
    o_verts = o_faces + 24 * cap
    o_mark = o_verts + 8 * n
    o_state = (o_mark + 4 * n + 255) & ~255
    total = o_state + 8 * HULL_STATE
    buf = _WS.get(dev, 3, total)
    base = buf.data_ptr()
    info = np.zeros(HULL_INFO, dtype=np.int64)
    flags = (1 if stamps else 0) | (2 if VERIFY[0] else 0)
    rc = L.h3d_hull(pts.data_ptr(), n, base + o_sorted, base + o_order, pws.data_ptr(), pwsb,
                    ws_lo.data_ptr(), ws_up.data_ptr(), wsb, base + o_raw, cap, base + o_faces,
                    base + o_verts, base + o_mark, base + o_state, flags, info.ctypes.data, s)
    routes = None
    if stamps:
        routes = np.zeros(STAMP_SLOTS, dtype=np.int32)
        L.h3d_profile_routes(routes.ctypes.data, STAMP_SLOTS)
    check_api(int(rc))
    out = HullOut()
    out.sorted_pts = buf[o_sorted:o_sorted + 24 * n].view(torch.float64).view(n, 3)
    out.order = buf[o_order:o_order + 8 * n].view(torch.int64)
    out.declined = int(info[0])
    out.perturbed = bool(info[5])
    out.k_lo, out.k_up = int(info[1]), int(info[2])
    out.level_rows, out.sort_ms, out.passes_ms = [], None, None
    if out.declined == E_VERIFY:
        d = int(info[7]) & ((1 << 64) - 1)
        raise VerifyError("fast path: a level wrote a group that fails the device checks "
                          f"(check {d >> 60}, level {(d >> 54) & 63}, pass {(d >> 53) & 1}, "
                          f"group {(d >> 20) & 0xffffffff}, item {d & 0xfffff})")
    if out.declined:
        FALLBACKS[0] += 1
        LAST_ERROR[0] = out.declined
        out.faces = out.vertices = None
        return out
    F, V = int(info[3]), int(info[4])
    out.faces = buf[o_faces:o_faces + 24 * F].view(torch.int64).view(F, 3)
    out.vertices = buf[o_verts:o_verts + 8 * V].view(torch.int64)
    if stamps:
        st = info[_STAMP_AT:_STAMP_AT + STAMP_SLOTS]
        out.level_rows = stamp_rows(st, routes)
        LAST_LEVEL_ROWS[:] = out.level_rows
        if st[0] > 0 and st[1] > 0:
            out.sort_ms = (int(st[1]) - int(st[0])) / 1e6
            LAST_SORT_MS[0] = out.sort_ms
        if st[1] > 0 and st[STAMP_END] > 0:
            out.passes_ms = (int(st[STAMP_END]) - int(st[1])) / 1e6
    return out


__all__ = ["run_both", "hull", "HullOut", "profile_enable", "profile_collect", "E_FASTPATH", "E_VERIFY", "VERIFY",
           "VerifyError", "verifying", "ctypes"]
