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


def profile_enable(on: bool) -> None:
    _lib.load().h3d_profile_enable(1 if on else 0)


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
    ws_up = _WS.get(dev, 1, wsb)
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


__all__ = ["run_both", "profile_enable", "profile_collect", "E_FASTPATH", "E_VERIFY", "VERIFY",
           "VerifyError", "verifying", "ctypes"]
