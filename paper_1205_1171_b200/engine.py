"""Device level scheduler for one hull pass (the B200 ``build_movie``).

The reference drives ``ceil(log2 n)`` merge levels from Python, one thread-
pool dispatch per level (pkg/src/hull3d/parallel.py:68-112).  Here a pass is
a sequence of stream-ordered launches over preallocated fixed-capacity
buffers; nothing is allocated per level and nothing is read back until the
facets are extracted.

Two engines produce the same final log (the merged log is canonical,
SURVEY.md F4):

* ``exact``: the seam kernels (csrc/seam.cu), one launch per level with the
  reference's sequential merge per job on the reference layout.  Used for
  per-level parity tests and as the reference-semantics mode.
* ``fast``: the fused path (csrc/fast.cu) -- see DESIGN.md.
"""

from __future__ import annotations

import time

import torch

from . import _lib
from .errors import check_merge, check_store

NIL = -1

# bench.py instrumentation: when a list, every merge-level launch appends
# (kernel name, pass index, level, device milliseconds)
PROFILE: list | None = None
# bench.py: leave the fast path's per-level device events with the calling
# thread instead of collecting them per call (one collection per timed loop,
# no per-call synchronisation inside the timed region)
PROFILE_DEFER = False
# bench.py: CUDA events around the lane-per-job kernel launches only (the
# dominant kernel's duration for the roofline), collected by the caller
KERNEL_EVENTS = False


def level_count(n: int) -> int:
    """parallel.py:27-31"""
    if n < 1:
        raise ValueError("no points")
    return (n - 1).bit_length()


def stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def record_start():
    if PROFILE is None:
        return None
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def record_end(e0, name: str, pass_idx: int, level: int, device=None) -> None:
    if e0 is None or PROFILE is None:
        return
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record()
    e1.synchronize()
    PROFILE.append((name, pass_idx, level, e0.elapsed_time(e1)))


def launch_count() -> int:
    return int(_lib.load().h3d_launch_count())


def sync_count() -> int:
    """Host synchronisations the library made so far (h3d_sync_count)."""
    return int(_lib.load().h3d_sync_count())


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


class ExactPass:
    """Reference-layout state of one pass: links (n,2) i32, two slot buffers."""

    def __init__(self, n: int, device: torch.device):
        self.n = n
        self.device = device
        self.links = torch.empty((n, 2), dtype=torch.int32, device=device)
        self.A = torch.full((2 * n,), NIL, dtype=torch.int32, device=device)
        self.B = torch.full((2 * n,), NIL, dtype=torch.int32, device=device)

    def init(self) -> None:
        L = _lib.load()
        check_store(L.h3d_seam_init_base_logs(_ptr(self.links), _ptr(self.A), self.n,
                                             stream_ptr(self.device)))

    def levels(self, pts: torch.Tensor, zsign: float, level_times=None):
        """Run every level; yields (level, out buffer) after each one."""
        L = _lib.load()
        src, dst = self.A, self.B
        s = stream_ptr(self.device)
        pidx = 0 if zsign > 0 else 1
        for lv in range(1, level_count(self.n) + 1):
            t0 = time.perf_counter()
            ev = record_start()
            check_merge(L.h3d_seam_run_level(_ptr(pts), zsign, _ptr(self.links), _ptr(src),
                                             _ptr(dst), self.n, lv, s))
            record_end(ev, "k_level_exact", pidx, lv, self.device)
            if level_times is not None:
                level_times.append(time.perf_counter() - t0)
            yield lv, dst
            src, dst = dst, src

    def run(self, pts: torch.Tensor, zsign: float, level_times=None) -> torch.Tensor:
        self.init()
        final = self.A
        for _, buf in self.levels(pts, zsign, level_times):
            final = buf
        return final

    def extract(self, final: torch.Tensor) -> torch.Tensor:
        L = _lib.load()
        limit = 2 * self.n
        faces = torch.empty((limit, 3), dtype=torch.int32, device=self.device)
        m = check_store(L.h3d_seam_extract_faces(_ptr(self.links), _ptr(final), 0, _ptr(faces),
                                                 limit, stream_ptr(self.device)))
        return faces[:m]


def run_pass_exact(pts: torch.Tensor, zsign: float, level_times=None) -> torch.Tensor:
    """Raw (prev, e, next) facet triples of one pass, sorted indices, int32."""
    n = pts.shape[0]
    st = ExactPass(n, pts.device)
    if n == 1:
        st.init()
        return torch.empty((0, 3), dtype=torch.int32, device=pts.device)
    final = st.run(pts, zsign, level_times)
    return st.extract(final)
