"""The reference's kernel-module seam, served by the B200 library.

Mirrors the module interface ``hull3d.kernels.active()`` returns
(pkg/src/hull3d/kernels.py:52-54, functions of _ckernels.pyx:231-375):
``IMPL``, ``NIL``, the ``E_*`` codes and the functions below, with the same
argument meaning, in-place mutation and negative-code returns -- but every
buffer is a CUDA tensor (pts f64 (n,3), links i32 (n,2), slots i32 (2n),
jobs i64 (m,3), faces i32 (limit,3)).  The calls are blocking, like the
reference's.  ``hull_recursive`` (the top-down serial solver) is not part of
the B200 path and is not provided.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .engine import stream_ptr

IMPL = "b200"
NIL = -1
E_OVERFLOW = -1
E_BRIDGE = -2
E_CHAIN = -3
E_COUNT = -4
E_UNTERMINATED = -5


def _chk(*tensors):
    for t in tensors:
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous()):
            raise TypeError("seam buffers must be contiguous CUDA tensors")
    return stream_ptr(tensors[0].device)


def act(links, i):
    s = _chk(links)
    return int(_lib.load().h3d_seam_act(links.data_ptr(), int(i), s))


def init_base_logs(links, slots, n):
    s = _chk(links, slots)
    return int(_lib.load().h3d_seam_init_base_logs(links.data_ptr(), slots.data_ptr(), int(n), s))


def find_initial_bridge(pts, links, u, v, limit):
    s = _chk(pts, links)
    out = (ctypes.c_int64 * 2)()
    _lib.load().h3d_seam_find_initial_bridge(pts.data_ptr(), links.data_ptr(), int(u), int(v),
                                             int(limit), ctypes.addressof(out), s)
    return int(out[0]), int(out[1])


def merge_movies(pts, links, in_slots, out_slots, L, M, R):
    s = _chk(pts, links, in_slots, out_slots)
    return int(_lib.load().h3d_seam_merge_movies(pts.data_ptr(), links.data_ptr(),
                                                 in_slots.data_ptr(), out_slots.data_ptr(),
                                                 int(L), int(M), int(R), s))


def merge_range(pts, links, in_slots, out_slots, jobs, lo, hi):
    s = _chk(pts, links, in_slots, out_slots, jobs)
    return int(_lib.load().h3d_seam_merge_range(pts.data_ptr(), links.data_ptr(),
                                                in_slots.data_ptr(), out_slots.data_ptr(),
                                                jobs.data_ptr(), int(lo), int(hi), s))


def replay(links, slots, off, count):
    s = _chk(links, slots)
    return int(_lib.load().h3d_seam_replay(links.data_ptr(), slots.data_ptr(), int(off),
                                           int(count), s))


def rewind_replay(links, slots, off, count):
    s = _chk(links, slots)
    return int(_lib.load().h3d_seam_rewind_replay(links.data_ptr(), slots.data_ptr(), int(off),
                                                  int(count), s))


def extract_faces(links, slots, off, faces):
    s = _chk(links, slots, faces)
    return int(_lib.load().h3d_seam_extract_faces(links.data_ptr(), slots.data_ptr(), int(off),
                                                  faces.data_ptr(), int(faces.shape[0]), s))


def log_length(slots, off, cap):
    s = _chk(slots)
    return int(_lib.load().h3d_seam_log_length(slots.data_ptr(), int(off), int(cap), s))


def copy_log(src, dst, off, cap):
    s = _chk(src, dst)
    return int(_lib.load().h3d_seam_copy_log(src.data_ptr(), dst.data_ptr(), int(off), int(cap), s))


def run_level(pts, links, in_slots, out_slots, n, level, zsign=1.0):
    """One whole level of build_movie in one launch (B200 addition)."""
    s = _chk(pts, links, in_slots, out_slots)
    return int(_lib.load().h3d_seam_run_level(pts.data_ptr(), float(zsign), links.data_ptr(),
                                              in_slots.data_ptr(), out_slots.data_ptr(), int(n),
                                              int(level), s))
