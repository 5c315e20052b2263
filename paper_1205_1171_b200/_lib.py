"""ctypes binding of ``lib/libhull3d_b200.so`` (declared in include/hull3d_b200.h).

There is no CPU fallback: if the library is missing or a CUDA device is not
available, the product path raises.  ``load()`` builds the library in-tree
when its sources are newer (nvcc cross-compiles without a GPU).
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import build as _build

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None

i64 = ctypes.c_int64
vp = ctypes.c_void_p
dbl = ctypes.c_double
sz = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/hull3d_b200.h
SIGNATURES: dict[str, tuple] = {
    "h3d_impl": (ctypes.c_char_p, []),
    "h3d_last_error": (ctypes.c_char_p, []),
    "h3d_launch_count": (i64, []),
    "h3d_sync_count": (i64, []),
    "h3d_profile_enable": (None, [ctypes.c_int32]),
    "h3d_profile_collect": (i64, [vp, vp, vp, i64]),
    "h3d_profile_stamps": (None, [vp]),
    "h3d_profile_routes": (i64, [vp, i64]),
    "h3d_fast_pass_workspace_bytes": (sz, [i64]),
    "h3d_fast_upper_workspace_bytes": (sz, [i64]),
    "h3d_fast_passes": (i64, [vp, i64, vp, vp, sz, vp, ctypes.c_int32, vp, vp]),
    "h3d_fast_passes_range": (i64, [vp, i64, i64, i64, ctypes.c_int32, ctypes.c_int32, vp, vp,
                                    sz, vp, ctypes.c_int32, vp]),
    "h3d_fast_layout": (i64, [i64, vp]),
    "h3d_tune": (i64, [ctypes.c_char_p, i64]),
    "h3d_fast_extract": (i64, [vp, vp, i64, i64, i64, vp, i64, vp, vp, vp]),
    "h3d_seam_act": (i64, [vp, i64, vp]),
    "h3d_seam_init_base_logs": (i64, [vp, vp, i64, vp]),
    "h3d_seam_find_initial_bridge": (i64, [vp, vp, i64, i64, i64, vp, vp]),
    "h3d_seam_merge_movies": (i64, [vp, vp, vp, vp, i64, i64, i64, vp]),
    "h3d_seam_merge_range": (i64, [vp, vp, vp, vp, vp, i64, i64, vp]),
    "h3d_seam_replay": (i64, [vp, vp, i64, i64, vp]),
    "h3d_seam_rewind_replay": (i64, [vp, vp, i64, i64, vp]),
    "h3d_seam_extract_faces": (i64, [vp, vp, i64, vp, i64, vp]),
    "h3d_seam_log_length": (i64, [vp, i64, i64, vp]),
    "h3d_seam_copy_log": (i64, [vp, vp, i64, i64, vp]),
    "h3d_seam_run_level": (i64, [vp, dbl, vp, vp, vp, i64, i64, vp]),
    "h3d_presort_workspace_bytes": (sz, [i64]),
    "h3d_presort": (i64, [vp, i64, vp, vp, vp, sz, vp, vp]),
    "h3d_orient_remap": (i64, [vp, i64, vp, vp, i64, vp, vp, vp, vp, sz, vp]),
    "h3d_orient_remap_ex": (i64, [vp, i64, vp, vp, i64, vp, vp, vp, vp, vp, sz, vp]),
    "h3d_presort_slab": (i64, [vp, i64, i64, i64, ctypes.c_int32, vp, vp, vp, sz, vp]),
    "h3d_presort_slab_workspace_bytes": (sz, [i64, i64]),
    "h3d_epilogue_workspace_bytes": (sz, [i64]),
    "h3d_hull": (i64, [vp, i64, vp, vp, vp, sz, vp, vp, sz, vp, i64, vp, vp, vp, vp, ctypes.c_int32,
                       vp, vp]),
    "h3d_prim_temp_bytes": (sz, [i64]),
    "h3d_radix_sort_pairs": (i64, [vp, vp, vp, vp, i64, ctypes.c_int32, ctypes.c_int32,
                                   ctypes.c_int32, ctypes.c_int32, vp, sz, vp]),
    "h3d_scan_i64": (i64, [vp, vp, i64, ctypes.c_int32, ctypes.c_int32, vp, sz, vp]),
    "h3d_select_flagged": (i64, [vp, i64, vp, vp, vp, sz, vp]),
}


def lib_path() -> str:
    return _build.LIB


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if _build.needs_build():
            _build.build()
        if not os.path.exists(_build.LIB):
            raise RuntimeError(f"B200 hull library missing: {_build.LIB}")
        L = ctypes.CDLL(_build.LIB)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


def last_error() -> str:
    return load().h3d_last_error().decode(errors="replace")
