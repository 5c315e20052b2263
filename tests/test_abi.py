"""The C-ABI library loads and exports every symbol include/hull3d_b200.h
declares (no compute calls: this runs on the CPU box)."""

from __future__ import annotations

import ctypes
import os
import re

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "hull3d_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(h3d_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "h3d_seam_merge_range" in syms and "h3d_presort" in syms
    assert len(syms) >= 15


def test_library_exports_every_declared_symbol():
    from paper_1205_1171_b200 import _lib

    L = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_ctypes_signatures_cover_header():
    from paper_1205_1171_b200 import _lib

    assert set(declared_symbols()) <= set(_lib.SIGNATURES)


def test_library_identity_and_host_only_calls():
    from paper_1205_1171_b200 import _lib

    L = _lib.load()
    assert L.h3d_impl() == b"b200"
    assert isinstance(L.h3d_last_error(), bytes)
    small = L.h3d_presort_workspace_bytes(1000)
    big = L.h3d_presort_workspace_bytes(1 << 24)
    assert 0 < small < big


def test_library_is_sm100a_only():
    from paper_1205_1171_b200 import build

    assert "arch=compute_100a,code=sm_100a" in build.ARCH
    assert "-fmad=false" in build.FLAGS
    blob = open(build.LIB, "rb").read()
    assert b"sm_100a" in blob or b"sm_100" in blob
    ctypes.CDLL(build.LIB)


def test_tune_leaf_depth_normalised():
    """leaf_b accepts 3 or 4 fused levels; anything below 3 turns the leaf
    kernel off (h3d_tune is host-only: no GPU needed)."""
    from paper_1205_1171_b200 import fast

    old = fast.tune("leaf_b", 2)
    try:
        assert fast.tune("leaf_b") == 0
        fast.tune("leaf_b", 9)
        assert fast.tune("leaf_b") == 4
        fast.tune("leaf_b", 3)
        assert fast.tune("leaf_b") == 3
    finally:
        fast.tune("leaf_b", old)
