"""Fused fast pass engine (placeholder: delegates to the exact engine until
csrc/fast.cu lands)."""

from __future__ import annotations

from .engine import run_pass_exact


def run_pass(pts, zsign, level_times=None):
    return run_pass_exact(pts, zsign, level_times)
