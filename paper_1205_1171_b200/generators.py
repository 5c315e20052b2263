"""Seed-deterministic synthetic clouds (restates pkg/src/hull3d/generators.py:18-46).

Same PCG64 stream and the same numpy calls in the same order, so a given
(n, dist, seed) gives bit-identical coordinates to the reference generator;
tests/test_host.py pins this against the reference and the golden digests.
``mixed`` is the BASELINE.md C5 definition (not in the reference).
"""

from __future__ import annotations

import numpy as np

DISTRIBUTIONS = ("ball", "sphere", "cube", "gauss", "mixed")
_SPHERE_JITTER = 1e-6


def generate(n: int, dist: str, seed: int) -> np.ndarray:
    if n < 1:
        raise ValueError("n must be >= 1")
    if dist == "mixed":
        # C5: ball of n - n/128 points plus an outlier shell of
        # n/128 points on a radius-2 sphere (2^27 -> 2^27-2^20 + 2^20)
        shell = max(1, n >> 7)
        return np.concatenate([generate(n - shell, "ball", seed),
                               2.0 * generate(shell, "sphere", seed + 1)])
    rng = np.random.Generator(np.random.PCG64(seed))
    if dist == "ball":
        dirs = rng.standard_normal((n, 3))
        norms = np.maximum(np.linalg.norm(dirs, axis=1, keepdims=True), 1e-300)
        radii = rng.random(n) ** (1.0 / 3.0)
        return dirs / norms * radii[:, None]
    if dist == "sphere":
        dirs = rng.standard_normal((n, 3))
        norms = np.maximum(np.linalg.norm(dirs, axis=1, keepdims=True), 1e-300)
        jitter = 1.0 + rng.uniform(-1.0, 1.0, n) * _SPHERE_JITTER
        return dirs / norms * jitter[:, None]
    if dist == "cube":
        return rng.uniform(-1.0, 1.0, (n, 3))
    if dist == "gauss":
        return rng.standard_normal((n, 3))
    raise ValueError(f"unknown distribution {dist!r}; expected one of {DISTRIBUTIONS}")


def integer_cloud(n: int, seed: int, half_range: int = 2**30) -> np.ndarray:
    """Integer-coordinate cloud (BASELINE.md "Integer" config): always takes
    the tie-perturbation path; reference-correct when the range >~ 2n."""
    rng = np.random.default_rng(seed)
    return rng.integers(-half_range, half_range, (n, 3)).astype(np.float64)
