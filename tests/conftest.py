"""Shared test setup.

Markers: ``gpu`` tests need a B200 (run on the GPU box with ``-m gpu``);
everything else runs on CPU.  The oracle (oracle/) is used here only as the
checker; golden fixtures come from the unmodified reference
(tests/golden/make_golden.py).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


class Small:
    """Accessor over tests/golden/small.npz."""

    def __init__(self):
        self.z = np.load(os.path.join(GOLDEN, "small.npz"))
        self.names = [str(s) for s in self.z["__names__"]]

    def case(self, name):
        z = self.z
        meta = z[f"{name}__meta"]
        return {
            "pts": z[f"{name}__pts"], "faces": z[f"{name}__faces"],
            "vertices": z[f"{name}__vertices"], "lower": int(meta[0]), "upper": int(meta[1]),
            "perturbed": bool(meta[2]), "general": bool(meta[3]),
        }


@pytest.fixture(scope="session")
def small():
    return Small()


@pytest.fixture(scope="session")
def levels_npz():
    return np.load(os.path.join(GOLDEN, "levels.npz"))


@pytest.fixture(scope="session")
def large_json():
    p = os.path.join(GOLDEN, "large.json")
    return json.load(open(p)) if os.path.exists(p) else {}


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as O

    O.lib()
    return O
