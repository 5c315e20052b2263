"""The hand-written device-wide primitives (csrc/prims.cuh) against numpy,
through the C ABI: the stable radix sort of (key, value) pairs is
np.argsort(kind="stable") (the presort's sort, api.py:97, and the lexsort
passes, api.py:86-87), the scans are np.cumsum / np.maximum.accumulate (the
tie-run heads, api.py:97-105), the flagged select is np.flatnonzero (the
vertex compaction behind np.unique, api.py:266).  Sizes straddle the tile
boundaries (4096 keys per 32-bit tile, 2816 per 64-bit tile, 2048 per scan
tile) and the chunked aggregate scan (> 2048 tiles)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_1205_1171_b200 import _lib
from paper_1205_1171_b200.engine import stream_ptr

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")


def _tmp(n):
    L = _lib.load()
    return torch.empty(int(L.h3d_prim_temp_bytes(n)), dtype=torch.uint8, device=DEV)


def _sort(keys: np.ndarray, begin: int, end: int, iota: bool, vals=None):
    L = _lib.load()
    n = keys.shape[0]
    kb = 8 if keys.dtype == np.uint64 else 4
    tdt = torch.int64 if kb == 8 else torch.int32
    k0 = torch.from_numpy(keys.view(np.int64 if kb == 8 else np.int32).copy()).to(DEV)
    k1 = torch.empty_like(k0)
    v0 = (torch.from_numpy(vals).to(DEV) if vals is not None
          else torch.full((max(n, 1),), -7, dtype=torch.int32, device=DEV))
    v1 = torch.empty_like(v0)
    tmp = _tmp(n)
    r = L.h3d_radix_sort_pairs(k0.data_ptr(), k1.data_ptr(), v0.data_ptr(), v1.data_ptr(), n, kb,
                               begin, end, 1 if iota else 0, tmp.data_ptr(), tmp.numel(),
                               stream_ptr(DEV))
    assert r in (0, 1), r
    torch.cuda.synchronize()
    ko, vo = (k1, v1) if r == 1 else (k0, v0)
    assert ko.dtype == tdt
    return ko.cpu().numpy().view(keys.dtype)[:n], vo.cpu().numpy()[:n]


def _digits(keys, begin, end):
    return (keys >> np.array(begin, dtype=keys.dtype)) & np.array((1 << (end - begin)) - 1, dtype=keys.dtype)


@pytest.mark.parametrize("n", [1, 2, 31, 4095, 4096, 4097, 100_003, 1 << 20])
@pytest.mark.parametrize("dist", ["uniform", "few", "sorted", "reversed"])
def test_radix_u32_stable_argsort(n, dist):
    rng = np.random.default_rng(n)
    if dist == "uniform":
        keys = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    elif dist == "few":
        keys = rng.integers(0, 5, n).astype(np.uint32) * np.uint32(0x01010101)
    elif dist == "sorted":
        keys = np.sort(rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32))
    else:
        keys = np.sort(rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32))[::-1].copy()
    ks, vs = _sort(keys, 0, 32, iota=True)
    perm = np.argsort(keys, kind="stable")
    assert np.array_equal(vs, perm.astype(np.int32))
    assert np.array_equal(ks, keys[perm])


@pytest.mark.parametrize("begin,end", [(0, 64), (0, 13), (8, 40), (61, 64)])
@pytest.mark.parametrize("n", [2815, 2816, 2817, 300_001])
def test_radix_u64_bit_ranges(n, begin, end):
    rng = np.random.default_rng(n + begin)
    keys = rng.integers(0, 2**63, n, dtype=np.int64).astype(np.uint64) * np.uint64(2)
    keys[::7] = keys[3]  # plenty of equal keys: stability matters
    vals = rng.integers(-2**31, 2**31, n).astype(np.int32)
    ks, vs = _sort(keys, begin, end, iota=False, vals=vals)
    perm = np.argsort(_digits(keys, begin, end), kind="stable")
    assert np.array_equal(vs, vals[perm])
    assert np.array_equal(ks, keys[perm])


@pytest.mark.parametrize("n", [1, 2047, 2048, 2049, 5_000_001])
@pytest.mark.parametrize("op_max,exclusive", [(0, 0), (0, 1), (1, 0)])
def test_scan_i64(n, op_max, exclusive):
    L = _lib.load()
    rng = np.random.default_rng(n)
    x = rng.integers(-10**6, 10**6, n).astype(np.int64)
    a = torch.from_numpy(x).to(DEV)
    out = torch.empty_like(a)
    tmp = _tmp(n)
    assert L.h3d_scan_i64(a.data_ptr(), out.data_ptr(), n, op_max, exclusive, tmp.data_ptr(),
                          tmp.numel(), stream_ptr(DEV)) == 0
    got = out.cpu().numpy()
    if op_max:
        exp = np.maximum.accumulate(x)
    else:
        exp = np.cumsum(x)
        if exclusive:
            exp = np.concatenate([[0], exp[:-1]])
    assert np.array_equal(got, exp)
    # in place
    assert L.h3d_scan_i64(a.data_ptr(), a.data_ptr(), n, op_max, exclusive, tmp.data_ptr(),
                          tmp.numel(), stream_ptr(DEV)) == 0
    assert np.array_equal(a.cpu().numpy(), exp)


@pytest.mark.parametrize("n", [1, 2048, 2049, 1 << 22])
@pytest.mark.parametrize("density", [0.0, 0.001, 0.5, 1.0])
def test_select_flagged(n, density):
    L = _lib.load()
    rng = np.random.default_rng(n)
    f = (rng.random(n) < density).astype(np.int32)
    flags = torch.from_numpy(f).to(DEV)
    out = torch.full((n,), -1, dtype=torch.int64, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    tmp = _tmp(n)
    assert L.h3d_select_flagged(flags.data_ptr(), n, out.data_ptr(), cnt.data_ptr(), tmp.data_ptr(),
                                tmp.numel(), stream_ptr(DEV)) == 0
    exp = np.flatnonzero(f)
    c = int(cnt.item())
    assert c == exp.size
    assert np.array_equal(out[:c].cpu().numpy(), exp)
