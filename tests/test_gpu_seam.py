"""The kernel-module seam on the B200 (csrc/seam.cu) against the reference's
own per-level buffers and links (tests/golden/levels.npz) and its
known-answer tests.  Mirrors pkg/tests/test_store.py / test_merge.py /
test_serial_parallel.py of the reference."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def cu(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


@pytest.fixture(scope="module")
def K():
    from paper_1205_1171_b200 import seam

    return seam


def test_seam_constants(K):
    assert K.IMPL == "b200" and K.NIL == -1
    assert (K.E_OVERFLOW, K.E_BRIDGE, K.E_CHAIN, K.E_COUNT, K.E_UNTERMINATED) == (-1, -2, -3, -4, -5)


def test_act_kats(K):
    links = cu(np.array([[-1, 1], [0, 2], [1, -1]], dtype=np.int32))
    assert K.act(links, 1) == 0
    h = links.cpu().numpy()
    assert h[0, 1] == 2 and h[2, 0] == 0 and h[1, 0] == 0 and h[1, 1] == 2
    assert K.act(links, 1) == 0
    h = links.cpu().numpy()
    assert h[0, 1] == 1 and h[2, 0] == 1
    assert K.act(links, 0) == K.E_CHAIN


def test_two_singletons_merge(K):
    # tests/test_merge.py:76-84
    pts = cu(np.array([[0.0, 1, 2], [1.0, -1, 0.5]]))
    links = torch.empty((2, 2), dtype=torch.int32, device="cuda")
    A = torch.full((4,), -1, dtype=torch.int32, device="cuda")
    B = torch.full((4,), -1, dtype=torch.int32, device="cuda")
    assert K.init_base_logs(links, A, 2) == 0
    assert K.merge_movies(pts, links, A, B, 0, 1, 2) == 0
    assert B[0].item() == -1
    assert links.cpu().numpy().tolist() == [[-1, 1], [0, -1]]


def test_bridge_hand_example(K):
    pts = cu(np.array([[0.0, 0, 0], [1, 0, -1], [2, 0, -1], [3, 0, 0]]))
    links = torch.empty((4, 2), dtype=torch.int32, device="cuda")
    A = torch.full((8,), -1, dtype=torch.int32, device="cuda")
    B = torch.full((8,), -1, dtype=torch.int32, device="cuda")
    K.init_base_logs(links, A, 4)
    assert K.merge_movies(pts, links, A, B, 0, 1, 2) == 0
    assert K.merge_movies(pts, links, A, B, 2, 3, 4) == 0
    assert K.find_initial_bridge(pts, links, 1, 2, 4) == (1, 2)


def test_run_level_matches_reference_buffers_and_links(K, levels_npz):
    """Every level's whole output buffer (stale slots included) and the whole
    link array equal the reference's, both passes (zsign on device)."""
    names = [str(s) for s in levels_npz["__names__"]]
    for name in names:
        P = levels_npz[f"{name}__pts"]
        n = len(P)
        upper = name.endswith("upper")
        base = P * np.array([1.0, 1.0, -1.0]) if upper else P  # un-negate: device negates
        pts = cu(base)
        links = torch.empty((n, 2), dtype=torch.int32, device="cuda")
        src = torch.full((2 * n,), -1, dtype=torch.int32, device="cuda")
        dst = torch.full((2 * n,), -1, dtype=torch.int32, device="cuda")
        K.init_base_logs(links, src, n)
        lv = 1
        while f"{name}__slots{lv}" in levels_npz:
            assert K.run_level(pts, links, src, dst, n, lv, -1.0 if upper else 1.0) == 0
            assert np.array_equal(dst.cpu().numpy(), levels_npz[f"{name}__slots{lv}"]), (name, lv)
            assert np.array_equal(links.cpu().numpy(), levels_npz[f"{name}__links{lv}"]), (name, lv)
            src, dst = dst, src
            lv += 1


def test_merge_range_and_extract_vs_oracle(K, oracle_mod):
    from paper_1205_1171_b200.generators import generate

    for n, dist in ((64, "ball"), (300, "gauss"), (1000, "sphere")):
        P = generate(n, dist, 5)
        P = P[np.lexsort((P[:, 2], P[:, 1], P[:, 0]))]
        pts = cu(P)
        links = torch.empty((n, 2), dtype=torch.int32, device="cuda")
        A = torch.full((2 * n,), -1, dtype=torch.int32, device="cuda")
        B = torch.full((2 * n,), -1, dtype=torch.int32, device="cuda")
        K.init_base_logs(links, A, n)
        src, dst = A, B
        lv = 1
        while (1 << lv) < 2 * n:
            size = 1 << lv
            half = size >> 1
            starts = np.arange(0, n, size)
            ends = np.minimum(starts + size, n)
            m = ends - starts > half
            jobs = np.column_stack((starts[m], starts[m] + half, ends[m])).astype(np.int64)
            assert K.merge_range(pts, links, src, dst, cu(jobs), 0, len(jobs)) == 0
            for c in starts[~m]:
                assert K.copy_log(src, dst, 2 * int(c), 2 * n - 2 * int(c)) >= 0
            src, dst = dst, src
            lv += 1
        k = K.log_length(src, 0, 2 * n)
        faces = torch.empty((2 * n, 3), dtype=torch.int32, device="cuda")
        before = links.clone()
        assert K.replay(links, src, 0, k) == 0
        assert K.rewind_replay(links, src, 0, k) == 0
        assert torch.equal(before, links)
        assert K.replay(links, src, 0, k + 1) == K.E_COUNT
        K.rewind_replay(links, src, 0, k)
        m = K.extract_faces(links, src, 0, faces)
        assert m == k
        expect = oracle_mod.hull_pass(P)
        assert np.array_equal(faces[:m].cpu().numpy(), expect)
