"""x-slab sharding plan and the group exchange protocol, on CPU: the plan
reproduces plan_level's merge tree exactly (pkg/src/hull3d/parallel.py:49-65),
and send_group / recv_group move compact groups intact between two gloo
ranks (world_size 2, 127.0.0.1)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1205_1171_b200.multigpu import GroupLayout, SlabPlan, recv_group, send_group


def plan_level(n, level):
    size = 1 << level
    half = size >> 1
    out = []
    for L in range(0, n, size):
        R = min(L + size, n)
        out.append((L, L + half, R) if R - L > half else ("carry", L))
    return out


@pytest.mark.parametrize("world", [1, 2, 4, 8, 3, 6])
@pytest.mark.parametrize("n", [4, 5, 16, 17, 100, 1000, 2**12, 2**12 + 3, 3 * 2**10])
def test_plan_reproduces_merge_tree(n, world):
    plan = SlabPlan(n, world)
    G = plan.G
    assert G >= 1 and G & (G - 1) == 0 and G <= world
    s = plan.slab_level
    assert s >= 1 or n < 2
    # slabs cover [0, n) disjointly and align with level-s groups
    covered = []
    for r in range(world):
        sl = plan.slab(r)
        if sl is not None:
            assert sl[0] % plan.S == 0
            covered.append(sl)
    covered.sort()
    assert covered[0][0] == 0 and covered[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))
    # local levels: every job of plan_level lies inside one slab
    for lv in range(1, s + 1):
        for job in plan_level(n, lv):
            L = job[1] if job[0] == "carry" else job[0]
            R = L + (1 << lv)
            owner = [sl for sl in covered if sl[0] <= L < sl[1]]
            assert len(owner) == 1 and min(R, n) <= owner[0][1]
    # cross levels: merges/carries happen exactly where plan_level puts them
    for lv in range(s + 1, plan.levels + 1):
        expect = plan_level(n, lv)
        got = []
        for r in range(world):
            role, peer = plan.role(lv, r)
            L = r * plan.S
            if role == "merge":
                got.append((L, L + (1 << (lv - 1)), min(n, L + (1 << lv))))
                assert plan.role(lv, peer) == ("send", r)
            elif role == "carry":
                got.append(("carry", L))
        assert sorted(got, key=str) == sorted(expect, key=str), (n, world, lv)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1205_1171_b200 import _lib

        wsb = int(_lib.load().h3d_fast_pass_workspace_bytes(n))
        ws = [torch.zeros(wsb, dtype=torch.uint8), torch.zeros(wsb, dtype=torch.uint8)]
        lays = [GroupLayout(ws[0], n), GroupLayout(ws[1], n)]
        level, g, buf = 5, 3, 1
        L = g << level
        sizes = [(20, 30), (17, 25)]
        if rank == 1:
            gen = torch.Generator().manual_seed(7)
            for p, lay in enumerate(lays):
                nS, k = sizes[p]
                lay.hdr_view(buf, g).copy_(torch.tensor([nS, k], dtype=torch.int32).view(torch.uint8))
                for v in (lay.lnk_view(buf, L, nS), lay.gid_view(buf, L, nS), lay.ev_view(buf, L, k)):
                    v.copy_(torch.randint(0, 256, (v.numel(),), generator=gen, dtype=torch.uint8))
            send_group(lays, buf, level, g, 0)
            q.put(("sent", [w.clone().numpy() for w in ws]))
        else:
            recv_group(lays, buf, level, g, 1)
            q.put(("recv", [w.clone().numpy() for w in ws]))
    finally:
        dist.destroy_process_group()


def test_group_exchange_gloo():
    n = 4096
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # everything the sender wrote arrived in the same slots; nothing else moved
    for a, b in zip(got["sent"], got["recv"]):
        assert np.array_equal(a, b)


def _rows_worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1205_1171_b200 import _lib
        from paper_1205_1171_b200.multigpu import gather_input

        # the sharded presort's exchange: a group's points travel with their
        # sorted rows and caller indices
        wsb = int(_lib.load().h3d_fast_pass_workspace_bytes(n))
        ws = [torch.zeros(wsb, dtype=torch.uint8), torch.zeros(wsb, dtype=torch.uint8)]
        lays = [GroupLayout(ws[0], n), GroupLayout(ws[1], n)]
        level, g, buf = 6, 1, 0
        L = g << level
        sizes = [(13, 21), (9, 14)]
        sp = torch.full((n, 3), float("nan"), dtype=torch.float64)
        od = torch.full((n,), -1, dtype=torch.int64)
        gen = torch.Generator().manual_seed(3)
        for p, lay in enumerate(lays):
            nS, k = sizes[p]
            lay.hdr_view(buf, g).copy_(torch.tensor([nS, k], dtype=torch.int32).view(torch.uint8))
            ids = (L + torch.randperm(1 << level, generator=gen)[:nS]).to(torch.int32)
            lay.gid_view(buf, L, nS).copy_(ids.view(torch.uint8))
        if rank == 1:
            sp.copy_(torch.randn((n, 3), generator=gen, dtype=torch.float64))
            od.copy_(torch.randperm(n, generator=gen))
            send_group(lays, buf, level, g, 0, (sp, od))
        else:
            recv_group(lays, buf, level, g, 1, (sp, od))
        # chunked input gather (uneven chunks for world 2 and n odd)
        pts = np.random.default_rng(9).uniform(-1, 1, (70001, 3))
        full = gather_input(pts, torch.device("cpu"), rank, world)
        q.put((rank, sp.numpy(), od.numpy(), bool(np.array_equal(full.numpy(), pts))))
    finally:
        dist.destroy_process_group()


def test_group_rows_and_input_gather_gloo():
    n = 4096
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, rest) for r, *rest in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sp1, od1, ok1 = got[1]
    sp0, od0, ok0 = got[0]
    assert ok0 and ok1
    moved = od0 >= 0
    assert 0 < moved.sum() <= 13 + 9
    assert np.array_equal(od0[moved], od1[moved])
    assert np.array_equal(sp0[moved], sp1[moved])
    assert np.isnan(sp0[~moved]).all()


def test_rank_memory_shrinks_with_world():
    """Per-rank device memory of the x-slab hull is O(n / G) apart from the
    replicated input and 32-bit presort keys (host arithmetic from the
    library's sizing functions; C5 = 2^27 points, its slab groups ~2^17)."""
    from paper_1205_1171_b200.multigpu import rank_memory_bytes

    one = rank_memory_bytes(2**27, 1, 2**20)
    eight = rank_memory_bytes(2**27, 8, 2**17)
    assert eight["total"] < one["total"] / 4
    assert eight["slab_passes"] <= one["slab_passes"] / 8 + 3 * 2**30  # + the fixed big-job scratch
    assert eight["total"] < 20 * 2**30
    # the O(n) parts are the input replica and the keys only
    assert eight["input_replica"] == 24 * 2**27
