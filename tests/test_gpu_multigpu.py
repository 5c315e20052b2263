"""The x-slab multi-GPU hull end to end.  The GPU box exposes one device, so
2 and 4 ranks share cuda:0 over gloo (groups staged through host memory);
the merge tree, the level ranges and the group exchange are the ones the
NCCL run uses.  Rank 0's result must equal the single-GPU result bit for
bit (and the reference's golden digest for C2)."""

from __future__ import annotations

import hashlib
import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make(n, kind, seed):
    """Test clouds: the generators' distributions, plus inputs the sharded
    presort must decline on every rank -- x ties ("int": a small integer
    range) and one long run of equal sort keys ("slab_x")."""
    from paper_1205_1171_b200.generators import generate, integer_cloud

    if kind == "int":
        return integer_cloud(n, seed, half_range=2**12)
    if kind == "slab_x":
        rng = np.random.default_rng(seed)
        p = rng.uniform(-1.0, 1.0, (n, 3))
        p[: n - 64, 0] = rng.uniform(0.0, 1e-12, n - 64)
        return p
    return generate(n, kind, seed)


def _worker(rank, world, port, cases, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["H3D_DIST_POISON"] = "1"  # rows a rank did not sort are NaN
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1205_1171_b200.generators import generate
        from paper_1205_1171_b200 import multigpu
        from paper_1205_1171_b200.multigpu import convex_hull_3d_distributed

        out = {}
        for n, dist_name, seed in cases:
            r = convex_hull_3d_distributed(make(n, dist_name, seed))
            if rank == 0:
                out[(n, dist_name, seed)] = (r.faces, r.vertices)
        multigpu.PHASES = []  # one call with phase events (bench.py's rank0_phases_ms)
        convex_hull_3d_distributed(generate(2**18, "ball", 4))
        phases = multigpu.PHASES
        multigpu.PHASES = None
        if rank == 0:
            out["sharded"] = multigpu.SHARDED_RUNS[0]
            out["phases"] = phases
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_distributed_equals_single_gpu(world, large_json):
    import paper_1205_1171_b200 as H
    from paper_1205_1171_b200.generators import generate

    # the 2^18 sphere sends its cross-rank levels through the time-split
    # pipeline (large merged logs), the others through the mini/warp merges
    cases = [(1000, "ball", 1), (3 * 1024 + 7, "sphere", 2), (5000, "cube", 3), (2**20, "ball", 0),
             (2**18, "sphere", 5), (70000, "int", 6), (70000, "slab_x", 7)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the two general-position cases >= SHARD_PRESORT_MIN points sort only
    # their own slabs (+ the phase-timed call); "int" and "slab_x" decline
    assert got.pop("sharded") == 3
    (ph,) = got.pop("phases")
    assert set(ph) == {"presort", "slab_levels", "cross_levels"} and min(ph.values()) >= 0
    for key, (faces, verts) in got.items():
        ref = H.convex_hull_3d(make(*key))
        assert np.array_equal(faces, ref.faces), key
        assert np.array_equal(verts, ref.vertices), key
    f, _ = got[(2**20, "ball", 0)]
    assert hashlib.sha256(np.ascontiguousarray(f).tobytes()).hexdigest() == \
        large_json["C2_ball_2^20"]["faces_sha256"]
