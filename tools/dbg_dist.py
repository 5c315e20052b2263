"""Run the distributed hull on one GPU with gloo (debugging):
python tools/dbg_dist.py WORLD N:KIND:SEED ..."""
import os
import socket
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def make(n, kind, seed):
    sys.path.insert(0, ROOT)
    from paper_1205_1171_b200.generators import generate, integer_cloud
    rng = np.random.default_rng(seed)
    if kind == "clusters":
        c = rng.uniform(-1, 1, (12, 3))
        return c[rng.integers(0, 12, n)] + rng.normal(0, 1e-7, (n, 3))
    if kind == "near_plane":
        p = rng.uniform(-1, 1, (n, 3))
        p[:, 2] = 0.2 * p[:, 0] - 0.4 * p[:, 1] + rng.normal(0, 1e-10, n)
        p[:8, 2] += 1.0
        return p
    if kind == "paraboloid":
        p = rng.uniform(-1, 1, (n, 3))
        p[:, 2] = p[:, 0] ** 2 + p[:, 1] ** 2
        return p
    if kind == "int_wide":
        return integer_cloud(n, seed)
    if kind == "int":
        return integer_cloud(n, seed, half_range=2**12)
    if kind == "slab_x":
        rng = np.random.default_rng(seed)
        p = rng.uniform(-1.0, 1.0, (n, 3))
        p[: n - 64, 0] = rng.uniform(0.0, 1e-12, n - 64)
        return p
    return generate(n, kind, seed)


def worker(rank, world, port, cases):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1205_1171_b200.multigpu import convex_hull_3d_distributed
    for n, kind, seed in cases:
        try:
            pts = make(n, kind, seed)
            r = convex_hull_3d_distributed(pts)
            if rank == 0:
                import paper_1205_1171_b200 as H
                try:
                    ref = H.convex_hull_3d(pts)
                    same = np.array_equal(r.faces, ref.faces) and np.array_equal(r.vertices, ref.vertices)
                except Exception as exc:  # noqa: BLE001
                    same = f"single GPU raised {type(exc).__name__}"
                print("rank0", n, kind, seed, "faces", len(r.faces), "same as 1 GPU:", same, flush=True)
        except Exception as exc:
            import traceback
            traceback.print_exc()
            print(f"rank {rank} case {(n, kind, seed)}: {type(exc).__name__}: {exc}", flush=True)
            os._exit(1)
    dist.destroy_process_group()


if __name__ == "__main__":
    world = int(sys.argv[1])
    cases = [(int(a.split(":")[0]), a.split(":")[1], int(a.split(":")[2])) for a in sys.argv[2:]]
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(r, world, port, cases)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
    print("exit codes", [p.exitcode for p in ps])
