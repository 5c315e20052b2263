"""Per-rank device time of the x-slab multi-GPU hull, emulated on ONE GPU
(NCCL needs one device per rank): for G = 2, 4, 8 time rank G-1's sharded
presort (h3d_presort_slab) plus its slab levels (h3d_fast_passes_range);
the cross levels (mini merges + point-to-point messages) come on top.
Usage: python tools/rank_time.py [C4|C2|C3]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1205_1171_b200 import _lib  # noqa: E402
from paper_1205_1171_b200.api import _Workspace, presort  # noqa: E402
from paper_1205_1171_b200.engine import stream_ptr  # noqa: E402
from paper_1205_1171_b200.fast import _WS  # noqa: E402
from paper_1205_1171_b200.generators import generate  # noqa: E402
from paper_1205_1171_b200.multigpu import SlabPlan  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
n, dist = {"C4": (1 << 24, "cube"), "C2": (1 << 20, "ball"), "C3": (1 << 20, "sphere"),
           "C5": (1 << 27, "mixed")}[cfg]
dev = torch.device("cuda", 0)
pts = torch.from_numpy(generate(n, dist, 0)).to(dev)
L = _lib.load()
s = stream_ptr(dev)
sp_full, _, _ = presort(pts)
wsb = int(L.h3d_fast_pass_workspace_bytes(n))
ws = [_WS.get(dev, 0, wsb), _WS.get(dev, 1, int(L.h3d_fast_upper_workspace_bytes(n)))]
err = torch.zeros(1, dtype=torch.int64, device=dev)
sp = torch.empty((n, 3), dtype=torch.float64, device=dev)
od = torch.empty(n, dtype=torch.int64, device=dev)
pws = _Workspace.get(dev, int(L.h3d_presort_workspace_bytes(n)))


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def full():
    L.h3d_fast_passes_range(sp_full.data_ptr(), n, 0, n, 1, (n - 1).bit_length(), ws[0].data_ptr(),
                            ws[1].data_ptr(), wsb, err.data_ptr(), 0, s)


print(f"{cfg}: 1 GPU presort {timed(lambda: presort(pts)):.3f} ms, all levels {timed(full):.3f} ms")
for G in (2, 4, 8):
    plan = SlabPlan(n, G)
    r = G - 1
    p0, p1 = plan.slab(r)
    sws = torch.empty(int(L.h3d_presort_slab_workspace_bytes(n, p1 - p0 + 1)), dtype=torch.uint8,
                      device=dev)

    def pre():
        L.h3d_presort_slab(pts.data_ptr(), n, p0 - 1, p1, 0, sp.data_ptr(), od.data_ptr(),
                           sws.data_ptr(), sws.numel(), s)

    n_r = p1 - p0
    wsb_r = int(L.h3d_fast_pass_workspace_bytes(n_r))
    ws_r = [torch.empty(wsb_r, dtype=torch.uint8, device=dev),
            torch.empty(int(L.h3d_fast_upper_workspace_bytes(n_r)), dtype=torch.uint8, device=dev)]
    rows_r = sp_full[p0:p1].contiguous()

    def slab():  # the slab as a problem of its own (multigpu.hull_distributed)
        L.h3d_fast_passes_range(rows_r.data_ptr(), n_r, 0, n_r, 1, plan.slab_level, ws_r[0].data_ptr(),
                                ws_r[1].data_ptr(), wsb_r, err.data_ptr(), 0, s)
    a, b = timed(pre), timed(slab)
    print(f"G={G} rank {r}: slab presort {a:.3f} ms + slab levels 1..{plan.slab_level} {b:.3f} ms"
          f" = {a + b:.3f} ms; err {int(err.item())}")
