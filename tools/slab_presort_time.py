"""Time h3d_presort (replicated) vs h3d_presort_slab (one rank's window of
n/G rows) on one GPU at C4's size."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1205_1171_b200 import _lib  # noqa: E402
from paper_1205_1171_b200.api import _Workspace, presort  # noqa: E402
from paper_1205_1171_b200.engine import stream_ptr  # noqa: E402

n = 1 << 24
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
pts = torch.rand((n, 3), dtype=torch.float64, device=dev, generator=g) * 2 - 1
L = _lib.load()
sp = torch.empty((n, 3), dtype=torch.float64, device=dev)
od = torch.empty(n, dtype=torch.int64, device=dev)
ws = _Workspace.get(dev, int(L.h3d_presort_workspace_bytes(n)))


def t(fn, reps=20):
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


print("replicated presort ms", round(t(lambda: presort(pts)), 3))
for G in (2, 4, 8):
    S = n // G
    for r in (0, G - 1):
        q0, p1 = max(0, r * S - 1), (r + 1) * S
        code = [0]

        def f():
            code[0] = L.h3d_presort_slab(pts.data_ptr(), n, q0, p1, 1 if r == 0 else 0,
                                         sp.data_ptr(), od.data_ptr(), ws.data_ptr(), ws.numel(),
                                         stream_ptr(dev))
        ms = t(f)
        print(f"G={G} rank={r} slab presort ms {ms:.3f} code {code[0]}")
