import sys

import torch

sys.path.insert(0, ".")
from paper_1205_1171_b200 import _lib  # noqa: E402
from paper_1205_1171_b200.api import _Workspace  # noqa: E402
from paper_1205_1171_b200.engine import stream_ptr  # noqa: E402

n = 1 << 24
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
pts = torch.rand((n, 3), dtype=torch.float64, device=dev, generator=g) * 2 - 1
L = _lib.load()
sp = torch.empty((n, 3), dtype=torch.float64, device=dev)
od = torch.empty(n, dtype=torch.int64, device=dev)
ws = _Workspace.get(dev, int(L.h3d_presort_workspace_bytes(n)))
S = n // 8
print(L.h3d_presort_slab(pts.data_ptr(), n, 7 * S - 1, n, 0, sp.data_ptr(), od.data_ptr(),
                         ws.data_ptr(), ws.numel(), stream_ptr(dev)))
