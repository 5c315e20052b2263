"""Lane-kernel SIMT efficiency estimate per level: mean merged child log
length / mean over 32-job warps of the longest (steps ~ log length).
python tools/simt_eff.py CONFIG [max_level]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1205_1171_b200 import _lib  # noqa: E402
from paper_1205_1171_b200.api import presort  # noqa: E402
from paper_1205_1171_b200.engine import stream_ptr  # noqa: E402
from paper_1205_1171_b200.generators import generate  # noqa: E402
from paper_1205_1171_b200.multigpu import GroupLayout  # noqa: E402

cfg = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
n, dist, seed, _ = bench.CONFIGS[cfg]
dev = torch.device("cuda", 0)
sp, _, _ = presort(torch.from_numpy(generate(n, dist, seed)).to(dev))
L = _lib.load()
wsb = int(L.h3d_fast_pass_workspace_bytes(n))
ws = [torch.empty(wsb, dtype=torch.uint8, device=dev) for _ in range(2)]
lay = GroupLayout(ws[0], n)
err = torch.zeros(1, dtype=torch.int64, device=dev)
L.h3d_fast_passes_range(sp.data_ptr(), n, 0, n, 1, 3, ws[0].data_ptr(), ws[1].data_ptr(), wsb,
                        err.data_ptr(), 0, stream_ptr(dev))
for lv in range(4, top + 1):
    b = (lv - 1) & 1
    g = (n + (1 << (lv - 1)) - 1) >> (lv - 1)
    o = lay.off[4 * b]
    hdr = lay.ws[o:o + 8 * g].view(torch.int32).view(g, 2).cpu().numpy().astype(np.int64)
    m = g // 2 * 2
    kin = hdr[:m:2, 1] + hdr[1:m:2, 1]
    w = kin[: len(kin) // 32 * 32].reshape(-1, 32)
    ws_max = w.max(axis=1)
    srt = np.sort(kin)[::-1][: len(kin) // 32 * 32].reshape(-1, 32).max(axis=1)
    print(f"level {lv}: jobs {len(kin)} mean kin {kin.mean():.1f} max {kin.max()} "
          f"eff {kin.mean() / ws_max.mean():.2f} (sorted {w.mean() / srt.mean():.2f})", flush=True)
    L.h3d_fast_passes_range(sp.data_ptr(), n, 0, n, lv, lv, ws[0].data_ptr(), ws[1].data_ptr(),
                            wsb, err.data_ptr(), 0, stream_ptr(dev))
