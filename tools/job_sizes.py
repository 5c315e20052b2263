"""Largest job per level (points nS, merged child log kin) of the fast path:
python tools/job_sizes.py [n] [dist]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1205_1171_b200 import _lib  # noqa: E402
from paper_1205_1171_b200.api import presort  # noqa: E402
from paper_1205_1171_b200.engine import stream_ptr  # noqa: E402
from paper_1205_1171_b200.generators import generate  # noqa: E402
from paper_1205_1171_b200.multigpu import GroupLayout  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
dist = sys.argv[2] if len(sys.argv) > 2 else "cube"
dev = torch.device("cuda", 0)
sp, _, _ = presort(torch.from_numpy(generate(n, dist, 0)).to(dev))
L = _lib.load()
wsb = int(L.h3d_fast_pass_workspace_bytes(n))
ws = [torch.zeros(wsb, dtype=torch.uint8, device=dev) for _ in range(2)]
lay = GroupLayout(ws[0], n)
err = torch.zeros(1, dtype=torch.int64, device=dev)
levels = (n - 1).bit_length()
L.h3d_fast_passes_range(sp.data_ptr(), n, 0, n, 1, 8, ws[0].data_ptr(), ws[1].data_ptr(), wsb,
                        err.data_ptr(), 0, stream_ptr(dev))
for lv in range(9, levels + 1):
    b = (lv - 1) & 1
    g = (n + (1 << (lv - 1)) - 1) >> (lv - 1)
    o = lay.off[4 * b]
    hdr = lay.ws[o:o + 8 * g].view(torch.int32).view(g, 2).cpu().numpy().astype(np.int64)
    m = g // 2 * 2
    nS = hdr[:m:2, 0] + hdr[1:m:2, 0]
    kin = hdr[:m:2, 1] + hdr[1:m:2, 1]
    print(f"level {lv}: jobs {m // 2} max nS {nS.max()} p99 nS {int(np.percentile(nS, 99))} "
          f"max kin {kin.max()} p99 kin {int(np.percentile(kin, 99))}")
    L.h3d_fast_passes_range(sp.data_ptr(), n, 0, n, lv, lv, ws[0].data_ptr(), ws[1].data_ptr(),
                            wsb, err.data_ptr(), 0, stream_ptr(dev))
