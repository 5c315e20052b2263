"""Debug: first level/group where the fast engine's log differs from the
oracle's (lower pass), for a given route."""
import ctypes
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1205_1171_b200 import _lib, fast  # noqa: E402
from paper_1205_1171_b200.api import presort  # noqa: E402
from paper_1205_1171_b200.engine import stream_ptr  # noqa: E402
from paper_1205_1171_b200.multigpu import GroupLayout  # noqa: E402
from oracle import oracle as O  # noqa: E402

route = dict(kv.split("=") for kv in sys.argv[1:])
rng = np.random.default_rng(11)
pts = rng.uniform(-1.0, 1.0, (20000, 3))
pts[:19990, 0] = rng.uniform(0.0, 1e-12, 19990)
sp, order, _ = presort(torch.from_numpy(pts).cuda())
spn = sp.cpu().numpy()
n = len(pts)
L = _lib.load()
wsb = int(L.h3d_fast_pass_workspace_bytes(n))
ws = [torch.zeros(wsb, dtype=torch.uint8, device="cuda") for _ in range(2)]
lay = GroupLayout(ws[0], n)
err = torch.zeros(1, dtype=torch.int64, device="cuda")
with fast.tuned(**{k: int(v) for k, v in route.items()}):
    for lv, kout, buf, links in O.level_logs(spn):
        err.zero_()
        r = L.h3d_fast_passes_range(sp.data_ptr(), n, 0, n, 1, lv, ws[0].data_ptr(), ws[1].data_ptr(),
                                    wsb, err.data_ptr(), 0, stream_ptr(sp.device))
        torch.cuda.synchronize()
        b = lv & 1
        bad = 0
        for g in range((n + (1 << lv) - 1) >> lv):
            Lg = g << lv
            hdr = lay.hdr_view(b, g).view(torch.int32).cpu().numpy()
            nS, k = int(hdr[0]), int(hdr[1])
            gid = lay.gid_view(b, Lg, nS).view(torch.int32).cpu().numpy()
            ev = lay.ev_view(b, Lg, k).cpu().numpy().view(np.int32).reshape(-1, 6)
            fb = gid[ev[:, 3]] if k else np.zeros(0, dtype=np.int32)
            exp = O.group_log(buf, Lg)
            if len(exp) != k or not np.array_equal(fb, exp):
                bad += 1
                if bad <= 2:
                    print(f"level {lv} group {g} L={Lg}: fast k={k} oracle k={len(exp)}")
                    print("  fast b  ", fb[:40].tolist())
                    print("  oracle b", exp[:40].tolist())
                    fa = gid[ev[:, 2]] if k else []
                    fc = gid[ev[:, 4]] if k else []
                    print("  fast a  ", list(fa[:40]))
                    print("  fast c  ", list(fc[:40]))
        print(f"level {lv}: err={int(err.item())} groups differing={bad}", flush=True)
        if bad:
            break
