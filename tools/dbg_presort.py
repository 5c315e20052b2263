"""Debug: device presort order vs numpy stable argsort on a clustered cloud."""
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1205_1171_b200 as H  # noqa: E402
from paper_1205_1171_b200 import fast  # noqa: E402
from paper_1205_1171_b200.api import presort  # noqa: E402
from oracle import oracle as O  # noqa: E402

rng = np.random.default_rng(11)
pts = rng.uniform(-1.0, 1.0, (20000, 3))
pts[:19990, 0] = rng.uniform(0.0, 1e-12, 19990)
sp, order, pert = presort(torch.from_numpy(pts).cuda())
exp_order = np.argsort(pts[:, 0], kind="stable")
print("perturbed", pert, "order equal:", np.array_equal(order.cpu().numpy(), exp_order))
exp = O.convex_hull_3d(pts)
f0 = fast.FALLBACKS[0]
r = H.convex_hull_3d(pts)
print("fast fallbacks", fast.FALLBACKS[0] - f0, "err", fast.LAST_ERROR[0])
print("faces equal", np.array_equal(r.faces, exp.faces), len(r.faces), len(exp.faces))
a = H.convex_hull_3d(pts, H.CudaBackend(0, engine="exact"))
print("exact engine equal", np.array_equal(a.faces, exp.faces), len(a.faces))
ref = O.reference()
if ref is not None:
    rr = ref.convex_hull_3d(pts)
    print("reference equal oracle", np.array_equal(rr.faces, exp.faces), len(rr.faces))
