import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_1205_1171_b200 as H
from paper_1205_1171_b200 import engine as E, fast
from paper_1205_1171_b200.generators import generate
n = int(sys.argv[1])
pts = torch.from_numpy(generate(n, "sphere", 3)).cuda()
prof = []
E.PROFILE = prof
try:
    H.convex_hull_3d(pts, return_device=True)
    torch.cuda.synchronize()
    print("ok")
except Exception as exc:
    print("ERR", exc)
E.PROFILE = None
for name, p, lv, t in prof:
    print(name, p, lv, round(t, 4))
