import ctypes, os, sys, json
sys.path.insert(0, '/root/repo')
import torch
import bench
import paper_1205_1171_b200 as H
from paper_1205_1171_b200 import _lib, fast
from paper_1205_1171_b200.generators import generate
L = _lib.load()
n, dist, seed, _ = bench.CONFIGS['C4']
pts = torch.from_numpy(generate(n, dist, seed)).cuda()
H.convex_hull_3d(pts, return_device=True)
torch.cuda.synchronize()
arr = (ctypes.c_longlong * 64)()
L.h3d_mini_dbg_read(arr)
v = list(arr)
print([v[i] - v[i-1] for i in range(1, 20) if v[i]])
