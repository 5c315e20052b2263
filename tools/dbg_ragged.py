import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1205_1171_b200 as H
from paper_1205_1171_b200.generators import generate
for n in [int(a) for a in sys.argv[1:]]:
    pts = generate(n, "sphere", 3)
    b = H.convex_hull_3d(pts)
    print(n, len(b.faces), flush=True)
