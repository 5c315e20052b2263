import sys, os; sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch, paper_1205_1171_b200 as H
from paper_1205_1171_b200 import fast
from paper_1205_1171_b200.api import presort
from paper_1205_1171_b200.generators import generate
for dist in ["sphere","ball","cube"]:
  for n in [4096, 20000, 777]:
    sp,_,_ = presort(torch.from_numpy(generate(n, dist, n+1)).cuda())
    for route in [{}, {"mini":0}, {"big_kin":1<<40}, {"leaf_b":0}]:
      try:
        with fast.tuned(**route), fast.verifying():
          fast.run_both(sp)
        print(dist, n, route, "ok")
      except Exception as e:
        print(dist, n, route, e)
