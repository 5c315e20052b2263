import sys

import torch

sys.path.insert(0, ".")
from paper_1205_1171_b200.api import presort  # noqa: E402

n = 1 << 24
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
pts = torch.rand((n, 3), dtype=torch.float64, device=dev, generator=g) * 2 - 1
presort(pts)
torch.cuda.synchronize()
