"""Time the hand-written device primitives (csrc/prims.cuh) at C4 size:
    python tools/prim_bench.py [n]"""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch  # noqa: E402

from paper_1205_1171_b200 import _lib  # noqa: E402
from paper_1205_1171_b200.engine import stream_ptr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
L = _lib.load()
dev = torch.device("cuda:0")
s = stream_ptr(dev)
tmp = torch.empty(int(L.h3d_prim_temp_bytes(n)), dtype=torch.uint8, device=dev)
for kb in (4, 8):
    keys = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32 if kb == 4 else torch.int64, device=dev)
    k0 = keys.clone(); k1 = torch.empty_like(keys)
    v0 = torch.empty(n, dtype=torch.int32, device=dev); v1 = torch.empty_like(v0)
    bits = 32 if kb == 4 else 64
    for _ in range(3):
        k0.copy_(keys)
        L.h3d_radix_sort_pairs(k0.data_ptr(), k1.data_ptr(), v0.data_ptr(), v1.data_ptr(), n, kb, 0, bits, 1,
                               tmp.data_ptr(), tmp.numel(), s)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        L.h3d_radix_sort_pairs(k0.data_ptr(), k1.data_ptr(), v0.data_ptr(), v1.data_ptr(), n, kb, 0, bits, 1,
                               tmp.data_ptr(), tmp.numel(), s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    byt = n * (kb + 4) * 2 * (bits // 8)
    print(f"radix u{8*kb} n={n}: {ms:.3f} ms  ({byt/ms/1e6:.0f} GB/s pass traffic)")
