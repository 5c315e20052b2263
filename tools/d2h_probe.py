"""D2H options for returning large int64 results as numpy arrays."""
import time

import numpy as np
import torch

F = 2_041_120
faces = torch.randint(0, 1 << 20, (F, 3), dtype=torch.int64, device="cuda")
torch.cuda.synchronize()


def bench(name, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    print(f"{name:40s} {(time.perf_counter() - t) / reps * 1e3:8.2f} ms", flush=True)
    return out


bench("tensor.cpu().numpy()", lambda: faces.cpu().numpy())


def pinned_new():
    h = torch.empty(faces.shape, dtype=faces.dtype, pin_memory=True)
    h.copy_(faces)
    return h.numpy()


bench("new pinned + copy_", pinned_new)


def np_into():
    a = np.empty((F, 3), dtype=np.int64)
    torch.from_numpy(a).copy_(faces)
    return a


bench("np.empty + from_numpy().copy_", np_into)


def np_into_touched():
    a = np.empty((F, 3), dtype=np.int64)
    a.reshape(-1)[::512] = 0  # touch every page first
    torch.from_numpy(a).copy_(faces)
    return a


bench("np.empty + touch + copy_", np_into_touched)

pool = torch.empty(faces.shape, dtype=faces.dtype, pin_memory=True)


def pinned_pool_then_copy():
    pool.copy_(faces)
    return pool.numpy().copy()


bench("pinned pool + numpy copy", pinned_pool_then_copy)
