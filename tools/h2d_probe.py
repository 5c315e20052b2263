import torch, time
for mb in (25, 100, 403):
    n = mb * (1 << 20) // 8
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 10
    t = time.perf_counter()
    for _ in range(10): x = h.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    dt2 = (time.perf_counter() - t) / 10
    print(mb, "MB copy_", round(dt * 1e3, 2), "ms", round(mb / 1024 / dt, 1), "GB/s; .to()", round(dt2 * 1e3, 2), "ms")
