import torch, time
n = 402653184 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunk = (n + k - 1) // k
    def go():
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i*chunk:(i+1)*chunk].copy_(h[i*chunk:(i+1)*chunk], non_blocking=True)
    for _ in range(3): go()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10): go()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 10
    print(k, "streams", round(dt * 1e3, 2), "ms", round(n * 8 / dt / 1e9, 1), "GB/s")
