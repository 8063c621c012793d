import torch, time
n = 336226108
h = torch.empty(n, dtype=torch.float32, pin_memory=True); h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
def run(k):
    streams = [torch.cuda.Stream() for _ in range(k)]
    parts = [(i * n // k, (i + 1) * n // k) for i in range(k)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        for s, (a, b) in zip(streams, parts):
            with torch.cuda.stream(s):
                d[a:b].copy_(h[a:b], non_blocking=True)
        torch.cuda.synchronize()
    return (time.perf_counter() - t0) / 5 * 1e3
for k in (1, 2, 4, 8, 1, 2):
    ms = run(k); print(k, "streams", round(ms, 2), "ms", round(4 * n / ms / 1e6, 1), "GB/s")
