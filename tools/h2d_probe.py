"""Dev: host->device bandwidth of a 512 MiB pinned copy, one stream vs split across streams."""
import torch, time
n = 512 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
def run(k):
    streams = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step = n // k
    for i, s in enumerate(streams):
        with torch.cuda.stream(s):
            d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
    torch.cuda.synchronize()
    return n / (time.perf_counter() - t0) / 1e9
for k in (1, 2, 4, 8, 1, 2, 4):
    print(k, "streams", round(run(k), 1), "GB/s", flush=True)
