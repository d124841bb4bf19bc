import time, torch
n = 1_024_000_000 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
def run(nstreams, direction):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    chunk = n // nstreams
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for r in range(3):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                if direction == "h2d": d[i*chunk:(i+1)*chunk].copy_(h[i*chunk:(i+1)*chunk], non_blocking=True)
                else: h[i*chunk:(i+1)*chunk].copy_(d[i*chunk:(i+1)*chunk], non_blocking=True)
    torch.cuda.synchronize(); t = (time.perf_counter() - t0) / 3
    return 8 * n / t / 1e9
for direction in ("h2d", "d2h"):
    for ns in (1, 2, 4):
        print(direction, ns, "streams:", round(run(ns, direction), 1), "GB/s")
# both directions at once
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.float64).pin_memory(); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); t = time.perf_counter() - t0
print("bidirectional: ", round(2 * 8 * n / t / 1e9, 1), "GB/s total")
