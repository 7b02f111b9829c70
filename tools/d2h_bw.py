import torch, time
n = 4 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    print("D2H GB/s", n / (time.perf_counter() - t0) / 1e9)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): h[: n // 2].copy_(d[: n // 2], non_blocking=True)
with torch.cuda.stream(s2): h[n // 2:].copy_(d[n // 2:], non_blocking=True)
torch.cuda.synchronize(); print("2 streams GB/s", n / (time.perf_counter() - t0) / 1e9)
