"""H2D / D2H pinned bandwidth alone and concurrently (for the e2e floor)."""
import time, torch
n = 1 << 30
h = torch.empty(n // 8, dtype=torch.float64, pin_memory=True); h2 = torch.empty_like(h, pin_memory=True)
d = torch.empty(n // 8, dtype=torch.float64, device="cuda"); d2 = torch.empty_like(d)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h2.copy_(d2, non_blocking=True))]:
    fn(); torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(4): fn()
    torch.cuda.synchronize(); print(name, 4 * n / (time.perf_counter() - t) / 1e9, "GB/s")
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(4):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); print("both", 4 * n / (time.perf_counter() - t) / 1e9, "GB/s per direction")
