"""Host <-> device copy rates on this box: H2D, D2H alone and concurrently (pinned, 2.75 GB)."""
import time
import torch

n = 344064000
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
gb = n * 8 / 1e9
for name, fn in (("H2D", lambda: d1.copy_(h1, non_blocking=True)), ("D2H", lambda: h2.copy_(d2, non_blocking=True))):
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"{name}: {gb / dt:.1f} GB/s", flush=True)
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"concurrent H2D + D2H: {2 * gb / dt:.1f} GB/s total ({dt * 1e3:.1f} ms for 2 x {gb:.2f} GB)", flush=True)
