"""PCIe probe: pinned H2D, D2H and concurrent H2D+D2H bandwidth (GB/s)."""
import time
import torch

n = 1 << 30
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name in ("h2d", "d2h", "both"):
    for it in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        if name in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d1.copy_(h1, non_blocking=True)
        if name in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    nb = n * (2 if name == "both" else 1)
    print(f"{name}: {nb / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms)")
