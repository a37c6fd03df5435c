"""Pinned host<->device copy bandwidth on this box (context for the e2e number)."""
import time, torch
n = 33_177_600
d = torch.empty(n, dtype=torch.uint8, device="cuda"); h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for name, f in (("d2h", lambda: h.copy_(d, non_blocking=True)), ("h2d", lambda: d.copy_(h, non_blocking=True))):
    for _ in range(3): f()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(50): f()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 50
    print(f"{name} {n/1e6:.1f} MB: {dt*1e3:.3f} ms = {n/dt/1e9:.1f} GB/s")
