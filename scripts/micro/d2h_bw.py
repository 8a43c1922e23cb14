"""Device-to-host copy rates on this box: pinned vs pageable destination (torch, 256 MB)."""
import time, torch
n = 256 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, h in (("pinned", torch.empty(n, dtype=torch.uint8, pin_memory=True)), ("pageable", torch.empty(n, dtype=torch.uint8))):
    h.fill_(1)
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        h.copy_(d, non_blocking=False); torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"D2H {name}: {n / dt / 1e9:.1f} GB/s")
a = torch.empty(n, dtype=torch.uint8); b = torch.empty(n, dtype=torch.uint8); b.fill_(2)
for rep in range(3):
    t = time.perf_counter(); a.copy_(b); dt = time.perf_counter() - t
print(f"host memcpy (torch, its own threads): {n / dt / 1e9:.1f} GB/s")
