"""Raw pinned H2D / D2H bandwidth on the box (context for the e2e number)."""
import torch, time
n = 120_000_000
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D {10*n/(time.perf_counter()-t)/1e9:.1f} GB/s", end="  ")
t = time.perf_counter()
for _ in range(10): h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"D2H {10*n/(time.perf_counter()-t)/1e9:.1f} GB/s")
