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
# H2D with a concurrent D2H of 1/6 the bytes (the e2e pipeline's 120 B in / 20 B out per pose)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
m = n // 6
h2 = torch.empty(m, dtype=torch.uint8).pin_memory()
d2 = torch.empty(m, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D with concurrent D2H: {10*n/(time.perf_counter()-t)/1e9:.1f} GB/s (in-direction)")
