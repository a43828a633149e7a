import torch, time
N = 256 << 20
src = torch.empty(N, dtype=torch.uint8).pin_memory()
dst = torch.empty(N, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
for ns in (1, 2, 4):
    for chunk in (16 << 20, 64 << 20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for rep in range(5):
            off = 0; k = 0
            while off < N:
                n = min(chunk, N - off)
                with torch.cuda.stream(streams[k % ns]):
                    dst[off:off + n].copy_(src[off:off + n], non_blocking=True)
                off += n; k += 1
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"streams {ns} chunk {chunk>>20} MiB: {5*N/dt/1e9:.1f} GB/s")
