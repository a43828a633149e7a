"""Time the host-pointer (e2e) scoring path piece by piece on the GPU box."""
import sys, time, ctypes
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_12232_b200 import _abi, synth, context, gridmaps
from paper_2509_12232_b200.backend import CudaBackend

torch.cuda.set_device(0)
spec = synth.config_grid_spec(1)
gset = gridmaps.build_grid_maps(synth.config_protein(1), spec, synth.CONFIGS[1].probe_types)
ctx = context.prepare_context(synth.config_ligand(1, 0), gset)
b = CudaBackend("fast", 0)
N = 1_000_000
genes = synth.random_genes(0, N, ctx.n_torsions, spec.origin, spec.upper)
pin = torch.from_numpy(genes).pin_memory()
outs = tuple(torch.empty(N, dtype=d).pin_memory() for d in (torch.float64, torch.float64, torch.float32))
outs_np = tuple(o.numpy() for o in outs)
gd = pin.cuda(); od = tuple(o.cuda() for o in outs)
for name, g, o in (("dev", gd, od), ("pinned", pin.numpy(), outs_np), ("pageable", genes, None)):
    for k in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        b.score_population_arrays(g, ctx, out=o)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(name, k, f"{dt*1e3:.2f} ms  {N/dt/1e6:.1f} M poses/s")
t0 = time.perf_counter(); x = pin.cuda(non_blocking=False); torch.cuda.synchronize(); print("torch H2D 120MB", (time.perf_counter()-t0)*1e3, "ms")
# fixed overhead vs size: slope = per-pose cost, intercept = per-call overhead
for n in (1 << 14, 1 << 17, 1 << 18, 1 << 19, N):
    g, o = pin.numpy()[:n], tuple(x[:n] for x in outs_np)
    b.score_population_arrays(g, ctx, out=o)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(10): b.score_population_arrays(g, ctx, out=o)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 10
    print(f"P={n:8d} {dt*1e3:.3f} ms  H2D-bound {n*120/54e9*1e3:.3f} ms")
