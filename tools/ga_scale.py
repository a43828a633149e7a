"""GA steady-state throughput vs batch size (replicated cfg2 ligands; GPU box)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_12232_b200 import context, gridmaps, synth
from paper_2509_12232_b200.backend import CudaBackend
from paper_2509_12232_b200.ga import GaConfig, _run
from paper_2509_12232_b200.screening import _shared_device_set

spec = synth.config_grid_spec(2)
gset = gridmaps.build_grid_maps(synth.config_protein(2), spec, synth.CONFIGS[2].probe_types)
uniq = [context.prepare_context(synth.config_ligand(2, i), gset) for i in range(64)]
b = CudaBackend("fast", 0)
ga = GaConfig(population_size=256, generations=200, translation_bounds=(spec.origin, spec.upper))
for n in (512, 2048, 8192):
    ctxs = [uniq[i % 64] for i in range(n)]
    grid, lset = _shared_device_set(b, gset, ctxs)
    gmax = 7 + max(c.n_torsions for c in ctxs)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _run(grid, lset, 0, n, ga, 0, 0, b._mode(), gmax, trace=False)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(n, f"{dt*1e3:.1f} ms", f"{n/dt:.0f} ligands/s", f"{n*256*201/dt/1e6:.1f} M evals/s")
