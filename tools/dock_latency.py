"""cfg0 single dock: wall time vs generations (fixed overhead vs per-generation cost)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_12232_b200 import gridmaps, synth
from paper_2509_12232_b200.backend import CudaBackend
from paper_2509_12232_b200.context import prepare_context
from paper_2509_12232_b200.ga import GaConfig, dock

spec = synth.config_grid_spec(0)
gset = gridmaps.build_grid_maps(synth.config_protein(0), spec, synth.CONFIGS[0].probe_types)
topo = synth.config_ligand(0, 0)
b = CudaBackend(mode="fast", device=0)
ctx = prepare_context(topo, gset)
for gens in (0, 10, 50, 200):
    cfg = GaConfig(population_size=100, generations=gens, seed=0)
    dock(topo, gset, cfg, backend=b, context=ctx)
    ts = []
    for _ in range(10):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = dock(topo, gset, cfg, backend=b, context=ctx)
        ts.append(time.perf_counter() - t0)
    print(f"generations {gens:4d}: {1e3*np.mean(sorted(ts)[:7]):.3f} ms")
