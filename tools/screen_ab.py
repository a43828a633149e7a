"""cfg2 screening (10k ligands, pop 256 x 200) ligands/s through vd_dock_batch, env as set."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_12232_b200 import gridmaps, hostprep, synth
from paper_2509_12232_b200.backend import CudaBackend
from paper_2509_12232_b200.ga import GaConfig, _run

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 200
spec = synth.config_grid_spec(2)
gset = gridmaps.build_grid_maps(synth.config_protein(2), spec, synth.CONFIGS[2].probe_types)
b = CudaBackend("fast", 0)
grid = b._grid_for_set(gset)
batch = hostprep.TopologyBatch.synth(2, 0, n)
lset = hostprep.ligand_set(hostprep.prepare_batch(batch, list(gset.maps)))
gmax = 7 + int(batch.n_torsions.max())
ga = GaConfig(population_size=256, generations=gens, translation_bounds=(spec.origin, spec.upper))
_run(grid, lset, 0, n, GaConfig(population_size=256, generations=1, translation_bounds=(spec.origin, spec.upper)), 0, 0, b._mode(), gmax, trace=False)
torch.cuda.synchronize(); t0 = time.perf_counter()
r = _run(grid, lset, 0, n, ga, 0, 0, b._mode(), gmax, trace=False)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"{n} ligands: {dt*1e3:.0f} ms  {n/dt:.0f} ligands/s  {n*256*(gens+1)/dt/1e6:.0f} M evals/s  checksum {float(np.sum(r[0].astype(np.float64))):.4f}")
