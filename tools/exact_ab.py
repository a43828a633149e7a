"""Exact-mode GA throughput on cfg2 ligands (pop 256 x G generations): ligands/s."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_12232_b200 import gridmaps, hostprep, synth, _abi
from paper_2509_12232_b200.backend import CudaBackend
from paper_2509_12232_b200.ga import GaConfig, _run

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 200
spec = synth.config_grid_spec(2)
gset = gridmaps.build_grid_maps(synth.config_protein(2), spec, synth.CONFIGS[2].probe_types)
b = CudaBackend("exact", 0)
grid = b._grid_for_set(gset)
batch = hostprep.TopologyBatch.synth(2, 0, n)
lset = hostprep.ligand_set(hostprep.prepare_batch(batch, grid.labels))
ga = GaConfig(population_size=256, generations=gens, translation_bounds=(spec.origin, spec.upper))
gmax = 7 + int(batch.n_torsions.max())
_run(grid, lset, 0, 16, GaConfig(population_size=256, generations=1, translation_bounds=(spec.origin, spec.upper)), 0, 0, _abi.MODE_EXACT, gmax, trace=False)
torch.cuda.synchronize(); t0 = time.perf_counter()
r = _run(grid, lset, 0, n, ga, 0, 0, _abi.MODE_EXACT, gmax, trace=False)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"exact GA {n} ligands x pop 256 x {gens}: {dt:.2f} s  {n/dt:.1f} ligands/s  best-sum {float(np.sum(r[0].astype(np.float64))):.6f}")
