"""cfg4 (128 atoms, 32 torsions, 126^3 grid, pop 512 x G) ligands/s for a batch of N ligands
(250 = one GPU's share of BASELINE cfg4 at 8 GPUs) with VD_GA_TEAM as set in the env."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_12232_b200 import gridmaps, hostprep, synth, _abi
from paper_2509_12232_b200.backend import CudaBackend
from paper_2509_12232_b200.ga import GaConfig, _run

n = int(sys.argv[1]) if len(sys.argv) > 1 else 250
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 300
spec = synth.config_grid_spec(4)
gset = gridmaps.build_grid_maps(synth.config_protein(4), spec, synth.CONFIGS[4].probe_types)
b = CudaBackend("fast", 0)
grid = b._grid_for_set(gset)
batch = hostprep.TopologyBatch.synth(4, 0, n)
lset = hostprep.ligand_set(hostprep.prepare_batch(batch, grid.labels))
ga = GaConfig(population_size=512, generations=gens, translation_bounds=(spec.origin, spec.upper))
gmax = 7 + int(batch.n_torsions.max())
_run(grid, lset, 0, 8, GaConfig(population_size=512, generations=1, translation_bounds=(spec.origin, spec.upper)), 0, 0, _abi.MODE_FAST, gmax, trace=False)
torch.cuda.synchronize(); t0 = time.perf_counter()
r = _run(grid, lset, 0, n, ga, 0, 0, _abi.MODE_FAST, gmax, trace=False)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"team={os.environ.get('VD_GA_TEAM', 'auto')} {n} ligands x pop 512 x {gens}: {dt:.3f} s  {n/dt:.1f} ligands/s  checksum {float(np.sum(r[0].astype(np.float64))):.4f}")
