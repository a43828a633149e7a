"""cfg4 stress (128 atoms, 32 torsions, 126^3 grid, pop 512 x 300): timing on the GPU box."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_12232_b200 import gridmaps, hostprep, synth
from paper_2509_12232_b200.backend import CudaBackend
from paper_2509_12232_b200.ga import GaConfig, _run

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 300
spec = synth.config_grid_spec(4)
t0 = time.perf_counter()
gset = gridmaps.build_grid_maps(synth.config_protein(4), spec, synth.CONFIGS[4].probe_types)
print("grid build 126^3 x 8000 atoms", round(time.perf_counter() - t0, 2), "s")
b = CudaBackend("fast", 0)
grid = b._grid_for_set(gset)
batch = hostprep.TopologyBatch.synth(4, 0, n)
arr = hostprep.prepare_batch(batch, list(gset.maps))
lset = hostprep.ligand_set(arr)
print("pairs/ligand", arr["pair_start"][-1] / n)
ga = GaConfig(population_size=512, generations=gens, translation_bounds=(spec.origin, spec.upper))
_run(grid, lset, 0, 4, GaConfig(population_size=512, generations=1, translation_bounds=(spec.origin, spec.upper)), 0, 0, b._mode(), 39, trace=False)
torch.cuda.synchronize(); t0 = time.perf_counter()
r = _run(grid, lset, 0, n, ga, 0, 0, b._mode(), 39, trace=False)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
ev = n * 512 * (gens + 1)
print(f"{n} ligands: {dt:.2f} s  {n/dt:.1f} ligands/s  {ev/dt/1e6:.1f} M evals/s  best {np.min(r[0]):.2f}")
# scoring kernel on a cfg4 ligand: 200k random poses
ctx_like = None
genes = synth.random_genes(0, 200_000, int(batch.n_torsions[0]), spec.origin, spec.upper)
from paper_2509_12232_b200 import _abi
P = len(genes)
out = (np.empty(P), np.empty(P), np.empty(P, np.float32))
gd = torch.from_numpy(genes).cuda(); od = tuple(torch.empty(P, dtype=t, device="cuda") for t in (torch.float64, torch.float64, torch.float32))
_abi.score_genes(grid, lset, 0, gd, *od)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5): _abi.score_genes(grid, lset, 0, gd, *od)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
print(f"cfg4 scoring: {P/dt/1e6:.1f} M poses/s ({dt*1e3:.2f} ms / 200k)")
