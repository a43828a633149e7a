import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2509_12232_b200 import gridmaps, hostprep, synth, _abi
from paper_2509_12232_b200.backend import CudaBackend
spec = synth.config_grid_spec(4)
gset = gridmaps.build_grid_maps(synth.config_protein(4), spec, synth.CONFIGS[4].probe_types)
b = CudaBackend("fast", 0)
grid = b._grid_for_set(gset)
batch = hostprep.TopologyBatch.synth(4, 0, 4)
lset = hostprep.ligand_set(hostprep.prepare_batch(batch, list(gset.maps)))
genes = synth.random_genes(0, 200_000, int(batch.n_torsions[0]), spec.origin, spec.upper)
P = len(genes)
gd = torch.from_numpy(genes).cuda(); od = tuple(torch.empty(P, dtype=t, device="cuda") for t in (torch.float64, torch.float64, torch.float32))
_abi.score_genes(grid, lset, 0, gd, *od)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10): _abi.score_genes(grid, lset, 0, gd, *od)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 10
print(f"cfg4 scoring: {P/dt/1e6:.1f} M poses/s ({dt*1e3:.2f} ms / 200k) checksum {float(od[2].double().sum()):.6e}")
