import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2509_12232_b200 import gridmaps, hostprep, synth, _abi
from paper_2509_12232_b200.backend import CudaBackend
from paper_2509_12232_b200.ga import GaConfig, _run
spec = synth.config_grid_spec(2)
gset = gridmaps.build_grid_maps(synth.config_protein(2), spec, synth.CONFIGS[2].probe_types)
b = CudaBackend("fast", 0)
grid = b._grid_for_set(gset)
batch = hostprep.TopologyBatch.synth(2, 0, 2000)
lset = hostprep.ligand_set(hostprep.prepare_batch(batch, list(gset.maps)))
gmax = 7 + int(batch.n_torsions.max())
ga = GaConfig(population_size=256, generations=5, translation_bounds=(spec.origin, spec.upper))
free0 = None
for it in range(30):
    _run(grid, lset, 0, 2000, ga, 0, 0, _abi.MODE_FAST, gmax, trace=False)
    torch.cuda.synchronize()
    free, tot = torch.cuda.mem_get_info()
    if it == 2: free0 = free
    if it in (2, 10, 29): print(it, "free MB", free // 2**20)
print("delta MB since iteration 2:", (free0 - free) // 2**20)
