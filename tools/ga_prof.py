"""One representative GA launch for profiling: cfg2 ligands of one size bucket (33-48 atoms)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_12232_b200 import gridmaps, hostprep, synth
from paper_2509_12232_b200.backend import CudaBackend
from paper_2509_12232_b200.ga import GaConfig, _run

gens = int(sys.argv[1]) if len(sys.argv) > 1 else 20
mode = sys.argv[2] if len(sys.argv) > 2 else "fast"
spec = synth.config_grid_spec(2)
gset = gridmaps.build_grid_maps(synth.config_protein(2), spec, synth.CONFIGS[2].probe_types)
b = CudaBackend(mode, 0)
grid = b._grid_for_set(gset)
full = hostprep.TopologyBatch.synth(2, 0, 6000)
keep = [l for l in range(len(full)) if 33 <= full.n_atoms[l] <= 48][:2048 if mode == "fast" else 512]
topos = [full.topology(l) for l in keep]
batch = hostprep.TopologyBatch.from_topologies(topos)
lset = hostprep.ligand_set(hostprep.prepare_batch(batch, list(gset.maps)))
ga = GaConfig(population_size=256, generations=gens, translation_bounds=(spec.origin, spec.upper))
r = _run(grid, lset, 0, len(topos), ga, 0, 0, b._mode(), 19, trace=False)
torch.cuda.synchronize()
print("ok", len(topos), float(np.min(r[0])))
