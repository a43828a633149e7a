"""GA throughput per atom-count bucket (cfg2 distribution, pop 256 x G generations; GPU box).
   python tools/ga_bucket.py [generations]   (VD_LIB selects a variant library)"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_12232_b200 import gridmaps, hostprep, synth
from paper_2509_12232_b200.backend import CudaBackend
from paper_2509_12232_b200.ga import GaConfig, _run

gens = int(sys.argv[1]) if len(sys.argv) > 1 else 200
spec = synth.config_grid_spec(2)
gset = gridmaps.build_grid_maps(synth.config_protein(2), spec, synth.CONFIGS[2].probe_types)
b = CudaBackend("fast", 0)
grid = b._grid_for_set(gset)
full = hostprep.TopologyBatch.synth(2, 0, 10000)
ga = GaConfig(population_size=256, generations=gens, translation_bounds=(spec.origin, spec.upper))
out = []
for lo, hi in ((0, 24), (25, 32), (33, 48), (49, 64)):
    keep = [l for l in range(len(full)) if lo <= full.n_atoms[l] <= hi]
    batch = hostprep.TopologyBatch.from_topologies([full.topology(l) for l in keep])
    lset = hostprep.ligand_set(hostprep.prepare_batch(batch, list(gset.maps)))
    gmax = 7 + int(batch.n_torsions.max())
    _run(grid, lset, 0, min(64, len(keep)), GaConfig(population_size=256, generations=2,
         translation_bounds=(spec.origin, spec.upper)), 0, 0, b._mode(), gmax, trace=False)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _run(grid, lset, 0, len(keep), ga, 0, 0, b._mode(), gmax, trace=False)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    out.append(f"[{lo}-{hi}] n={len(keep)} {dt*1e3:.0f} ms {len(keep)/dt:.0f} lig/s")
print(" | ".join(out))
