"""Score-kernel throughput for cfg2-distribution ligands of each GA size bucket (GPU box):
   1M random poses per ligand against the cfg2 64^3 grid."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_12232_b200 import _abi, gridmaps, hostprep, synth
from paper_2509_12232_b200.backend import CudaBackend

spec = synth.config_grid_spec(2)
gset = gridmaps.build_grid_maps(synth.config_protein(2), spec, synth.CONFIGS[2].probe_types)
b = CudaBackend("fast", 0)
grid = b._grid_for_set(gset)
full = hostprep.TopologyBatch.synth(2, 0, 2000)
P = 1 << 20
out = []
for lo, hi in ((0, 24), (25, 32), (33, 48), (49, 64)):
    cand = [l for l in range(len(full)) if lo <= full.n_atoms[l] <= hi]
    l = cand[len(cand) // 2]
    batch = hostprep.TopologyBatch.from_topologies([full.topology(l)])
    arr = hostprep.prepare_batch(batch, list(gset.maps))
    lset = hostprep.ligand_set(arr)
    genes = synth.random_genes(l, P, int(batch.n_torsions[0]), spec.origin, spec.upper)
    gd = torch.from_numpy(genes).cuda()
    od = tuple(torch.empty(P, dtype=t, device="cuda") for t in (torch.float64, torch.float64, torch.float32))
    _abi.score_genes(grid, lset, 0, gd, *od)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5): _abi.score_genes(grid, lset, 0, gd, *od)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
    out.append(f"[{lo}-{hi}] N={int(batch.n_atoms[0])} P={int(arr['pair_start'][-1])} {P/dt/1e6:.0f} M/s")
print(" | ".join(out))
