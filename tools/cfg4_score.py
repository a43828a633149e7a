"""cfg4 scoring kernel only: 200k random poses of one 128-atom / 32-torsion ligand (GPU box)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_12232_b200 import _abi, gridmaps, hostprep, synth
from paper_2509_12232_b200.backend import CudaBackend

spec = synth.config_grid_spec(4)
gset = gridmaps.build_grid_maps(synth.config_protein(4), spec, synth.CONFIGS[4].probe_types)
b = CudaBackend("fast", 0)
grid = b._grid_for_set(gset)
batch = hostprep.TopologyBatch.synth(4, 0, 1)
arr = hostprep.prepare_batch(batch, list(gset.maps))
lset = hostprep.ligand_set(arr)
P = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
genes = synth.random_genes(0, P, int(batch.n_torsions[0]), spec.origin, spec.upper)
gd = torch.from_numpy(genes).cuda()
od = tuple(torch.empty(P, dtype=t, device="cuda") for t in (torch.float64, torch.float64, torch.float32))
_abi.score_genes(grid, lset, 0, gd, *od)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5): _abi.score_genes(grid, lset, 0, gd, *od)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
npairs = int(arr["pair_start"][-1]); na = int(batch.n_atoms[0])
fl = 32 * npairs + 107 * na
print(f"cfg4 scoring: N={na} P={npairs} {P/dt/1e6:.2f} M poses/s ({dt*1e3:.2f} ms / {P}); "
      f"{fl*P/dt/1e12:.2f} TFLOP/s model; MUFU ceiling {148*1.965e9*16/(4*npairs)/1e6:.0f} M poses/s")
