"""Small invocations of every hot kernel shape for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck: one tool per gpurun call).  No torch: the library through ctypes.

  score_kernel  TPP 4 role split (cfg1 fixture, 40 atoms, resident pairs), TPP 8 with
                streamed pair tiles (128-atom fixture), TPP 1 exact; z-pair, brick and
                plain grid layouts; host-buffer pipeline path
  pose_kernel   TPP 1 / 4 / 8
  ga_kernel     fast packed (incl. the 3-CTA r3 variant), fast plain, exact
  grid_kernel   small device grid build
Usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

import fixtures as fx  # noqa: E402
from paper_2509_12232_b200 import _abi, gridmaps, hostprep, synth  # noqa: E402
from paper_2509_12232_b200.backend import CudaBackend  # noqa: E402
from paper_2509_12232_b200.context import prepare_context  # noqa: E402
from paper_2509_12232_b200.ga import GaConfig, dock, _run  # noqa: E402


def main():
    _abi.ensure_device(0)
    for layout, env in (("brick", {"VD_BRICK_BUDGET_MB": "100000"}),
                        ("zpair", {"VD_BRICK_BUDGET_MB": "0"}), ("plain", {"VD_NO_PACK": "1"})):
        os.environ.update(env)
        for name, n in (("cfg1", 130), ("big", 66)):
            c = fx.pop_case(name)
            g2 = gridmaps.GridMapSet(c["grid"].spec, dict(c["grid"].maps))  # fresh device grid
            ctx = prepare_context(c["topo"], g2, table=fx.TABLE)
            for mode in ("fast", "exact"):
                b = CudaBackend(mode=mode, device=0)
                b.score_population_arrays(c["genes"][:n], ctx)
            grid, ligs = CudaBackend(mode="fast", device=0).prepared(ctx)
            for tpp in (4, 8):
                _abi.debug_pose_genes(ligs, 0, c["genes"][:n], tpp)
            CudaBackend(mode="fast", device=0).pose_population(c["genes"][:n], ctx)
            for mode in ("fast", "exact"):
                dock(c["topo"], g2, GaConfig(population_size=40, generations=2, seed=1),
                     backend=CudaBackend(mode=mode, device=0), context=ctx)
        for k in env:
            del os.environ[k]
    # r3 variant + multi-bucket concurrent launches on a small cfg2-like batch
    c = fx.pop_case("cfg1")
    b = CudaBackend(mode="fast", device=0)
    grid = b._grid_for_set(c["grid"])
    batch = hostprep.TopologyBatch.synth(2, 0, 12)
    try:
        arrays = hostprep.prepare_batch(batch, grid.labels, table=fx.TABLE)
        lset = hostprep.ligand_set(arrays)
        s = c["grid"].spec
        _run(grid, lset, 0, 12, GaConfig(population_size=64, generations=2,
                                         translation_bounds=(s.origin, s.upper)),
             0, 0, _abi.MODE_FAST, 7 + int(batch.n_torsions.max()))
    except ValueError:
        pass
    # device grid builder
    prot = synth.make_protein(3, 300)
    gridmaps.build_grid_maps(prot, gridmaps.GridSpec.centered((0, 0, 0), (9, 9, 9), 0.8), ["C", "HD"])
    print("sanitize case done")


if __name__ == "__main__":
    main()
