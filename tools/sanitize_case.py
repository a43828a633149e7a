"""Small invocations of every hot kernel shape, with all outputs saved, for the checked-
build comparison (tests/test_gpu_checked.py; compute-sanitizer is closed on this pool).

  score_kernel  TPP 4 role split (cfg1 fixture, 40 atoms, resident pairs), TPP 16 and 8
                with streamed pair tiles (128-atom fixture), TPP 8 exact; yz-brick, z-pair
                and plain grid layouts; the host-buffer pipeline path
  pose_kernel   TPP 1 / 4 / 8 / 16
  ga_kernel     fast packed, fast plain, exact, several shape groups at once, the same
                batch through the generation-synchronous path (pop_score_kernel +
                ga_step_kernel); ga_team_kernel (6 cfg4 ligands: one ligand over 8 CTAs)
  grid_kernel   a small device grid build; MUGD load (transpose kernel)
Usage: [VD_LIB=.../libvdb200_checked.so] python tools/sanitize_case.py OUT.npz
Prints the checked build's device flag word (0 = no bounds/invariant failure).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import ctypes  # noqa: E402

import numpy as np  # noqa: E402

import fixtures as fx  # noqa: E402
from paper_2509_12232_b200 import _abi, gridmaps, hostprep, synth  # noqa: E402
from paper_2509_12232_b200.backend import CudaBackend  # noqa: E402
from paper_2509_12232_b200.context import prepare_context  # noqa: E402
from paper_2509_12232_b200.ga import GaConfig, _run, dock  # noqa: E402


def main(out_path):
    _abi.ensure_device(0)
    out = {}
    for layout, env in (("brick", {"VD_BRICK_BUDGET_MB": "100000"}),
                        ("zpair", {"VD_BRICK_BUDGET_MB": "0"}), ("plain", {"VD_NO_PACK": "1"})):
        os.environ.update(env)
        for name, n in (("cfg1", 130), ("big", 66)):
            c = fx.pop_case(name)
            g2 = gridmaps.GridMapSet(c["grid"].spec, dict(c["grid"].maps))  # fresh device grid
            ctx = prepare_context(c["topo"], g2, table=fx.TABLE)
            for mode in ("fast", "exact"):
                b = CudaBackend(mode=mode, device=0)
                for k, v in zip("eat", b.score_population_arrays(c["genes"][:n], ctx)):
                    out[f"{layout}_{name}_{mode}_score_{k}"] = v
            _, ligs = CudaBackend(mode="fast", device=0).prepared(ctx)
            if name == "big":  # > 96 atoms launch with 16 subs: keep the 8-sub shape covered
                os.environ["VD_TPP"] = "8"
                for k, v in zip("eat", CudaBackend(mode="fast", device=0).score_population_arrays(
                        c["genes"][:n], ctx)):
                    out[f"{layout}_{name}_fast_score8_{k}"] = v
                del os.environ["VD_TPP"]
            for tpp in (4, 8, 16):
                out[f"{layout}_{name}_pose{tpp}"] = _abi.debug_pose_genes(ligs, 0, c["genes"][:n], tpp)
            out[f"{layout}_{name}_pose1"] = CudaBackend(mode="fast", device=0).pose_population(
                c["genes"][:n], ctx)
            for mode in ("fast", "exact"):
                r = dock(c["topo"], g2, GaConfig(population_size=40, generations=3, seed=1),
                         backend=CudaBackend(mode=mode, device=0), context=ctx)
                out[f"{layout}_{name}_{mode}_ga_genes"] = r.best_genotype
                out[f"{layout}_{name}_{mode}_ga_trace"] = r.trace
        for k in env:
            del os.environ[k]
    # several GA shape groups at once (concurrent launches) on a cfg2 batch
    spec = gridmaps.GridSpec.centered((0.0, 0.0, 0.0), (40, 40, 40), 0.375)
    gset = gridmaps.build_grid_maps(synth.make_protein(5, 1500), spec, synth.CONFIGS[2].probe_types)
    out["grid_maps_sample"] = np.stack([gset.maps[l][::7, ::5, ::3] for l in gset.maps])
    b = CudaBackend(mode="fast", device=0)
    grid = b._grid_for_set(gset)
    batch = hostprep.TopologyBatch.synth(2, 0, 40)
    arrays = hostprep.prepare_batch(batch, grid.labels)
    lset = hostprep.ligand_set(arrays)
    # the persistent kernels (one CTA per ligand, 4 / 8 subs with the role split) ...
    os.environ["VD_GA_SYNC"] = "0"
    r = _run(grid, lset, 0, 40, GaConfig(population_size=64, generations=3,
                                         translation_bounds=(spec.origin, spec.upper)),
             0, 0, _abi.MODE_FAST, 7 + int(batch.n_torsions.max()))
    del os.environ["VD_GA_SYNC"]
    for k, v in zip(("bt", "be", "ba", "bg", "tr", "ne"), r):
        out[f"batch_ga_{k}"] = v
    # ... and the same batch through the default generation-synchronous path (pop_score_kernel +
    # ga_step_kernel; bit-identical to the persistent kernels by design)
    r = _run(grid, lset, 0, 40, GaConfig(population_size=64, generations=3,
                                         translation_bounds=(spec.origin, spec.upper)),
             0, 0, _abi.MODE_FAST, 7 + int(batch.n_torsions.max()))
    for k, v in zip(("bt", "be", "ba", "bg", "tr", "ne"), r):
        out[f"sync_ga_{k}"] = v
        assert np.array_equal(np.asarray(v).view(np.uint8), np.asarray(out[f"batch_ga_{k}"]).view(np.uint8)), k
    # large ligands in a small batch: the team kernel (a ligand's population over 8 CTAs)
    b4 = hostprep.TopologyBatch.synth(4, 0, 6)
    l4 = hostprep.ligand_set(hostprep.prepare_batch(b4, grid.labels))
    r = _run(grid, l4, 0, 6, GaConfig(population_size=96, generations=2,
                                       translation_bounds=(spec.origin, spec.upper)),
             0, 0, _abi.MODE_FAST, 7 + int(b4.n_torsions.max()))
    for k, v in zip(("bt", "be", "ba", "bg", "tr", "ne"), r):
        out[f"team_ga_{k}"] = v
    mg = gridmaps.load_grid_set(fx.GOLDEN / "ref_grid_odd.mugd")
    out["mugd_odd"] = mg.device_grid.download()
    flags = ctypes.c_uint32(0)
    checked = _abi.lib().vd_debug_check_flags(ctypes.byref(flags), 1)
    selftest = ctypes.c_uint32(0)
    _abi.lib().vd_debug_check_flags(ctypes.byref(selftest), -1)
    np.savez(out_path, **out)
    print(f"sanitize case done: checked_build={checked} flags=0x{flags.value:x} "
          f"selftest=0x{selftest.value:x} arrays={len(out)}")
    return 0 if flags.value == 0 else 3


if __name__ == "__main__":
    sys.exit(main(sys.argv[1] if len(sys.argv) > 1 else "sanitize_out.npz"))
