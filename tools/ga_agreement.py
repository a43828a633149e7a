"""Full-length GA agreement, device vs oracle GA with the same Philox keys, at BASELINE
lengths (cfg0 pop 100 x 50 seed 0; cfg2 pop 256 x 200; cfg4 pop 512 x 300), in fast and
exact modes.  Prints one JSON line per (cfg, mode).  Usage: python tools/ga_agreement.py
[n_cfg2] [n_cfg4]"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import oracle, parity  # noqa: E402
from paper_2509_12232_b200 import _abi, hostprep  # noqa: E402
from paper_2509_12232_b200.ga import GaConfig, _run  # noqa: E402
from test_gpu_baseline import workload_grid  # noqa: E402


def run(cfg, count, pop, gens, first=0):
    gset, grid, stack, _ = workload_grid(cfg)
    batch = hostprep.TopologyBatch.synth(cfg, first, count)
    arrays = hostprep.prepare_batch(batch, grid.labels)
    lset = hostprep.ligand_set(arrays)
    ligs = oracle.ligands_from_arrays(arrays, stack, gset.spec)
    ga = GaConfig(population_size=pop, generations=gens,
                  translation_bounds=(gset.spec.origin, gset.spec.upper))
    params = oracle.ga_params(ga, gset.spec.origin, gset.spec.upper)
    t0 = time.perf_counter()
    ref = oracle.dock_many(ligs, params, 0, first, n_threads=0)
    t_or = time.perf_counter() - t0
    gmax = 7 + int(lset.n_torsions.max())
    for name, mode in (("fast", _abi.MODE_FAST), ("exact", _abi.MODE_EXACT)):
        bt, be, ba, bg, tr, ne = _run(grid, lset, 0, count, ga, 0, first, mode, gmax, trace=False)
        ag = parity.ga_agreement(ligs, params, 0, first, bt, bg, oracle_out=ref)
        rs = parity.rescore_summary(ligs, bt, be, ba, bg)
        ag.pop("_oracle_best_total")
        rms = ag.pop("_rmsd")
        print(json.dumps({"cfg": cfg, "mode": name, "pop": pop, "generations": gens, **ag,
                          "rescore": rs, "oracle_s": round(t_or, 1),
                          "rmsd_of_disagreeing": [round(float(x), 2) for x in rms[~np.isnan(rms)][:20]]}),
              flush=True)


def run_cfg0():
    from paper_2509_12232_b200 import synth
    from paper_2509_12232_b200.backend import CudaBackend
    from paper_2509_12232_b200.context import prepare_context
    from paper_2509_12232_b200.ga import dock

    gset, _, _, _ = workload_grid(0)
    topo = synth.config_ligand(0, 0)
    ctx = prepare_context(topo, gset)
    lig = oracle.Ligand(ctx)
    cfg = GaConfig(population_size=100, generations=50, seed=0)
    g, bt, *_ = oracle.dock(lig, oracle.ga_params(cfg, gset.spec.origin, gset.spec.upper), 0, 0)
    for mode in ("fast", "exact"):
        r = dock(topo, gset, cfg, backend=CudaBackend(mode=mode, device=0), context=ctx)
        tol = bool(parity.within_tol([r.best_score.total], [bt])[0])
        print(json.dumps({"cfg": 0, "mode": mode, "device_best": r.best_score.total,
                          "oracle_best": float(bt), "within_tol": tol,
                          "bit_identical": bool(np.float32(r.best_score.total) == bt),
                          "rmsd": parity.rmsd(lig, r.best_genotype, g)}), flush=True)


if __name__ == "__main__":
    n2 = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    n4 = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    _abi.ensure_device(0)
    run_cfg0()
    run(2, n2, 256, 200)
    run(4, n4, 512, 300)
