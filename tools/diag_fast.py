"""Diagnose FAST-mode tolerance failures on random cfg1 poses (GPU box)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import fixtures as fx
from oracle import oracle
from paper_2509_12232_b200 import synth
from paper_2509_12232_b200.backend import CudaBackend

c = fx.pop_case("cfg1")
spec = c["grid"].spec
genes = synth.random_genes(0, 300_000, c["ctx"].n_torsions, spec.origin, spec.upper)[::7]
fast = CudaBackend("fast", 0)
exact = CudaBackend("exact", 0)
e, a, t = fast.score_population_arrays(genes, c["ctx"])
xe, xa, xt = exact.score_population_arrays(genes, c["ctx"])
we, wa, wt = oracle.dock_population(oracle.Ligand(c["ctx"]), genes, n_threads=0)
for name, g, w in (("total", t, wt), ("inter", e, we), ("intra", a, wa), ("x_total", xt, wt)):
    ok = fx.within_tol(g, w)
    rel = np.abs(g.astype(np.float64) - w) / np.maximum(np.abs(w), 1e-30)
    print(name, "fail", int((~ok).sum()), "of", len(ok), "max rel", float(rel.max()))
bad = np.flatnonzero(~fx.within_tol(t, wt))[:10]
for k in bad:
    print(k, "tot", t[k], wt[k], "inter", e[k], we[k], "intra", a[k], wa[k])
