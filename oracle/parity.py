"""GA parity checks against the oracle (TEST INFRASTRUCTURE ONLY: used by tests/
and by bench.py after its timed regions, never by the product path).

The north star's GA criterion (BASELINE.json): full GA runs on the same seeded
Philox streams agree on best energies within 1e-3 kcal/mol or 1e-4 relative, or
on best-pose RMSD <= 0.5 A where float reordering flips a selection.  Reference:
vd/ga.py:180-235 (dock), pkg/tests/test_ga.py:135-228 (GA contract).
"""

from __future__ import annotations

import numpy as np

from . import oracle

REL, ABS = 1e-4, 1e-3


def within_tol(got, want, rel=REL, abs_=ABS):
    """|d| <= 1e-3 kcal/mol OR |d|/|E_ref| <= 1e-4, per element."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    d = np.abs(got - want)
    return (d <= abs_) | (d <= rel * np.abs(want))


def rescore(ligs, genes, n_threads=0):
    """Oracle (inter64, intra64, total32) of one genotype row per ligand."""
    from concurrent.futures import ThreadPoolExecutor

    n = len(ligs)
    inter, intra = np.empty(n), np.empty(n)
    total = np.empty(n, np.float32)

    def one(l):
        G = 7 + ligs[l].n_torsions
        e, a, t = oracle.dock_population(ligs[l], genes[l:l + 1, :G])
        inter[l], intra[l], total[l] = e[0], a[0], t[0]

    with ThreadPoolExecutor(max(1, n_threads or oracle.cores())) as ex:
        list(ex.map(one, range(n)))
    return inter, intra, total


def rmsd(lig, genes_a, genes_b) -> float:
    """Best-pose RMSD (A) between two genotypes of one ligand (exact oracle poses)."""
    G = 7 + lig.n_torsions
    p = oracle.pose_population(lig, np.stack([genes_a[:G], genes_b[:G]]))
    return float(np.sqrt(((p[0] - p[1]) ** 2).sum(axis=0).mean()))


def rescore_summary(ligs, best_total, best_inter, best_intra, best_genes, n_threads=0) -> dict:
    """Re-score every returned best genotype with the oracle: the device's reported
    best_total / inter / intra must be the oracle's energies of that genotype."""
    e, a, t = rescore(ligs, best_genes, n_threads)
    ok_t = within_tol(best_total, t)
    ok = ok_t & within_tol(best_inter, e) & within_tol(best_intra, a)
    d = np.abs(np.asarray(best_total, np.float64) - t.astype(np.float64))
    return {"ligands": int(len(ligs)), "best_rescored_within_tol": int(ok.sum()),
            "max_abs_diff_total": float(d.max()) if len(d) else 0.0,
            "max_rel_diff_total": float((d / np.maximum(np.abs(t), 1e-30)).max()) if len(d) else 0.0}


def ga_agreement(ligs, params, seed, base, best_total, best_genes, n_threads=0,
                 oracle_out=None) -> dict:
    """Full-length GA agreement, fast device GA vs the oracle GA with the same keys:
    per ligand, best_total within tolerance, else best-pose RMSD <= 0.5 A."""
    if oracle_out is None:
        oracle_out = oracle.dock_many(ligs, params, seed, base, n_threads=n_threads)
    og, obt = oracle_out[0], oracle_out[1]
    tol = within_tol(best_total, obt)
    rms = np.full(len(ligs), np.nan)
    for l in np.flatnonzero(~tol):
        rms[l] = rmsd(ligs[l], best_genes[l], og[l])
    by_rmsd = (~tol) & (rms <= 0.5)
    diff = np.asarray(best_total, np.float64) - obt.astype(np.float64)
    return {"ligands": int(len(ligs)), "within_tol": int(tol.sum()), "within_rmsd_0.5": int(by_rmsd.sum()),
            "agree": int((tol | by_rmsd).sum()),
            "bit_identical_best": int(np.sum(np.asarray(best_total, np.float32) == obt)),
            "device_better": int(np.sum(diff < 0) - np.sum((diff < 0) & tol)),
            "oracle_better": int(np.sum(diff > 0) - np.sum((diff > 0) & tol)),
            "median_best_total_device": float(np.median(best_total)),
            "median_best_total_oracle": float(np.median(obt)),
            "_oracle_best_total": obt, "_rmsd": rms}
