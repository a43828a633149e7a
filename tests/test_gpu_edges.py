"""Edge cases of the device path against the oracle: sizes at and past the shape limits,
degenerate ligands and batches, everything out of the box.  Reference behaviour:
vd/scoring/simd.py (no size limit on the CPU), vd/ga.py:180-235, vd/screening.py:165-244
(an empty batch is an error there; an empty slice of a batch is a no-op here).
Tolerance (north star): |d| <= 1e-3 kcal/mol or |d|/|E| <= 1e-4; exact mode bit for bit."""

from __future__ import annotations

import numpy as np
import pytest

import fixtures as fx
from oracle import oracle, parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def grid():
    from paper_2509_12232_b200 import gridmaps, synth

    spec = gridmaps.GridSpec.centered((0.0, 0.0, 0.0), (50, 46, 54), 0.4)
    return gridmaps.build_grid_maps(synth.make_protein(21, 2500, half_extent=16.0), spec,
                                    synth.CONFIGS[2].probe_types)


def _score_vs_oracle(topo, gset, n, seed, lo_hi=None):
    from paper_2509_12232_b200 import synth
    from paper_2509_12232_b200.backend import CudaBackend
    from paper_2509_12232_b200.context import prepare_context

    ctx = prepare_context(topo, gset)
    lo, hi = lo_hi or (gset.spec.origin, gset.spec.upper)
    genes = synth.random_genes(seed, n, ctx.n_torsions, lo, hi)
    want = oracle.dock_population(oracle.Ligand(ctx), genes, n_threads=0)
    for mode in ("fast", "exact"):
        got = CudaBackend(mode=mode, device=0).score_population_arrays(genes, ctx)
        for g, w, what in zip(got, want, ("inter", "intra", "total")):
            if mode == "exact":
                assert np.array_equal(g, w), (mode, what)
            ok = parity.within_tol(g, w)
            assert ok.all(), (mode, what, int((~ok).sum()))
    return ctx


@pytest.mark.parametrize("heavy,hd,tors", [(225, 75, 40), (300, 100, 12)])
def test_large_ligands_score_like_the_oracle(grid, heavy, hd, tors):
    """300-400 atoms (past cfg4's 128; TPP 8 with 16 pose pairs per CTA, streamed pairs:
    ~45k-80k of them) and 40 torsions."""
    from paper_2509_12232_b200 import synth

    _score_vs_oracle(synth.make_ligand(7, heavy, hd, tors), grid, 1024, 5)


def test_ligand_too_large_for_the_pose_tile_is_a_clean_error(grid):
    from paper_2509_12232_b200 import synth
    from paper_2509_12232_b200.backend import CudaBackend
    from paper_2509_12232_b200.context import prepare_context

    ctx = prepare_context(synth.make_ligand(3, 1500, 500, 10), grid)
    genes = synth.random_genes(1, 8, ctx.n_torsions, grid.spec.origin, grid.spec.upper)
    with pytest.raises(RuntimeError, match="too large"):
        CudaBackend(mode="fast", device=0).score_population_arrays(genes, ctx)
    # the library is still usable afterwards
    _score_vs_oracle(synth.make_ligand(4, 20, 6, 3), grid, 64, 2)


def test_single_atom_ligand_scores_and_docks(grid):
    """N = 1, no pairs, no torsions: inter only; the GA still runs its generations."""
    from paper_2509_12232_b200 import synth
    from paper_2509_12232_b200.backend import CudaBackend
    from paper_2509_12232_b200.ga import GaConfig, dock

    topo = synth.make_ligand(3, 1, 0, 0)
    ctx = _score_vs_oracle(topo, grid, 256, 9)
    cfg = GaConfig(population_size=32, generations=5, seed=4)
    r = dock(topo, grid, cfg, backend=CudaBackend(mode="exact", device=0), context=ctx)
    g, bt, *_ = oracle.dock(oracle.Ligand(ctx), oracle.ga_params(cfg, grid.spec.origin,
                                                               grid.spec.upper), 4, 0)
    assert r.best_score.total == float(bt) and np.array_equal(r.best_genotype, g)
    assert r.best_score.intra == 0.0


def test_every_atom_out_of_the_box(grid):
    """Translations far outside the box: every atom takes the 1e4 * (distance + 1) penalty."""
    from paper_2509_12232_b200 import synth

    far = (np.asarray(grid.spec.upper) + 30.0, np.asarray(grid.spec.upper) + 60.0)
    ctx = _score_vs_oracle(synth.make_ligand(8, 24, 8, 5), grid, 512, 3, lo_hi=far)
    assert ctx.n_atoms == 32


def test_empty_population_and_empty_ligand_range(grid):
    from paper_2509_12232_b200 import _abi, hostprep, synth
    from paper_2509_12232_b200.backend import CudaBackend
    from paper_2509_12232_b200.context import prepare_context
    from paper_2509_12232_b200.ga import GaConfig, _run

    b = CudaBackend(mode="fast", device=0)
    ctx = prepare_context(synth.make_ligand(2, 20, 5, 4), grid)
    e, a, t = b.score_population_arrays(np.empty((0, 7 + ctx.n_torsions)), ctx)
    assert e.shape == a.shape == t.shape == (0,)
    g = b._grid_for_set(grid)
    batch = hostprep.TopologyBatch.synth(2, 0, 3)
    lset = hostprep.ligand_set(hostprep.prepare_batch(batch, g.labels))
    ga = GaConfig(population_size=16, generations=2,
                  translation_bounds=(grid.spec.origin, grid.spec.upper))
    out = _run(g, lset, 1, 0, ga, 0, 0, _abi.MODE_FAST, 7 + int(batch.n_torsions.max()))
    assert all(len(x) == 0 for x in out if x is not None)


@pytest.mark.parametrize("pop", [2, 3, 65, 257])
def test_ga_odd_and_tiny_populations_match_oracle(grid, pop):
    """Populations that leave a half-filled pose pair / tile (and pop = 2, the minimum):
    exact mode equals the oracle GA bit for bit."""
    from paper_2509_12232_b200 import synth
    from paper_2509_12232_b200.backend import CudaBackend
    from paper_2509_12232_b200.context import prepare_context
    from paper_2509_12232_b200.ga import GaConfig, dock

    topo = synth.make_ligand(12, 26, 8, 6)
    ctx = prepare_context(topo, grid)
    cfg = GaConfig(population_size=pop, generations=4, seed=6, elitism_count=1)
    r = dock(topo, grid, cfg, backend=CudaBackend(mode="exact", device=0), context=ctx)
    g, bt, *_, trace, ne = oracle.dock(oracle.Ligand(ctx), oracle.ga_params(
        cfg, grid.spec.origin, grid.spec.upper), 6, 0)
    assert np.array_equal(r.trace.view(np.uint32), trace.view(np.uint32))
    assert np.array_equal(r.best_genotype, g) and r.n_evaluations == ne == pop * 5
    fast = dock(topo, grid, cfg, backend=CudaBackend(mode="fast", device=0), context=ctx)
    assert fast.n_evaluations == pop * 5 and np.isfinite(fast.best_score.total)
