"""GPU GA: device docking vs the restated CPU GA oracle, plus the reference's GA
contract (pkg/tests/test_ga.py:135-228, test_acceptance.py:211-248)."""

from __future__ import annotations

import numpy as np
import pytest

import fixtures as fx
from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    from paper_2509_12232_b200.backend import CudaBackend

    return {"fast": CudaBackend(mode="fast", device=0), "exact": CudaBackend(mode="exact", device=0)}


def _oracle_dock(c, cfg, seed, lig_index=0):
    lo, hi = c["grid"].spec.origin, c["grid"].spec.upper
    return oracle.dock(oracle.Ligand(c["ctx"]), oracle.ga_params(cfg, lo, hi), seed, lig_index)


@pytest.mark.parametrize("name", ["cfg0", "cfg1", "rigid", "refgen"])
def test_exact_mode_ga_is_stream_exact(cuda, name):
    """Same Philox stream + reference-exact scoring => identical trajectories."""
    from paper_2509_12232_b200.ga import GaConfig, dock

    c = fx.pop_case(name)
    cfg = GaConfig(population_size=48, generations=12, seed=5)
    res = dock(c["topo"], c["grid"], cfg, backend=cuda["exact"], context=c["ctx"])
    g, bt, be, ba, trace, ne = _oracle_dock(c, cfg, 5)
    assert np.array_equal(res.trace.view(np.uint32), trace.view(np.uint32))
    assert np.array_equal(res.best_genotype, g)
    assert res.best_score.total == float(bt)
    assert res.n_evaluations == ne == 48 * 13


@pytest.mark.parametrize("name", ["cfg0", "cfg1"])
def test_fast_mode_ga_within_tolerance_or_rmsd(cuda, name):
    from paper_2509_12232_b200.ga import GaConfig, dock

    c = fx.pop_case(name)
    cfg = GaConfig(population_size=64, generations=30, seed=11)
    res = dock(c["topo"], c["grid"], cfg, backend=cuda["fast"], context=c["ctx"])
    g, bt, *_ = _oracle_dock(c, cfg, 11)
    if not fx.within_tol([res.best_score.total], [bt]).all():
        lig = oracle.Ligand(c["ctx"])
        p_dev = oracle.pose_population(lig, res.best_genotype[None])[0]
        p_ref = oracle.pose_population(lig, g[None])[0]
        rmsd = float(np.sqrt(((p_dev - p_ref) ** 2).sum(axis=0).mean()))
        assert rmsd <= 0.5, (res.best_score.total, bt, rmsd)


def test_contract_monotone_trace_count_determinism(cuda):
    from paper_2509_12232_b200.ga import GaConfig, dock

    c = fx.pop_case("cfg0")
    cfg = GaConfig(population_size=16, generations=25, seed=2)
    r1 = dock(c["topo"], c["grid"], cfg, backend=cuda["fast"], context=c["ctx"])
    r2 = dock(c["topo"], c["grid"], cfg, backend=cuda["fast"], context=c["ctx"])
    assert np.all(np.diff(r1.trace) <= 0)
    assert len(r1.trace) == cfg.generations + 1
    assert r1.n_evaluations == 16 * 26
    assert np.array_equal(r1.best_genotype, r2.best_genotype)
    assert np.array_equal(r1.trace.view(np.uint32), r2.trace.view(np.uint32))
    r3 = dock(c["topo"], c["grid"], GaConfig(population_size=16, generations=25, seed=3),
              backend=cuda["fast"], context=c["ctx"])
    assert not np.array_equal(r1.best_genotype, r3.best_genotype)
    from paper_2509_12232_b200 import backend

    re = backend.score_pose(c["topo"], r1.best_genotype, c["grid"], backend=cuda["fast"],
                            context=c["ctx"])
    assert re.total == pytest.approx(r1.best_score.total, abs=1e-4)


def test_constant_landscape_trace(cuda):
    from paper_2509_12232_b200 import chem, gridmaps, topology
    from paper_2509_12232_b200.ga import GaConfig, dock

    custom = chem.parse_parameter_table("C 4.0 0.0 0.0 0.0 0\n")
    spec = gridmaps.GridSpec.centered((0, 0, 0), (5, 5, 5), 1.0)
    z = np.zeros(spec.dims, np.float32)
    gset = gridmaps.GridMapSet(spec, {"C": z, chem.ELEC_LABEL: z, chem.DESOLV_LABEL: z})
    coords = np.zeros((3, 3), np.float32)
    coords[0] = [-1.0, 0.0, 1.0]
    topo = topology.LigandTopology(coords, np.zeros(3, np.int32), np.zeros(3, np.float32),
                                   np.array([[0, 1], [1, 2]], np.int32),
                                   (topology.RotatableBond(0, 1, np.array([1, 2], np.int32)),))
    res = dock(topo, gset, GaConfig(population_size=10, generations=15, seed=1),
               backend=cuda["fast"], table=custom)
    assert np.all(res.trace == float(np.float32(chem.TermWeights().tors)))


def test_single_atom_converges_to_minimum_node(cuda):
    """pkg/tests/test_ga.py:195-228: 20/20 seeds park the atom within 2 spacings."""
    from paper_2509_12232_b200 import chem, gridmaps, topology
    from paper_2509_12232_b200.ga import GaConfig, dock

    custom = chem.parse_parameter_table("C 4.0 0.0 0.0 0.0 0\n")
    spec = gridmaps.GridSpec.centered((0, 0, 0), (9, 9, 9), 0.5)
    target = (6, 3, 2)
    ax, ay, az = np.meshgrid(np.arange(9), np.arange(9), np.arange(9), indexing="ij")
    m = (0.5 * np.sqrt((ax - 6.0) ** 2 + (ay - 3.0) ** 2 + (az - 2.0) ** 2)).astype(np.float32)
    m[target] = -50.0
    z = np.zeros(spec.dims, np.float32)
    gset = gridmaps.GridMapSet(spec, {"C": m, chem.ELEC_LABEL: z, chem.DESOLV_LABEL: z})
    topo = topology.LigandTopology(np.zeros((3, 1), np.float32), np.zeros(1, np.int32),
                                   np.zeros(1, np.float32), np.empty((0, 2), np.int32))
    txyz = np.array([spec.origin[k] + target[k] * spec.spacing for k in range(3)])
    hits = 0
    for seed in range(20):
        cfg = GaConfig(population_size=40, generations=200, seed=seed, elitism_count=1)
        r = dock(topo, gset, cfg, backend=cuda["fast"], table=custom)
        hits += np.linalg.norm(r.best_genotype[:3] - txyz) <= 2 * spec.spacing
    assert hits == 20


def test_batch_equals_single_and_is_shard_independent(cuda):
    """Ligand i keyed (seed, i): one batched launch == per-ligand launches == any split."""
    from paper_2509_12232_b200 import synth
    from paper_2509_12232_b200.ga import GaConfig
    from paper_2509_12232_b200.screening import ScreenConfig, screen_batch

    c = fx.pop_case("cfg1")
    ligs = [(f"l{i}", synth.config_ligand(2, i)) for i in range(12)]
    cfg = ScreenConfig(ga=GaConfig(population_size=32, generations=8), backend="cuda",
                       global_seed=4)
    whole = screen_batch(ligs, c["grid"], cfg)
    from paper_2509_12232_b200 import ga as gam

    for i in (0, 5, 11):
        r = gam.dock(ligs[i][1], c["grid"], cfg.ga, backend="cuda", seed_key=(4, i))
        assert np.array_equal(r.best_genotype, whole[i].result.best_genotype)
        assert r.best_score == whole[i].result.best_score
    # emulate a 3-rank split: each shard docked by its own launch with its global base
    from dataclasses import replace

    from paper_2509_12232_b200 import backend as bk
    from paper_2509_12232_b200.context import prepare_context
    from paper_2509_12232_b200.screening import _shared_device_set, shard_range

    b = bk.get_backend("cuda")
    ctxs = [prepare_context(t, c["grid"]) for _, t in ligs]
    grid, lset = _shared_device_set(b, c["grid"], ctxs)
    ga = replace(cfg.ga, translation_bounds=(c["grid"].spec.origin, c["grid"].spec.upper))
    gmax = 7 + max(t.n_torsions for _, t in ligs)
    full = gam._run(grid, lset, 0, len(ligs), ga, 4, 0, b._mode(), gmax, trace=False)
    for rank in range(3):
        lo, hi = shard_range(len(ligs), rank, 3)
        part = gam._run(grid, lset, lo, hi - lo, ga, 4, lo, b._mode(), gmax, trace=False)
        assert np.array_equal(part[3], full[3][lo:hi])
        assert np.array_equal(part[0], full[0][lo:hi])


def test_exact_batch_matches_oracle_dock_many(cuda):
    from paper_2509_12232_b200 import synth
    from paper_2509_12232_b200.context import prepare_context
    from paper_2509_12232_b200.ga import GaConfig
    from paper_2509_12232_b200.screening import ScreenConfig, screen_batch

    c = fx.pop_case("cfg1")
    ligs = [(f"l{i}", synth.config_ligand(2, i)) for i in range(6)]
    ga = GaConfig(population_size=24, generations=6)
    got = screen_batch(ligs, c["grid"], ScreenConfig(ga=ga, backend="cuda-exact", global_seed=9))
    lo, hi = c["grid"].spec.origin, c["grid"].spec.upper
    ors = [oracle.Ligand(prepare_context(t, c["grid"])) for _, t in ligs]
    g, bt, be, ba, ne = oracle.dock_many(ors, oracle.ga_params(ga, lo, hi), 9, 0)
    for i, e in enumerate(got):
        G = 7 + ligs[i][1].n_torsions
        assert np.array_equal(e.result.best_genotype, g[i, :G])
        assert e.result.best_score.total == float(bt[i])


def test_cfg4_ligand_exact_ga_matches_oracle(cuda):
    """128-atom / 32-torsion ligand (cfg4 shape): device GA == oracle GA, bit for bit."""
    from paper_2509_12232_b200 import hostprep
    from paper_2509_12232_b200.context import prepare_context
    from paper_2509_12232_b200.ga import GaConfig, dock

    c = fx.pop_case("cfg1")
    topo = hostprep.TopologyBatch.synth(4, 7, 1).topology(0)
    ctx = prepare_context(topo, c["grid"])
    cfg = GaConfig(population_size=24, generations=3, seed=1)
    res = dock(topo, c["grid"], cfg, backend=cuda["exact"], context=ctx)
    lo, hi = c["grid"].spec.origin, c["grid"].spec.upper
    g, bt, *_, trace, ne = oracle.dock(oracle.Ligand(ctx), oracle.ga_params(cfg, lo, hi), 1, 0)
    assert np.array_equal(res.trace.view(np.uint32), trace.view(np.uint32))
    assert np.array_equal(res.best_genotype, g)


def test_screen_batch_records_failures_in_place(cuda):
    """A ligand whose atom type has no map fails alone (vd/screening.py:195-244)."""
    from paper_2509_12232_b200 import synth
    from paper_2509_12232_b200.ga import GaConfig
    from paper_2509_12232_b200.screening import ScreenConfig, screen_batch
    from paper_2509_12232_b200.topology import LigandTopology

    c = fx.pop_case("cfg1")
    good = synth.config_ligand(2, 3)
    bad = LigandTopology(good.coords0, np.full(good.n_atoms, fx.TABLE.index_of("S")),
                         good.charge, good.bonds, good.rotatable_bonds)
    maps = {k: v for k, v in c["grid"].maps.items() if k != "S"}
    from paper_2509_12232_b200 import gridmaps

    g = gridmaps.GridMapSet(c["grid"].spec, maps)
    out = screen_batch([("a", good), ("b", bad), ("c", good)], g,
                       ScreenConfig(ga=GaConfig(population_size=16, generations=3)))
    assert out[0].error is None and out[2].error is None
    assert out[1].result is None and "no map" in out[1].error
    assert out[0].seed_key == (0, 0) and out[2].seed_key == (0, 2)


@pytest.mark.parametrize("kw", [dict(elitism_count=3, tournament_size=3),
                                dict(elitism_count=0, tournament_size=1, crossover_rate=0.0),
                                dict(mutation_rate=0.3, crossover_rate=1.0, population_size=33),
                                dict(population_size=2, generations=4)])
def test_exact_ga_operator_variants_match_oracle(cuda, kw):
    from paper_2509_12232_b200.ga import GaConfig, dock

    c = fx.pop_case("refgen")
    base = dict(population_size=40, generations=6, seed=13)
    base.update(kw)
    cfg = GaConfig(**base)
    res = dock(c["topo"], c["grid"], cfg, backend=cuda["exact"], context=c["ctx"])
    g, bt, *_, trace, ne = _oracle_dock(c, cfg, 13)
    assert np.array_equal(res.trace.view(np.uint32), trace.view(np.uint32))
    assert np.array_equal(res.best_genotype, g)
    assert res.n_evaluations == ne


@pytest.mark.parametrize("layout", ["plain", "zpair", "brick"])
def test_fast_mode_ga_identical_on_every_grid_layout(cuda, layout, monkeypatch):
    """The GA kernel is instantiated per grid layout (packed: pipelined brick / z-pair
    gathers; plain: z-pair loads with the out-of-box early return, e.g. cfg4's 126^3 grid).
    Corner values, lerps and the atom summation order are the same, so a fast-mode GA run
    is bit-identical on every layout."""
    from paper_2509_12232_b200 import gridmaps
    from paper_2509_12232_b200.backend import CudaBackend
    from paper_2509_12232_b200.context import prepare_context
    from paper_2509_12232_b200.ga import GaConfig, dock

    env = {"plain": ("VD_NO_PACK", "1"), "zpair": ("VD_BRICK_BUDGET_MB", "0"),
           "brick": ("VD_BRICK_BUDGET_MB", "100000")}
    c = fx.pop_case("cfg1")
    cfg = GaConfig(population_size=64, generations=8, seed=21)

    def run(lay):
        monkeypatch.setenv(*env[lay])
        g2 = gridmaps.GridMapSet(c["grid"].spec, dict(c["grid"].maps))  # fresh device grid
        ctx = prepare_context(c["topo"], g2)
        r = dock(c["topo"], g2, cfg, backend=CudaBackend(mode="fast", device=0), context=ctx)
        monkeypatch.undo()
        return r

    got, ref = run(layout), run("plain" if layout != "plain" else "brick")
    assert np.array_equal(got.trace.view(np.uint32), ref.trace.view(np.uint32))
    assert np.array_equal(got.best_genotype, ref.best_genotype)


def test_generation_synchronous_path_is_bit_identical_to_persistent_kernels(cuda, monkeypatch):
    """Batches that fill the GPU run every generation as two launches over all ligands
    (pop_score_kernel at the score kernel's shapes + ga_step_kernel); smaller batches and
    teams run the persistent kernels.  Both use a ligand's own sub-thread count and the same
    role split, operators and random streams, so which path a batch takes never shows:
    every output of a 96-ligand cfg2 batch is identical byte for byte."""
    from paper_2509_12232_b200 import _abi, gridmaps, hostprep, synth
    from paper_2509_12232_b200.ga import GaConfig, _run

    spec = synth.config_grid_spec(2)
    gset = gridmaps.build_grid_maps(synth.config_protein(2), spec, synth.CONFIGS[2].probe_types)
    grid = cuda["fast"]._grid_for_set(gset)
    batch = hostprep.TopologyBatch.synth(2, 0, 96)
    assert batch.n_atoms.min() <= 24 and batch.n_atoms.max() >= 56  # several shape groups
    lset = hostprep.ligand_set(hostprep.prepare_batch(batch, grid.labels))
    ga = GaConfig(population_size=256, generations=20, elitism_count=2,
                  translation_bounds=(spec.origin, spec.upper))
    gmax = 7 + int(batch.n_torsions.max())

    def run(sync):
        monkeypatch.setenv("VD_GA_SYNC", sync)
        return _run(grid, lset, 0, 96, ga, 4, 0, _abi.MODE_FAST, gmax)

    a, b = run("0"), run("1")
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
    # odd populations (half-filled pose pairs and tiles), no elites
    ga2 = GaConfig(population_size=67, generations=6, elitism_count=0,
                   translation_bounds=(spec.origin, spec.upper))
    monkeypatch.setenv("VD_GA_SYNC", "0")
    a = _run(grid, lset, 0, 24, ga2, 9, 100, _abi.MODE_FAST, gmax)
    monkeypatch.setenv("VD_GA_SYNC", "1")
    b = _run(grid, lset, 0, 24, ga2, 9, 100, _abi.MODE_FAST, gmax)
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))


def test_concurrent_host_threads_dock_batches_of_shared_shapes(cuda):
    """Four host threads dock different slices of a cfg2 batch at once (the reference's
    screen_batch worker pool does this, one ligand per call).  The generation-synchronous
    path sets a per-function carveout before each of its launches and the slices share
    kernel functions: results must equal the sequential ones byte for byte."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2509_12232_b200 import _abi, gridmaps, hostprep, synth
    from paper_2509_12232_b200.ga import GaConfig, _run

    spec = synth.config_grid_spec(2)
    gset = gridmaps.build_grid_maps(synth.config_protein(2), spec, synth.CONFIGS[2].probe_types)
    grid = cuda["fast"]._grid_for_set(gset)
    batch = hostprep.TopologyBatch.synth(2, 0, 64)
    lset = hostprep.ligand_set(hostprep.prepare_batch(batch, grid.labels))
    ga = GaConfig(population_size=128, generations=12, translation_bounds=(spec.origin, spec.upper))
    gmax = 7 + int(batch.n_torsions.max())
    slices = [(0, 16), (16, 16), (32, 16), (48, 16), (5, 1), (40, 3)]

    def work(sl):
        return _run(grid, lset, sl[0], sl[1], ga, 11, sl[0], _abi.MODE_FAST, gmax)

    want = [work(sl) for sl in slices]
    with ThreadPoolExecutor(max_workers=4) as ex:
        got = list(ex.map(work, slices * 3))
    for k, g in enumerate(got):
        for x, y in zip(g, want[k % len(slices)]):
            assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
    whole = _run(grid, lset, 0, 64, ga, 11, 0, _abi.MODE_FAST, gmax)
    for sl, w in zip(slices, want):
        assert np.array_equal(w[0], whole[0][sl[0]:sl[0] + sl[1]])   # batch-independent results
        assert np.array_equal(w[3], whole[3][sl[0]:sl[0] + sl[1]])


@pytest.mark.parametrize("team", ["2", "4", "8"])
def test_team_split_ga_is_bit_identical(cuda, team, monkeypatch):
    """Large ligands in small batches split one ligand's population over a team of CTAs
    (ga_team_kernel: fitness through global memory, two team barriers per generation).
    Selection, RNG and scoring are unchanged, so every output equals the one-CTA GA's."""
    from paper_2509_12232_b200 import _abi, gridmaps, hostprep, synth
    from paper_2509_12232_b200.ga import GaConfig, _run

    spec = gridmaps.GridSpec.centered((0.0, 0.0, 0.0), (56, 56, 56), 0.375)
    gset = gridmaps.build_grid_maps(synth.make_protein(11, 2500, half_extent=14.0), spec,
                                    synth.CONFIGS[4].probe_types)
    grid = cuda["fast"]._grid_for_set(gset)
    batch = hostprep.TopologyBatch.synth(4, 3, 10)
    lset = hostprep.ligand_set(hostprep.prepare_batch(batch, grid.labels))
    gmax = 7 + int(batch.n_torsions.max())
    # pop 100: slices of 100 / team individuals, odd tile tails; elitism 3 crosses slices
    ga = GaConfig(population_size=100, generations=6, elitism_count=3,
                  translation_bounds=(spec.origin, spec.upper))

    def run(t):
        monkeypatch.setenv("VD_GA_TEAM", t)
        r = _run(grid, lset, 0, 10, ga, 9, 40, _abi.MODE_FAST, gmax)
        monkeypatch.delenv("VD_GA_TEAM")
        return r

    one, split = run("1"), run(team)
    for x, y in zip(one, split):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
