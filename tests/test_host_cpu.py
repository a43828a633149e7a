"""CPU tests of host logic: registry plumbing, sharding + record gather over a
real 2-rank gloo group, GA operators of the restated oracle GA (the reference's
pkg/tests/test_ga.py properties), RNG transforms, MUGD I/O, mirror validation."""

from __future__ import annotations

import ctypes
import io
import math
import os
import socket
import types

import numpy as np
import pytest

import fixtures as fx
from oracle import oracle
from paper_2509_12232_b200 import chem, gridmaps, topology
from paper_2509_12232_b200.ga import GaConfig
from paper_2509_12232_b200.screening import REC_HEAD, gather_records, pack_records, shard_range


# --- sharding / gather --------------------------------------------------------------
@pytest.mark.parametrize("n,world", [(1, 1), (10, 3), (100000, 8), (7, 8), (12, 2)])
def test_shard_range_partitions(n, world):
    seen = []
    for r in range(world):
        lo, hi = shard_range(n, r, world)
        assert 0 <= lo <= hi <= n
        seen.extend(range(lo, hi))
    assert seen == list(range(n))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather_worker(rank, world, port, n, q, widths=(4, 4)):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(n, rank, world)
    m = hi - lo
    idx = np.arange(lo, hi, dtype=np.float64)
    rec = pack_records(idx.astype(np.float32), idx * 2, idx * 3, np.full(m, 7),
                       np.tile(idx[:, None], (1, widths[rank])), np.ones(m))
    out = gather_records(rec, n, dist)
    q.put((rank, out))
    dist.destroy_process_group()


def test_gather_records_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    n, world, port = 11, 2, _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        out = got[r]
        assert out.shape == (n, REC_HEAD + 4)
        np.testing.assert_array_equal(out[:, 0], np.arange(n, dtype=np.float32))
        np.testing.assert_array_equal(out[:, 1], 2.0 * np.arange(n))
        np.testing.assert_array_equal(out[:, 4], np.ones(n))
        np.testing.assert_array_equal(out[:, REC_HEAD], np.arange(n))


def test_gather_records_gloo_world2_ragged_gene_widths():
    """Ranks whose shards hold different max torsion counts (gene widths 7+3 and 7+9) agree
    on the widest record; the narrower rank's genes are zero-padded."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    n, world, port = 9, 2, _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, n, q, (3, 9)))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lo1, _ = shard_range(n, 1, world)
    for r in range(world):
        out = got[r]
        assert out.shape == (n, REC_HEAD + 9)
        np.testing.assert_array_equal(out[:, 0], np.arange(n, dtype=np.float32))
        np.testing.assert_array_equal(out[:lo1, REC_HEAD + 3:], 0.0)
        np.testing.assert_array_equal(out[lo1:, REC_HEAD + 8], np.arange(lo1, n))


# --- reference registry plumbing -------------------------------------------------
def test_register_into_reference_style_registry_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present: covered by GPU tests")
    from paper_2509_12232_b200.backend import register_reference_backend

    class BackendUnavailable(RuntimeError):
        pass

    mod = types.SimpleNamespace(_REGISTRY={}, BackendUnavailable=BackendUnavailable)

    def _load_backends():
        if mod._REGISTRY:
            return
        mod._REGISTRY["simd"] = object()

    mod._load_backends = _load_backends
    entry = register_reference_backend(mod)
    assert "simd" in mod._REGISTRY  # stock backends loaded before ours
    assert isinstance(entry, BackendUnavailable)


# --- restated GA (oracle) properties: pkg/tests/test_ga.py ------------------------
@pytest.fixture(scope="module")
def lig12():
    return fx.pop_case("cfg0")


def _params(**kw):
    base = dict(population_size=20, generations=10, seed=3)
    base.update(kw)
    cfg = GaConfig(**base)
    return oracle.ga_params(cfg, (-2.0, -2.0, -2.0), (2.0, 2.0, 2.0)), cfg


def test_ga_init_properties():
    p, _ = _params(population_size=200)
    a = oracle.init_population(p, 5, (3, 0))
    b = oracle.init_population(p, 5, (3, 0))
    np.testing.assert_array_equal(a, b)
    assert np.all(a[:, :3] >= -2.0) and np.all(a[:, :3] <= 2.0)
    np.testing.assert_allclose(np.linalg.norm(a[:, 3:7], axis=1), 1.0, atol=1e-12)
    assert np.all(a[:, 7:] >= -math.pi) and np.all(a[:, 7:] < math.pi)
    c = oracle.init_population(p, 5, (3, 1))
    assert not np.array_equal(a, c)  # key separates ligands (test_ga.py:231-237)


def test_ga_degenerate_operators_resample_parents():
    p, _ = _params(crossover_rate=0.0, mutation_rate=0.0, tournament_size=1, elitism_count=1)
    pop = oracle.init_population(p, 3, (1, 0))
    fit = np.arange(p.pop, dtype=np.float64)
    new = oracle.next_generation(p, 3, pop, fit, 0, (1, 0))
    np.testing.assert_array_equal(new[0], pop[0])
    rows = {tuple(r) for r in pop}
    assert all(tuple(r) in rows for r in new)


def test_ga_elites_survive_stable_order():
    p, _ = _params(elitism_count=2)
    pop = oracle.init_population(p, 3, (2, 0))
    fit = np.linspace(5.0, -3.0, p.pop)
    fit[3] = fit[-1]  # tie with the best: stable order keeps index 3 second
    new = oracle.next_generation(p, 3, pop, fit, 0, (2, 0))
    np.testing.assert_array_equal(new[0], pop[3])
    np.testing.assert_array_equal(new[1], pop[p.pop - 1])


def test_ga_operator_rates_within_binomial_bounds():
    p, cfg = _params(population_size=30, crossover_rate=0.7, mutation_rate=0.05)
    pop = oracle.init_population(p, 3, (9, 0))
    fit = np.random.default_rng(9).standard_normal(p.pop)
    counts = oracle.OrGaCounts()
    for gen in range(400):
        oracle.next_generation(p, 3, pop, fit, gen, (9, 0), counts)
    n = counts.children
    for observed, rate, total in ((counts.crossovers, cfg.crossover_rate, n),
                                  (counts.gene_mutations, cfg.mutation_rate, counts.genes_seen)):
        mean, sigma = rate * total, math.sqrt(total * rate * (1 - rate))
        assert abs(observed - mean) <= 3 * sigma, (observed, mean, sigma)


def test_ga_rotation_genes_stay_decodable():
    p, _ = _params(mutation_rate=0.5)
    pop = oracle.init_population(p, 3, (5, 0))
    fit = np.random.default_rng(5).standard_normal(p.pop)
    for gen in range(20):
        pop = oracle.next_generation(p, 3, pop, fit, gen, (5, 0))
    assert np.all(np.linalg.norm(pop[:, 3:7], axis=1) > 1e-6)


def test_oracle_dock_contract(lig12):
    c = lig12
    cfg = GaConfig(population_size=16, generations=25, seed=2)
    p = oracle.ga_params(cfg, c["grid"].spec.origin, c["grid"].spec.upper)
    lig = oracle.Ligand(c["ctx"])
    g1, bt1, *_, tr1, ne = oracle.dock(lig, p, 2, 0)
    g2, bt2, *_, tr2, _ = oracle.dock(lig, p, 2, 0)
    assert np.all(np.diff(tr1) <= 0) and len(tr1) == 26 and ne == 16 * 26
    np.testing.assert_array_equal(g1, g2)
    np.testing.assert_array_equal(tr1.view(np.uint32), tr2.view(np.uint32))
    _, _, tot = oracle.dock_population(lig, g1[None])
    assert tot[0] == bt1


# --- RNG transforms -------------------------------------------------------------------
def test_rng_transcendentals_accurate():
    L = oracle.lib()
    for x in np.concatenate([np.geomspace(2.0**-53, 1.0, 200), [0.5, 0.999999, 1.0]]):
        assert abs(L.or_log(float(x)) - math.log(x)) <= 4e-16 * max(1.0, abs(math.log(x)))
    for u in np.linspace(0.0, 1.0, 1001, endpoint=False):
        assert abs(L.or_cos2pi(float(u)) - math.cos(2 * math.pi * u)) <= 1e-15
    z = np.array([L.or_normal(c, 1, 2, 4, 7, 3) for c in range(20000)])
    assert abs(z.mean()) < 0.05 and abs(z.std() - 1.0) < 0.03


def _numpy_philox_at(key, counter):
    """numpy's Philox positioned so its next block is `counter` (numpy bumps the
    counter before each block)."""
    prev = list(counter)
    for w in range(4):
        if prev[w] > 0:
            prev[w] -= 1
            break
        prev[w] = 2**64 - 1
    return np.random.Philox(key=np.array(key, np.uint64), counter=np.array(prev, np.uint64))


@pytest.mark.parametrize("seed,lig,phase,gen", [(0, 0, 1, 0), (2**63 + 11, 99_999, 3, 199),
                                                (7, 12_345, 4, 57)])
def test_oracle_stream_pinned_to_numpy(seed, lig, phase, gen):
    """The oracle's counter map, uniform and integer transforms against numpy itself:
    word (idx, slot) = Philox(key=(seed, lig)) block (slot//4, idx, gen, phase) [slot%4];
    uniform = Generator.random on that block; integer = floor(w * n / 2^64)."""
    n_idx, n_slot = 64, 12
    words = oracle.rng_words(seed, lig, phase, gen, n_idx, n_slot)
    L = oracle.lib()
    L.or_rng_uniform.restype = ctypes.c_double
    L.or_rng_uniform.argtypes = [ctypes.c_uint64]
    L.or_rng_below.restype = ctypes.c_uint64
    L.or_rng_below.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    for idx in range(0, n_idx, 7):
        for blk in range(n_slot // 4):
            ctr = (blk, idx, gen, phase)
            raw = _numpy_philox_at((seed, lig), ctr).random_raw(4)
            np.testing.assert_array_equal(words[idx, 4 * blk:4 * blk + 4], raw)
            u = np.random.Generator(_numpy_philox_at((seed, lig), ctr)).random(4)
            got = np.array([L.or_rng_uniform(int(w)) for w in raw])
            np.testing.assert_array_equal(got, u)
            for n in (2, 100, 257, 8192):
                assert [L.or_rng_below(int(w), n) for w in raw] == [(int(w) * n) >> 64 for w in raw]


def test_oracle_normals_distribution():
    """1e5 Box-Muller normals of the oracle stream: N(0, 1) by Kolmogorov-Smirnov."""
    from scipy import stats

    z = oracle.rng_normals(5, 77, 4, 3, 25_000, 4).ravel()
    assert stats.kstest(z, "norm").pvalue > 1e-3
    assert abs(z.mean()) < 0.015 and abs(z.std() - 1.0) < 0.01


# --- mirror validation / formats --------------------------------------------------------
def test_gaconfig_invariants():
    assert GaConfig().population_size == 100 and GaConfig().generations == 1000
    for bad in (dict(population_size=1), dict(elitism_count=100, population_size=100),
                dict(crossover_rate=1.5), dict(tournament_size=0), dict(generations=-1)):
        with pytest.raises(ValueError):
            GaConfig(**bad)


def test_decode_genotype_errors():
    from paper_2509_12232_b200.pose import decode_genotype

    topo = fx.pop_case("rigid")["topo"]
    with pytest.raises(ValueError, match="does not match"):
        decode_genotype(np.zeros(8), topo)
    with pytest.raises(ValueError, match="all zero"):
        decode_genotype(np.zeros(7), topo)
    with pytest.raises(ValueError, match="non-finite"):
        decode_genotype(np.array([0, 0, 0, 1.0, 0, 0, np.nan]), topo)


def test_mugd_round_trip_bitwise():
    g = fx.grid_from(fx.load("grids_small"), "b__")
    buf = io.BytesIO()
    gridmaps.write_grid_set(g, buf)
    back = gridmaps.read_grid_set(buf.getvalue())
    assert list(back.maps) == list(g.maps)
    for k in g.maps:
        assert np.array_equal(back.maps[k].view(np.uint32), g.maps[k].view(np.uint32))
    with pytest.raises(gridmaps.GridFormatError, match="bad magic"):
        gridmaps.read_grid_set(b"XXXX" + buf.getvalue()[4:])
    with pytest.raises(gridmaps.GridFormatError, match="trailing"):
        gridmaps.read_grid_set(buf.getvalue() + b"\0")


def test_trilinear_lookup_exact_at_nodes():
    g = fx.grid_from(fx.load("golden_case"))  # 17^3 at 0.5 A: dyadic, nodes exact
    m = g.maps["C"]
    s = g.spec
    for node in [(0, 0, 0), (3, 5, 2), (16, 16, 16)]:
        p = [s.origin[k] + node[k] * s.spacing for k in range(3)]
        assert gridmaps.trilinear_lookup(m, s, p) == float(m[node])


def test_prepare_context_errors():
    from paper_2509_12232_b200.context import prepare_context

    c = fx.pop_case("cfg0")
    maps = {k: v for k, v in c["grid"].maps.items() if k != "HD"}
    with pytest.raises(ValueError, match="no map for ligand atom type"):
        prepare_context(c["topo"], gridmaps.GridMapSet(c["grid"].spec, maps))
    maps = {k: v for k, v in c["grid"].maps.items() if k != chem.ELEC_LABEL}
    with pytest.raises(ValueError, match="missing the '@elec' map"):
        prepare_context(c["topo"], gridmaps.GridMapSet(c["grid"].spec, maps))


def test_ring_bond_not_rotatable():
    t = topology.LigandTopology(np.zeros((3, 3), np.float32), np.zeros(3, np.int32),
                                np.zeros(3, np.float32), np.array([[0, 1], [1, 2], [0, 2]]),
                                (topology.RotatableBond(0, 1, np.empty(0, np.int32)),))
    with pytest.raises(ValueError, match="lies on a ring"):
        topology.build_fragment_masks(t)


def test_bench_records_csv_byte_stable_and_parseable():
    """vd/bench.py:322-341 CSV rules; columns == the reference's BenchRecord fields."""
    from paper_2509_12232_b200 import benchrecords as br

    fl, by = br.modeled_work(608, 40, 256, 200)
    assert fl == 256 * 200 * (32 * 608 + 107 * 40)
    recs = [br.make_record("cfg2", "cuda", [2.0, 1.0, 1.1, 0.9], 10, fl, by, warmup_discard=1),
            br.make_record("cfg2", "reference", [500.0, 400.0], 10, fl, by)]
    br.fill_speedups(recs)
    assert recs[0].speedup_vs_reference == pytest.approx(450.0 / 1.0)
    a = br.emit_csv(recs)
    b = br.emit_csv(list(reversed(recs)))
    assert a == b and a.splitlines()[0].split(",") == br.BENCH_CSV_COLUMNS
    assert br.BENCH_CSV_COLUMNS == ["scenario", "backend", "threads", "mean_ms", "stddev_ms", "cv",
                                    "ligands_per_s", "modeled_flops", "modeled_bytes",
                                    "modeled_ai", "speedup_vs_reference", "n_samples",
                                    "lane_utilization", "status"]
    back = br.parse_csv(a)
    assert br.emit_csv(back) == a


# --- bench.py launcher (the driver's N-GPU contract) ------------------------------------
def test_bench_self_launches_gpus_ranks_gloo():
    """`python bench.py --gpus 2` without torchrun starts 2 ranks through
    torch.distributed.run; every rank joins one group and rank 0 prints n_gpus == 2."""
    import json
    import subprocess
    import sys

    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                        "--launch-check"], capture_output=True, text=True, env=env, timeout=240)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["max_over_ranks"] == 2.0 and d["screen_ligands"] == 100000
    bad = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                          "--launch-check"], capture_output=True, text=True,
                         env={**env, "WORLD_SIZE": "1"}, timeout=120)
    assert bad.returncode != 0 and "WORLD_SIZE=1" in bad.stderr
