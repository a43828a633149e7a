"""GPU parity: the CUDA scoring path (through the C-ABI) against the reference
fixtures and the CPU oracle.  Restates the reference's scoring contract tests
(pkg/tests/test_scoring.py) for the `cuda` backend.

Tolerances: EXACT mode reproduces the reference's canonical sequences and
must agree to 1e-6 relative (in practice bit-for-bit); FAST mode must meet
the north-star rule |d| <= 1e-3 kcal/mol or |d|/|E| <= 1e-4 per pose.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import fixtures as fx
from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    from paper_2509_12232_b200.backend import CudaBackend

    return {"fast": CudaBackend(mode="fast", device=0), "exact": CudaBackend(mode="exact", device=0)}


def test_native_library_is_the_one_loaded():
    from paper_2509_12232_b200 import _abi

    lib = _abi.lib()
    assert lib._name.endswith("libvdb200.so")
    assert _abi.launches() >= 0


@pytest.mark.parametrize("name", fx.POP_NAMES)
def test_poses_bitwise_vs_reference(cuda, name):
    c = fx.pop_case(name)
    got = cuda["exact"].pose_population(c["genes"][: len(c["poses"])], c["ctx"])
    assert np.array_equal(got.view(np.uint32), c["poses"].view(np.uint32))


@pytest.mark.parametrize("name", fx.POP_NAMES)
def test_exact_mode_matches_reference(cuda, name):
    c = fx.pop_case(name)
    e, a, t = cuda["exact"].score_population_arrays(c["genes"], c["ctx"])
    for got, want in ((e, c["inter"]), (a, c["intra"]), (t.astype(np.float64), c["total"])):
        rel = np.abs(got - want) / np.maximum(1.0, np.abs(want))
        assert rel.max() <= 1e-6, rel.max()
    # bit-exact on (nearly) every pose: only libm ulp differences may flip a rounding
    assert np.mean(t.view(np.uint32) == c["total"].view(np.uint32)) >= 0.99


@pytest.mark.parametrize("name", fx.POP_NAMES)
def test_fast_mode_within_north_star_tolerance(cuda, name):
    c = fx.pop_case(name)
    e, a, t = cuda["fast"].score_population_arrays(c["genes"], c["ctx"])
    assert fx.within_tol(t, c["total"]).all()
    assert fx.within_tol(e, c["inter"]).all()
    assert fx.within_tol(a, c["intra"]).all()


def test_golden_vector(cuda):
    d, topo, gset, ctx = fx.golden_case()
    from paper_2509_12232_b200 import backend

    want = d["expected"]
    for mode in ("fast", "exact"):
        bd = backend.score_pose(topo, d["genotype"], gset, backend=cuda[mode], context=ctx)
        got = np.array([bd.inter, bd.intra, bd.torsional, bd.total])
        assert np.all(np.abs(got - want) / np.maximum(1.0, np.abs(want)) < 1e-4), (mode, got)


def test_score_poses_path_matches_fixture(cuda):
    c = fx.pop_case("cfg0")
    e, a = cuda["exact"].score_many(c["poses"], c["ctx"])
    n = len(c["poses"])
    np.testing.assert_allclose(e, c["inter"][:n], rtol=1e-6)
    np.testing.assert_allclose(a, c["intra"][:n], rtol=1e-6)


def _node_fixture():
    from paper_2509_12232_b200 import chem, gridmaps, topology

    rng = np.random.default_rng(7)
    spec = gridmaps.GridSpec(origin=(-2.0, -2.0, -2.0), spacing=0.5, dims=(9, 9, 9))
    custom = chem.parse_parameter_table("C 4.0 0.15 33.51 0.0 0\n")
    maps = {"C": rng.uniform(-3, 3, spec.dims).astype(np.float32),
            chem.ELEC_LABEL: rng.uniform(-3, 3, spec.dims).astype(np.float32),
            chem.DESOLV_LABEL: rng.uniform(-3, 3, spec.dims).astype(np.float32)}
    gset = gridmaps.GridMapSet(spec, maps)
    nodes = [(0, 0, 0), (3, 7, 2), (8, 8, 8), (4, 1, 6)]
    coords = np.array([[spec.origin[k] + n[k] * spec.spacing for n in nodes] for k in range(3)],
                      np.float32)
    topo = topology.LigandTopology(coords, np.zeros(4, np.int32), np.zeros(4, np.float32),
                                   np.array([[k, k + 1] for k in range(3)], np.int32))
    return gset, custom, topo, nodes


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_atoms_on_nodes_reproduce_map_values(cuda, mode):
    """pkg/tests/test_scoring.py:48-71 (node-exact, '==')."""
    from paper_2509_12232_b200 import backend

    gset, custom, topo, nodes = _node_fixture()
    got = backend.inter_energy(topo.coords0, topo.type_index, topo.charge, gset,
                               backend=cuda[mode], table=custom)
    want = float(np.float32(sum(float(gset.maps["C"][n]) for n in nodes)))
    assert got == want
    one = backend.inter_energy(topo.coords0[:, :1], topo.type_index[:1], topo.charge[:1], gset,
                               backend=cuda[mode], table=custom)
    assert one == float(gset.maps["C"][nodes[0]])


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_out_of_box_penalty(cuda, mode):
    """pkg/tests/test_scoring.py:73-86."""
    from paper_2509_12232_b200 import backend

    gset, custom, _, _ = _node_fixture()
    coords = np.array([[gset.spec.upper[0] + 2.0], [0.0], [0.0]], np.float32)
    got = backend.inter_energy(coords, np.zeros(1, np.int32), np.zeros(1, np.float32), gset,
                               backend=cuda[mode], table=custom)
    assert got == pytest.approx(1e4 * 3.0, rel=1e-6)


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_intra_empty_and_equilibrium_pair(cuda, mode):
    """pkg/tests/test_scoring.py:101-120."""
    from paper_2509_12232_b200 import backend, chem, topology

    empty = topology.NonbondPairList.empty()
    coords = np.zeros((3, 4), np.float32)
    coords[0] = [0, 1.5, 3.0, 4.5]
    assert backend.intra_energy(coords, empty, backend=cuda[mode]) == 0.0
    custom = chem.parse_parameter_table("C 4.0 0.15 0.0 0.0 0\n")
    c5 = np.zeros((3, 5), np.float32)
    c5[0] = [0.0, 1.0, 2.0, 3.0, 4.0]
    topo = topology.LigandTopology(c5, np.zeros(5, np.int32), np.zeros(5, np.float32),
                                   np.array([[k, k + 1] for k in range(4)], np.int32))
    pl = topology.build_nonbond_pairlist(topo, custom)
    assert pl.pairs() == [(0, 4)]
    w = chem.TermWeights()
    got = backend.intra_energy(topo.coords0, pl, weights=w, backend=cuda[mode])
    assert got == pytest.approx(w.vdw * -0.15, rel=1e-5)


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_constant_landscape_only_torsional(cuda, mode):
    """pkg/tests/test_scoring.py:176-200."""
    from paper_2509_12232_b200 import backend, chem, gridmaps, topology

    custom = chem.parse_parameter_table("C 4.0 0.0 0.0 0.0 0\n")
    spec = gridmaps.GridSpec.centered((0, 0, 0), (9, 9, 9), 1.0)
    z = np.zeros(spec.dims, np.float32)
    gset = gridmaps.GridMapSet(spec, {"C": z, chem.ELEC_LABEL: z, chem.DESOLV_LABEL: z})
    coords = np.zeros((3, 3), np.float32)
    coords[0] = [0.0, 1.0, 2.0]
    topo = topology.LigandTopology(coords, np.zeros(3, np.int32), np.zeros(3, np.float32),
                                   np.array([[0, 1], [1, 2]], np.int32),
                                   (topology.RotatableBond(0, 1, np.array([1, 2], np.int32)),))
    w = chem.TermWeights()
    bd = backend.score_pose(topo, np.array([0, 0, 0, 1.0, 0, 0, 0, 0.4]), gset, weights=w,
                            backend=cuda[mode], table=custom)
    assert bd.inter == 0.0 and bd.intra == 0.0
    assert bd.total == float(np.float32(w.tors * 1))


def test_intra_invariant_under_rigid_change(cuda):
    """pkg/tests/test_scoring.py:202-211 / test_acceptance.py geometry invariants."""
    c = fx.pop_case("cfg1")
    rng = np.random.default_rng(23)
    T = c["ctx"].n_torsions
    tors = rng.uniform(-math.pi, math.pi, T)
    rows = [np.concatenate([rng.uniform(-2, 2, 3), rng.normal(size=4), tors]) for _ in range(16)]
    _, a, _ = cuda["fast"].score_population_arrays(np.array(rows), c["ctx"])
    assert np.max(np.abs(a - a[0]) / max(1.0, abs(a[0]))) < 1e-4


def test_large_batch_vs_oracle_and_pipeline(cuda):
    """300k cfg1-like random poses (crosses the 2^17-pose host pipeline chunk) vs oracle."""
    from paper_2509_12232_b200 import synth

    c = fx.pop_case("cfg1")
    spec = c["grid"].spec
    genes = synth.random_genes(0, 300_000, c["ctx"].n_torsions, spec.origin, spec.upper)
    e, a, t = cuda["fast"].score_population_arrays(genes, c["ctx"])
    sub = slice(0, 300_000, 7)
    we, wa, wt = oracle.dock_population(oracle.Ligand(c["ctx"]), genes[sub], n_threads=0)
    assert fx.within_tol(t[sub], wt).all()
    assert fx.within_tol(e[sub], we).all() and fx.within_tol(a[sub], wa).all()


def test_device_pointers_match_host_pointers(cuda):
    import torch

    c = fx.pop_case("cfg0")
    g = torch.from_numpy(c["genes"]).cuda()
    P = g.shape[0]
    out = (torch.empty(P, dtype=torch.float64, device="cuda"),
           torch.empty(P, dtype=torch.float64, device="cuda"),
           torch.empty(P, dtype=torch.float32, device="cuda"))
    cuda["fast"].score_population_arrays(g, c["ctx"], out=out)
    torch.cuda.synchronize()
    e, a, t = cuda["fast"].score_population_arrays(c["genes"], c["ctx"])
    assert np.array_equal(out[2].cpu().numpy(), t) and np.array_equal(out[0].cpu().numpy(), e)


def test_reference_context_accepted(cuda):
    """A ScoringContext carrying its own map stack (the reference's layout) scores identically."""
    from paper_2509_12232_b200.context import ScoringContext
    import dataclasses

    c = fx.pop_case("refgen")
    ctx = c["ctx"]
    ref_like = dataclasses.replace(ctx, grid_set=None, explicit_stack=ctx.map_stack)
    e1, a1, t1 = cuda["exact"].score_population_arrays(c["genes"], ctx)
    e2, a2, t2 = cuda["exact"].score_population_arrays(c["genes"], ref_like)
    assert np.array_equal(t1, t2) and np.array_equal(e1, e2) and np.array_equal(a1, a2)
    assert isinstance(ref_like, ScoringContext)


@pytest.mark.parametrize("case", ["a", "b"])
def test_grid_builder_vs_reference(case):
    from paper_2509_12232_b200 import chem, gridmaps

    d = fx.load("grids_small")
    p = f"{case}__"
    prot = fx.protein_from(d, p)
    ref = fx.grid_from(d, p)
    probes = [l for l in ref.maps if not l.startswith("@")]
    got = gridmaps.build_grid_maps(prot, ref.spec, probes, chem.TermWeights(), fx.TABLE)
    for label in ref.maps:
        w = ref.maps[label].astype(np.float64)
        g = got.maps[label].astype(np.float64)
        rel = np.abs(g - w) / np.maximum(np.abs(w), 1e-4)
        assert rel.max() < 1e-4, (label, rel.max())


LAYOUTS = {"plain": ("VD_NO_PACK", "1"), "zpair": ("VD_BRICK_BUDGET_MB", "0"),
           "brick": ("VD_BRICK_BUDGET_MB", "100000")}


def _score_with_layout(c, layout, monkeypatch):
    from paper_2509_12232_b200 import gridmaps
    from paper_2509_12232_b200.backend import CudaBackend
    from paper_2509_12232_b200.context import prepare_context

    monkeypatch.setenv(*LAYOUTS[layout])
    g2 = gridmaps.GridMapSet(c["grid"].spec, dict(c["grid"].maps))  # fresh device grid
    ctx = prepare_context(c["topo"], g2)
    return CudaBackend(mode="fast", device=0).score_population_arrays(c["genes"], ctx)


@pytest.mark.parametrize("name", ["cfg1", "big"])
@pytest.mark.parametrize("layout", sorted(LAYOUTS))
def test_fast_mode_every_grid_layout(cuda, name, layout, monkeypatch):
    """Each gather layout -- plain (n_maps, nx, ny, nz) maps (the packed copy would not stay
    L2-resident, e.g. cfg4's 126^3 grid), z-pair type maps (cfg1) and yz-brick type maps
    (cfg2) -- agrees with the reference, and the inter energies are bit-identical across
    layouts (same corner values, same lerp arithmetic, same summation order)."""
    c = fx.pop_case(name)
    e, a, t = _score_with_layout(c, layout, monkeypatch)
    assert fx.within_tol(t, c["total"]).all()
    assert fx.within_tol(e, c["inter"]).all()
    monkeypatch.undo()
    e0, _, _ = _score_with_layout(c, "plain", monkeypatch)
    assert np.array_equal(e.view(np.uint64), e0.view(np.uint64))


@pytest.mark.parametrize("tpp", ["1", "2", "4", "8", "16"])
def test_fast_mode_every_launch_shape(cuda, tpp, monkeypatch):
    """Every threads-per-pose-pair shape gives the same poses and in-tolerance energies."""
    from paper_2509_12232_b200.backend import CudaBackend

    monkeypatch.setenv("VD_TPP", tpp)
    c = fx.pop_case("big")
    b = CudaBackend(mode="fast", device=0)
    e, a, t = b.score_population_arrays(c["genes"], c["ctx"])
    assert fx.within_tol(t, c["total"]).all()


@pytest.mark.parametrize("heavy", [16, 30, 40, 48])
def test_fast_mode_role_split_balance(cuda, heavy):
    """The score kernel's role split hands the last atoms to the pair subs (few pairs per
    atom, e.g. 21 atoms / 129 pairs) or the last pairs to the gather subs (many pairs per
    atom, e.g. 64 atoms / 1,750 resident pairs).  Both hand-overs agree with the oracle."""
    from paper_2509_12232_b200 import synth
    from paper_2509_12232_b200.context import prepare_context

    c = fx.pop_case("cfg1")
    topo = synth.make_ligand(100 + heavy, heavy, heavy // 3, 6)
    ctx = prepare_context(topo, c["grid"])
    spec = c["grid"].spec
    genes = synth.random_genes(heavy, 4096, ctx.n_torsions, spec.origin, spec.upper)
    e, a, t = cuda["fast"].score_population_arrays(genes, ctx)
    we, wa, wt = oracle.dock_population(oracle.Ligand(ctx), genes, n_threads=0)
    assert fx.within_tol(t, wt).all()
    assert fx.within_tol(e, we).all()
    assert fx.within_tol(a, wa).all()


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_alternating_ligand_sizes_reuse_launch_setup(cuda, mode):
    """Launch set-up is cached per kernel shape; a larger ligand after a smaller one of the same
    shape must still get its shared-memory limit (large -> small -> large, host buffers)."""
    big, small = fx.pop_case("cfg1"), fx.pop_case("cfg0")
    first = cuda[mode].score_population_arrays(big["genes"], big["ctx"])
    cuda[mode].score_population_arrays(small["genes"], small["ctx"])
    cuda[mode].score_many(small["poses"], small["ctx"])
    again = cuda[mode].score_population_arrays(big["genes"], big["ctx"])
    for x, y in zip(first, again):
        assert np.array_equal(np.asarray(x), np.asarray(y))


def test_concurrent_threads_different_ligands(cuda):
    """The reference's screen_batch drives one backend from several Python threads
    (vd/screening.py:116-161): concurrent calls on ligands of different sizes must neither
    fail (kernel attributes are process-wide) nor change any result."""
    from concurrent.futures import ThreadPoolExecutor

    cases = [fx.pop_case(n) for n in ("cfg1", "cfg0", "big", "refgen")]
    want = [cuda["fast"].score_population_arrays(c["genes"], c["ctx"]) for c in cases]

    def work(k):
        c = cases[k % len(cases)]
        return k % len(cases), cuda["fast"].score_population_arrays(c["genes"], c["ctx"])

    with ThreadPoolExecutor(max_workers=4) as ex:
        for k, got in ex.map(work, range(24)):
            for x, y in zip(got, want[k]):
                assert np.array_equal(np.asarray(x), np.asarray(y))


def test_reference_contexts_share_deduplicated_device_maps():
    """300 contexts that each carry a private copy of the same map stack (what the
    reference's screen_batch keeps alive, vd/screening.py:195-203) upload the maps once:
    device memory stays flat and every context scores exactly as with the shared grid."""
    import dataclasses

    import torch

    from paper_2509_12232_b200 import hostprep, synth
    from paper_2509_12232_b200.backend import CudaBackend
    from paper_2509_12232_b200.context import prepare_context

    c = fx.pop_case("cfg1")
    gset = c["grid"]
    b = CudaBackend(mode="fast", device=0)
    batch = hostprep.TopologyBatch.synth(2, 0, 300)
    ctxs = []
    free0 = torch.cuda.mem_get_info(0)[0]
    for l in range(len(batch)):
        try:
            ctx = prepare_context(batch.topology(l), gset, table=fx.TABLE)
        except ValueError:
            continue  # type without a map in the small fixture grid
        own = np.array(ctx.map_stack, copy=True)  # a private copy per context
        ref_like = dataclasses.replace(ctx, grid_set=None, explicit_stack=own)
        genes = synth.random_genes(l, 64, ctx.n_torsions, gset.spec.origin, gset.spec.upper)
        got = b.score_population_arrays(genes, ref_like)
        want = b.score_population_arrays(genes, ctx)
        for x, y in zip(got, want):
            assert np.array_equal(x, y)
        ctxs.append(ref_like)
    assert len(ctxs) >= 100
    used = free0 - torch.cuda.mem_get_info(0)[0]
    assert b._pool.n_device_maps() <= len(gset.maps)
    assert used < 256 << 20, f"{used / 2**20:.0f} MiB for {len(ctxs)} contexts"


def test_short_lived_threads_reuse_staging_pipes(cuda):
    """Worker threads that come and go (a fresh pool per screen_batch call) lease staging
    pipelines from one process-wide pool: the count is bounded by the concurrency, not by
    how many threads ever called."""
    import threading

    from paper_2509_12232_b200 import _abi

    c = fx.pop_case("cfg0")
    want = cuda["fast"].score_population_arrays(c["genes"], c["ctx"])
    before = _abi.lib().vd_pipe_count(0)
    for _ in range(10):
        ts = []
        errs = []

        def work():
            got = cuda["fast"].score_population_arrays(c["genes"], c["ctx"])
            if not all(np.array_equal(x, y) for x, y in zip(got, want)):
                errs.append("mismatch")

        for _ in range(3):
            ts.append(threading.Thread(target=work))
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errs
    assert _abi.lib().vd_pipe_count(0) - before <= 3


@pytest.mark.parametrize("tag", ["b", "odd"])
def test_mugd_file_loads_straight_to_device(cuda, tag):
    """A MUGD stream written by the reference's write_grid_set (vd/grids.py:232-258) goes
    file -> pinned staging -> device transpose (csrc/vd_mugd.cu): the device stack equals
    the reference's maps bit for bit, and scoring through the loaded set equals scoring
    through the host-read set."""
    from paper_2509_12232_b200 import gridmaps, synth
    from paper_2509_12232_b200.context import prepare_context

    d = fx.load("mugd_cases")
    path = fx.GOLDEN / f"ref_grid_{tag}.mugd"
    dset = gridmaps.load_grid_set(path)
    stack = dset.device_grid.download()
    assert np.array_equal(stack.view(np.uint32), d[f"{tag}__stack"].view(np.uint32))
    assert list(dset.maps) == [str(l) for l in d[f"{tag}__labels"]]
    hset = gridmaps.read_grid_set(path)
    assert dset.spec == hset.spec
    if tag == "b":
        topo = synth.make_ligand(5, 18, 6, 4)
        genes = synth.random_genes(9, 2048, topo.n_torsions, hset.spec.origin, hset.spec.upper)
        a = cuda["exact"].score_population_arrays(genes, prepare_context(topo, dset, table=fx.TABLE))
        b = cuda["exact"].score_population_arrays(genes, prepare_context(topo, hset, table=fx.TABLE))
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
