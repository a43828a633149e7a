"""The reference's own entry points driven through the backend seam, on CPU.

Imports the REFERENCE package from /root/reference (present in the build container only;
skipped elsewhere), registers `CudaBackend` into its registry with
`register_reference_backend` (vd/scoring/__init__.py:210-247), and runs the reference's
`score_population` (:330-346), `score_pose` (:317-327), `ga.dock` (vd/ga.py:180-235) and
`screen_batch` with 3 worker threads (vd/screening.py:165-244).

No GPU here, so the native layer under the backend is a stub: `_abi`'s grid, ligand-set
and score functions are replaced by Python fakes that score with the CPU oracle
(bit-exact with the reference's simd backend, tests/test_oracle_golden.py).  What is under
test is everything above the C-ABI: how CudaBackend turns reference ScoringContexts into
device grids and ligand records (map-slot -> grid-map indices, elec/desolv indices, content
deduplication of the per-context map stacks), its caching under concurrent workers, and the
protocol members the reference calls.  Every result must equal the reference's simd
backend bit for bit.
"""

from __future__ import annotations

import os
import sys
import tempfile
import threading
import types
from pathlib import Path

import numpy as np
import pytest

REF_SRC = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF_SRC.exists(), reason="reference tree not present")


@pytest.fixture(scope="module")
def ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "vd_numba_cache"))
    sys.path.insert(0, str(REF_SRC))
    from vecdock import ga, grids, io_formats, model, scoring, screening

    table = io_formats.default_parameter_table()
    rng = np.random.default_rng(8)
    n = 300
    coords = rng.uniform(-9, 9, (3, n)).astype(np.float32)
    keep = np.linalg.norm(coords, axis=0) > 5.0
    labels = ["C", "N", "OA", "SA", "HD"]
    types_ = np.array([table.index_of(labels[k]) for k in rng.integers(0, 5, n)], np.int32)
    prot = model.Protein(coords=np.ascontiguousarray(coords[:, keep]), type_index=types_[keep],
                         charge=rng.uniform(-0.5, 0.5, int(keep.sum())).astype(np.float32))
    spec = grids.GridSpec.centered((0.0, 0.0, 0.0), (17, 17, 17), 0.5)
    gset = grids.build_grid_maps(prot, spec, ["C", "A", "N", "NA", "OA", "SA", "HD"], table=table)
    return types.SimpleNamespace(ga=ga, grids=grids, io=io_formats, model=model, scoring=scoring,
                                 screening=screening, table=table, gset=gset)


def _ref_topology(ref, topo):
    return ref.model.LigandTopology(
        coords0=topo.coords0, type_index=topo.type_index, charge=topo.charge, bonds=topo.bonds,
        rotatable_bonds=tuple(ref.model.RotatableBond(rb.axis_a, rb.axis_b, rb.fragment)
                              for rb in topo.rotatable_bonds))


class _Stub:
    """The C-ABI layer under CudaBackend, restated on the CPU oracle (test-only)."""

    def __init__(self):
        self.grids_made = 0
        self.sets_made = 0
        self.lock = threading.Lock()

    def install(self, monkeypatch):
        from paper_2509_12232_b200 import _abi

        stub = self

        class FakeGrid:
            def __init__(self, stack, lo, hi, spacing, labels=None):
                with stub.lock:
                    stub.grids_made += 1
                self.stack = np.ascontiguousarray(stack, np.float32)
                self.n_maps = self.stack.shape[0]
                self.labels = labels
                self.layout = "plain"

        class FakeSet:
            def __init__(self, contexts, atom_maps, elec, desolv):
                with stub.lock:
                    stub.sets_made += 1
                self.contexts, self.atom_maps = contexts, atom_maps
                self.elec, self.desolv = elec, desolv
                self.n_atoms = np.array([c.n_atoms for c in contexts])

        def ligand(grid, ligs, lig):
            from oracle import oracle

            view = ligs.contexts[lig]
            geo = view._c  # the reference context behind the padded view
            c = types.SimpleNamespace(**{k: getattr(view, k) for k in dir(view)
                                         if not k.startswith("_")})
            for k in ("dims", "box_lo", "box_hi", "spacing"):
                setattr(c, k, getattr(geo, k))
            return oracle.Ligand(c, grid.stack, ligs.atom_maps[lig], ligs.elec, ligs.desolv)

        def score_poses(grid, ligs, lig, poses, inter, intra, mode=0, stream=None):
            from oracle import oracle

            inter[:], intra[:] = oracle.score_poses(ligand(grid, ligs, lig), poses)

        def score_genes(grid, ligs, lig, genes, inter, intra, total, mode=0, stream=None):
            from oracle import oracle

            e, a, t = oracle.dock_population(ligand(grid, ligs, lig), genes)
            inter[:], intra[:] = e, a
            if total is not None:
                total[:] = t

        monkeypatch.setattr(_abi, "lib", lambda: object())
        monkeypatch.setattr(_abi, "ensure_device", lambda device=None: 0)
        monkeypatch.setattr(_abi, "grid_from_stack", FakeGrid)
        monkeypatch.setattr(_abi, "LigandSet", FakeSet)
        monkeypatch.setattr(_abi, "score_genes", score_genes)
        monkeypatch.setattr(_abi, "score_poses", score_poses)


@pytest.fixture
def cuda(ref, monkeypatch):
    from paper_2509_12232_b200.backend import register_reference_backend

    stub = _Stub()
    stub.install(monkeypatch)
    ref.scoring._load_backends()
    saved = dict(ref.scoring._REGISTRY)
    b = register_reference_backend(ref.scoring, "cuda")
    assert "simd" in ref.scoring._REGISTRY and b is ref.scoring.get_backend("cuda")
    yield b, stub
    ref.scoring._REGISTRY.clear()
    ref.scoring._REGISTRY.update(saved)


def _ligand(ref, k, n_tors=5):
    from paper_2509_12232_b200 import synth

    return _ref_topology(ref, synth.make_ligand(100 + k, 14 + k, 5, n_tors))


def test_score_population_and_score_pose_through_the_seam(ref, cuda):
    from paper_2509_12232_b200 import synth

    topo = _ligand(ref, 0)
    ctx = ref.scoring.prepare_context(topo, ref.gset, table=ref.table)
    s = ref.gset.spec
    genes = synth.random_genes(3, 257, topo.n_torsions, s.origin, s.upper)
    got = ref.scoring.score_population(topo, genes, ctx, backend="cuda")
    want = ref.scoring.score_population(topo, genes, ctx, backend="simd")
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
    a = ref.scoring.score_pose(topo, genes[5], ref.gset, backend="cuda", table=ref.table)
    b = ref.scoring.score_pose(topo, genes[5], ref.gset, backend="simd", table=ref.table)
    assert a == b


def test_ga_dock_through_the_seam(ref, cuda):
    topo = _ligand(ref, 1)
    cfg = ref.ga.GaConfig(population_size=24, generations=6, seed=4)
    got = ref.ga.dock(topo, ref.gset, cfg, backend="cuda", table=ref.table)
    want = ref.ga.dock(topo, ref.gset, cfg, backend="simd", table=ref.table)
    assert np.array_equal(got.best_genotype, want.best_genotype)
    assert np.array_equal(got.trace, want.trace) and got.best_score == want.best_score


def test_screen_batch_threads_share_one_deduplicated_grid(ref, cuda):
    b, stub = cuda
    entries = tuple((f"lig{k}", _ligand(ref, k, n_tors=k % 4)) for k in range(8))
    batch = ref.io.LigandBatch(entries=entries, provenance="synthetic")
    ga = ref.ga.GaConfig(population_size=16, generations=3)
    got = ref.screening.screen_batch(batch, ref.gset, ref.screening.ScreenConfig(
        worker_count=3, ga=ga, backend="cuda", global_seed=2), table=ref.table)
    want = ref.screening.screen_batch(batch, ref.gset, ref.screening.ScreenConfig(
        worker_count=1, ga=ga, backend="simd", global_seed=2), table=ref.table)
    for g, w in zip(got, want):
        assert g.error is None and w.error is None
        assert np.array_equal(g.result.best_genotype, w.result.best_genotype)
        assert g.result.best_score == w.result.best_score
    # 8 contexts, each with a private copy of up to 9 maps: only the grid set's distinct
    # maps reach the device, in a handful of grid rebuilds
    assert b._pool.n_device_maps() <= len(ref.gset.maps)
    assert stub.grids_made <= len(ref.gset.maps)
    assert stub.sets_made == len(entries)


def test_prepared_is_single_flight_under_concurrent_workers(ref, cuda):
    b, stub = cuda
    topo = _ligand(ref, 3)
    ctx = ref.scoring.prepare_context(topo, ref.gset, table=ref.table)
    go = threading.Barrier(8)
    out = []

    def worker():
        go.wait()
        out.append(b.prepared(ctx))

    ts = [threading.Thread(target=worker) for _ in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert stub.sets_made == 1
    assert all(o is out[0] for o in out)
