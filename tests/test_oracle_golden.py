"""Pin the CPU oracle and the host-side preparation against the reference.

Every expectation here was produced by the reference itself
(tests/golden/make_golden.py); these tests run on CPU only.
"""

from __future__ import annotations

import numpy as np
import pytest

import fixtures as fx
from oracle import oracle
from paper_2509_12232_b200 import chem, context, topology

CTX_COMPARE = ("atom_slot", "charge", "desolv_factor", "box_lo", "box_hi", "pair_i", "pair_j",
               "pair_a", "pair_b", "pair_hb", "pair_qq", "pair_desolv", "pose_centered0",
               "frag_index", "frag_start", "frag_axis_a", "frag_axis_b")


def assert_ctx_bitwise(ctx, ref):
    for f in CTX_COMPARE:
        got, want = np.asarray(getattr(ctx, f)), ref[f]
        assert got.dtype == want.dtype or f == "pair_hb", (f, got.dtype, want.dtype)
        np.testing.assert_array_equal(got, want, err_msg=f)
        if got.dtype.kind == "f":
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), f
    assert np.float32(ctx.torsional32) == ref["torsional32"]
    assert len(ctx.map_labels) == int(ref["map_slots"])


class TestGoldenScore:
    """pkg/tests/data/golden_score.json via pkg/tests/test_scoring.py:220-247."""

    def test_context_matches_reference(self):
        d, topo, gset, ctx = fx.golden_case()
        assert_ctx_bitwise(ctx, fx.ref_ctx_arrays(d))

    def test_oracle_matches_reference_and_golden_vector(self):
        d, topo, gset, ctx = fx.golden_case()
        lig = oracle.Ligand(ctx)
        e, a, t = oracle.dock_population(lig, d["genotype"][None, :])
        bd = context.ScoreBreakdown.from_components(e[0], a[0], ctx.torsional32)
        got = np.array([bd.inter, bd.intra, bd.torsional, bd.total])
        # bit-exact against the reference run here ...
        np.testing.assert_array_equal(got, d["ref_breakdown"])
        assert np.float32(t[0]) == np.float32(bd.total)
        # ... and the reference's own known-answer vector at its tolerance
        want = d["expected"]
        assert np.all(np.abs(got - want) / np.maximum(1.0, np.abs(want)) < 1e-4)

    def test_atoms_outside_box(self):
        d, topo, gset, ctx = fx.golden_case()
        pose = oracle.pose_population(oracle.Ligand(ctx), d["genotype"][None, :])[0]
        lo, hi = np.asarray(ctx.box_lo), np.asarray(ctx.box_hi)
        outside = ~np.all((pose >= lo[:, None]) & (pose <= hi[:, None]), axis=0)
        assert int(outside.sum()) == int(d["atoms_outside_box"])


@pytest.mark.parametrize("name", fx.POP_NAMES)
class TestPopulationFixtures:
    def test_context_bitwise(self, name):
        c = fx.pop_case(name)
        assert_ctx_bitwise(c["ctx"], c["ref_ctx"])

    def test_poses_bitwise(self, name):
        c = fx.pop_case(name)
        got = oracle.pose_population(oracle.Ligand(c["ctx"]), c["genes"][: len(c["poses"])])
        assert np.array_equal(got.view(np.uint32), c["poses"].view(np.uint32))

    def test_scores_bitwise(self, name):
        c = fx.pop_case(name)
        e, a, t = oracle.dock_population(oracle.Ligand(c["ctx"]), c["genes"], n_threads=2)
        assert np.array_equal(e.view(np.uint64), c["inter"].view(np.uint64))
        assert np.array_equal(a.view(np.uint64), c["intra"].view(np.uint64))
        assert np.array_equal(t.view(np.uint32), c["total"].view(np.uint32))

    def test_score_poses_path(self, name):
        c = fx.pop_case(name)
        lig = oracle.Ligand(c["ctx"])
        e, a = oracle.score_poses(lig, c["poses"])
        n = len(c["poses"])
        assert np.array_equal(e, c["inter"][:n]) and np.array_equal(a, c["intra"][:n])


def test_pairlists_and_masks_bitwise():
    d = fx.load("pairlists")
    gset_labels = chem.default_parameter_table().labels
    for trial in range(int(d["n_trials"])):
        p = f"t{trial}__"
        ref_topo = fx.topo_from(d, p)
        # rebuild fragments with the mirror BFS and compare
        axes = d[p + "axes"]
        mine = topology.with_fragments(
            topology.LigandTopology(ref_topo.coords0, ref_topo.type_index, ref_topo.charge,
                                    ref_topo.bonds), [tuple(a) for a in axes])
        for r_ref, r_mine in zip(ref_topo.rotatable_bonds, mine.rotatable_bonds):
            np.testing.assert_array_equal(r_mine.fragment, r_ref.fragment)
        pl = topology.build_nonbond_pairlist(mine, fx.TABLE)
        for f, k in (("a_coef", "pl_a"), ("b_coef", "pl_b"), ("qq_product", "pl_qq"),
                     ("desolv_coeff", "pl_dsl")):
            got = getattr(pl, f)
            assert np.array_equal(got.view(np.uint32), d[p + k].view(np.uint32)), (trial, f)
        np.testing.assert_array_equal(pl.i, d[p + "ctx_pair_i"])
        np.testing.assert_array_equal(pl.j, d[p + "ctx_pair_j"])
        z = np.zeros((3, 3, 3), np.float32)
        from paper_2509_12232_b200 import gridmaps

        gset = gridmaps.GridMapSet(gridmaps.GridSpec.centered((0, 0, 0), (3, 3, 3), 1.0),
                                   {l: z for l in gset_labels + [chem.ELEC_LABEL, chem.DESOLV_LABEL]})
        ctx = context.prepare_context(mine, gset, table=fx.TABLE)
        assert_ctx_bitwise(ctx, fx.ref_ctx_arrays(d, p))


def test_philox_matches_numpy():
    d = fx.load("philox")
    for row in d["blocks"]:
        key, counter, want = row[:2], row[2:6], row[6:]
        got = oracle.philox_block(counter, key)
        np.testing.assert_array_equal(got, want)
    # Generator.random() == (raw >> 11) * 2^-53 (the uniform transform of or_rng.c and vd_rng.h)
    u = (d["random_raw"] >> np.uint64(11)).astype(np.float64) * 2.0**-53
    np.testing.assert_array_equal(u, d["random_u"])


@pytest.mark.parametrize("case", ["a", "b"])
def test_grid_builder_oracle_vs_reference(case):
    d = fx.load("grids_small")
    p = f"{case}__"
    prot = fx.protein_from(d, p)
    gset = fx.grid_from(d, p)
    labels = [str(l) for l in d[p + "grid_labels"]]
    probes = [l for l in labels if not l.startswith("@")]
    maps = oracle.build_grid(prot, gset.spec.origin, gset.spec.spacing, gset.spec.dims, probes,
                             chem.TermWeights(), fx.TABLE, n_threads=2)
    want = d[p + "grid_maps"]
    order = probes + [chem.ELEC_LABEL, chem.DESOLV_LABEL]
    for k, l in enumerate(order):
        w = want[labels.index(l)].astype(np.float64)
        g = maps[k].astype(np.float64)
        rel = np.abs(g - w) / np.maximum(np.abs(w), 1e-4)
        assert rel.max() < 1e-6, (l, rel.max())
