"""C++ batched host prep (csrc/vd_host.cpp) == per-ligand prepare_context, bit for bit,
and == the reference's contexts stored in the fixtures."""

from __future__ import annotations

import numpy as np
import pytest

import fixtures as fx
from paper_2509_12232_b200 import chem, hostprep
from paper_2509_12232_b200.context import prepare_context

FIELDS = {"desolv_factor": "desolv_factor", "pair_i": "pair_i", "pair_j": "pair_j",
          "pair_a": "pair_a", "pair_b": "pair_b", "pair_qq": "pair_qq",
          "pair_desolv": "pair_desolv", "frag_index": "frag_index"}


def _compare(batch, ctxs, labels):
    arr = hostprep.prepare_batch(batch, labels, table=fx.TABLE)
    for l, ctx in enumerate(ctxs):
        a0, a1 = batch.atom_start[l], batch.atom_start[l + 1]
        p0, p1 = arr["pair_start"][l], arr["pair_start"][l + 1]
        got_c0 = arr["centered0"][3 * a0:3 * a1].reshape(-1, 3).T
        assert np.array_equal(got_c0.view(np.uint32), ctx.pose_centered0.view(np.uint32)), l
        assert np.array_equal(arr["desolv_factor"][a0:a1].view(np.uint32),
                              np.asarray(ctx.desolv_factor).view(np.uint32))
        for k in ("pair_i", "pair_j"):
            np.testing.assert_array_equal(arr[k][p0:p1], getattr(ctx, k))
        for k in ("pair_a", "pair_b", "pair_qq", "pair_desolv"):
            assert np.array_equal(arr[k][p0:p1].view(np.uint32),
                                  np.asarray(getattr(ctx, k)).view(np.uint32)), (l, k)
        np.testing.assert_array_equal(arr["pair_hb"][p0:p1].astype(bool), ctx.pair_hb)
        t0, t1 = batch.tors_start[l], batch.tors_start[l + 1]
        fl = arr["frag_lo"][t0:t1] - (arr["frag_lo"][t0] if t1 > t0 else 0)
        np.testing.assert_array_equal(fl, ctx.frag_start[:-1])
        if t1 > t0:
            f0, f1 = arr["frag_lo"][t0], arr["frag_hi"][t1 - 1]
            np.testing.assert_array_equal(arr["frag_index"][f0:f1], ctx.frag_index)
        assert arr["torsional32"][l] == ctx.torsional32
        slot_map = [labels.index(x) for x in ctx.map_labels]
        np.testing.assert_array_equal(arr["atom_map"][a0:a1],
                                      np.array(slot_map)[ctx.atom_slot])


def test_fixture_ligands_bitwise():
    cases = [fx.pop_case(n) for n in fx.POP_NAMES]
    topos = [c["topo"] for c in cases]
    ctxs = [c["ctx"] for c in cases]
    labels = list(cases[0]["grid"].maps)
    _compare(hostprep.TopologyBatch.from_topologies(topos), ctxs, labels)


def test_random_trees_bitwise():
    d = fx.load("pairlists")
    topos = [fx.topo_from(d, f"t{k}__") for k in range(int(d["n_trials"]))]
    z = np.zeros((3, 3, 3), np.float32)
    from paper_2509_12232_b200 import gridmaps

    labels = fx.TABLE.labels + [chem.ELEC_LABEL, chem.DESOLV_LABEL]
    g = gridmaps.GridMapSet(gridmaps.GridSpec.centered((0, 0, 0), (3, 3, 3), 1.0),
                            {l: z for l in labels})
    ctxs = [prepare_context(t, g, table=fx.TABLE) for t in topos]
    _compare(hostprep.TopologyBatch.from_topologies(topos), ctxs, labels)


@pytest.mark.parametrize("cfg", [2, 4])
def test_synth_batches_valid_and_bitwise(cfg):
    b = hostprep.TopologyBatch.synth(cfg, 100, 12)
    again = hostprep.TopologyBatch.synth(cfg, 100, 12)
    assert np.array_equal(b.xyz, again.xyz) and np.array_equal(b.axes, again.axes)
    part = hostprep.TopologyBatch.synth(cfg, 105, 3)
    s = slice(b.atom_start[5], b.atom_start[8])
    assert np.array_equal(part.type_index, b.type_index[s])  # index-keyed stream
    n = b.n_atoms
    if cfg == 2:
        heavy = np.rint(n / (4.0 / 3.0))
        assert n.min() >= 21 and n.max() <= 64 and b.n_torsions.max() <= 12
    else:
        assert np.all(n == 128) and np.all(b.n_torsions == 32)
    assert abs(float(b.charge.sum())) < 1e-3 * len(b)
    from paper_2509_12232_b200.topology import build_nonbond_pairlist

    topos = [b.topology(l) for l in range(len(b))]
    for t in topos:  # bonds ~1.5 A (heavy) / 1.0-1.1 A (HD)
        d = np.linalg.norm(t.coords0[:, t.bonds[:, 0]] - t.coords0[:, t.bonds[:, 1]], axis=0)
        assert d.min() > 0.95 and d.max() < 1.65
    labels = fx.TABLE.labels + [chem.ELEC_LABEL, chem.DESOLV_LABEL]
    z = np.zeros((3, 3, 3), np.float32)
    from paper_2509_12232_b200 import gridmaps

    g = gridmaps.GridMapSet(gridmaps.GridSpec.centered((0, 0, 0), (3, 3, 3), 1.0),
                            {l: z for l in labels})
    _compare(b, [prepare_context(t, g, table=fx.TABLE) for t in topos], labels)


def test_oracle_ligands_from_arrays_score_like_contexts():
    """oracle.ligands_from_arrays (the CSR set the device gets, over one shared map stack)
    scores bit-identically to oracle.Ligand over prepare_context's per-ligand stack."""
    from oracle import oracle
    from paper_2509_12232_b200 import gridmaps, synth

    spec = gridmaps.GridSpec.centered((0.0, 0.0, 0.0), (9, 10, 11), 1.5)
    rng = np.random.default_rng(4)
    labels = list(synth.CONFIGS[2].probe_types) + [chem.ELEC_LABEL, chem.DESOLV_LABEL]
    gset = gridmaps.GridMapSet(spec, {l: rng.normal(0, 3, spec.dims).astype(np.float32)
                                      for l in labels})
    batch = hostprep.TopologyBatch.synth(2, 11, 5)
    arrays = hostprep.prepare_batch(batch, labels)
    stack = np.stack([gset.maps[l] for l in labels])
    ligs = oracle.ligands_from_arrays(arrays, stack, spec)
    for l in range(len(batch)):
        ctx = prepare_context(batch.topology(l), gset)
        genes = synth.random_genes(l, 64, ctx.n_torsions, spec.origin, spec.upper)
        got = oracle.dock_population(ligs[l], genes)
        want = oracle.dock_population(oracle.Ligand(ctx), genes)
        for g, w in zip(got, want):
            assert np.array_equal(g, w), l
