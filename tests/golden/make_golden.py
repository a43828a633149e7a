"""Generate the parity fixtures in tests/golden/ by running the REFERENCE.

Run here (the reference exists only in this container, never on the GPU box):

    python tests/golden/make_golden.py

It imports vecdock from /root/reference/pkg/src read-only (NUMBA_CACHE_DIR is
pointed outside the reference tree so numba's cache=True kernels never write
into it), feeds it inputs built by this repo's own generators, and stores the
reference's outputs: per-pose inter64/intra64/total32 from the `simd`
backend (the fastest CPU path, bitwise equal to `reference`/`scalar` per
pkg/test_output.txt:228), poses from pose.pose_population, scoring contexts
from scoring.prepare_context, pair lists / fragment masks from vecdock.model,
grid maps from grids.build_grid_maps, and raw numpy Philox blocks.
"""

from __future__ import annotations

import json
import math
import os
import sys
import tempfile
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "vd_numba_cache"))
REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
sys.path.insert(0, str(REF_SRC))
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from vecdock import grids as rgrids  # noqa: E402
from vecdock import io_formats as rio  # noqa: E402
from vecdock import model as rmodel  # noqa: E402
from vecdock import scoring as rscoring  # noqa: E402
from vecdock.pose import pose_population as rpose_population  # noqa: E402

from paper_2509_12232_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent
TABLE = rio.default_parameter_table()


def ref_topology(topo):
    """Convert a mirror LigandTopology into the reference's record type."""
    return rmodel.LigandTopology(
        coords0=topo.coords0, type_index=topo.type_index, charge=topo.charge, bonds=topo.bonds,
        rotatable_bonds=tuple(rmodel.RotatableBond(rb.axis_a, rb.axis_b, rb.fragment)
                              for rb in topo.rotatable_bonds))


def topo_arrays(prefix, topo):
    rb = topo.rotatable_bonds
    frag = [np.asarray(r.fragment, np.int32) for r in rb]
    return {
        f"{prefix}coords0": topo.coords0, f"{prefix}type_index": topo.type_index,
        f"{prefix}charge": topo.charge, f"{prefix}bonds": topo.bonds,
        f"{prefix}axes": np.array([[r.axis_a, r.axis_b] for r in rb], np.int32).reshape(-1, 2),
        f"{prefix}frag_start": np.concatenate([[0], np.cumsum([f.size for f in frag])]).astype(np.int32),
        f"{prefix}frag_index": np.concatenate(frag).astype(np.int32) if frag else np.empty(0, np.int32),
    }


CTX_FIELDS = ("atom_slot", "charge", "desolv_factor", "box_lo", "box_hi", "pair_i", "pair_j",
              "pair_a", "pair_b", "pair_hb", "pair_qq", "pair_desolv", "pose_centered0",
              "frag_index", "frag_start", "frag_axis_a", "frag_axis_b")


def ctx_arrays(prefix, ctx):
    d = {f"{prefix}ctx_{f}": np.asarray(getattr(ctx, f)) for f in CTX_FIELDS}
    d[f"{prefix}ctx_torsional32"] = np.float32(ctx.torsional32)
    d[f"{prefix}ctx_map_slots"] = np.int32(ctx.map_stack.shape[0])
    return d


def grid_arrays(prefix, gset):
    labels = list(gset.maps)
    return {
        f"{prefix}grid_labels": np.array(labels),
        f"{prefix}grid_maps": np.stack([gset.maps[l] for l in labels]).astype(np.float32),
        f"{prefix}grid_origin": np.array(gset.spec.origin, np.float64),
        f"{prefix}grid_spacing": np.float64(gset.spec.spacing),
        f"{prefix}grid_dims": np.array(gset.spec.dims, np.int32),
    }


def protein_arrays(prefix, p):
    return {f"{prefix}prot_coords": p.coords, f"{prefix}prot_type": p.type_index,
            f"{prefix}prot_charge": p.charge}


def gene_batch(rng, n, T, lo, hi, margin=2.0):
    t = rng.uniform(np.asarray(lo) - margin, np.asarray(hi) + margin, (n, 3))
    q = rng.normal(size=(n, 4))
    th = rng.uniform(-math.pi, math.pi, (n, T))
    g = np.concatenate([t, q, th], axis=1)
    # edge rows: identity pose at the box centre, non-unit quaternion, far outside,
    # torsions beyond +-pi, a pose exactly at the lower box corner
    c = 0.5 * (np.asarray(lo) + np.asarray(hi))
    g[0] = np.concatenate([c, [1.0, 0, 0, 0], np.zeros(T)])
    g[1] = np.concatenate([c, [3.0, -1.0, 0.5, 2.0], np.full(T, 0.7)])
    g[2] = np.concatenate([np.asarray(hi) + 25.0, [0.2, 0.9, -0.3, 0.1], np.full(T, -2.5)])
    g[3] = np.concatenate([c, [0.5, 0.5, 0.5, 0.5], np.linspace(-7.0, 9.0, T)])
    g[4] = np.concatenate([np.asarray(lo), [1.0, 0, 0, 0], np.zeros(T)])
    return np.ascontiguousarray(g)


def make_golden_case():
    golden = json.loads((REF_TESTS / "data" / "golden_score.json").read_text())
    sys.path.insert(0, str(REF_TESTS))
    from conftest import make_pocket_protein  # the reference's own fixture helper

    protein = make_pocket_protein(golden["protein"]["seed"], golden["protein"]["n_atoms"],
                                  golden["protein"]["shell_radius"], table=TABLE)
    spec = rgrids.GridSpec.centered(golden["grid"]["center"], golden["grid"]["dims"],
                                    golden["grid"]["spacing"])
    gset = rgrids.build_grid_maps(protein, spec, probe_types=TABLE.labels, table=TABLE)
    lig = rio.generate_synthetic_ligand(golden["ligand"]["seed"], golden["ligand"]["n_atoms"],
                                        golden["ligand"]["n_torsions"])
    genes = np.array(golden["genotype"], np.float64)
    bd = rscoring.score_pose(lig, genes, gset, backend="simd", table=TABLE)
    ctx = rscoring.prepare_context(lig, gset, table=TABLE)
    d = {}
    d.update(topo_arrays("", lig))
    d.update(protein_arrays("", protein))
    d.update(grid_arrays("", gset))
    d.update(ctx_arrays("", ctx))
    d["genotype"] = genes
    d["expected"] = np.array([golden["expected"][k] for k in ("inter", "intra", "torsional",
                                                              "total")], np.float64)
    d["ref_breakdown"] = np.array([bd.inter, bd.intra, bd.torsional, bd.total], np.float64)
    d["atoms_outside_box"] = np.int32(golden["atoms_outside_box"])
    np.savez_compressed(OUT / "golden_case.npz", **d)
    print("golden_case", bd)


def make_pop_cases():
    """Population scoring fixtures on one shared grid (mirror generators as inputs)."""
    protein = synth.make_protein(77, 700, half_extent=14.0, pocket_radius=7.0)
    rprot = rmodel.Protein(protein.coords, protein.type_index, protein.charge)
    spec = rgrids.GridSpec.centered((0.0, 0.0, 0.0), (21, 21, 21), 0.7)
    probes = TABLE.labels
    gset = rgrids.build_grid_maps(rprot, spec, probe_types=probes, table=TABLE)
    ligands = {
        "cfg0": synth.make_ligand(0, 24, 8, 6),
        "cfg1": synth.make_ligand(1, 30, 10, 8),
        "rigid": synth.make_ligand(2, 16, 5, 0),
        "refgen": None,
        "big": synth.make_ligand(4, 96, 32, 32),
    }
    rng = np.random.default_rng(20251020)
    d = {}
    d.update(protein_arrays("", protein))
    d.update(grid_arrays("", gset))
    names = []
    for name, topo in ligands.items():
        if topo is None:
            rtopo = rio.generate_synthetic_ligand(31, 30, 5)
        else:
            rtopo = ref_topology(topo)
        ctx = rscoring.prepare_context(rtopo, gset, table=TABLE)
        n = 48 if name == "big" else 256
        genes = gene_batch(rng, n, rtopo.n_torsions, spec.origin, spec.upper)
        inter, intra, total = rscoring.score_population(rtopo, genes, ctx, backend="simd")
        poses = rpose_population(rtopo, genes[:32])
        p = f"{name}__"
        d.update(topo_arrays(p, rtopo))
        d.update(ctx_arrays(p, ctx))
        d[p + "genes"] = genes
        d[p + "inter"] = inter
        d[p + "intra"] = intra
        d[p + "total"] = total
        d[p + "poses"] = poses
        names.append(name)
        print(name, rtopo.n_atoms, rtopo.n_torsions, ctx.n_pairs,
              "total range", float(total.min()), float(total.max()))
    d["names"] = np.array(names)
    np.savez_compressed(OUT / "pop_cases.npz", **d)


def make_pairlists():
    """Pair lists + fragment masks on random trees (test_acceptance.py:121-157 shape)."""
    rng = np.random.default_rng(6)
    spec = rgrids.GridSpec.centered((0, 0, 0), (3, 3, 3), 1.0)
    zero = np.zeros(spec.dims, np.float32)
    gset = rgrids.GridMapSet(spec, {l: zero for l in TABLE.labels} | {
        rgrids.ELEC_LABEL: zero, rgrids.DESOLV_LABEL: zero})
    d = {}
    for trial in range(60):
        n = int(rng.integers(2, 29))
        parents = [int(rng.integers(0, k)) for k in range(1, n)]
        bonds = np.array([[p, k + 1] for k, p in enumerate(parents)], np.int32).reshape(-1, 2)
        probe = rmodel.LigandTopology(
            coords0=rng.uniform(-4, 4, (3, n)).astype(np.float32),
            type_index=rng.integers(0, len(TABLE), n).astype(np.int32),
            charge=rng.uniform(-0.5, 0.5, n).astype(np.float32),
            bonds=bonds,
            rotatable_bonds=tuple(rmodel.RotatableBond(int(a), int(b), np.empty(0, np.int32))
                                  for a, b in bonds.tolist()))
        masks = rmodel.build_fragment_masks(probe)
        topo = rmodel.LigandTopology(
            probe.coords0, probe.type_index, probe.charge, probe.bonds,
            tuple(rmodel.RotatableBond(r.axis_a, r.axis_b, m)
                  for r, m in zip(probe.rotatable_bonds, masks)))
        ctx = rscoring.prepare_context(topo, gset, table=TABLE)
        p = f"t{trial}__"
        d.update(topo_arrays(p, topo))
        d.update(ctx_arrays(p, ctx))
        pl = rmodel.build_nonbond_pairlist(topo, TABLE)
        d[p + "pl_a"] = pl.a_coef
        d[p + "pl_b"] = pl.b_coef
        d[p + "pl_qq"] = pl.qq_product
        d[p + "pl_dsl"] = pl.desolv_coeff
    d["n_trials"] = np.int32(60)
    np.savez_compressed(OUT / "pairlists.npz", **d)


def make_philox():
    rows = []
    for key in ((0, 0), (7, 3), (2**63 + 5, 12345), (0, 99), (1 << 40, 1)):
        for counter in ((1, 0, 0, 0), (2, 0, 0, 0), (5, 17, 3, 1), (0, 1, 0, 0),
                        (123456789, 42, 199, 3), (2**64 - 1, 0, 0, 4)):
            prev = list(counter)
            # numpy increments the 256-bit counter before each block: start one below
            for w in range(4):
                if prev[w] > 0:
                    prev[w] -= 1
                    break
                prev[w] = 2**64 - 1
            bg = np.random.Philox(key=np.array(key, np.uint64), counter=np.array(prev, np.uint64))
            raw = bg.random_raw(4)
            rows.append(list(key) + list(counter) + [int(v) for v in raw])
    arr = np.array(rows, dtype=np.uint64)
    # Generator.random() == (raw >> 11) * 2^-53 on the same stream
    g = np.random.Generator(np.random.Philox(key=np.array([7, 3], np.uint64)))
    u = g.random(4)
    raw = np.random.Philox(key=np.array([7, 3], np.uint64)).random_raw(4)
    np.savez_compressed(OUT / "philox.npz", blocks=arr, random_u=u, random_raw=raw)


def make_grids_small():
    sys.path.insert(0, str(REF_TESTS))
    from conftest import make_pocket_protein, make_protein
    from vecdock.energy import TermWeights

    d = {}
    a = make_protein(3, 5, extent=2.0, table=TABLE)
    spec_a = rgrids.GridSpec.centered((0.0, 0.0, 0.0), (8, 8, 8), 0.6)
    ga = rgrids.build_grid_maps(a, spec_a, ["C", "OA", "HD"], TermWeights(), TABLE)
    d.update(protein_arrays("a__", a))
    d.update(grid_arrays("a__", ga))
    b = make_pocket_protein(41, 50, radius=5.5, table=TABLE)
    spec_b = rgrids.GridSpec.centered((0.0, 0.0, 0.0), (16, 16, 16), 0.55)
    gb = rgrids.build_grid_maps(b, spec_b, TABLE.labels, TermWeights(), TABLE)
    d.update(protein_arrays("b__", b))
    d.update(grid_arrays("b__", gb))
    np.savez_compressed(OUT / "grids_small.npz", **d)


def make_mugd():
    """MUGD streams written by the REFERENCE's write_grid_set (vd/grids.py:232-258), with
    the maps they hold: the grids_small 'b' set (16^3 x 9 maps, built by the reference) and
    a random non-cubic one (13 x 7 x 37, 3 maps) for the device transpose's edges."""
    sys.path.insert(0, str(REF_TESTS))
    from conftest import make_pocket_protein

    b = make_pocket_protein(41, 50, radius=5.5, table=TABLE)
    spec_b = rgrids.GridSpec.centered((0.0, 0.0, 0.0), (16, 16, 16), 0.55)
    gb = rgrids.build_grid_maps(b, spec_b, TABLE.labels, table=TABLE)
    rgrids.write_grid_set(gb, OUT / "ref_grid_b.mugd")
    rng = np.random.default_rng(77)
    spec_r = rgrids.GridSpec((-1.25, 0.5, 3.0), 0.375, (13, 7, 37))
    maps_r = {l: rng.normal(0, 5, spec_r.dims).astype(np.float32) for l in ("C", "@elec", "@desolv")}
    gr = rgrids.GridMapSet(spec=spec_r, maps=maps_r)
    rgrids.write_grid_set(gr, OUT / "ref_grid_odd.mugd")
    d = {}
    for tag, g in (("b", gb), ("odd", gr)):
        d[f"{tag}__labels"] = np.array(list(g.maps))
        d[f"{tag}__stack"] = np.stack([g.maps[l] for l in g.maps]).astype(np.float32)
        d[f"{tag}__origin"] = np.array(g.spec.origin)
        d[f"{tag}__spacing"] = np.float64(g.spec.spacing)
        d[f"{tag}__dims"] = np.array(g.spec.dims)
    np.savez_compressed(OUT / "mugd_cases.npz", **d)


if __name__ == "__main__":
    make_mugd()
    make_golden_case()
    make_pop_cases()
    make_pairlists()
    make_philox()
    make_grids_small()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
