"""Rebuild mirror records from the reference-generated fixtures in tests/golden/."""

from __future__ import annotations

from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2509_12232_b200 import chem, context, gridmaps, topology

GOLDEN = Path(__file__).resolve().parent / "golden"
TABLE = chem.default_parameter_table()


@lru_cache(maxsize=None)
def load(name: str):
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def topo_from(d, p=""):
    axes = d[p + "axes"]
    fs, fi = d[p + "frag_start"], d[p + "frag_index"]
    rbs = tuple(topology.RotatableBond(int(a), int(b), fi[fs[k]:fs[k + 1]].astype(np.int32))
                for k, (a, b) in enumerate(axes))
    return topology.LigandTopology(d[p + "coords0"], d[p + "type_index"], d[p + "charge"],
                                   d[p + "bonds"], rbs)


def protein_from(d, p=""):
    return topology.Protein(d[p + "prot_coords"], d[p + "prot_type"], d[p + "prot_charge"])


def grid_from(d, p=""):
    spec = gridmaps.GridSpec(tuple(d[p + "grid_origin"]), float(d[p + "grid_spacing"]),
                             tuple(int(v) for v in d[p + "grid_dims"]))
    labels = [str(l) for l in d[p + "grid_labels"]]
    return gridmaps.GridMapSet(spec, {l: d[p + "grid_maps"][k] for k, l in enumerate(labels)})


def ref_ctx_arrays(d, p=""):
    pre = p + "ctx_"
    return {k[len(pre):]: d[k] for k in d if k.startswith(pre)}


def golden_case():
    d = load("golden_case")
    topo = topo_from(d)
    gset = grid_from(d)
    ctx = context.prepare_context(topo, gset, table=TABLE)
    return d, topo, gset, ctx


def pop_case(name: str):
    d = load("pop_cases")
    p = f"{name}__"
    topo = topo_from(d, p)
    gset = grid_from(d)
    ctx = context.prepare_context(topo, gset, table=TABLE)
    return {
        "topo": topo, "grid": gset, "ctx": ctx, "genes": d[p + "genes"],
        "inter": d[p + "inter"], "intra": d[p + "intra"], "total": d[p + "total"],
        "poses": d[p + "poses"], "ref_ctx": ref_ctx_arrays(d, p),
    }


POP_NAMES = ("cfg0", "cfg1", "rigid", "refgen", "big")


def within_tol(got, want, rel=1e-4, abs_=1e-3):
    """North-star rule: |d| <= 1e-3 kcal/mol OR |d|/|E_ref| <= 1e-4 (per element)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    d = np.abs(got - want)
    return (d <= abs_) | (d <= rel * np.abs(want))
