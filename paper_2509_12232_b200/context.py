"""The kernel input record (`ScoringContext`) and its host preparation.

Mirror of vd/scoring/__init__.py:51-207 with the reference's field names so a
context built here and one built by the reference are interchangeable for
`CudaBackend`.  One B200-driven difference: the per-ligand `map_stack`
copy (vd/scoring/__init__.py:158-161, ~18 MB per ligand at 80^3) is built
lazily, only if a CPU consumer asks for it; the device path addresses the
shared, once-uploaded grid through `map_labels` instead.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import chem
from .gridmaps import GridMapSet
from .topology import LigandTopology, NonbondPairList, build_nonbond_pairlist


class BackendUnavailable(RuntimeError):
    """vd/scoring/__init__.py:47-48"""


@dataclass(frozen=True)
class ScoreBreakdown:
    """f32 score parts; total = f32(f32(inter + intra) + tors) (vd/scoring/__init__.py:51-66)."""

    inter: float
    intra: float
    torsional: float
    total: float

    @classmethod
    def from_components(cls, inter64, intra64, torsional32):
        e, a, t = np.float32(inter64), np.float32(intra64), np.float32(torsional32)
        return cls(float(e), float(a), float(t), float(np.float32(np.float32(e + a) + t)))


@dataclass(frozen=True)
class ScoringContext:
    """Weight-folded per-ligand inputs (field set of vd/scoring/__init__.py:69-114)."""

    atom_slot: np.ndarray
    charge: np.ndarray
    desolv_factor: np.ndarray
    box_lo: np.ndarray
    box_hi: np.ndarray
    spacing: np.float32
    dims: tuple
    penalty_scale: np.float32
    pair_i: np.ndarray | None
    pair_j: np.ndarray | None
    pair_a: np.ndarray | None
    pair_b: np.ndarray | None
    pair_hb: np.ndarray | None
    pair_qq: np.ndarray | None
    pair_desolv: np.ndarray | None
    intra_cutoff2: np.float32
    torsional32: np.float32
    n_atoms: int
    pose_centered0: np.ndarray
    frag_index: np.ndarray
    frag_start: np.ndarray
    frag_axis_a: np.ndarray
    frag_axis_b: np.ndarray
    # B200 additions: the shared grid and the label of every stack slot
    grid_set: GridMapSet | None = field(default=None, compare=False, repr=False)
    map_labels: tuple = ()
    explicit_stack: np.ndarray | None = field(default=None, compare=False, repr=False)

    @property
    def map_stack(self) -> np.ndarray:
        if self.explicit_stack is not None:
            return self.explicit_stack
        cached = self.__dict__.get("_stack_cache")
        if cached is None:
            cached = np.ascontiguousarray(
                np.stack([self.grid_set.maps[l] for l in self.map_labels]), dtype=np.float32)
            object.__setattr__(self, "_stack_cache", cached)
        return cached

    @property
    def n_pairs(self) -> int:
        return 0 if self.pair_i is None else int(self.pair_i.shape[0])

    @property
    def n_torsions(self) -> int:
        return int(self.frag_axis_a.shape[0])


def fold_pairs(pairlist: NonbondPairList, weights: chem.TermWeights):
    """Fold term weights into per-pair coefficients (vd/scoring/__init__.py:117-130)."""
    hb = pairlist.is_hbond
    w = np.where(hb, np.float32(weights.hbond), np.float32(weights.vdw))
    cq = np.float32(weights.elec * chem.ELEC_SCALE)
    return (pairlist.i, pairlist.j,
            (w * pairlist.a_coef).astype(np.float32),
            (w * pairlist.b_coef).astype(np.float32),
            hb,
            (cq * pairlist.qq_product).astype(np.float32),
            (np.float32(weights.desolv) * pairlist.desolv_coeff).astype(np.float32))


def prepare_context(topology: LigandTopology, grid_set: GridMapSet, weights=None, table=None,
                    pairlist: NonbondPairList | None = None, intra_cutoff: float | None = None,
                    penalty_scale: float = chem.BOX_PENALTY_SCALE) -> ScoringContext:
    """Scoring context for one topology against one grid set (vd/scoring/__init__.py:133-207)."""
    weights = weights or chem.TermWeights()
    table = table or chem.default_parameter_table()
    if pairlist is None:
        pairlist = build_nonbond_pairlist(topology, table)

    labels = [table[int(t)].type_label for t in topology.type_index]
    needed = sorted(set(labels))
    for label in needed:
        if label not in grid_set.maps:
            raise ValueError(f"grid set has no map for ligand atom type {label!r}")
    for reserved in (chem.ELEC_LABEL, chem.DESOLV_LABEL):
        if reserved not in grid_set.maps:
            raise ValueError(f"grid set is missing the {reserved!r} map")
    slot = {l: k for k, l in enumerate(needed)}

    solpar = table.solpar_array()[topology.type_index]
    dsf = (solpar + np.float32(chem.QASP) * np.abs(topology.charge)).astype(np.float32)
    spec = grid_set.spec
    pi, pj, pa, pb, phb, pqq, pdsl = fold_pairs(pairlist, weights)
    cut2 = np.float32(np.inf) if intra_cutoff is None else np.float32(intra_cutoff * intra_cutoff)

    frags = [np.asarray(rb.fragment, dtype=np.int32) for rb in topology.rotatable_bonds]
    frag_start = np.zeros(len(frags) + 1, dtype=np.int32)
    frag_start[1:] = np.cumsum([f.size for f in frags], dtype=np.int64)
    frag_index = np.concatenate(frags).astype(np.int32) if frags else np.empty(0, np.int32)

    return ScoringContext(
        atom_slot=np.array([slot[l] for l in labels], dtype=np.int32),
        charge=topology.charge,
        desolv_factor=dsf,
        box_lo=np.asarray(spec.origin, dtype=np.float32),
        box_hi=np.asarray(spec.upper, dtype=np.float32),
        spacing=np.float32(spec.spacing),
        dims=spec.dims,
        penalty_scale=np.float32(penalty_scale),
        pair_i=pi, pair_j=pj, pair_a=pa, pair_b=pb, pair_hb=phb, pair_qq=pqq, pair_desolv=pdsl,
        intra_cutoff2=cut2,
        torsional32=np.float32(weights.tors * topology.n_torsions),
        n_atoms=topology.n_atoms,
        pose_centered0=(topology.coords0 - topology.centroid0[:, None]).astype(np.float32),
        frag_index=frag_index,
        frag_start=frag_start,
        frag_axis_a=np.array([rb.axis_a for rb in topology.rotatable_bonds], dtype=np.int32),
        frag_axis_b=np.array([rb.axis_b for rb in topology.rotatable_bonds], dtype=np.int32),
        grid_set=grid_set,
        map_labels=tuple(needed) + (chem.ELEC_LABEL, chem.DESOLV_LABEL),
    )
