"""Ligand / receptor records and the topology-derived host preprocessing.

Host-side mirror of vd/model.py with the same public names and error
behaviour, re-implemented around dense boolean reachability matrices (a
ligand has <= a few hundred atoms, so an n x n bool matrix is tiny and the
whole pair selection is three matrix products instead of n Python BFS runs).

* LigandTopology / RotatableBond / Protein ... vd/model.py:42-125
* NonbondPairList .......................... vd/model.py:128-149
* build_fragment_masks ..................... vd/model.py:174-192
* bond_separation .......................... vd/model.py:195-213
* build_nonbond_pairlist ................... vd/model.py:216-269
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import chem


def _coords3(x) -> np.ndarray:
    a = np.asarray(x, dtype=np.float32)
    if a.ndim != 2 or a.shape[0] != 3:
        raise ValueError(f"coords must have shape (3, n_atoms), got {a.shape}")
    return a


@dataclass(frozen=True)
class RotatableBond:
    """Bond (axis_a, axis_b); `fragment` = sorted atoms on axis_b's side (axis_b included)."""

    axis_a: int
    axis_b: int
    fragment: np.ndarray


@dataclass(frozen=True)
class LigandTopology:
    coords0: np.ndarray          # (3, n) f32 reference conformation
    type_index: np.ndarray       # (n,) i32
    charge: np.ndarray           # (n,) f32
    bonds: np.ndarray            # (B, 2) i32, sorted per row
    rotatable_bonds: tuple = ()

    def __post_init__(self):
        c = _coords3(self.coords0)
        n = c.shape[1]
        t = np.asarray(self.type_index, dtype=np.int32)
        q = np.asarray(self.charge, dtype=np.float32)
        b = np.sort(np.asarray(self.bonds, dtype=np.int32).reshape(-1, 2), axis=1)
        set_ = object.__setattr__
        set_(self, "coords0", c)
        set_(self, "type_index", t)
        set_(self, "charge", q)
        set_(self, "bonds", b)
        set_(self, "rotatable_bonds", tuple(self.rotatable_bonds))
        if n < 1:
            raise ValueError("ligand needs at least one atom")
        if t.shape != (n,) or q.shape != (n,):
            raise ValueError("type_index/charge length must match atom count")
        if b.size and (b.min() < 0 or b.max() >= n):
            raise ValueError(f"bond index out of range for {n} atoms")
        for rb in self.rotatable_bonds:
            if not (0 <= rb.axis_a < n and 0 <= rb.axis_b < n):
                raise ValueError(f"rotatable bond ({rb.axis_a}, {rb.axis_b}) out of range")

    @property
    def n_atoms(self) -> int:
        return self.coords0.shape[1]

    @property
    def n_torsions(self) -> int:
        return len(self.rotatable_bonds)

    @property
    def centroid0(self) -> np.ndarray:
        # fp64 mean rounded once to f32 (vd/model.py:100-103); numpy's mean is
        # used on purpose so the pairwise-summation order is the reference's.
        return self.coords0.mean(axis=1, dtype=np.float64).astype(np.float32)


@dataclass(frozen=True)
class Protein:
    coords: np.ndarray
    type_index: np.ndarray
    charge: np.ndarray

    def __post_init__(self):
        set_ = object.__setattr__
        set_(self, "coords", _coords3(self.coords))
        set_(self, "type_index", np.asarray(self.type_index, dtype=np.int32))
        set_(self, "charge", np.asarray(self.charge, dtype=np.float32))
        if self.coords.shape[1] < 1:
            raise ValueError("receptor needs at least one atom")
        if not np.isfinite(self.coords).all():
            raise ValueError("receptor coordinates must be finite")

    @property
    def n_atoms(self) -> int:
        return self.coords.shape[1]


@dataclass(frozen=True)
class NonbondPairList:
    i: np.ndarray
    j: np.ndarray
    a_coef: np.ndarray
    b_coef: np.ndarray
    is_hbond: np.ndarray
    qq_product: np.ndarray
    desolv_coeff: np.ndarray

    @property
    def n_pairs(self) -> int:
        return int(self.i.shape[0])

    def pairs(self):
        return list(zip(self.i.tolist(), self.j.tolist()))

    @classmethod
    def empty(cls):
        z32 = np.empty(0, np.float32)
        return cls(np.empty(0, np.int32), np.empty(0, np.int32), z32, z32.copy(),
                   np.empty(0, bool), z32.copy(), z32.copy())


def adjacency_matrix(n: int, bonds: np.ndarray) -> np.ndarray:
    adj = np.zeros((n, n), dtype=bool)
    if len(bonds):
        adj[bonds[:, 0], bonds[:, 1]] = True
        adj[bonds[:, 1], bonds[:, 0]] = True
    return adj


def _side_of(adj: np.ndarray, start: int, cut_a: int, cut_b: int) -> np.ndarray:
    """Boolean mask of atoms reachable from `start` with edge (cut_a, cut_b) removed."""
    g = adj.copy()
    g[cut_a, cut_b] = g[cut_b, cut_a] = False
    seen = np.zeros(adj.shape[0], dtype=bool)
    seen[start] = True
    frontier = seen.copy()
    while frontier.any():
        nxt = g[frontier].any(axis=0) & ~seen
        seen |= nxt
        frontier = nxt
    return seen


def build_fragment_masks(topology: LigandTopology):
    """Per rotatable bond: sorted atoms reachable from axis_b without the bond."""
    adj = adjacency_matrix(topology.n_atoms, topology.bonds)
    out = []
    for rb in topology.rotatable_bonds:
        side = _side_of(adj, rb.axis_b, rb.axis_a, rb.axis_b)
        if side[rb.axis_a]:
            raise ValueError(
                f"bond ({rb.axis_a}, {rb.axis_b}) lies on a ring; removing it does not "
                "split the graph, so it is not rotatable")
        out.append(np.flatnonzero(side).astype(np.int32))
    return out


def _hop_distances(n: int, bonds: np.ndarray, max_depth: int) -> np.ndarray:
    """(n, n) int matrix of bond-graph separations; max_depth+1 means 'farther'."""
    adj = adjacency_matrix(n, bonds).astype(np.int32)
    dist = np.full((n, n), max_depth + 1, dtype=np.int32)
    np.fill_diagonal(dist, 0)
    reach = np.eye(n, dtype=np.int32)
    for d in range(1, max_depth + 1):
        reach = ((reach @ adj) > 0).astype(np.int32)
        newly = (reach > 0) & (dist > d)
        dist[newly] = d
    return dist


def bond_separation(topology: LigandTopology, max_depth: int):
    """{(i, j): separation} for i < j within max_depth bonds."""
    d = _hop_distances(topology.n_atoms, topology.bonds, max_depth)
    ii, jj = np.nonzero(np.triu(d <= max_depth, k=1))
    return {(int(a), int(b)): int(d[a, b]) for a, b in zip(ii, jj)}


def nonbond_pairs(n: int, bonds: np.ndarray):
    """(i, j) with i < j and separation >= 4 bonds, row-major order."""
    d = _hop_distances(n, np.asarray(bonds, dtype=np.int64).reshape(-1, 2), 3)
    ii, jj = np.nonzero(np.triu(d > 3, k=1))
    return ii.astype(np.int32), jj.astype(np.int32)


def build_nonbond_pairlist(topology: LigandTopology, params) -> NonbondPairList:
    """Non-bonded pairs with Lorentz-Berthelot mixing; 12-10 for donor-H x acceptor."""
    table = list(params)
    t = topology.type_index
    bad = np.flatnonzero((t < 0) | (t >= len(table)))
    if bad.size:
        raise ValueError(f"atom {int(bad[0])} has unknown atom type index {int(t[bad[0]])}")
    pi, pj = nonbond_pairs(topology.n_atoms, topology.bonds)

    col = lambda name, dt=np.float64: np.array([getattr(p, name) for p in table], dtype=dt)
    r_eq_t, eps_t, vol_t, sol_t = col("r_eq"), col("eps"), col("volume"), col("solpar")
    don_t, acc_t = col("hbond_donor", bool), col("hbond_acceptor", bool)

    ti, tj = t[pi], t[pj]
    r_eq = 0.5 * (r_eq_t[ti] + r_eq_t[tj])
    eps = np.sqrt(eps_t[ti] * eps_t[tj])
    hb = (don_t[ti] & acc_t[tj]) | (acc_t[ti] & don_t[tj])
    lj_a, lj_b = chem.lj_coefficients(r_eq, eps)
    hb_a, hb_b = chem.hb_coefficients(r_eq, eps)
    q = topology.charge.astype(np.float64)
    qi, qj = q[pi], q[pj]
    dsl = chem.desolvation_coefficient(sol_t[ti], vol_t[ti], qi, sol_t[tj], vol_t[tj], qj)
    return NonbondPairList(
        i=pi, j=pj,
        a_coef=np.where(hb, hb_a, lj_a).astype(np.float32),
        b_coef=np.where(hb, hb_b, lj_b).astype(np.float32),
        is_hbond=hb,
        qq_product=(qi * qj).astype(np.float32),
        desolv_coeff=dsl.astype(np.float32),
    )


def with_fragments(topology: LigandTopology, axes) -> LigandTopology:
    """Topology whose rotatable bonds (axis pairs) carry their BFS fragments."""
    probe = LigandTopology(topology.coords0, topology.type_index, topology.charge,
                           topology.bonds,
                           tuple(RotatableBond(int(a), int(b), np.empty(0, np.int32))
                                 for a, b in axes))
    masks = build_fragment_masks(probe)
    return LigandTopology(topology.coords0, topology.type_index, topology.charge,
                          topology.bonds,
                          tuple(RotatableBond(rb.axis_a, rb.axis_b, m)
                                for rb, m in zip(probe.rotatable_bonds, masks)))
