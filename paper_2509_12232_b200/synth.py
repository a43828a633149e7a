"""Seeded synthetic inputs standing in for the BASELINE.json configurations.

The paper's datasets (MEDIATE subset, a PDBbind complex) are not available,
and the reference ships no generator with the BASELINE distributions, so the
recipes of SURVEY.md Appendix B are implemented here.  Everything is a pure
function of its seed (numpy Philox), identical on every host, and emits the
mirror's own `LigandTopology` / `Protein` records.

Seeds: protein 1000 + cfg; ligand = its index; pose batch 0; GA global seed 0.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import chem
from .gridmaps import GridSpec
from .topology import LigandTopology, Protein, with_fragments

HEAVY_TYPES = ("C", "A", "N", "NA", "OA", "SA")
DONOR_HOSTS = ("N", "NA", "OA", "SA")      # HD binds to N/O/S (parameters.txt:3)
PROTEIN_TYPES = ("C", "N", "OA", "SA", "HD")
PROTEIN_FRACS = (0.60, 0.15, 0.15, 0.02, 0.08)
TETRA = math.radians(109.5)


def _rng(*key) -> np.random.Generator:
    k = (list(key) + [0, 0])[:2]
    return np.random.Generator(np.random.Philox(key=np.array(k, dtype=np.uint64)))


def _unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _place(rng, xyz, placed, parent, grand, length, n_try=24):
    """Child position at `length` from parent with a ~tetrahedral angle to the
    grandparent bond and a random dihedral; best clearance of n_try draws."""
    p = xyz[parent]
    if grand < 0:
        dirs = _unit(rng.standard_normal((n_try, 3)))
    else:
        b = _unit(p - xyz[grand])
        ang = TETRA + np.radians(rng.uniform(-8.0, 8.0, n_try))
        ref = np.array([1.0, 0.0, 0.0]) if abs(b[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
        e1 = _unit(np.cross(b, ref))
        e2 = np.cross(b, e1)
        phi = rng.uniform(0.0, 2.0 * math.pi, n_try)
        # angle(parent->grand, parent->child) = ang  =>  child dir has -cos(ang) along b
        dirs = (-np.cos(ang))[:, None] * b + np.sin(ang)[:, None] * (
            np.cos(phi)[:, None] * e1 + np.sin(phi)[:, None] * e2)
    cand = p + length * dirs
    others = [k for k in placed if k != parent]
    if not others:
        return cand[0]
    d = np.linalg.norm(cand[:, None, :] - xyz[others][None, :, :], axis=-1).min(axis=1)
    ok = np.flatnonzero(d >= 2.0)
    return cand[ok[0]] if ok.size else cand[int(np.argmax(d))]


def make_ligand(seed: int, n_heavy: int, n_hd: int, n_torsions: int,
                table: chem.ParameterTable | None = None) -> LigandTopology:
    """Random heavy-atom tree + HD leaves, ~1.5 A bonds, tetrahedral-ish angles.

    Rotatable bonds are non-terminal heavy-heavy tree edges (capped by how many
    exist), oriented root-outward and declared in breadth order so nested
    fragments compose.  Charges U(-0.4, 0.4) re-centred to net zero.
    """
    table = table or chem.default_parameter_table()
    rng = _rng(seed)
    n = n_heavy + n_hd
    if n_heavy < 1:
        raise ValueError("need at least one heavy atom")
    # heavy-atom tree: a backbone chain then branches on atoms with free valence
    backbone = min(n_heavy, max(n_torsions + 2, (3 * n_heavy) // 5))
    parent = [-1] * n
    kids = [0] * n
    for k in range(1, n_heavy):
        if k < backbone:
            parent[k] = k - 1
        else:
            open_ = [a for a in range(k) if kids[a] < 3]
            parent[k] = open_[int(rng.integers(len(open_)))]
        kids[parent[k]] += 1
    types = [HEAVY_TYPES[int(i)] for i in rng.integers(0, len(HEAVY_TYPES), n_heavy)]
    # HD leaves on donor-capable heavy atoms with free valence (retype if short)
    hosts = []
    for h in range(n_hd):
        cand = [a for a in range(n_heavy) if types[a] in DONOR_HOSTS and kids[a] < 3]
        if not cand:
            spare = [a for a in range(n_heavy) if kids[a] < 3]
            if not spare:
                raise ValueError("no free valence left for HD atoms")
            a = spare[int(rng.integers(len(spare)))]
            types[a] = DONOR_HOSTS[int(rng.integers(len(DONOR_HOSTS)))]
            cand = [a]
        a = cand[int(rng.integers(len(cand)))]
        parent[n_heavy + h] = a
        kids[a] += 1
        hosts.append(a)
    types += ["HD"] * n_hd

    xyz = np.zeros((n, 3))
    placed = [0]
    order = list(range(1, n_heavy)) + list(range(n_heavy, n))
    for k in order:
        length = (1.5 + 0.05 * float(np.clip(rng.standard_normal(), -2, 2))) if k < n_heavy \
            else float(rng.uniform(1.0, 1.1))
        xyz[k] = _place(rng, xyz, placed, parent[k], parent[parent[k]] if parent[k] >= 0 else -1,
                        length)
        placed.append(k)

    bonds = np.array([[parent[k], k] for k in range(1, n)], dtype=np.int32).reshape(-1, 2)
    heavy_deg = np.zeros(n_heavy, dtype=np.int64)
    for k in range(1, n_heavy):
        heavy_deg[k] += 1
        heavy_deg[parent[k]] += 1
    eligible = [k for k in range(1, n_heavy) if heavy_deg[k] >= 2 and heavy_deg[parent[k]] >= 2]
    t = min(n_torsions, len(eligible))
    chosen = sorted(rng.choice(len(eligible), size=t, replace=False).tolist()) if t else []
    depth = np.zeros(n, dtype=np.int64)
    for k in range(1, n):
        depth[k] = depth[parent[k]] + 1
    axes = sorted(((parent[eligible[c]], eligible[c]) for c in chosen),
                  key=lambda ab: (depth[ab[1]], ab[1]))

    q = rng.uniform(-0.4, 0.4, n)
    q = (q - q.mean()).astype(np.float32)
    topo = LigandTopology(
        coords0=xyz.T.astype(np.float32),
        type_index=np.array([table.index_of(s) for s in types], dtype=np.int32),
        charge=q,
        bonds=bonds,
    )
    return with_fragments(topo, axes)


def make_protein(seed: int, n_atoms: int, half_extent: float = 20.0, pocket_radius: float = 10.0,
                 table: chem.ParameterTable | None = None) -> Protein:
    """Atoms uniform in a cube, excluding a central pocket sphere (Appendix B)."""
    table = table or chem.default_parameter_table()
    rng = _rng(seed)
    pts = np.empty((0, 3))
    while len(pts) < n_atoms:
        c = rng.uniform(-half_extent, half_extent, (2 * n_atoms, 3))
        pts = np.concatenate([pts, c[np.linalg.norm(c, axis=1) >= pocket_radius]])
    pts = pts[:n_atoms]
    kinds = rng.choice(len(PROTEIN_TYPES), size=n_atoms, p=PROTEIN_FRACS)
    tindex = np.array([table.index_of(PROTEIN_TYPES[k]) for k in kinds], dtype=np.int32)
    return Protein(coords=pts.T.astype(np.float32), type_index=tindex,
                   charge=rng.uniform(-0.5, 0.5, n_atoms).astype(np.float32))


def random_genes(seed: int, n: int, n_torsions: int, lo, hi) -> np.ndarray:
    """(n, 7+T) fp64: t ~ U(box), q = normalised N(0,1)^4, theta ~ U(-pi, pi)."""
    rng = _rng(seed)
    t = rng.uniform(np.asarray(lo, dtype=np.float64), np.asarray(hi, dtype=np.float64), (n, 3))
    q = rng.standard_normal((n, 4))
    q /= np.sqrt((q * q).sum(axis=1))[:, None]
    th = rng.uniform(-math.pi, math.pi, (n, n_torsions))
    return np.ascontiguousarray(np.concatenate([t, q, th], axis=1))


@dataclass(frozen=True)
class Config:
    name: str
    grid_dims: int
    protein_atoms: int
    probe_types: tuple
    spacing: float = 0.375


PROBES_7 = ("C", "A", "N", "NA", "OA", "SA", "HD")
CONFIGS = {
    0: Config("cfg0-single-dock", 48, 2000, PROBES_7),
    1: Config("cfg1-score-1M", 80, 4000, PROBES_7),
    2: Config("cfg2-screen-10k", 64, 3000, PROBES_7),
    3: Config("cfg3-screen-100k", 64, 3000, PROBES_7),
    4: Config("cfg4-stress-128", 126, 8000, PROBES_7 + ("S",)),
}


def config_grid_spec(cfg: int) -> GridSpec:
    c = CONFIGS[cfg]
    return GridSpec.centered((0.0, 0.0, 0.0), (c.grid_dims,) * 3, c.spacing)


def config_protein(cfg: int) -> Protein:
    return make_protein(1000 + cfg, CONFIGS[cfg].protein_atoms)


def config_ligand(cfg: int, index: int = 0) -> LigandTopology:
    """Ligand `index` of configuration `cfg` (seed = index, per Appendix B)."""
    if cfg == 0:
        return make_ligand(index, 24, 8, 6)
    if cfg == 1:
        return make_ligand(index, 30, 10, 8)
    if cfg in (2, 3):
        r = _rng(0x5C2EE9, index)
        heavy = int(r.integers(16, 49))
        return make_ligand(index, heavy, int(round(heavy / 3)), int(r.integers(0, 13)))
    if cfg == 4:
        return make_ligand(index, 96, 32, 32)
    raise ValueError(f"unknown config {cfg}")
