"""Genotype decoding (host validation) and pose generation (device).

Mirror of vd/pose.py.  `decode_genotype` / `quaternion_matrix` are the
reference's host-side helpers (vd/pose.py:29-61); `apply_pose` and
`pose_population` (vd/pose.py:119-205) run the bit-exact device pose stage
(csrc/vd_device.cuh build_pose) -- there is no CPU path.
"""

from __future__ import annotations

import math

import numpy as np

RIGID_GENES = 7


def genotype_length(topology) -> int:
    return RIGID_GENES + topology.n_torsions


def decode_genotype(genes, topology):
    g = np.asarray(genes, dtype=np.float64)
    want = genotype_length(topology)
    if g.shape != (want,):
        raise ValueError(
            f"genotype length {g.shape} does not match 7 + {topology.n_torsions} torsions")
    if not np.isfinite(g).all():
        raise ValueError("genotype contains non-finite genes")
    q = g[3:7]
    n = math.sqrt(float((q * q).sum()))
    if n < 1e-12:
        raise ValueError("rotation genes are all zero; orientation undefined")
    return g[:3].copy(), q / n, g[7:].copy()


def quaternion_matrix(q) -> np.ndarray:
    w, x, y, z = (float(v) for v in q)
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ], dtype=np.float64).astype(np.float32)


class _PoseContext:
    """The pose-stage subset of a ScoringContext for a bare topology."""

    def __init__(self, topology):
        n = topology.n_atoms
        self.n_atoms = n
        self.pose_centered0 = (topology.coords0 - topology.centroid0[:, None]).astype(np.float32)
        frags = [np.asarray(rb.fragment, np.int32) for rb in topology.rotatable_bonds]
        self.frag_start = np.concatenate([[0], np.cumsum([f.size for f in frags])]).astype(np.int32)
        self.frag_index = np.concatenate(frags).astype(np.int32) if frags else np.empty(0, np.int32)
        self.frag_axis_a = np.array([rb.axis_a for rb in topology.rotatable_bonds], np.int32)
        self.frag_axis_b = np.array([rb.axis_b for rb in topology.rotatable_bonds], np.int32)
        self.n_torsions = len(frags)
        z = np.zeros(n, np.float32)
        self.charge = self.desolv_factor = z
        self.pair_i = self.pair_j = np.empty(0, np.int32)
        self.pair_a = self.pair_b = self.pair_qq = self.pair_desolv = np.empty(0, np.float32)
        self.pair_hb = np.empty(0, bool)
        self.n_pairs = 0
        self.torsional32 = np.float32(0)
        self.intra_cutoff2 = np.float32(np.inf)
        self.penalty_scale = np.float32(1e4)


_pose_sets = {}


def pose_population(topology, genes: np.ndarray) -> np.ndarray:
    """(pop, 7+T) fp64 genes -> (pop, 3, n) f32 poses on the device, bit-exact."""
    from . import _abi
    import weakref

    g = np.ascontiguousarray(genes, dtype=np.float64)
    if g.ndim != 2 or g.shape[1] != genotype_length(topology):
        raise ValueError(f"population gene length {g.shape[-1]} != {genotype_length(topology)}")
    q = g[:, 3:7]
    if (np.sqrt((q * q).sum(axis=1)) < 1e-12).any():
        raise ValueError("rotation genes are all zero for some individual")
    key = id(topology)
    ligs = _pose_sets.get(key)
    if ligs is None:
        ctx = _PoseContext(topology)
        ligs = _abi.LigandSet([ctx], [np.zeros(ctx.n_atoms, np.int32)], 0, 0)
        _pose_sets[key] = ligs
        weakref.finalize(topology, _pose_sets.pop, key, None)
    out = np.empty((g.shape[0], 3, topology.n_atoms), np.float32)
    _abi.pose_genes(ligs, 0, g, out)
    return out


def apply_pose(topology, genes) -> np.ndarray:
    """Docked (3, n) f32 coordinates of one genotype (vd/pose.py:119-134)."""
    decode_genotype(genes, topology)
    return pose_population(topology, np.asarray(genes, np.float64)[None, :])[0]
