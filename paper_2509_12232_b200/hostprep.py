"""Batched host preprocessing and synthetic ligand batches in C++ (csrc/vd_host.cpp).

`TopologyBatch` is a CSR of ligand topologies; `prepare_batch` turns one into
the vd_ligand_arrays record set that `_abi.LigandSet.from_arrays` uploads --
bit-identical to running `context.prepare_context` per ligand (tested), but
OpenMP-parallel in C++ instead of ~1.4-5.5 ms of Python per ligand
(SURVEY.md 8a row 6, 8f row 2).  `TopologyBatch.synth` draws the cfg2/3/4
ligand distributions of SURVEY Appendix B on a counter-keyed stream, so rank r
can generate exactly its index range.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi, chem
from .topology import LigandTopology, RotatableBond

SYNTH_SEED = 0x5EED
HEAVY = ("C", "A", "N", "NA", "OA", "SA")
SYNTH_RECIPES = {  # heavy lo/hi, HD ratio, torsion lo/hi  (BASELINE.json configs)
    2: (16, 48, 1.0 / 3.0, 0, 12),
    3: (16, 48, 1.0 / 3.0, 0, 12),
    4: (96, 96, 1.0 / 3.0, 32, 32),
}


def _cs(counts, dtype=np.int64):
    out = np.zeros(len(counts) + 1, dtype=dtype)
    np.cumsum(counts, out=out[1:])
    return out


@dataclass
class TopologyBatch:
    atom_start: np.ndarray   # [L+1] i32
    xyz: np.ndarray          # per ligand (3, n) f32, concatenated
    type_index: np.ndarray   # [sumN] i32
    charge: np.ndarray       # [sumN] f32
    bond_start: np.ndarray   # [L+1] i32
    bonds: np.ndarray        # [sumB, 2] i32
    tors_start: np.ndarray   # [L+1] i32
    axes: np.ndarray         # [sumT, 2] i32 (axis_a, axis_b)

    def __len__(self):
        return len(self.atom_start) - 1

    @property
    def n_atoms(self):
        return np.diff(self.atom_start)

    @property
    def n_torsions(self):
        return np.diff(self.tors_start)

    @classmethod
    def from_topologies(cls, topos):
        na = [t.n_atoms for t in topos]
        nb = [len(t.bonds) for t in topos]
        nt = [t.n_torsions for t in topos]
        return cls(
            atom_start=_cs(na, np.int32), bond_start=_cs(nb, np.int32),
            tors_start=_cs(nt, np.int32),
            xyz=np.concatenate([np.ascontiguousarray(t.coords0, np.float32).ravel() for t in topos]),
            type_index=np.concatenate([t.type_index for t in topos]).astype(np.int32),
            charge=np.concatenate([t.charge for t in topos]).astype(np.float32),
            bonds=np.concatenate([np.asarray(t.bonds, np.int32).reshape(-1, 2) for t in topos]),
            axes=np.array([[rb.axis_a, rb.axis_b] for t in topos for rb in t.rotatable_bonds],
                          np.int32).reshape(-1, 2),
        )

    @classmethod
    def synth(cls, cfg: int, first: int, count: int, table=None, seed: int = SYNTH_SEED):
        """Ligands [first, first+count) of configuration `cfg` (2, 3 or 4)."""
        table = table or chem.default_parameter_table()
        h_lo, h_hi, ratio, t_lo, t_hi = SYNTH_RECIPES[cfg]
        L = _abi.host_lib()
        na = np.empty(count, np.int32)
        tmax = np.empty(count, np.int32)
        L.vd_synth_count(seed, first, count, h_lo, h_hi, ratio, t_lo, t_hi, na.ctypes.data,
                         tmax.ctypes.data)
        atom_start = _cs(na, np.int32)
        n = int(atom_start[-1])
        xyz = np.empty(3 * n, np.float32)
        types = np.empty(n, np.int32)
        charge = np.empty(n, np.float32)
        bonds = np.empty((n - count, 2), np.int32)
        nt = np.empty(count, np.int32)
        axes = np.empty((count * t_hi, 2), np.int32)
        heavy = np.array([table.index_of(l) for l in HEAVY], np.int32)
        L.vd_synth_fill(seed, first, count, h_lo, h_hi, ratio, t_lo, t_hi, heavy.ctypes.data,
                        table.index_of("HD"), atom_start.ctypes.data, xyz.ctypes.data,
                        types.ctypes.data, charge.ctypes.data, bonds.ctypes.data,
                        nt.ctypes.data, axes.ctypes.data)
        keep = np.concatenate([np.arange(k * t_hi, k * t_hi + nt[k]) for k in range(count)]) \
            if count else np.empty(0, np.int64)
        return cls(atom_start=atom_start, xyz=xyz, type_index=types, charge=charge,
                   bond_start=(atom_start - np.arange(count + 1)).astype(np.int32), bonds=bonds,
                   tors_start=_cs(nt, np.int32), axes=axes[keep.astype(np.int64)])

    def topology(self, l: int) -> LigandTopology:
        """The mirror LigandTopology of ligand l (fragments via the host BFS)."""
        from .topology import with_fragments

        a0, a1 = self.atom_start[l], self.atom_start[l + 1]
        n = a1 - a0
        topo = LigandTopology(self.xyz[3 * a0:3 * a1].reshape(3, n), self.type_index[a0:a1],
                              self.charge[a0:a1],
                              self.bonds[self.bond_start[l]:self.bond_start[l + 1]])
        return with_fragments(topo, [tuple(x) for x in
                                     self.axes[self.tors_start[l]:self.tors_start[l + 1]]])


def prepare_batch(batch: TopologyBatch, map_labels, weights=None, table=None,
                  penalty_scale: float = chem.BOX_PENALTY_SCALE, intra_cutoff=None) -> dict:
    """vd_ligand_arrays-shaped arrays for every ligand of `batch`.

    `map_labels` lists the device grid's map labels in order; each atom's type
    map is looked up by label, exactly as prepare_context's slot -> stack mapping.
    """
    weights = weights or chem.TermWeights()
    table = table or chem.default_parameter_table()
    labels = list(map_labels)
    where = {l: k for k, l in enumerate(labels)}
    for reserved in (chem.ELEC_LABEL, chem.DESOLV_LABEL):
        if reserved not in where:
            raise ValueError(f"grid set is missing the {reserved!r} map")
    type_map = np.array([where.get(e.type_label, -1) for e in table], np.int32)
    used = np.unique(batch.type_index)
    missing = [table[int(t)].type_label for t in used if type_map[t] < 0]
    if missing:
        raise ValueError(f"grid set has no map for ligand atom type {missing[0]!r}")
    L = _abi.host_lib()
    nl = len(batch)
    npairs = np.empty(nl, np.int64)
    nfrag = np.empty(nl, np.int64)
    rc = L.vd_prepare_count(nl, batch.atom_start.ctypes.data, batch.xyz.ctypes.data,
                            batch.bond_start.ctypes.data, batch.bonds.ctypes.data,
                            batch.tors_start.ctypes.data, batch.axes.ctypes.data,
                            npairs.ctypes.data, nfrag.ctypes.data)
    if rc:
        raise ValueError("a rotatable bond lies on a ring; removing it does not split the graph")
    pair_start, frag_start = _cs(npairs), _cs(nfrag)
    P, F, N, T = int(pair_start[-1]), int(frag_start[-1]), int(batch.atom_start[-1]), \
        int(batch.tors_start[-1])
    out = dict(
        centered0=np.empty(3 * N, np.float32), desolv_factor=np.empty(N, np.float32),
        atom_map=np.empty(N, np.int32), pair_i=np.empty(P, np.int32),
        pair_j=np.empty(P, np.int32), pair_a=np.empty(P, np.float32),
        pair_b=np.empty(P, np.float32), pair_qq=np.empty(P, np.float32),
        pair_desolv=np.empty(P, np.float32), pair_hb=np.empty(P, np.uint8),
        frag_lo=np.empty(T, np.int32), frag_hi=np.empty(T, np.int32),
        frag_index=np.empty(F, np.int32), torsional32=np.empty(nl, np.float32),
    )
    tt = _abi.atom_type_array(table)
    w = _abi.VdWeights(weights.vdw, weights.hbond, weights.elec, weights.desolv)
    order = ("centered0", "desolv_factor", "atom_map", "pair_i", "pair_j", "pair_a", "pair_b",
             "pair_qq", "pair_desolv", "pair_hb", "frag_lo", "frag_hi", "frag_index",
             "torsional32")
    rc = L.vd_prepare_fill(nl, batch.atom_start.ctypes.data, batch.xyz.ctypes.data,
                           batch.type_index.ctypes.data, batch.charge.ctypes.data,
                           batch.bond_start.ctypes.data, batch.bonds.ctypes.data,
                           batch.tors_start.ctypes.data, batch.axes.ctypes.data,
                           C.cast(tt, C.c_void_p), len(table), type_map.ctypes.data,
                           C.byref(w), float(weights.tors), pair_start.ctypes.data,
                           frag_start.ctypes.data, *[out[k].ctypes.data for k in order])
    if rc:
        raise ValueError("host preparation failed (atom type without a map or ring bond)")
    cut2 = np.float32(np.inf) if intra_cutoff is None else np.float32(intra_cutoff ** 2)
    out.update(
        atom_start=batch.atom_start.astype(np.int32), pair_start=pair_start.astype(np.int32),
        tors_start=batch.tors_start.astype(np.int32), charge=batch.charge,
        axis_a=np.ascontiguousarray(batch.axes[:, 0]), axis_b=np.ascontiguousarray(batch.axes[:, 1]),
        intra_cutoff2=np.full(nl, cut2, np.float32),
        penalty_scale=np.full(nl, np.float32(penalty_scale), np.float32),
    )
    out["_elec"], out["_desolv"] = where[chem.ELEC_LABEL], where[chem.DESOLV_LABEL]
    return out


def ligand_set(arrays: dict) -> "_abi.LigandSet":
    keep = {k: v for k, v in arrays.items() if not k.startswith("_")}
    return _abi.LigandSet.from_arrays(keep, arrays["_elec"], arrays["_desolv"])
