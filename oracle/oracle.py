"""ctypes front of the CPU oracle (oracle/vd_oracle.c, oracle/vd_ga_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, never by the product package.  Every function
takes the same context record the product consumes (a ScoringContext from
either the reference or paper_2509_12232_b200.context) so both sides score
identical inputs.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "libvdoracle.so"
_lib = None

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C")


class OrLigand(C.Structure):
    _fields_ = [
        ("maps", C.c_void_p), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
        ("lo", C.c_float * 3), ("hi", C.c_float * 3), ("spacing", C.c_float),
        ("penalty", C.c_float),
        ("n_atoms", C.c_int), ("atom_map", C.c_void_p), ("elec_map", C.c_int),
        ("desolv_map", C.c_int), ("charge", C.c_void_p), ("dsf", C.c_void_p),
        ("n_pairs", C.c_int), ("pi", C.c_void_p), ("pj", C.c_void_p), ("pa", C.c_void_p),
        ("pb", C.c_void_p), ("pqq", C.c_void_p), ("pdsl", C.c_void_p), ("phb", C.c_void_p),
        ("cut2", C.c_float), ("lane", C.c_int),
        ("centered0", C.c_void_p), ("n_torsions", C.c_int), ("frag_start", C.c_void_p),
        ("frag_index", C.c_void_p), ("axis_a", C.c_void_p), ("axis_b", C.c_void_p),
    ]


class OrGaParams(C.Structure):
    _fields_ = [
        ("pop", C.c_int), ("generations", C.c_int), ("tournament", C.c_int),
        ("elitism", C.c_int), ("cx_rate", C.c_double), ("mut_rate", C.c_double),
        ("sigma_t", C.c_double), ("sigma_r", C.c_double), ("sigma_tor", C.c_double),
        ("lo", C.c_double * 3), ("hi", C.c_double * 3),
    ]


class OrGaCounts(C.Structure):
    _fields_ = [("children", C.c_int64), ("crossovers", C.c_int64),
                ("gene_mutations", C.c_int64), ("genes_seen", C.c_int64)]


class OrAtomType(C.Structure):
    _fields_ = [("r_eq", C.c_double), ("eps", C.c_double), ("volume", C.c_double),
                ("solpar", C.c_double), ("donor", C.c_int), ("acceptor", C.c_int)]


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        vp, i64, i32, f32 = C.c_void_p, C.c_int64, C.c_int, C.c_float
        L.or_dock_population.argtypes = [vp, vp, i64, i32, vp, vp, vp, f32, i32]
        L.or_score_poses.argtypes = [vp, vp, i64, vp, vp, i32]
        L.or_pose_population.argtypes = [vp, vp, i64, i32, vp]
        L.or_build_grid.argtypes = [vp, vp, vp, i32, vp, i32, vp, i32,
                                    C.c_double, C.c_double, C.c_double, C.c_double,
                                    i32, i32, i32, C.c_double, C.c_double, C.c_double,
                                    C.c_double, C.c_double, vp, i32]
        L.or_philox_block.argtypes = [C.c_uint64] * 6 + [vp]
        L.or_log.argtypes = [C.c_double]
        L.or_log.restype = C.c_double
        L.or_cos2pi.argtypes = [C.c_double]
        L.or_cos2pi.restype = C.c_double
        L.or_normal.argtypes = [C.c_uint64] * 6
        L.or_normal.restype = C.c_double
        L.or_rng_words.argtypes = [C.c_uint64, C.c_uint64, i32, i64, i64, i64, vp]
        L.or_rng_normals.argtypes = [C.c_uint64, C.c_uint64, i32, i64, i64, i64, vp]
        L.or_init_population.argtypes = [vp, i32, C.c_uint64, C.c_uint64, vp]
        L.or_next_generation.argtypes = [vp, i32, vp, vp, i32, C.c_uint64, C.c_uint64, vp, vp]
        L.or_dock.argtypes = [vp, vp, C.c_uint64, C.c_uint64, f32, vp, vp, vp, vp, vp, vp]
        L.or_dock_many.argtypes = [vp, i32, vp, C.c_uint64, i64, vp, i32, vp, vp, vp, vp, vp, i32]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data if a is not None and a.size else None


class Ligand:
    """or_ligand over a scoring context; keeps every array it points at alive.

    `maps`/`atom_map`/`elec_map`/`desolv_map` default to the context's own
    map stack (slot indices); pass a shared (m, nx, ny, nz) stack and global
    indices to score many ligands against one grid without copies.
    """

    def __init__(self, ctx, maps=None, atom_map=None, elec_map=None, desolv_map=None, lane=8):
        if maps is None:
            maps = ctx.map_stack
            atom_map = ctx.atom_slot
            elec_map, desolv_map = maps.shape[0] - 2, maps.shape[0] - 1
        keep = dict(
            maps=np.ascontiguousarray(maps, dtype=np.float32),
            atom_map=np.ascontiguousarray(atom_map, dtype=np.int32),
            charge=np.ascontiguousarray(ctx.charge, dtype=np.float32),
            dsf=np.ascontiguousarray(ctx.desolv_factor, dtype=np.float32),
            centered0=np.ascontiguousarray(ctx.pose_centered0, dtype=np.float32),
            frag_start=np.ascontiguousarray(ctx.frag_start, dtype=np.int32),
            frag_index=np.ascontiguousarray(ctx.frag_index, dtype=np.int32),
            axis_a=np.ascontiguousarray(ctx.frag_axis_a, dtype=np.int32),
            axis_b=np.ascontiguousarray(ctx.frag_axis_b, dtype=np.int32),
        )
        n_pairs = 0 if ctx.pair_i is None else int(ctx.pair_i.shape[0])
        if n_pairs:
            keep.update(
                pi=np.ascontiguousarray(ctx.pair_i, dtype=np.int32),
                pj=np.ascontiguousarray(ctx.pair_j, dtype=np.int32),
                pa=np.ascontiguousarray(ctx.pair_a, dtype=np.float32),
                pb=np.ascontiguousarray(ctx.pair_b, dtype=np.float32),
                pqq=np.ascontiguousarray(ctx.pair_qq, dtype=np.float32),
                pdsl=np.ascontiguousarray(ctx.pair_desolv, dtype=np.float32),
                phb=np.ascontiguousarray(ctx.pair_hb, dtype=np.uint8),
            )
        self._keep = keep
        nx, ny, nz = (int(d) for d in ctx.dims)
        s = OrLigand()
        s.maps = _ptr(keep["maps"])
        s.nx, s.ny, s.nz = nx, ny, nz
        s.lo[:] = [float(v) for v in np.asarray(ctx.box_lo, np.float32)]
        s.hi[:] = [float(v) for v in np.asarray(ctx.box_hi, np.float32)]
        s.spacing = float(np.float32(ctx.spacing))
        s.penalty = float(np.float32(ctx.penalty_scale))
        s.n_atoms = int(ctx.n_atoms)
        s.atom_map = _ptr(keep["atom_map"])
        s.elec_map, s.desolv_map = int(elec_map), int(desolv_map)
        s.charge, s.dsf = _ptr(keep["charge"]), _ptr(keep["dsf"])
        s.n_pairs = n_pairs
        for f in ("pi", "pj", "pa", "pb", "pqq", "pdsl", "phb"):
            setattr(s, f, _ptr(keep[f]) if n_pairs else None)
        s.cut2 = float(np.float32(ctx.intra_cutoff2))
        s.lane = int(lane)
        s.centered0 = _ptr(keep["centered0"])
        s.n_torsions = int(keep["axis_a"].shape[0])
        for f in ("frag_start", "frag_index", "axis_a", "axis_b"):
            setattr(s, f, _ptr(keep[f]))
        self.struct = s
        self.n_atoms = s.n_atoms
        self.n_torsions = s.n_torsions
        self.torsional32 = np.float32(ctx.torsional32)


class _CsrContext:
    """One ligand of a vd_ligand_arrays CSR set, in the ScoringContext field names."""

    def __init__(self, a: dict, l: int, spec):
        s0, s1 = int(a["atom_start"][l]), int(a["atom_start"][l + 1])
        p0, p1 = int(a["pair_start"][l]), int(a["pair_start"][l + 1])
        t0, t1 = int(a["tors_start"][l]), int(a["tors_start"][l + 1])
        self.n_atoms = s1 - s0
        self.charge = a["charge"][s0:s1]
        self.desolv_factor = a["desolv_factor"][s0:s1]
        self.pose_centered0 = a["centered0"][3 * s0:3 * s1].reshape(-1, 3).T  # atom-major -> (3, n)
        self.atom_map = a["atom_map"][s0:s1]
        for f in ("pair_i", "pair_j", "pair_a", "pair_b", "pair_qq", "pair_desolv", "pair_hb"):
            setattr(self, f, a[f][p0:p1])
        self.n_pairs = p1 - p0
        lo, hi = a["frag_lo"][t0:t1], a["frag_hi"][t0:t1]
        f0 = int(lo[0]) if t1 > t0 else 0
        self.frag_start = np.concatenate([[0], np.cumsum(hi - lo)]).astype(np.int32)
        self.frag_index = np.concatenate([a["frag_index"][x:y] for x, y in zip(lo, hi)]) \
            if t1 > t0 else np.empty(0, np.int32)
        assert t1 == t0 or np.array_equal(lo - f0, self.frag_start[:-1])
        self.frag_axis_a, self.frag_axis_b = a["axis_a"][t0:t1], a["axis_b"][t0:t1]
        self.dims = tuple(int(d) for d in spec.dims)
        self.box_lo = np.asarray(spec.origin, np.float32)
        self.box_hi = np.asarray(spec.upper, np.float32)
        self.spacing = np.float32(spec.spacing)
        self.penalty_scale = np.float32(a["penalty_scale"][l])
        self.intra_cutoff2 = np.float32(a["intra_cutoff2"][l])
        self.torsional32 = np.float32(a["torsional32"][l])


def ligands_from_arrays(arrays: dict, maps: np.ndarray, spec, which=None) -> list:
    """Oracle ligands over a shared (m, nx, ny, nz) map stack for ligands `which` (default all)
    of a vd_ligand_arrays CSR set (hostprep.prepare_batch, bit-identical to prepare_context),
    with the same global map indices the device set uses."""
    stack = np.ascontiguousarray(maps, dtype=np.float32)
    n = len(arrays["atom_start"]) - 1
    out = []
    for l in (range(n) if which is None else which):
        c = _CsrContext(arrays, int(l), spec)
        out.append(Ligand(c, stack, c.atom_map, arrays["_elec"], arrays["_desolv"]))
    return out


def dock_population(lig: Ligand, genes: np.ndarray, n_threads: int = 1):
    """(inter64, intra64, total32) per genotype row -- SimdBackend.dock_population + totals."""
    g = np.ascontiguousarray(genes, dtype=np.float64)
    P, G = g.shape
    inter = np.empty(P, np.float64)
    intra = np.empty(P, np.float64)
    total = np.empty(P, np.float32)
    lib().or_dock_population(C.byref(lig.struct), g.ctypes.data, P, G, inter.ctypes.data,
                             intra.ctypes.data, total.ctypes.data, float(lig.torsional32),
                             int(n_threads))
    return inter, intra, total


def score_poses(lig: Ligand, poses: np.ndarray, n_threads: int = 1):
    p = np.ascontiguousarray(poses, dtype=np.float32)
    inter = np.empty(p.shape[0], np.float64)
    intra = np.empty(p.shape[0], np.float64)
    lib().or_score_poses(C.byref(lig.struct), p.ctypes.data, p.shape[0], inter.ctypes.data,
                         intra.ctypes.data, int(n_threads))
    return inter, intra


def pose_population(lig: Ligand, genes: np.ndarray) -> np.ndarray:
    g = np.ascontiguousarray(genes, dtype=np.float64)
    out = np.empty((g.shape[0], 3, lig.n_atoms), np.float32)
    lib().or_pose_population(C.byref(lig.struct), g.ctypes.data, g.shape[0], g.shape[1],
                             out.ctypes.data)
    return out


def atom_type_table(table):
    arr = (OrAtomType * len(table))()
    for k, e in enumerate(table):
        arr[k].r_eq, arr[k].eps, arr[k].volume, arr[k].solpar = e.r_eq, e.eps, e.volume, e.solpar
        arr[k].donor, arr[k].acceptor = int(e.hbond_donor), int(e.hbond_acceptor)
    return arr


def build_grid(protein, origin, spacing, dims, probe_types, weights, table, cutoff=8.0,
               n_threads=0) -> np.ndarray:
    """(n_probe + 2, nx, ny, nz) f32: probe maps, then elec, then desolv."""
    tt = atom_type_table(table)
    probe = np.array([table.index_of(l) for l in probe_types], dtype=np.int32)
    coords = np.ascontiguousarray(protein.coords, dtype=np.float32)
    ptype = np.ascontiguousarray(protein.type_index, dtype=np.int32)
    charge = np.ascontiguousarray(protein.charge, dtype=np.float32)
    nx, ny, nz = (int(d) for d in dims)
    out = np.empty((len(probe) + 2, nx, ny, nz), np.float32)
    lib().or_build_grid(coords.ctypes.data, ptype.ctypes.data, charge.ctypes.data,
                        coords.shape[1], C.cast(tt, C.c_void_p), len(table), probe.ctypes.data,
                        len(probe), float(origin[0]), float(origin[1]), float(origin[2]),
                        float(spacing), nx, ny, nz, float(weights.vdw), float(weights.hbond),
                        float(weights.elec), float(weights.desolv), float(cutoff),
                        out.ctypes.data, int(n_threads))
    return out


def philox_block(counter, key) -> np.ndarray:
    out = np.empty(4, np.uint64)
    lib().or_philox_block(*[int(c) for c in counter], int(key[0]), int(key[1]), out.ctypes.data)
    return out


def rng_words(seed: int, lig_index: int, phase: int, gen: int, n_idx: int,
              n_slot: int) -> np.ndarray:
    """Words of the restated GA stream (or_rng.c): [idx][slot] at (phase, gen)."""
    out = np.empty((n_idx, n_slot), np.uint64)
    lib().or_rng_words(int(seed), int(lig_index), int(phase), int(gen), int(n_idx), int(n_slot),
                       out.ctypes.data)
    return out


def rng_normals(seed: int, lig_index: int, phase: int, gen: int, n_idx: int,
                n_comp: int) -> np.ndarray:
    out = np.empty((n_idx, n_comp), np.float64)
    lib().or_rng_normals(int(seed), int(lig_index), int(phase), int(gen), int(n_idx),
                         int(n_comp), out.ctypes.data)
    return out


def ga_params(cfg, lo, hi) -> OrGaParams:
    p = OrGaParams()
    p.pop, p.generations = cfg.population_size, cfg.generations
    p.tournament, p.elitism = cfg.tournament_size, cfg.elitism_count
    p.cx_rate, p.mut_rate = cfg.crossover_rate, cfg.mutation_rate
    p.sigma_t = cfg.mutation_sigma_translation
    p.sigma_r = cfg.mutation_sigma_rotation
    p.sigma_tor = cfg.mutation_sigma_torsion
    p.lo[:] = [float(v) for v in lo]
    p.hi[:] = [float(v) for v in hi]
    return p


def init_population(params: OrGaParams, n_torsions: int, key) -> np.ndarray:
    out = np.empty((params.pop, 7 + n_torsions), np.float64)
    lib().or_init_population(C.byref(params), n_torsions, int(key[0]), int(key[1]),
                             out.ctypes.data)
    return out


def next_generation(params: OrGaParams, n_torsions: int, pop: np.ndarray, fitness: np.ndarray,
                    gen: int, key, counts: OrGaCounts | None = None) -> np.ndarray:
    cur = np.ascontiguousarray(pop, np.float64)
    fit = np.ascontiguousarray(fitness, np.float64)
    out = np.empty_like(cur)
    lib().or_next_generation(C.byref(params), n_torsions, cur.ctypes.data, fit.ctypes.data,
                             int(gen), int(key[0]), int(key[1]), out.ctypes.data,
                             C.byref(counts) if counts is not None else None)
    return out


def dock(lig: Ligand, params: OrGaParams, seed: int, lig_index: int):
    """Restated GA dock: (best_genes, best_total32, inter64, intra64, trace, n_evals)."""
    G = 7 + lig.n_torsions
    genes = np.empty(G, np.float64)
    bt = C.c_float()
    be, ba = C.c_double(), C.c_double()
    trace = np.empty(params.generations + 1, np.float32)
    ne = C.c_int64()
    lib().or_dock(C.byref(lig.struct), C.byref(params), int(seed), int(lig_index),
                  float(lig.torsional32), genes.ctypes.data, C.byref(bt), C.byref(be),
                  C.byref(ba), trace.ctypes.data, C.byref(ne))
    return genes, np.float32(bt.value), be.value, ba.value, trace, int(ne.value)


def dock_many(ligs, params: OrGaParams, seed: int, lig_index_base: int = 0, n_threads: int = 0):
    n = len(ligs)
    arr = (OrLigand * n)(*[l.struct for l in ligs])
    gmax = 7 + max(l.n_torsions for l in ligs)
    tors = np.array([l.torsional32 for l in ligs], np.float32)
    genes = np.zeros((n, gmax), np.float64)
    bt = np.empty(n, np.float32)
    be = np.empty(n, np.float64)
    ba = np.empty(n, np.float64)
    ne = np.empty(n, np.int64)
    lib().or_dock_many(C.cast(arr, C.c_void_p), n, C.byref(params), int(seed),
                       int(lig_index_base), tors.ctypes.data, gmax, genes.ctypes.data,
                       bt.ctypes.data, be.ctypes.data, ba.ctypes.data, ne.ctypes.data,
                       int(n_threads))
    return genes, bt, be, ba, ne


def cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
