"""ctypes binding of libvdb200.so (include/vecdock_b200.h).

This is the only place the package touches native code.  There is no CPU
fallback: if the library or a CUDA device is missing, `lib()` raises
`BackendUnavailable` and nothing silently degrades.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .context import BackendUnavailable

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libvdb200.so"
if os.environ.get("VD_LIB"):  # A/B tuning only: a variant build of the same library
    LIB_PATH = Path(os.environ["VD_LIB"]).resolve()

MODE_FAST = 0
MODE_EXACT = 1

_lock = threading.Lock()
_lib = None
_tls = threading.local()


class VdLigandArrays(C.Structure):
    _fields_ = [
        ("n_ligands", C.c_int32),
        ("atom_start", C.c_void_p), ("pair_start", C.c_void_p), ("tors_start", C.c_void_p),
        ("centered0", C.c_void_p), ("charge", C.c_void_p), ("desolv_factor", C.c_void_p),
        ("atom_map", C.c_void_p), ("pair_i", C.c_void_p), ("pair_j", C.c_void_p),
        ("pair_a", C.c_void_p), ("pair_b", C.c_void_p), ("pair_qq", C.c_void_p),
        ("pair_desolv", C.c_void_p), ("pair_hb", C.c_void_p), ("axis_a", C.c_void_p),
        ("axis_b", C.c_void_p), ("frag_lo", C.c_void_p), ("frag_hi", C.c_void_p),
        ("frag_index", C.c_void_p), ("torsional32", C.c_void_p), ("intra_cutoff2", C.c_void_p),
        ("penalty_scale", C.c_void_p), ("elec_map", C.c_int32), ("desolv_map", C.c_int32),
    ]


class VdAtomType(C.Structure):
    _fields_ = [("r_eq", C.c_double), ("eps", C.c_double), ("volume", C.c_double),
                ("solpar", C.c_double), ("donor", C.c_int32), ("acceptor", C.c_int32)]


class VdWeights(C.Structure):
    _fields_ = [("vdw", C.c_double), ("hbond", C.c_double), ("elec", C.c_double),
                ("desolv", C.c_double)]


class VdMugdInfo(C.Structure):
    _fields_ = [("n_maps", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("origin", C.c_float * 3), ("spacing", C.c_float), ("labels_bytes", C.c_int32)]


class VdGaParams(C.Structure):
    _fields_ = [("pop", C.c_int32), ("generations", C.c_int32), ("tournament", C.c_int32),
                ("elitism", C.c_int32), ("cx_rate", C.c_double), ("mut_rate", C.c_double),
                ("sigma_t", C.c_double), ("sigma_r", C.c_double), ("sigma_tor", C.c_double),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3)]


EXPORTS = (
    "vd_abi_version", "vd_last_error", "vd_device_count", "vd_init", "vd_grid_create",
    "vd_grid_build", "vd_grid_n_maps", "vd_grid_layout", "vd_grid_download", "vd_grid_destroy",
    "vd_ligands_create", "vd_ligands_n_torsions", "vd_ligands_destroy", "vd_score_genes",
    "vd_score_poses", "vd_pose_genes", "vd_dock_batch", "vd_last_launch_count", "vd_pipe_count", "vd_debug_check_flags",
    "vd_prepare_count", "vd_prepare_fill", "vd_synth_count", "vd_synth_fill",
    "vd_mugd_read_header", "vd_grid_load_mugd",
    "vd_debug_rng", "vd_debug_ga_init", "vd_debug_ga_breed", "vd_debug_pose_genes",
)


def load_library(path: Path = LIB_PATH):
    """dlopen + prototypes; no device needed (used by the CPU symbol test)."""
    if not path.exists():
        raise BackendUnavailable(
            f"{path.name} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(str(path))
    vp, i32, i64, u64 = C.c_void_p, C.c_int, C.c_int64, C.c_uint64
    L.vd_last_error.restype = C.c_char_p
    L.vd_abi_version.restype = i32
    L.vd_device_count.argtypes = [vp]
    L.vd_init.argtypes = [i32]
    L.vd_grid_create.argtypes = [vp, i32, i32, i32, i32, vp, vp, C.c_float, vp]
    L.vd_grid_build.argtypes = [vp, vp, vp, i32, vp, i32, vp, i32, vp, C.c_double, i32, i32,
                                i32, vp, C.c_double, vp]
    L.vd_grid_n_maps.argtypes = [vp]
    L.vd_grid_layout.argtypes = [vp]
    L.vd_mugd_read_header.argtypes = [C.c_char_p, vp, vp, i32]
    L.vd_grid_load_mugd.argtypes = [C.c_char_p, vp]
    L.vd_grid_download.argtypes = [vp, vp]
    L.vd_grid_destroy.argtypes = [vp]
    L.vd_ligands_create.argtypes = [vp, vp]
    L.vd_ligands_n_torsions.argtypes = [vp, i32]
    L.vd_ligands_destroy.argtypes = [vp]
    L.vd_score_genes.argtypes = [vp, vp, i32, vp, i64, vp, vp, vp, i32, vp]
    L.vd_score_poses.argtypes = [vp, vp, i32, vp, i64, vp, vp, i32, vp]
    L.vd_pose_genes.argtypes = [vp, i32, vp, i64, vp, vp]
    L.vd_dock_batch.argtypes = [vp, vp, i32, i32, vp, u64, i64, i32, vp, vp, vp, vp, i32, vp,
                                vp, vp]
    L.vd_last_launch_count.argtypes = [vp]
    L.vd_pipe_count.argtypes = [i32]
    L.vd_debug_check_flags.argtypes = [vp, i32]
    L.vd_prepare_count.argtypes = [i32] + [vp] * 8
    L.vd_prepare_fill.argtypes = [i32] + [vp] * 8 + [vp, i32, vp, vp, C.c_double] + [vp] * 16
    L.vd_synth_count.argtypes = [u64, i64, i32, i32, i32, C.c_double, i32, i32, vp, vp]
    L.vd_synth_fill.argtypes = [u64, i64, i32, i32, i32, C.c_double, i32, i32, vp, i32] + [vp] * 7
    L.vd_debug_rng.argtypes = [i32, u64, u64, i32, i64, i64, i32, vp]
    L.vd_debug_ga_init.argtypes = [vp, i32, u64, u64, vp]
    L.vd_debug_ga_breed.argtypes = [vp, i32, vp, vp, i32, u64, u64, vp]
    L.vd_debug_pose_genes.argtypes = [vp, i32, vp, i64, i32, vp]
    return L


_host_lib = None


def host_lib():
    """The library for host-only entry points (no device required)."""
    global _host_lib
    if _host_lib is None:
        _host_lib = _lib if _lib is not None else load_library()
    return _host_lib


def lib():
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                L = load_library()
                n = C.c_int(0)
                if L.vd_device_count(C.byref(n)) != 0 or n.value < 1:
                    raise BackendUnavailable("no CUDA device visible to libvdb200")
                _lib = L
    return _lib


def check(rc: int, what: str):
    if rc != 0:
        raise RuntimeError(f"{what}: {lib().vd_last_error().decode()}")


def ensure_device(device: int | None = None) -> int:
    """Bind the calling thread to `device` (default: torch's current device or 0)."""
    if device is None:
        device = getattr(_tls, "device", None)
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0")) if _torch_current() is None \
                else _torch_current()
    if getattr(_tls, "device", None) != device:
        check(lib().vd_init(int(device)), "vd_init")
        _tls.device = device
    return device


def _torch_current():
    try:
        import torch

        if torch.cuda.is_available() and torch.cuda.is_initialized():
            return torch.cuda.current_device()
    except Exception:
        pass
    return None


def launches() -> int:
    v = C.c_int64()
    lib().vd_last_launch_count(C.byref(v))
    return int(v.value)


def _p(a):
    return None if a is None else a.ctypes.data


def ptr_of(x):
    """Raw pointer of a numpy array or a torch tensor (host or device)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return int(x.data_ptr())


# --- grids ----------------------------------------------------------------------
class DeviceGrid:
    """Owned vd_grid handle."""

    def __init__(self, handle, n_maps, dims, lo, hi, spacing, labels=None):
        self.handle = handle
        self.n_maps = n_maps
        self.dims = tuple(dims)
        self.lo, self.hi, self.spacing = lo, hi, spacing
        self.labels = labels

    LAYOUTS = {0: "plain", 1: "brick", 2: "zpair"}

    @property
    def layout(self) -> str:
        """Gather layout chosen at creation: "plain", "brick" (yz-bricks) or "zpair"."""
        return self.LAYOUTS[int(lib().vd_grid_layout(self.handle))]

    def download(self) -> np.ndarray:
        out = np.empty((self.n_maps,) + self.dims, np.float32)
        check(lib().vd_grid_download(self.handle, out.ctypes.data), "vd_grid_download")
        return out

    def close(self):
        if self.handle:
            lib().vd_grid_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def grid_from_stack(stack: np.ndarray, lo, hi, spacing, labels=None) -> DeviceGrid:
    ensure_device()
    s = np.ascontiguousarray(stack, dtype=np.float32)
    lo32 = np.ascontiguousarray(lo, dtype=np.float32)
    hi32 = np.ascontiguousarray(hi, dtype=np.float32)
    h = C.c_void_p()
    check(lib().vd_grid_create(s.ctypes.data, s.shape[0], s.shape[1], s.shape[2], s.shape[3],
                               lo32.ctypes.data, hi32.ctypes.data, float(np.float32(spacing)),
                               C.byref(h)), "vd_grid_create")
    return DeviceGrid(h, s.shape[0], s.shape[1:], lo32, hi32, np.float32(spacing), labels)


def atom_type_array(table):
    arr = (VdAtomType * len(table))()
    for k, e in enumerate(table):
        arr[k].r_eq, arr[k].eps, arr[k].volume, arr[k].solpar = e.r_eq, e.eps, e.volume, e.solpar
        arr[k].donor, arr[k].acceptor = int(e.hbond_donor), int(e.hbond_acceptor)
    return arr


def build_grid_device(protein, spec, probe_types, weights, table, cutoff) -> DeviceGrid:
    ensure_device()
    tt = atom_type_array(table)
    probe = np.array([table.index_of(l) for l in probe_types], np.int32)
    xyz = np.ascontiguousarray(protein.coords, np.float32)
    rt = np.ascontiguousarray(protein.type_index, np.int32)
    rq = np.ascontiguousarray(protein.charge, np.float32)
    origin = np.asarray(spec.origin, np.float64)
    w = VdWeights(weights.vdw, weights.hbond, weights.elec, weights.desolv)
    h = C.c_void_p()
    nx, ny, nz = spec.dims
    check(lib().vd_grid_build(xyz.ctypes.data, rt.ctypes.data, rq.ctypes.data, xyz.shape[1],
                              C.cast(tt, C.c_void_p), len(table), probe.ctypes.data, len(probe),
                              origin.ctypes.data, float(spec.spacing), nx, ny, nz, C.byref(w),
                              float(cutoff), C.byref(h)), "vd_grid_build")
    labels = list(probe_types) + ["@elec", "@desolv"]
    return DeviceGrid(h, len(probe) + 2, spec.dims, np.asarray(spec.origin, np.float32),
                      np.asarray(spec.upper, np.float32), np.float32(spec.spacing), labels)


def _mugd_check(rc: int, what: str):
    if rc == -2:
        from .gridmaps import GridFormatError

        raise GridFormatError(lib_err())
    check(rc, what)


def lib_err() -> str:
    msg = host_lib().vd_last_error()
    return msg.decode() if msg else ""


def mugd_header(path) -> tuple:
    """(VdMugdInfo, [labels]) of a MUGD file (host-only: no device needed)."""
    L = host_lib()
    info = VdMugdInfo()
    p = os.fsencode(os.fspath(path))
    rc = L.vd_mugd_read_header(p, C.byref(info), None, 0)
    if rc == -2:
        from .gridmaps import GridFormatError

        raise GridFormatError(lib_err())
    if rc:
        raise OSError(lib_err())
    buf = C.create_string_buffer(max(1, info.labels_bytes))
    if L.vd_mugd_read_header(p, C.byref(info), buf, len(buf)):
        raise OSError(lib_err())
    labels = buf.raw[:info.labels_bytes].split(b"\0")[:-1] if info.labels_bytes else []
    return info, [l.decode("utf-8") for l in labels]


def grid_from_mugd(path, device=None) -> DeviceGrid:
    """A MUGD file straight into a device grid (pinned staging + device transpose)."""
    info, labels = mugd_header(path)
    ensure_device(device)
    h = C.c_void_p()
    _mugd_check(lib().vd_grid_load_mugd(os.fsencode(os.fspath(path)), C.byref(h)),
                "vd_grid_load_mugd")
    dims = (info.nx, info.ny, info.nz)
    origin = tuple(float(v) for v in info.origin)
    upper = tuple(o + (d - 1) * float(info.spacing) for o, d in zip(origin, dims))
    return DeviceGrid(h, info.n_maps, dims, np.asarray(origin, np.float32),
                      np.asarray(upper, np.float32), np.float32(info.spacing), labels)


def build_grid(protein, spec, probe_types, weights, table, cutoff, device=None) -> np.ndarray:
    ensure_device(device)
    g = build_grid_device(protein, spec, probe_types, weights, table, cutoff)
    try:
        return g.download()
    finally:
        g.close()


# --- ligand sets -------------------------------------------------------------------
class LigandSet:
    """Owned vd_ligands handle over a list of scoring contexts (CSR)."""

    @classmethod
    def from_arrays(cls, keep: dict, elec_map: int, desolv_map: int):
        """Build directly from vd_ligand_arrays-shaped numpy arrays (hostprep batches)."""
        ensure_device()
        self = cls.__new__(cls)
        a = VdLigandArrays()
        a.n_ligands = len(keep["atom_start"]) - 1
        for k, v in keep.items():
            setattr(a, k, v.ctypes.data if v.size else None)
        a.elec_map, a.desolv_map = int(elec_map), int(desolv_map)
        h = C.c_void_p()
        check(lib().vd_ligands_create(C.byref(a), C.byref(h)), "vd_ligands_create")
        self.handle = h
        self.n_ligands = a.n_ligands
        self.n_atoms = np.diff(keep["atom_start"])
        self.n_torsions = np.diff(keep["tors_start"])
        return self

    def __init__(self, contexts, atom_maps, elec_map: int, desolv_map: int):
        ensure_device()
        L = len(contexts)
        na = [int(c.n_atoms) for c in contexts]
        npr = [c.n_pairs for c in contexts]
        nt = [c.n_torsions for c in contexts]
        cs = lambda v: np.concatenate([[0], np.cumsum(v)]).astype(np.int32)
        self.atom_start, self.pair_start, self.tors_start = cs(na), cs(npr), cs(nt)
        cat = lambda xs, dt: (np.concatenate([np.asarray(x, dt).ravel() for x in xs])
                              if xs else np.empty(0, dt))
        centered = cat([np.asarray(c.pose_centered0, np.float32).T for c in contexts], np.float32)
        pair_src = [c for c in contexts if c.n_pairs]
        frag_lo, frag_hi, frag_idx, off = [], [], [], 0
        for c in contexts:
            fs = np.asarray(c.frag_start, np.int64)
            frag_lo.append(fs[:-1] + off)
            frag_hi.append(fs[1:] + off)
            frag_idx.append(np.asarray(c.frag_index, np.int32))
            off += int(fs[-1]) if len(fs) else 0
        keep = dict(
            atom_start=self.atom_start, pair_start=self.pair_start, tors_start=self.tors_start,
            centered0=centered,
            charge=cat([c.charge for c in contexts], np.float32),
            desolv_factor=cat([c.desolv_factor for c in contexts], np.float32),
            atom_map=cat(atom_maps, np.int32),
            pair_i=cat([c.pair_i for c in pair_src], np.int32),
            pair_j=cat([c.pair_j for c in pair_src], np.int32),
            pair_a=cat([c.pair_a for c in pair_src], np.float32),
            pair_b=cat([c.pair_b for c in pair_src], np.float32),
            pair_qq=cat([c.pair_qq for c in pair_src], np.float32),
            pair_desolv=cat([c.pair_desolv for c in pair_src], np.float32),
            pair_hb=cat([c.pair_hb for c in pair_src], np.uint8),
            axis_a=cat([c.frag_axis_a for c in contexts], np.int32),
            axis_b=cat([c.frag_axis_b for c in contexts], np.int32),
            frag_lo=cat(frag_lo, np.int32), frag_hi=cat(frag_hi, np.int32),
            frag_index=cat(frag_idx, np.int32),
            torsional32=np.array([c.torsional32 for c in contexts], np.float32),
            intra_cutoff2=np.array([c.intra_cutoff2 for c in contexts], np.float32),
            penalty_scale=np.array([c.penalty_scale for c in contexts], np.float32),
        )
        a = VdLigandArrays()
        a.n_ligands = L
        for k, v in keep.items():
            setattr(a, k, v.ctypes.data if v.size else None)
        a.elec_map, a.desolv_map = int(elec_map), int(desolv_map)
        h = C.c_void_p()
        check(lib().vd_ligands_create(C.byref(a), C.byref(h)), "vd_ligands_create")
        self.handle = h
        self.n_ligands = L
        self.n_atoms = np.array(na)
        self.n_torsions = np.array(nt)

    def close(self):
        if self.handle:
            lib().vd_ligands_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def score_genes(grid: DeviceGrid, ligs: LigandSet, lig: int, genes, inter, intra, total,
                mode: int = MODE_FAST, stream=None):
    P = genes.shape[0]
    check(lib().vd_score_genes(grid.handle, ligs.handle, int(lig), ptr_of(genes), int(P),
                               ptr_of(inter), ptr_of(intra), ptr_of(total), int(mode),
                               stream), "vd_score_genes")


def score_poses(grid: DeviceGrid, ligs: LigandSet, lig: int, poses, inter, intra,
                mode: int = MODE_FAST, stream=None):
    check(lib().vd_score_poses(grid.handle, ligs.handle, int(lig), ptr_of(poses),
                               int(poses.shape[0]), ptr_of(inter), ptr_of(intra), int(mode),
                               stream), "vd_score_poses")


def pose_genes(ligs: LigandSet, lig: int, genes, out, stream=None):
    check(lib().vd_pose_genes(ligs.handle, int(lig), ptr_of(genes), int(genes.shape[0]),
                              ptr_of(out), stream), "vd_pose_genes")


def dock_batch(grid: DeviceGrid, ligs: LigandSet, first: int, count: int, params: VdGaParams,
               seed: int, lig_index_base: int, mode: int, best_total, best_inter, best_intra,
               best_genes, trace, n_evals, stream=None):
    check(lib().vd_dock_batch(grid.handle, ligs.handle, int(first), int(count), C.byref(params),
                              int(seed) & ((1 << 64) - 1), int(lig_index_base), int(mode),
                              ptr_of(best_total), ptr_of(best_inter), ptr_of(best_intra),
                              ptr_of(best_genes), int(best_genes.shape[1]), ptr_of(trace),
                              ptr_of(n_evals), stream), "vd_dock_batch")


# ---- test probes (vd_debug_*): the GA's device draws / operators on chosen inputs ----
def debug_rng_words(seed: int, lig_index: int, phase: int, gen: int, n_idx: int,
                    n_slot: int) -> np.ndarray:
    out = np.empty((n_idx, n_slot), np.uint64)
    check(lib().vd_debug_rng(0, int(seed), int(lig_index), int(phase), int(gen), int(n_idx),
                             int(n_slot), out.ctypes.data), "vd_debug_rng")
    return out


def debug_rng_normals(seed: int, lig_index: int, phase: int, gen: int, n_idx: int,
                      n_comp: int) -> np.ndarray:
    out = np.empty((n_idx, n_comp), np.float64)
    check(lib().vd_debug_rng(1, int(seed), int(lig_index), int(phase), int(gen), int(n_idx),
                             int(n_comp), out.ctypes.data), "vd_debug_rng")
    return out


def debug_ga_init(params: VdGaParams, n_torsions: int, seed: int, lig_index: int) -> np.ndarray:
    out = np.empty((params.pop, 7 + n_torsions), np.float64)
    check(lib().vd_debug_ga_init(C.byref(params), int(n_torsions), int(seed), int(lig_index),
                                 out.ctypes.data), "vd_debug_ga_init")
    return out


def debug_ga_breed(params: VdGaParams, n_torsions: int, cur: np.ndarray, fitness: np.ndarray,
                   gen: int, seed: int, lig_index: int) -> np.ndarray:
    cur = np.ascontiguousarray(cur, np.float64)
    fit = np.ascontiguousarray(fitness, np.float32)
    out = np.empty((params.pop - params.elitism, 7 + n_torsions), np.float64)
    check(lib().vd_debug_ga_breed(C.byref(params), int(n_torsions), cur.ctypes.data,
                                  fit.ctypes.data, int(gen), int(seed), int(lig_index),
                                  out.ctypes.data), "vd_debug_ga_breed")
    return out


def debug_pose_genes(ligs: LigandSet, lig: int, genes: np.ndarray, tpp: int) -> np.ndarray:
    """(P, 3, N) poses from the fast score kernel's TPP = 4/8 pose stage."""
    g = np.ascontiguousarray(genes, np.float64)
    out = np.empty((g.shape[0], 3, int(ligs.n_atoms[lig])), np.float32)
    check(lib().vd_debug_pose_genes(ligs.handle, int(lig), g.ctypes.data, int(g.shape[0]),
                                    int(tpp), out.ctypes.data), "vd_debug_pose_genes")
    return out
