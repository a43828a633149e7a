"""The `cuda` compute backend and the scoring entry points.

`CudaBackend` satisfies the reference's duck-typed backend protocol
(vd/scoring/__init__.py:210-247 registry; members used at
vd/scoring/__init__.py:275,309,325-343, vd/screening.py:181-182,
vd/bench.py:246-247): `name`, `lane_width`, `inter_one`, `intra_one`,
`score_many`, `dock_population`, `warmup`.  It accepts a ScoringContext built
by either the reference or this package.  Device state (grid maps, the
ligand's CSR record) is uploaded once per grid / context and cached.

The module-level functions mirror vd/scoring/__init__.py:234-346 (same names,
arguments, rounding and errors) with `cuda` as the default backend.
"""

from __future__ import annotations

import os
import threading
import weakref

import numpy as np

from . import _abi, chem
from .context import BackendUnavailable, ScoreBreakdown, ScoringContext, fold_pairs, prepare_context
from .topology import LigandTopology, NonbondPairList

DEFAULT_BACKEND = "cuda"
BACKEND_ENV_VAR = "VECDOCK_BACKEND"
_MODES = {"fast": _abi.MODE_FAST, "exact": _abi.MODE_EXACT}


class _DeviceCache:
    """id(obj) -> value, dropped when obj is garbage collected.  Single-flight: when
    several threads ask for the same object at once (the reference's screen_batch workers
    share one backend, vd/screening.py:212-222), one builds and the others wait for it."""

    def __init__(self):
        self._d = {}
        self._inflight = {}
        self._lock = threading.Lock()

    def get(self, obj, make):
        key = id(obj)
        while True:
            with self._lock:
                hit = self._d.get(key)
                if hit is not None:
                    return hit
                ev = self._inflight.get(key)
                owner = ev is None
                if owner:
                    ev = self._inflight[key] = threading.Event()
            if owner:
                break
            ev.wait()  # the owner finished (or failed: then this thread retries as owner)
        try:
            val = make()
            with self._lock:
                self._d[key] = val
            try:
                weakref.finalize(obj, self._d.pop, key, None)
            except TypeError:  # not weak-referenceable: keep for process lifetime
                pass
            return val
        finally:
            with self._lock:
                self._inflight.pop(key, None)
            ev.set()


class _MapPool:
    """Device grids for reference ScoringContexts, deduplicated by content.

    A reference context carries a private copy of its maps (`map_stack`, the sorted
    needed type maps then @elec/@desolv, vd/scoring/__init__.py:158-161), and the
    reference's screen_batch keeps one context per ligand alive for the whole batch
    (vd/screening.py:195-203).  Uploading each stack would cost ~10-50 MB of device memory
    per ligand.  Instead every distinct map (same grid geometry, equal values) is uploaded
    once into a shared grid; a context only maps its slots to indices of that grid.  When
    a context brings a map not seen before, the pool's grid is rebuilt with it appended
    (grids already handed out stay valid for the contexts that hold them)."""

    def __init__(self):
        self._lock = threading.Lock()
        self._pools = {}

    @staticmethod
    def _digest(m):
        import hashlib

        sample = np.ascontiguousarray(m[::3, ::3, ::3])
        return hashlib.blake2b(sample.tobytes(), digest_size=16).digest()

    def resolve(self, ctx):
        """(DeviceGrid, slot -> grid map index) for a context's map stack."""
        stack = np.asarray(ctx.map_stack, np.float32)
        key = (stack.shape[1:], tuple(np.asarray(ctx.box_lo, np.float32).tolist()),
               tuple(np.asarray(ctx.box_hi, np.float32).tolist()), float(np.float32(ctx.spacing)))
        with self._lock:
            st = self._pools.setdefault(key, {"maps": [], "by_digest": {}, "grid": None})
            where = []
            for k in range(stack.shape[0]):
                m = stack[k]
                cands = st["by_digest"].setdefault(self._digest(m), [])
                idx = next((i for i in cands if np.array_equal(st["maps"][i], m)), None)
                if idx is None:
                    idx = len(st["maps"])
                    st["maps"].append(np.array(m, np.float32, copy=True))
                    cands.append(idx)
                where.append(idx)
            if st["grid"] is None or st["grid"].n_maps < len(st["maps"]):
                st["grid"] = _abi.grid_from_stack(np.stack(st["maps"]), key[1], key[2], key[3])
            return st["grid"], np.asarray(where, np.int32)

    def n_device_maps(self) -> int:
        with self._lock:
            return sum(len(st["maps"]) for st in self._pools.values())


class CudaBackend:
    """B200 backend (thread-per-pose fused kernels, see csrc/vd_device.cuh)."""

    name = "cuda"
    lane_width = 32

    def __init__(self, mode: str = "fast", device: int | None = None):
        if mode not in _MODES:
            raise ValueError(f"mode must be one of {sorted(_MODES)}")
        self.mode = mode
        self.device = device
        self._grids = _DeviceCache()
        self._ligs = _DeviceCache()
        self._pool = _MapPool()
        _abi.lib()  # raise BackendUnavailable now, not mid-run

    # -- device state ------------------------------------------------------
    def _grid_for_set(self, grid_set):
        dg = getattr(grid_set, "device_grid", None)
        if dg is not None:  # loaded straight onto the device (gridmaps.load_grid_set)
            return dg

        def make():
            labels = list(grid_set.maps)
            stack = np.stack([grid_set.maps[l] for l in labels])
            s = grid_set.spec
            return _abi.grid_from_stack(stack, np.asarray(s.origin, np.float32),
                                        np.asarray(s.upper, np.float32), s.spacing, labels)
        return self._grids.get(grid_set, make)

    def prepared(self, ctx):
        """(DeviceGrid, LigandSet) for a context (cached per context object)."""
        _abi.ensure_device(self.device)

        def make():
            n = int(ctx.n_atoms)
            gs = getattr(ctx, "grid_set", None)
            if gs is not None:
                grid = self._grid_for_set(gs)
                where = {l: k for k, l in enumerate(grid.labels)}
                slot_to_map = np.array([where[l] for l in ctx.map_labels], np.int32)
                atom_map = slot_to_map[np.asarray(ctx.atom_slot, np.int64)]
                elec, desolv = where[chem.ELEC_LABEL], where[chem.DESOLV_LABEL]
            else:  # a reference ScoringContext: its private map stack, deduplicated
                grid, where = self._pool.resolve(ctx)
                atom_map = where[np.asarray(ctx.atom_slot, np.int64)]
                elec, desolv = int(where[-2]), int(where[-1])
            view = _PaddedContext(ctx, n)
            atom_map = _pad(atom_map, n, np.int32)
            return grid, _abi.LigandSet([view], [atom_map], elec, desolv)
        return self._ligs.get(ctx, make)

    def _mode(self):
        return _MODES[self.mode]

    # -- backend protocol ----------------------------------------------------
    def dock_population(self, genes: np.ndarray, ctx):
        inter, intra, _ = self.score_population_arrays(genes, ctx)
        return inter, intra

    def score_population_arrays(self, genes, ctx, out=None):
        """(inter64, intra64, total32); genes/outputs may be numpy or torch (host/device)."""
        grid, ligs = self.prepared(ctx)
        g = genes if not isinstance(genes, np.ndarray) else np.ascontiguousarray(genes, np.float64)
        P = g.shape[0]
        if out is None:
            out = (np.empty(P, np.float64), np.empty(P, np.float64), np.empty(P, np.float32))
        _abi.score_genes(grid, ligs, 0, g, *out, mode=self._mode())
        return out

    def score_many(self, poses: np.ndarray, ctx):
        grid, ligs = self.prepared(ctx)
        p = np.ascontiguousarray(poses, np.float32)
        inter = np.empty(p.shape[0], np.float64)
        intra = np.empty(p.shape[0], np.float64)
        _abi.score_poses(grid, ligs, 0, p, inter, intra, mode=self._mode())
        return inter, intra

    def inter_one(self, pose: np.ndarray, ctx) -> float:
        e, _ = self.score_many(np.asarray(pose, np.float32)[None], ctx)
        return float(e[0])

    def intra_one(self, pose: np.ndarray, ctx) -> float:
        if ctx.pair_i is None:
            raise ValueError("context has no pair list (inter-only context)")
        _, a = self.score_many(np.asarray(pose, np.float32)[None], ctx)
        return float(a[0])

    def pose_population(self, genes: np.ndarray, ctx) -> np.ndarray:
        _, ligs = self.prepared(ctx)
        g = np.ascontiguousarray(genes, np.float64)
        out = np.empty((g.shape[0], 3, int(ctx.n_atoms)), np.float32)
        _abi.pose_genes(ligs, 0, g, out)
        return out

    def warmup(self, ctx=None):
        _abi.ensure_device(self.device)
        if ctx is not None:
            self.prepared(ctx)


def _pad(a, n, dtype):
    a = np.asarray(a, dtype).ravel()
    if a.shape[0] >= n:
        return a[:n]
    return np.concatenate([a, np.zeros(n - a.shape[0], dtype)])


class _PaddedContext:
    """Context view whose per-atom arrays cover n_atoms (the reference's
    intra_energy() context carries empty atom arrays, vd/scoring/__init__.py:282-307)."""

    def __init__(self, ctx, n):
        self._c = ctx
        self.n_atoms = n
        self.charge = _pad(ctx.charge, n, np.float32)
        self.desolv_factor = _pad(ctx.desolv_factor, n, np.float32)
        c0 = np.asarray(ctx.pose_centered0, np.float32)
        if c0.shape[1] != n:
            c0 = np.zeros((3, n), np.float32)
        self.pose_centered0 = c0
        empty_i = np.empty(0, np.int32)
        empty_f = np.empty(0, np.float32)
        has = ctx.pair_i is not None
        self.pair_i = ctx.pair_i if has else empty_i
        self.pair_j = ctx.pair_j if has else empty_i
        self.pair_a = ctx.pair_a if has else empty_f
        self.pair_b = ctx.pair_b if has else empty_f
        self.pair_qq = ctx.pair_qq if has else empty_f
        self.pair_desolv = ctx.pair_desolv if has else empty_f
        self.pair_hb = ctx.pair_hb if has else np.empty(0, bool)
        self.n_pairs = int(self.pair_i.shape[0])
        self.frag_axis_a, self.frag_axis_b = ctx.frag_axis_a, ctx.frag_axis_b
        self.frag_start, self.frag_index = ctx.frag_start, ctx.frag_index
        self.n_torsions = int(np.asarray(ctx.frag_axis_a).shape[0])
        self.torsional32 = ctx.torsional32
        self.intra_cutoff2 = ctx.intra_cutoff2
        self.penalty_scale = ctx.penalty_scale


# --- registry mirror (vd/scoring/__init__.py:210-247) --------------------------------
_REGISTRY: dict = {}
_REG_LOCK = threading.Lock()


def _load_backends():
    with _REG_LOCK:
        if _REGISTRY:
            return
        for key, mode in (("cuda", "fast"), ("cuda-exact", "exact")):
            try:
                _REGISTRY[key] = CudaBackend(mode=mode)
            except (BackendUnavailable, OSError) as exc:
                _REGISTRY[key] = BackendUnavailable(f"{key} backend unavailable: {exc}")


def list_backends():
    _load_backends()
    return [k for k, v in _REGISTRY.items() if not isinstance(v, BackendUnavailable)]


def get_backend(name=None):
    _load_backends()
    if name is None:
        name = os.environ.get(BACKEND_ENV_VAR) or DEFAULT_BACKEND
    if isinstance(name, str):
        key = name.lower()
        if key not in _REGISTRY:
            raise ValueError(f"unknown backend {name!r}; choose from {sorted(_REGISTRY)}")
        found = _REGISTRY[key]
        if isinstance(found, BackendUnavailable):
            raise found
        return found
    return name


def register_reference_backend(scoring_module, name: str = "cuda", mode: str = "fast"):
    """Plug CudaBackend into the REFERENCE's registry (vd/scoring/__init__.py:210-226).

    `_load_backends()` is called first: it early-returns on a non-empty
    registry, so registering before it would hide the stock backends.
    """
    scoring_module._load_backends()
    try:
        scoring_module._REGISTRY[name] = CudaBackend(mode=mode)
    except (BackendUnavailable, OSError) as exc:
        scoring_module._REGISTRY[name] = scoring_module.BackendUnavailable(str(exc))
    return scoring_module._REGISTRY[name]


# --- scoring entry points (vd/scoring/__init__.py:250-346) ------------------------------
def inter_energy(pose, type_index, charges, grid_set, backend=None, table=None) -> float:
    table = table or chem.default_parameter_table()
    topo = LigandTopology(pose, type_index, np.asarray(charges, np.float32),
                          np.empty((0, 2), np.int32))
    ctx = prepare_context(topo, grid_set, table=table, pairlist=NonbondPairList.empty())
    b = get_backend(backend)
    return float(np.float32(b.inter_one(np.asarray(pose, np.float32), ctx)))


def intra_energy(pose, pairlist: NonbondPairList, weights=None, backend=None) -> float:
    weights = weights or chem.TermWeights()
    pi, pj, pa, pb, phb, pqq, pdsl = fold_pairs(pairlist, weights)
    n = int(np.asarray(pose).shape[-1])
    z = np.zeros(n, np.float32)
    ctx = ScoringContext(
        atom_slot=np.zeros(n, np.int32), charge=z, desolv_factor=z,
        box_lo=np.zeros(3, np.float32), box_hi=np.ones(3, np.float32),
        spacing=np.float32(1.0), dims=(2, 2, 2), penalty_scale=np.float32(chem.BOX_PENALTY_SCALE),
        pair_i=pi, pair_j=pj, pair_a=pa, pair_b=pb, pair_hb=phb, pair_qq=pqq, pair_desolv=pdsl,
        intra_cutoff2=np.float32(np.inf), torsional32=np.float32(0.0), n_atoms=n,
        pose_centered0=np.zeros((3, n), np.float32), frag_index=np.empty(0, np.int32),
        frag_start=np.zeros(1, np.int32), frag_axis_a=np.empty(0, np.int32),
        frag_axis_b=np.empty(0, np.int32),
        explicit_stack=np.zeros((2, 2, 2, 2), np.float32),
    )
    b = get_backend(backend)
    return float(np.float32(b.intra_one(np.asarray(pose, np.float32), ctx)))


def score_pose(topology, genotype, grid_set, weights=None, backend=None, table=None,
               context=None) -> ScoreBreakdown:
    from .pose import decode_genotype

    ctx = context or prepare_context(topology, grid_set, weights=weights, table=table)
    b = get_backend(backend)
    decode_genotype(genotype, topology)  # the reference's validation (vd/pose.py:29-47)
    g = np.asarray(genotype, np.float64)[None, :]
    if hasattr(b, "dock_population"):
        e, a = b.dock_population(g, ctx)
    else:
        from .pose import apply_pose

        pose = apply_pose(topology, genotype)
        e, a = np.array([b.inter_one(pose, ctx)]), np.array([b.intra_one(pose, ctx)])
    return ScoreBreakdown.from_components(e[0], a[0], ctx.torsional32)


def score_population(topology, genes: np.ndarray, context, backend=None):
    """(inter64, intra64, total32) for a population (vd/scoring/__init__.py:330-346)."""
    b = get_backend(backend)
    if hasattr(b, "score_population_arrays"):
        return b.score_population_arrays(genes, context)
    inter64, intra64 = b.dock_population(np.ascontiguousarray(genes, np.float64), context)
    tot = (inter64.astype(np.float32) + intra64.astype(np.float32)) + context.torsional32
    return inter64, intra64, tot.astype(np.float32)
