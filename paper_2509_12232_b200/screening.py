"""Batch virtual screening on one or many B200s.

Mirror of vd/screening.py (ScreenConfig, ScreenEntry, screen_batch,
write_screen_csv; :35-282).  The reference runs one `dock` per ligand on a
work-stealing CPU thread pool (:67-162); here the whole batch is ONE
persistent GA kernel launch per GPU (csrc/vd_ga.cu), and with
torch.distributed initialised the ligands are split into contiguous index
ranges over ranks.  Ligand i always uses seed key (global_seed, i), so
results are bit-identical for any rank count.  The only communication is
one all-gather of fixed-size per-ligand records (NCCL over NVLink on GPUs,
gloo in the CPU tests).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field, replace

import numpy as np

from . import _abi
from .context import ScoreBreakdown, prepare_context
from .ga import DockingResult, GaConfig, _run

REC_HEAD = 5  # best_total, inter64, intra64, n_evals, ok


@dataclass(frozen=True)
class ScreenConfig:
    worker_count: int = 1          # accepted for API parity; the GPU needs no CPU workers
    pin_workers: bool = False
    pin_map: tuple | None = None
    ga: GaConfig = field(default_factory=GaConfig)
    backend: str | None = None
    global_seed: int = 0

    def __post_init__(self):
        if self.worker_count < 1:
            raise ValueError("worker_count must be >= 1")


@dataclass
class ScreenEntry:
    name: str
    result: DockingResult | None
    error: str | None
    wall_ms: float
    seed_key: tuple


def shard_range(n: int, rank: int, world: int):
    """Contiguous, even split of [0, n) by ligand index."""
    per = math.ceil(n / world) if world > 0 else n
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


def _dist():
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return dist
    except Exception:
        pass
    return None


def pack_records(bt, be, ba, ne, bg, ok) -> np.ndarray:
    """(n, REC_HEAD + gstride) f64 per-ligand records for the gather."""
    n = len(bt)
    rec = np.zeros((n, REC_HEAD + bg.shape[1]), np.float64)
    rec[:, 0] = bt
    rec[:, 1] = be
    rec[:, 2] = ba
    rec[:, 3] = ne
    rec[:, 4] = ok
    rec[:, REC_HEAD:] = bg
    return rec


def gather_records(rec: np.ndarray, n_total: int, dist=None, device=None) -> np.ndarray:
    """All-gather equal-size shards of records (rank r holds shard_range(n_total, r, W))."""
    if dist is None:
        return rec
    import torch

    world = dist.get_world_size()
    per = math.ceil(n_total / world)
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    # ranks may hold different max torsion counts (gene widths): agree on the widest
    w = torch.tensor([rec.shape[1]], dtype=torch.int64, device=dev)
    dist.all_reduce(w, op=dist.ReduceOp.MAX)
    width = int(w.item())
    buf = np.zeros((per, width), np.float64)
    buf[: rec.shape[0], : rec.shape[1]] = rec
    t = torch.from_numpy(buf).to(dev)
    out = torch.empty((world * per, width), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(out, t)
    return out.cpu().numpy()[:n_total]


def screen_batch(batch, grid_set, config: ScreenConfig, weights=None, table=None) -> list:
    """Dock every ligand; one ScreenEntry per ligand in input order (vd/screening.py:165-244)."""
    from .backend import get_backend

    entries = list(batch.entries if hasattr(batch, "entries") else batch)
    if not entries:
        raise ValueError("batch is empty")
    b = get_backend(config.backend)
    b.warmup()
    ga = config.ga
    if ga.translation_bounds is None:
        ga = replace(ga, translation_bounds=(grid_set.spec.origin, grid_set.spec.upper))
    dist = _dist()
    rank, world = (dist.get_rank(), dist.get_world_size()) if dist else (0, 1)
    n = len(entries)
    lo, hi = shard_range(n, rank, world)
    gmax = 7 + max(t.n_torsions for _, t in entries)

    # host prep for this shard: the C++ batch path (csrc/vd_host.cpp, bit-identical to
    # prepare_context); if any ligand fails it, fall back per ligand so failures are
    # recorded in place and the batch continues (vd/screening.py:195-203)
    from . import hostprep

    errors = {}
    good = list(range(lo, hi))
    t0 = time.perf_counter()
    grid = b._grid_for_set(grid_set)
    ligs = None
    try:
        batch = hostprep.TopologyBatch.from_topologies([entries[i][1] for i in good])
        ligs = hostprep.ligand_set(
            hostprep.prepare_batch(batch, grid.labels, weights=weights, table=table))
    except Exception:
        # per-ligand Python contexts (stored fragments, exact reference semantics)
        ctxs, ok_idx = [], []
        for idx in good:
            try:
                ctxs.append(prepare_context(entries[idx][1], grid_set, weights=weights,
                                            table=table))
                ok_idx.append(idx)
            except Exception as exc:
                errors[idx] = f"{type(exc).__name__}: {exc}"
        good = ok_idx
        if good:
            _, ligs = _shared_device_set(b, grid_set, ctxs)
    m = hi - lo
    bt = np.full(m, np.nan, np.float32)
    be = np.full(m, np.nan)
    ba = np.full(m, np.nan)
    ne = np.zeros(m, np.int64)
    bg = np.zeros((m, gmax))
    ok = np.zeros(m)
    if good:
        # ligand index i keys its stream (global_seed, i): consecutive index runs share a launch
        for run_lo, run_hi in _runs(good):
            k0 = good.index(run_lo)
            r = _run(grid, ligs, k0, run_hi - run_lo, ga, config.global_seed, run_lo, b._mode(),
                     gmax, trace=False)
            s = slice(run_lo - lo, run_hi - lo)
            bt[s], be[s], ba[s], bg[s], ne[s] = r[0], r[1], r[2], r[3], r[5]
            ok[s] = 1
    wall_ms = (time.perf_counter() - t0) * 1e3 / max(1, m)

    rec = pack_records(bt, be, ba, ne, bg, ok)
    allrec = gather_records(rec, n, dist)
    out = []
    for idx, (name, topo) in enumerate(entries):
        r = allrec[idx]
        key = (config.global_seed, idx)
        if r[4] != 1:
            err = errors.get(idx) or "ligand failed on its rank"
            out.append(ScreenEntry(name, None, err, float("nan"), key))
            continue
        G = 7 + topo.n_torsions
        tors32 = np.float32(_tors_weight(weights) * topo.n_torsions)
        res = DockingResult(
            best_genotype=r[REC_HEAD:REC_HEAD + G].copy(),
            best_score=ScoreBreakdown.from_components(r[1], r[2], tors32),
            trace=np.empty(0, np.float32),
            n_evaluations=int(r[3]),
            seed_key=key,
        )
        out.append(ScreenEntry(name, res, None, wall_ms, key))
    return out


def _tors_weight(weights):
    from .chem import TermWeights

    return (weights or TermWeights()).tors


def _runs(indices):
    """Maximal runs of consecutive integers in a sorted list -> [(lo, hi), ...]."""
    runs = []
    for i in indices:
        if runs and runs[-1][1] == i:
            runs[-1][1] += 1
        else:
            runs.append([i, i + 1])
    return [tuple(r) for r in runs]


def _shared_device_set(backend, grid_set, ctxs):
    grid = backend._grid_for_set(grid_set)
    where = {l: k for k, l in enumerate(grid.labels)}
    maps = []
    for c in ctxs:
        slot_to_map = np.array([where[l] for l in c.map_labels], np.int32)
        maps.append(slot_to_map[np.asarray(c.atom_slot, np.int64)])
    ligs = _abi.LigandSet(ctxs, maps, where["@elec"], where["@desolv"])
    return grid, ligs


SCREEN_CSV_COLUMNS = ["name", "best_total", "inter", "intra", "torsional", "generations",
                      "wall_ms", "seed"]


def write_screen_csv(entries, sink, generations: int | None = None) -> None:
    """vd/screening.py:247-282 column set."""
    import csv

    own = isinstance(sink, str) or hasattr(sink, "__fspath__")
    f = open(sink, "w", newline="") if own else sink
    try:
        w = csv.writer(f)
        w.writerow(SCREEN_CSV_COLUMNS)
        for e in entries:
            seed = f"{e.seed_key[0]}:{e.seed_key[1]}"
            if e.result is None:
                w.writerow([e.name, "nan", "nan", "nan", "nan", 0, f"{e.wall_ms:.3f}", seed])
                continue
            s = e.result.best_score
            gens = len(e.result.trace) - 1 if len(e.result.trace) else (generations or 0)
            w.writerow([e.name, repr(s.total), repr(s.inter), repr(s.intra), repr(s.torsional),
                        gens, f"{e.wall_ms:.3f}", seed])
    finally:
        if own:
            f.close()
