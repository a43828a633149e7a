"""Genetic-algorithm docking, run entirely on the device.

Mirror of vd/ga.py: `GaConfig` (same fields, defaults and validation,
vd/ga.py:25-52), `DockingResult` (:65-71) and `dock` (:180-235).  The loop
(init, score, elitism, tournament, crossover, mutation, renormalisation)
is one persistent CUDA kernel (csrc/vd_ga.cu); the host only uploads the
ligand and reads back the best genotype, its score parts and the trace.

Randomness: the reference keys numpy's Philox with (seed, ligand_index)
(vd/ga.py:74-77) and consumes it sequentially; here the same key drives a
counter-addressed Philox4x64-10 stream (csrc/vd_rng.h), so a run is a pure
function of (seed key, config, inputs) on any number of GPUs.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from . import _abi
from .context import ScoreBreakdown, prepare_context


@dataclass(frozen=True)
class GaConfig:
    population_size: int = 100
    generations: int = 1000
    tournament_size: int = 2
    crossover_rate: float = 0.8
    mutation_rate: float = 0.02
    mutation_sigma_translation: float = 0.5
    mutation_sigma_rotation: float = 0.1
    mutation_sigma_torsion: float = 0.2
    elitism_count: int = 1
    seed: int = 0
    translation_bounds: tuple | None = None

    def __post_init__(self):
        if self.population_size < 2:
            raise ValueError("population_size must be >= 2")
        if not (0 <= self.elitism_count < self.population_size):
            raise ValueError("elitism_count must be in [0, population_size)")
        for name in ("crossover_rate", "mutation_rate"):
            v = getattr(self, name)
            if not (0.0 <= v <= 1.0):
                raise ValueError(f"{name} must be in [0, 1], got {v}")
        if self.tournament_size < 1:
            raise ValueError("tournament_size must be >= 1")
        if self.generations < 0:
            raise ValueError("generations must be >= 0")


@dataclass(frozen=True)
class DockingResult:
    best_genotype: np.ndarray
    best_score: ScoreBreakdown
    trace: np.ndarray
    n_evaluations: int
    seed_key: tuple


def bounds_of(config: GaConfig):
    if config.translation_bounds is None:
        raise ValueError("config.translation_bounds unset; pass the grid box")
    lo = np.asarray(config.translation_bounds[0], dtype=np.float64)
    hi = np.asarray(config.translation_bounds[1], dtype=np.float64)
    if (hi <= lo).any():
        raise ValueError(f"degenerate translation box: lo={lo}, hi={hi}")
    return lo, hi


def ga_params(config: GaConfig) -> _abi.VdGaParams:
    lo, hi = bounds_of(config)
    p = _abi.VdGaParams()
    p.pop, p.generations = config.population_size, config.generations
    p.tournament, p.elitism = config.tournament_size, config.elitism_count
    p.cx_rate, p.mut_rate = config.crossover_rate, config.mutation_rate
    p.sigma_t = config.mutation_sigma_translation
    p.sigma_r = config.mutation_sigma_rotation
    p.sigma_tor = config.mutation_sigma_torsion
    p.lo[:] = [float(v) for v in lo]
    p.hi[:] = [float(v) for v in hi]
    return p


def make_seed_key(global_seed: int, ligand_index: int = 0) -> tuple:
    """The (key0, key1) pair of vd/ga.py:74-77's make_rng."""
    return (int(global_seed), int(ligand_index))


def seed_key_of_rng(rng) -> tuple | None:
    """Recover (seed, ligand) from a numpy Philox Generator made by the reference's make_rng."""
    try:
        st = rng.bit_generator.state
        if st.get("bit_generator") == "Philox":
            k = st["state"]["key"]
            return (int(k[0]), int(k[1]))
    except Exception:
        pass
    return None


def dock(topology, grid_set, config: GaConfig | None = None, backend=None, weights=None,
         table=None, rng=None, seed_key=None, context=None) -> DockingResult:
    """Run the GA for one ligand on the device (vd/ga.py:180-235 semantics)."""
    from .backend import get_backend

    config = config or GaConfig()
    if config.translation_bounds is None:
        config = replace(config, translation_bounds=(grid_set.spec.origin, grid_set.spec.upper))
    if seed_key is None and rng is not None:
        seed_key = seed_key_of_rng(rng)
    if seed_key is None:
        seed_key = (config.seed, 0)
    ctx = context or prepare_context(topology, grid_set, weights=weights, table=table)
    b = get_backend(backend)
    grid, ligs = b.prepared(ctx)
    G = 7 + ctx.n_torsions
    out = _run(grid, ligs, 0, 1, config, seed_key[0], seed_key[1], b._mode(), G)
    bt, be, ba, bg, tr, ne = out
    return DockingResult(
        best_genotype=bg[0, :G].copy(),
        best_score=ScoreBreakdown.from_components(be[0], ba[0], ctx.torsional32),
        trace=tr[0].copy(),
        n_evaluations=int(ne[0]),
        seed_key=tuple(seed_key),
    )


def _run(grid, ligs, first, count, config, seed, base, mode, gstride, trace=True):
    bt = np.empty(count, np.float32)
    be = np.empty(count, np.float64)
    ba = np.empty(count, np.float64)
    bg = np.zeros((count, gstride), np.float64)
    tr = np.empty((count, config.generations + 1), np.float32) if trace else None
    ne = np.empty(count, np.int64)
    _abi.dock_batch(grid, ligs, first, count, ga_params(config), seed, base, mode, bt, be, ba,
                    bg, tr, ne)
    return bt, be, ba, bg, tr, ne
