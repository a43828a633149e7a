"""The device GA's randomness and operators, draw for draw, against the oracle's
independent restatement (oracle/or_rng.c, oracle/vd_ga_oracle.c; no product
source is compiled into the oracle).

Each test runs the GA kernel's own device functions through the vd_debug_*
probes (csrc/vd_ga.cu) on >= 1e5 draws per phase and requires bit equality.
The oracle stream itself is pinned to numpy's Philox/Generator and to libm in
tests/test_host_cpu.py.  Reference draw sites: vd/ga.py:74-77 (key),
:90-109 (init), :139-174 (breed).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

PH_INIT_U, PH_INIT_N, PH_BREED_U, PH_BREED_N = 1, 2, 3, 4


@pytest.fixture(scope="module")
def abi():
    from paper_2509_12232_b200 import _abi

    _abi.ensure_device(0)
    return _abi


def _vd_params(abi, pop, elitism=1, tournament=2, cx=0.8, mut=0.02, lo=(-11.8, -9.0, -7.5),
               hi=(11.8, 9.0, 7.5)):
    p = abi.VdGaParams()
    p.pop, p.generations, p.tournament, p.elitism = pop, 1, tournament, elitism
    p.cx_rate, p.mut_rate = cx, mut
    p.sigma_t, p.sigma_r, p.sigma_tor = 0.5, 0.1, 0.4
    p.lo[:], p.hi[:] = list(lo), list(hi)
    q = oracle.OrGaParams()
    for f, _ in abi.VdGaParams._fields_:
        if f in ("lo", "hi"):
            getattr(q, f)[:] = list(getattr(p, f))
        else:
            setattr(q, f, getattr(p, f))
    return p, q


@pytest.mark.parametrize("phase", [PH_INIT_U, PH_INIT_N, PH_BREED_U, PH_BREED_N])
@pytest.mark.parametrize("seed,lig,gen", [(0, 0, 0), (2**63 + 11, 99_999, 199)])
def test_words_bit_identical(abi, phase, seed, lig, gen):
    n_idx, n_slot = 4096, 32  # 131,072 words
    dev = abi.debug_rng_words(seed, lig, phase, gen, n_idx, n_slot)
    ref = oracle.rng_words(seed, lig, phase, gen, n_idx, n_slot)
    assert np.array_equal(dev, ref)


@pytest.mark.parametrize("phase", [PH_INIT_N, PH_BREED_N])
@pytest.mark.parametrize("seed,lig,gen", [(0, 0, 0), (7, 12_345, 57)])
def test_normals_bit_identical(abi, phase, seed, lig, gen):
    n_idx, n_comp = 32768, 4  # 131,072 normals
    dev = abi.debug_rng_normals(seed, lig, phase, gen, n_idx, n_comp)
    ref = oracle.rng_normals(seed, lig, phase, gen, n_idx, n_comp)
    assert np.array_equal(dev.view(np.uint64), ref.view(np.uint64))
    assert abs(ref.mean()) < 0.02 and abs(ref.std() - 1.0) < 0.02


@pytest.mark.parametrize("T", [0, 12, 32])
def test_init_population_bit_identical(abi, T):
    p, q = _vd_params(abi, pop=8192)
    for seed, lig in ((0, 0), (3, 4321)):
        dev = abi.debug_ga_init(p, T, seed, lig)
        ref = oracle.init_population(q, T, (seed, lig))
        assert np.array_equal(dev.view(np.uint64), ref.view(np.uint64)), (T, seed, lig)


def _population(rng, pop, T, degenerate=0):
    g = np.empty((pop, 7 + T))
    g[:, :3] = rng.uniform(-10, 10, (pop, 3))
    q = rng.standard_normal((pop, 4))
    g[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
    g[:, 7:] = rng.uniform(-np.pi, np.pi, (pop, T))
    if degenerate:
        g[:degenerate, 3:7] *= 1e-12  # |q| < 1e-9 after crossover -> parent-1 fallback
    return g


@pytest.mark.parametrize("kw", [dict(), dict(mut=0.35), dict(elitism=5, tournament=3, cx=0.5),
                                dict(tournament=1, cx=1.0, mut=0.6)])
def test_breed_bit_identical(abi, kw):
    """Tournament ints, crossover flag/cuts, mutation flags and normals: ~2e5+ draws."""
    rng = np.random.default_rng(17)
    pop, T = 8192, 12
    p, q = _vd_params(abi, pop=pop, **kw)
    cur = _population(rng, pop, T, degenerate=64)
    fit = np.round(rng.normal(0, 50, pop)).astype(np.float32)  # many ties: first index wins
    for gen, (seed, lig) in ((0, (0, 0)), (123, (5, 777))):
        dev = abi.debug_ga_breed(p, T, cur, fit, gen, seed, lig)
        ref = oracle.next_generation(q, T, cur, fit.astype(np.float64), gen, (seed, lig))
        assert np.array_equal(dev.view(np.uint64), ref[p.elitism:].view(np.uint64)), (kw, gen)
