"""BenchRecord CSV rows for the `cuda` backend.

Same columns, modeled flop/byte constants and byte-stable CSV rules as the
reference's harness (vd/bench.py:118-171, 322-341), so the reference's report
tooling (`vecdock-report speedup|roofline`, pkg/frontend/src/roofline.ts:28-30)
and its `speedup_vs_reference` column work unchanged on GPU rows.
"""

from __future__ import annotations

import csv
import io
import math
from dataclasses import dataclass, fields

import numpy as np


@dataclass
class BenchRecord:
    scenario: str
    backend: str
    threads: int
    mean_ms: float
    stddev_ms: float
    cv: float
    ligands_per_s: float
    modeled_flops: float
    modeled_bytes: float
    modeled_ai: float
    speedup_vs_reference: float
    n_samples: int
    lane_utilization: float
    status: str = "ok"


BENCH_CSV_COLUMNS = [f.name for f in fields(BenchRecord)]

# the reference's stated model (vd/bench.py:139-171): exp/sqrt/div count as 1 flop
PAIR_FLOP_COUNT = 32
ATOM_FLOP_COUNT = 107
PAIR_BYTE_COUNT = 46
ATOM_BYTE_COUNT = 120


def modeled_work(n_pairs: int, n_atoms: int, population: int, generations: int):
    """(flops, bytes) of one docking run: population * generations evaluations
    (the initial-population pass is excluded, as in vd/bench.py:174-186)."""
    ev = float(population) * generations
    return (ev * (PAIR_FLOP_COUNT * n_pairs + ATOM_FLOP_COUNT * n_atoms),
            ev * (PAIR_BYTE_COUNT * n_pairs + ATOM_BYTE_COUNT * n_atoms))


def make_record(scenario: str, backend: str, samples_ms, n_ligands: int, flops: float,
                nbytes: float, warmup_discard: int = 0, lane_utilization: float = 1.0,
                threads: int = 1) -> BenchRecord:
    """Summary over samples[warmup_discard:] (vd/bench.py:279-281)."""
    s = np.asarray(samples_ms, dtype=np.float64)[warmup_discard:]
    mean = float(s.mean())
    sd = float(s.std(ddof=1)) if len(s) > 1 else 0.0
    return BenchRecord(scenario=scenario, backend=backend, threads=threads, mean_ms=mean,
                       stddev_ms=sd, cv=sd / mean if mean else math.nan,
                       ligands_per_s=n_ligands / (mean / 1e3), modeled_flops=float(flops),
                       modeled_bytes=float(nbytes),
                       modeled_ai=float(flops) / float(nbytes) if nbytes else math.nan,
                       speedup_vs_reference=math.nan, n_samples=len(s),
                       lane_utilization=float(lane_utilization))


def fill_speedups(records):
    """speedup_vs_reference = reference mean / backend mean at equal threads."""
    ref = {(r.scenario, r.threads): r for r in records
           if r.backend == "reference" and r.status == "ok"}
    for r in records:
        if r.status != "ok":
            continue
        base = ref.get((r.scenario, r.threads))
        if r.backend == "reference":
            r.speedup_vs_reference = 1.0
        elif base is not None:
            r.speedup_vs_reference = base.mean_ms / r.mean_ms
    return records


def _fmt(v):
    return repr(v) if isinstance(v, float) else str(v)


def emit_csv(records, sink=None) -> str:
    out = io.StringIO()
    w = csv.writer(out, lineterminator="\n")
    w.writerow(BENCH_CSV_COLUMNS)
    for r in sorted(records, key=lambda r: (r.scenario, r.backend, r.threads)):
        w.writerow([_fmt(getattr(r, k)) for k in BENCH_CSV_COLUMNS])
    text = out.getvalue()
    if sink is not None:
        own = isinstance(sink, str) or hasattr(sink, "__fspath__")
        f = open(sink, "w", newline="") if own else sink
        try:
            f.write(text)
        finally:
            if own:
                f.close()
    return text


def parse_csv(text: str):
    rows = list(csv.reader(io.StringIO(text)))
    if not rows or rows[0] != BENCH_CSV_COLUMNS:
        raise ValueError("not a BenchRecord CSV (header mismatch)")
    types = {f.name: f.type for f in fields(BenchRecord)}
    out = []
    for row in rows[1:]:
        kw = {}
        for k, v in zip(BENCH_CSV_COLUMNS, row):
            t = types[k]
            kw[k] = int(v) if t in (int, "int") else float(v) if t in (float, "float") else v
        out.append(BenchRecord(**kw))
    return out
