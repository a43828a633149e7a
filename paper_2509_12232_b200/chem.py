"""Force-field constants, term weights and the atom-type parameter table.

Host-side mirror of the reference's model chemistry.  The numbers are the
reference's (they *are* the scoring function); the code is ours.

* constants ........ vd/energy.py:17-34
* TermWeights ...... vd/energy.py:37-54
* closed forms ..... vd/energy.py:57-109 (used by host prep and the grid builder)
* AtomParams ....... vd/model.py:19-39
* ParameterTable ... vd/io_formats.py:34-123, data vd/data/parameters.txt:4-13
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# --- constants (vd/energy.py:17-34) ---------------------------------------
ELEC_SCALE = 332.06363            # kcal/mol * A / e^2
DIEL_A = -8.5525                  # Mehler-Solmajer sigmoidal dielectric
DIEL_B = 78.4 - DIEL_A
DIEL_K = 7.7839
DIEL_LAMBDA = 0.003627
DIEL_LAMB = DIEL_LAMBDA * DIEL_B  # folded exponent, vd/scoring/__init__.py:42
DESOLV_SIGMA = 3.6
DESOLV_DENOM = 2.0 * DESOLV_SIGMA * DESOLV_SIGMA
QASP = 0.01097
MIN_R2 = 0.01
MIN_R = 0.1
BOX_PENALTY_SCALE = 1.0e4         # vd/scoring/__init__.py:44

ELEC_LABEL = "@elec"              # vd/grids.py:22-23
DESOLV_LABEL = "@desolv"


@dataclass(frozen=True)
class TermWeights:
    """AutoDock4 free-energy term weights (vd/energy.py:37-54)."""

    vdw: float = 0.1662
    hbond: float = 0.1209
    elec: float = 0.1406
    desolv: float = 0.1322
    tors: float = 0.2983

    def __post_init__(self):
        for name in ("vdw", "hbond", "elec", "desolv", "tors"):
            v = getattr(self, name)
            if not (np.isfinite(v) and v >= 0):
                raise ValueError(f"term weight {name!r} must be finite and >= 0, got {v}")


# --- closed forms (float64; vd/energy.py:57-109) -----------------------------
# Same float64 expression shapes as the reference so folded f32 coefficients
# come out bit-identical (numpy power for integer exponents goes through pow).
def lj_coefficients(r_eq, eps):
    r = np.asarray(r_eq, dtype=np.float64)
    return eps * r**12, 2.0 * eps * r**6


def hb_coefficients(r_eq, eps):
    r = np.asarray(r_eq, dtype=np.float64)
    return 5.0 * eps * r**12, 6.0 * eps * r**10


def distance_dielectric(r):
    r = np.asarray(r, dtype=np.float64)
    return DIEL_A + DIEL_B / (1.0 + DIEL_K * np.exp(-DIEL_LAMBDA * DIEL_B * r))


def desolvation_coefficient(sol_i, vol_i, q_i, sol_j, vol_j, q_j):
    return sol_i * vol_j + sol_j * vol_i + QASP * (np.abs(q_i) * vol_j + np.abs(q_j) * vol_i)


# --- atom types ---------------------------------------------------------------
@dataclass(frozen=True)
class AtomParams:
    type_label: str
    r_eq: float
    eps: float
    volume: float
    solpar: float
    hbond_acceptor: bool = False
    hbond_donor: bool = False

    def __post_init__(self):
        if not self.type_label:
            raise ValueError("atom type label must be non-empty")
        if not self.r_eq > 0:
            raise ValueError(f"type {self.type_label!r}: r_eq must be > 0, got {self.r_eq}")
        if self.eps < 0 or self.volume < 0:
            raise ValueError(f"type {self.type_label!r}: eps and volume must be >= 0")


class ParameterTable:
    """Ordered atom-type table, indexable by position or label."""

    def __init__(self, entries):
        entries = list(entries)
        if not entries:
            raise ValueError("parameter table is empty")
        self._entries = entries
        self._index = {}
        for k, e in enumerate(entries):
            if e.type_label in self._index:
                raise ValueError(f"duplicate atom type label(s): [{e.type_label!r}]")
            self._index[e.type_label] = k

    def __len__(self):
        return len(self._entries)

    def __iter__(self):
        return iter(self._entries)

    def __contains__(self, label):
        return label in self._index

    def __getitem__(self, key):
        return self._entries[self._index[key]] if isinstance(key, str) else self._entries[key]

    def index_of(self, label: str) -> int:
        try:
            return self._index[label]
        except KeyError:
            raise KeyError(f"unknown atom type label {label!r}") from None

    @property
    def labels(self):
        return [e.type_label for e in self._entries]

    def column(self, name: str, dtype=np.float64) -> np.ndarray:
        return np.array([getattr(e, name) for e in self._entries], dtype=dtype)

    def solpar_array(self) -> np.ndarray:
        return self.column("solpar", np.float32)


def parse_parameter_table(text: str) -> ParameterTable:
    """Whitespace table: label r_eq eps volume solpar hbond(0|A|D); '#' comments."""
    rows = []
    for n, raw in enumerate(text.splitlines(), start=1):
        body = raw.partition("#")[0].split()
        if not body:
            continue
        if len(body) != 6:
            raise ValueError(f"line {n}: expected 6 fields, got {len(body)}")
        label, r_eq, eps, vol, sol, flag = body
        if flag not in ("0", "A", "D"):
            raise ValueError(f"line {n}: hbond flag must be 0, A, or D, got {flag!r}")
        rows.append(AtomParams(label, float(r_eq), float(eps), float(vol), float(sol),
                               hbond_acceptor=flag == "A", hbond_donor=flag == "D"))
    return ParameterTable(rows)


# AutoDock4-convention defaults (values of vd/data/parameters.txt:4-13).
_DEFAULT_ROWS = (
    ("C", 4.00, 0.150, 33.5103, -0.00143, "0"),
    ("A", 4.00, 0.150, 33.5103, -0.00052, "0"),
    ("N", 3.50, 0.160, 22.4493, -0.00162, "0"),
    ("NA", 3.50, 0.160, 22.4493, -0.00162, "A"),
    ("O", 3.20, 0.200, 17.1573, -0.00251, "0"),
    ("OA", 3.20, 0.200, 17.1573, -0.00251, "A"),
    ("H", 2.00, 0.020, 0.0000, 0.00051, "0"),
    ("HD", 2.00, 0.020, 0.0000, 0.00051, "D"),
    ("S", 4.00, 0.200, 33.5103, -0.00214, "0"),
    ("SA", 4.00, 0.200, 33.5103, -0.00214, "A"),
)
_DEFAULT_TABLE = None


def default_parameter_table() -> ParameterTable:
    global _DEFAULT_TABLE
    if _DEFAULT_TABLE is None:
        _DEFAULT_TABLE = ParameterTable(
            AtomParams(l, r, e, v, s, hbond_acceptor=f == "A", hbond_donor=f == "D")
            for l, r, e, v, s, f in _DEFAULT_ROWS
        )
    return _DEFAULT_TABLE
