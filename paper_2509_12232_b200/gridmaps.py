"""Receptor grid maps: lattice spec, map set, MUGD file I/O, device builder.

Host-side mirror of vd/grids.py (same names, argument meaning and error
messages).  The map *builder* is the B200 kernel `vd_build_grid`
(csrc/gridbuild.cu); this module only validates inputs and moves arrays.

* GridSpec .............. vd/grids.py:38-80
* GridMapSet ............ vd/grids.py:83-119
* build_grid_maps ....... vd/grids.py:122-202 (device: csrc/gridbuild.cu)
* trilinear_lookup ...... vd/grids.py:205-229
* write/read_grid_set ... vd/grids.py:232-303 (MUGD; x-fastest payloads)
* load_grid_set ......... read_grid_set straight to the device (csrc/vd_mugd.cu)
"""

from __future__ import annotations

import io
import struct
from dataclasses import dataclass

import numpy as np

from . import chem
from .chem import DESOLV_LABEL, ELEC_LABEL

MAGIC = b"MUGD"
VERSION = 1
DEFAULT_CUTOFF = 8.0
DEFAULT_SPACING = 0.375


class GridFormatError(ValueError):
    pass


@dataclass(frozen=True)
class GridSpec:
    origin: tuple
    spacing: float
    dims: tuple

    def __post_init__(self):
        if not self.spacing > 0:
            raise ValueError(f"spacing must be > 0, got {self.spacing}")
        if any(int(d) < 2 for d in self.dims):
            raise ValueError(f"need >= 2 nodes per axis, got dims {self.dims}")
        object.__setattr__(self, "origin", tuple(float(v) for v in self.origin))
        object.__setattr__(self, "dims", tuple(int(d) for d in self.dims))

    @property
    def upper(self):
        return tuple(o + (d - 1) * self.spacing for o, d in zip(self.origin, self.dims))

    @property
    def n_nodes(self) -> int:
        return int(np.prod(self.dims))

    def axes(self):
        return tuple(self.origin[k] + self.spacing * np.arange(self.dims[k], dtype=np.float64)
                     for k in range(3))

    def contains(self, point) -> bool:
        p = np.asarray(point, dtype=np.float64)
        return bool(np.all(p >= np.asarray(self.origin)) and np.all(p <= np.asarray(self.upper)))

    @classmethod
    def centered(cls, center, dims, spacing: float) -> "GridSpec":
        dims = tuple(int(d) for d in dims)
        return cls(tuple(float(c) - (d - 1) * spacing / 2.0 for c, d in zip(center, dims)),
                   spacing, dims)


@dataclass(frozen=True)
class GridMapSet:
    """Same-shaped f32 maps keyed by label; C-order (x, y, z), z fastest."""

    spec: GridSpec
    maps: dict

    def __post_init__(self):
        fixed = {}
        for label, arr in self.maps.items():
            a = np.ascontiguousarray(arr, dtype=np.float32)
            if a.shape != self.spec.dims:
                raise ValueError(f"map {label!r} has shape {a.shape}, expected {self.spec.dims}")
            if not np.isfinite(a).all():
                raise ValueError(f"map {label!r} contains non-finite values")
            a.flags.writeable = False
            fixed[label] = a
        object.__setattr__(self, "maps", fixed)

    @property
    def elec_map(self):
        return self.maps[ELEC_LABEL]

    @property
    def desolv_map(self):
        return self.maps[DESOLV_LABEL]

    @property
    def type_labels(self):
        return [k for k in self.maps if not k.startswith("@")]


def trilinear_lookup(map_array: np.ndarray, spec: GridSpec, point) -> float:
    """fp64 8-corner interpolation at an in-box point (cell clamped to the lattice)."""
    u = (np.asarray(point, dtype=np.float64) - np.asarray(spec.origin)) / spec.spacing
    cell = np.clip(np.floor(u).astype(np.int64), 0, np.asarray(spec.dims) - 2)
    f = u - cell
    block = map_array[cell[0]:cell[0] + 2, cell[1]:cell[1] + 2, cell[2]:cell[2] + 2].astype(np.float64)
    for axis in range(3):  # collapse x, then y, then z
        t = float(f[axis])
        block = block[0] * (1.0 - t) + block[1] * t
    return float(block)


def build_grid_maps(protein, spec: GridSpec, probe_types, weights=None, table=None,
                    cutoff: float = DEFAULT_CUTOFF, device: int | None = None) -> GridMapSet:
    """AutoGrid-style maps built on the GPU (csrc/gridbuild.cu).

    fp64 direct sum over receptor atoms in receptor order per node, so the
    result is deterministic; cutoff applies to vdW/H-bond/desolvation only.
    """
    weights = weights or chem.TermWeights()
    table = table or chem.default_parameter_table()
    probe_types = list(probe_types)
    if not probe_types:
        raise ValueError("probe_types must be non-empty")
    for label in probe_types:
        if label not in table:
            raise ValueError(f"probe type {label!r} not in parameter table")
    if float(np.abs(protein.coords).max()) > 1e4:
        raise ValueError("receptor coordinate magnitude exceeds 1e4 A; refusing to grid")
    from . import _abi

    maps = _abi.build_grid(protein, spec, probe_types, weights, table, cutoff, device)
    out = {label: maps[k] for k, label in enumerate(probe_types)}
    out[ELEC_LABEL] = maps[len(probe_types)]
    out[DESOLV_LABEL] = maps[len(probe_types) + 1]
    return GridMapSet(spec=spec, maps=out)


# --- MUGD little-endian container --------------------------------------------
def write_grid_set(grid_set: GridMapSet, sink) -> None:
    own = isinstance(sink, str) or hasattr(sink, "__fspath__")
    f = open(sink, "wb") if own else sink
    try:
        s = grid_set.spec
        f.write(MAGIC + struct.pack("<I3I3ffI", VERSION, *s.dims, *s.origin, s.spacing,
                                    len(grid_set.maps)))
        for label, arr in grid_set.maps.items():
            raw = label.encode("utf-8")
            f.write(struct.pack("<H", len(raw)) + raw)
            f.write(np.asarray(arr, dtype="<f4").transpose(2, 1, 0).tobytes())
    finally:
        if own:
            f.close()


def _take(src, n, what):
    b = src.read(n)
    if len(b) != n:
        raise GridFormatError(f"unexpected end of MUGD stream while reading {what}")
    return b


def read_grid_set(source) -> GridMapSet:
    own = False
    if isinstance(source, (bytes, bytearray)):
        source = io.BytesIO(source)
    elif isinstance(source, str) or hasattr(source, "__fspath__"):
        source, own = open(source, "rb"), True
    try:
        magic = _take(source, 4, "magic")
        if magic != MAGIC:
            raise GridFormatError(f"bad magic {magic!r}, expected {MAGIC!r}")
        (version,) = struct.unpack("<I", _take(source, 4, "version"))
        if version != VERSION:
            raise GridFormatError(f"unsupported MUGD version {version}, expected {VERSION}")
        dims = struct.unpack("<3I", _take(source, 12, "dims"))
        origin = struct.unpack("<3f", _take(source, 12, "origin"))
        (spacing,) = struct.unpack("<f", _take(source, 4, "spacing"))
        (count,) = struct.unpack("<I", _take(source, 4, "map count"))
        spec = GridSpec(origin, spacing, dims)
        nx, ny, nz = dims
        maps = {}
        for _ in range(count):
            (ln,) = struct.unpack("<H", _take(source, 2, "label length"))
            label = _take(source, ln, "label").decode("utf-8")
            flat = np.frombuffer(_take(source, 4 * nx * ny * nz, f"payload of map {label!r}"),
                                 dtype="<f4")
            maps[label] = np.ascontiguousarray(flat.reshape(nz, ny, nx).transpose(2, 1, 0))
        if source.read(1):
            raise GridFormatError("trailing bytes after final map payload (size mismatch)")
        return GridMapSet(spec, maps)
    finally:
        if own:
            source.close()


class _DeviceMaps(dict):
    """Label -> map view of a device-loaded set: the keys are known from the header,
    the host values are downloaded once, on first access (the device path never needs
    them; the oracle and the reference-style map_stack do)."""

    def __init__(self, dgrid):
        super().__init__()
        self._dgrid = dgrid
        self._labels = list(dgrid.labels)
        self._host = None

    def _fill(self):
        if self._host is None:
            stack = self._dgrid.download()
            for k, l in enumerate(self._labels):
                a = stack[k]
                a.flags.writeable = False
                dict.__setitem__(self, l, a)
            self._host = True

    def __contains__(self, label):
        return label in self._labels

    def __iter__(self):
        return iter(self._labels)

    def __len__(self):
        return len(self._labels)

    def keys(self):
        return list(self._labels)

    def __getitem__(self, label):
        if label not in self._labels:
            raise KeyError(label)
        self._fill()
        return dict.__getitem__(self, label)

    def items(self):
        self._fill()
        return [(l, dict.__getitem__(self, l)) for l in self._labels]

    def values(self):
        return [v for _, v in self.items()]


class DeviceGridMapSet:
    """A GridMapSet whose maps were loaded onto the device from a MUGD file."""

    def __init__(self, spec: GridSpec, dgrid):
        self.spec = spec
        self.device_grid = dgrid
        self.maps = _DeviceMaps(dgrid)

    @property
    def elec_map(self):
        return self.maps[ELEC_LABEL]

    @property
    def desolv_map(self):
        return self.maps[DESOLV_LABEL]

    @property
    def type_labels(self):
        return [k for k in self.maps if not k.startswith("@")]


def load_grid_set(source, device: int | None = None) -> DeviceGridMapSet:
    """read_grid_set (vd/grids.py:269-303) with the payloads going file -> pinned host
    staging -> device, transposed there to the z-fastest layout (csrc/vd_mugd.cu).  Same
    GridFormatError messages as read_grid_set."""
    from . import _abi

    dgrid = _abi.grid_from_mugd(source, device)
    info, _ = _abi.mugd_header(source)
    spec = GridSpec(tuple(float(v) for v in info.origin), float(info.spacing),
                    (info.nx, info.ny, info.nz))
    return DeviceGridMapSet(spec, dgrid)
