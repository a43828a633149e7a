"""MUGD grid files (vd/grids.py:232-303; format pinned by pkg/tests/test_grids.py:206-272)
against streams written by the REFERENCE's write_grid_set (tests/golden/make_golden.py):
the mirror's host reader and the native header parser of the device loader
(csrc/vd_mugd.cu), including the reference's GridFormatError cases."""

from __future__ import annotations

import shutil
import struct

import numpy as np
import pytest

import fixtures as fx
from paper_2509_12232_b200 import _abi, gridmaps

CASES = ("b", "odd")


def _path(tag):
    return fx.GOLDEN / f"ref_grid_{tag}.mugd"


@pytest.mark.parametrize("tag", CASES)
def test_host_reader_reads_reference_stream(tag):
    d = fx.load("mugd_cases")
    g = gridmaps.read_grid_set(_path(tag))
    assert list(g.maps) == [str(l) for l in d[f"{tag}__labels"]]
    for k, l in enumerate(g.maps):
        assert np.array_equal(g.maps[l].view(np.uint32), d[f"{tag}__stack"][k].view(np.uint32))
    assert g.spec.dims == tuple(int(x) for x in d[f"{tag}__dims"])
    assert np.array_equal(np.float32(g.spec.origin), np.float32(d[f"{tag}__origin"]))


@pytest.mark.parametrize("tag", CASES)
def test_native_header_matches_reference_stream(tag):
    d = fx.load("mugd_cases")
    info, labels = _abi.mugd_header(_path(tag))
    assert labels == [str(l) for l in d[f"{tag}__labels"]]
    assert (info.nx, info.ny, info.nz) == tuple(int(x) for x in d[f"{tag}__dims"])
    assert np.array_equal(np.float32(list(info.origin)), np.float32(d[f"{tag}__origin"]))
    assert np.float32(info.spacing) == np.float32(d[f"{tag}__spacing"])


def _variants(tmp_path):
    raw = _path("odd").read_bytes()
    out = {}
    out["bad magic"] = b"MUGX" + raw[4:]
    out["unsupported MUGD version 2"] = raw[:4] + struct.pack("<I", 2) + raw[8:]
    out["unexpected end of MUGD stream while reading payload of map '@elec'"] = raw[:-13 * 7 * 37 * 4 - 100]
    out["unexpected end of MUGD stream while reading dims"] = raw[:10]
    out["trailing bytes after final map payload"] = raw + b"\0"
    paths = {}
    for k, (msg, blob) in enumerate(out.items()):
        p = tmp_path / f"v{k}.mugd"
        p.write_bytes(blob)
        paths[msg] = p
    return paths


def test_format_errors_match_reference_messages(tmp_path):
    for msg, p in _variants(tmp_path).items():
        with pytest.raises(gridmaps.GridFormatError, match=msg.split(" '")[0]):
            gridmaps.read_grid_set(p)
        with pytest.raises(gridmaps.GridFormatError) as e:
            _abi.mugd_header(p)
        assert msg in str(e.value), (msg, str(e.value))


def test_header_of_missing_file_is_oserror(tmp_path):
    with pytest.raises(OSError):
        _abi.mugd_header(tmp_path / "nope.mugd")
    shutil.copy(_path("b"), tmp_path / "ok.mugd")
    assert _abi.mugd_header(tmp_path / "ok.mugd")[0].n_maps == len(fx.load("mugd_cases")["b__labels"])
