"""CPU-side checks of the native boundary: the library loads without a GPU and
exports exactly the entry points include/vecdock_b200.h declares."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "vecdock_b200.h"
LIB = ROOT / "paper_2509_12232_b200" / "libvdb200.so"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vd_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists():
        pytest.fail(f"{LIB.name} not built: run __graft_entry__.build()")
    return ctypes.CDLL(str(LIB))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("vd_score_genes", "vd_score_poses", "vd_dock_batch", "vd_grid_build",
              "vd_ligands_create", "vd_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_the_exports():
    from paper_2509_12232_b200 import _abi

    assert set(_abi.EXPORTS) == set(declared_symbols())
    L = _abi.load_library()
    assert L.vd_abi_version() == 1


def test_no_device_reports_error_not_crash(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    n = ctypes.c_int(-1)
    rc = lib.vd_device_count(ctypes.byref(n))
    assert rc != 0 or n.value == 0
    lib.vd_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.vd_last_error(), bytes)


def test_product_refuses_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_2509_12232_b200 import BackendUnavailable
    from paper_2509_12232_b200.backend import CudaBackend

    with pytest.raises(BackendUnavailable):
        CudaBackend()
