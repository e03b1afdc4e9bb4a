"""The C-ABI library loads and exports every symbol include/rbffd_b200.h
declares; parameter validation happens before any CUDA call.  CPU only: no
compute call is made here."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2107_03632_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "rbffd_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rbf_[a-z_]+)\s*\(", text)))


def test_library_builds_and_loads():
    lib = _lib.load()
    assert lib.rbf_version() == 1


def test_every_declared_symbol_is_exported():
    lib = _lib.load()
    syms = declared_symbols()
    assert set(syms) == set(_lib.EXPORTED)
    for name in syms:
        assert hasattr(lib, name), name


def test_status_codes_match_header():
    text = HEADER.read_text()
    for name in ("RBF_OK", "RBF_ERR_CUDA", "RBF_ERR_PARAM", "RBF_ERR_INSTABILITY",
                 "RBF_ERR_TIMEOUT", "RBF_RENUMBER_MORTON", "RBF_NO_RESIDENT", "RBF_NO_PDL"):
        m = re.search(rf"#define {name} (\S+)", text)
        assert m, name
        assert int(m.group(1).rstrip("u"), 0) == getattr(_lib, name)


def test_plan_info_layout():
    text = HEADER.read_text()
    body = re.search(r"typedef struct rbf_plan_info \{(.*?)\} rbf_plan_info;", text, re.S).group(1)
    fields = re.findall(r"\b(\w+)\s*[;,]", re.sub(r"/\*.*?\*/", "", body, flags=re.S))
    assert [f for f, _ in _lib.PlanInfo._fields_] == fields


@pytest.mark.parametrize(
    "N,N_i,n",
    [(0, 0, 1), (10, 11, 3), (10, 5, 0), (2**31, 1, 1)],
)
def test_plan_create_rejects_bad_sizes_before_touching_cuda(N, N_i, n):
    lib = _lib.load()
    h = ctypes.c_void_p()
    z = np.zeros(16)
    rc = lib.rbf_plan_create(ctypes.byref(h), N, N_i, n, z.ctypes.data, z.ctypes.data,
                             z.ctypes.data, z.ctypes.data, None, 0, 0)
    assert rc == _lib.RBF_ERR_PARAM
    assert _lib.last_error(lib)


def test_plan_create_rejects_bad_interior_before_touching_cuda():
    lib = _lib.load()
    h = ctypes.c_void_p()
    rows = np.zeros((2, 3), dtype=np.int64)
    w = np.zeros((2, 3))
    f = np.zeros(2)
    for interior in (np.array([1, 1]), np.array([-1, 2]), np.array([2, 9])):
        interior = interior.astype(np.int64)
        rc = lib.rbf_plan_create(ctypes.byref(h), 5, 2, 3, interior.ctypes.data, rows.ctypes.data,
                                 w.ctypes.data, f.ctypes.data, None, 0, 0)
        assert rc == _lib.RBF_ERR_PARAM, interior
    rc = lib.rbf_plan_create(ctypes.byref(h), 5, 2, 3, np.array([3, 4]).ctypes.data,
                             rows.ctypes.data, w.ctypes.data, f.ctypes.data, None, 0,
                             _lib.RBF_RENUMBER_MORTON)
    assert rc == _lib.RBF_ERR_PARAM  # morton without positions


def test_sass_is_native_sm100a_without_fma_in_the_update():
    """The library carries sm_100a SASS; the 15-wide step kernel's update uses
    separate DMUL/DADD (DFMA only appears in the residual's IEEE division)."""
    import shutil
    import subprocess

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not on PATH")
    out = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out
    parts = re.split(r"\n\s+Function : ", out)
    body = next(p for p in parts if p.startswith("_ZN3rbf18step_stream_kernelILi15E"))
    assert len(re.findall(r"\bDMUL\b", body)) >= 16
    assert len(re.findall(r"\bDADD\b", body)) >= 17
