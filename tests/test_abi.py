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


def _sass_with_lines(tmp_path):
    """nvdisasm -g of every sm_100a cubin in the library: {kernel: [lines]}."""
    import shutil
    import subprocess

    if not (shutil.which("cuobjdump") and shutil.which("nvdisasm")):
        pytest.skip("cuobjdump / nvdisasm not on PATH")
    subprocess.run(["cuobjdump", "-xelf", "all", str(_lib.LIB_PATH)], cwd=tmp_path, check=True,
                   capture_output=True)
    kernels = {}
    for cubin in sorted(tmp_path.glob("*.sm_100a.cubin")):
        text = subprocess.run(["nvdisasm", "-g", "-c", str(cubin)], capture_output=True, text=True,
                              check=True).stdout
        cur = None
        for line in text.splitlines():
            m = re.match(r"^\.text\.(\S+):", line)
            if m:
                cur = kernels.setdefault(m.group(1), [])
            elif cur is not None:
                cur.append(line)
    return kernels


UPDATE_KERNELS = ("step_tma_kernel", "step_stream_kernel", "grid_loop_kernel", "cluster_loop_kernel",
                  "resident_loop_kernel", "pair_tma_kernel", "stream_loop_kernel", "part_loop_kernel")
UNROLLED = ("step_tma_kernel", "stream_loop_kernel", "part_loop_kernel")


def test_sass_is_native_sm100a_without_fma_in_the_update(tmp_path):
    """Every kernel that runs the update (all widths, all loop variants, the
    production TMA ring included) is sm_100a SASS whose only DFMAs are the
    IEEE division of the steady residual (max|u2-u1| / dt): either on a
    source line that calls __ddiv_rn or inside CUDA's out-of-line division
    subroutine.  numba compiles the update to separate fmul/fadd (SURVEY.md
    A.3); a contracted DFMA in the dot product would change bits."""
    kernels = _sass_with_lines(tmp_path)
    src_cache = {}

    def src_line(path, no):
        if path not in src_cache:
            src_cache[path] = Path(path).read_text().splitlines() if Path(path).exists() else []
        lines = src_cache[path]
        return lines[no - 1] if 0 < no <= len(lines) else ""

    checked = 0
    for name, body in kernels.items():
        if not any(k in name for k in UPDATE_KERNELS):
            continue
        checked += 1
        where, sub = None, None
        n_dmul = n_dadd = 0
        for line in body:
            m = re.match(r'^\s*//## File "([^"]+)", line (\d+)', line)
            if m:
                where = (m.group(1), int(m.group(2)))
                continue
            m = re.match(r"^(\$\S+):\s*$", line)
            if m:
                sub = m.group(1)
                continue
            if re.search(r"\bDMUL\b", line):
                n_dmul += 1
            if re.search(r"\bDADD\b", line):
                n_dadd += 1
            if re.search(r"\bDFMA\b", line):
                if sub is not None:
                    assert "div_rn_f64" in sub, (name, sub, line)
                else:
                    assert where is not None and "__ddiv_rn" in src_line(*where), (name, where, line)
        m = re.search(r"ILi(\d+)E", name)
        nj = int(m.group(1)) if m else 0
        if nj > 0 and any(k in name for k in UNROLLED):  # unrolled chain: nj products, nj + 2 sums
            assert n_dmul >= nj and n_dadd >= nj + 2, (name, n_dmul, n_dadd)
    assert checked >= 24 * 8, checked
    # the production kernels of the benchmarked widths are among them
    for k in ("_ZN3rbf15step_tma_kernelILi15ELi15ELi1ELi2E", "_ZN3rbf18stream_loop_kernelILi15ELi15ELi2E",
              "_ZN3rbf18stream_loop_kernelILi30ELi15ELi2E", "_ZN3rbf18stream_loop_kernelILi56ELi8ELi4E",
              "_ZN3rbf16part_loop_kernelILi15ELi15ELi2E"):
        assert any(name.startswith(k) for name in kernels), k
