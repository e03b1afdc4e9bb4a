"""ctypes binding of the C ABI in include/rbffd_b200.h (librbffd_b200.so).

There is deliberately no fallback: if the shared library is missing or cannot
be loaded the import of the solver fails loudly.  Build it with
``python -c "import __graft_entry__ as g; g.build()"`` or ``make -C
paper_2107_03632_b200/csrc``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "librbffd_b200.so"

RBF_OK = 0
RBF_ERR_CUDA = 1
RBF_ERR_PARAM = 2
RBF_ERR_INSTABILITY = 4
RBF_ERR_TIMEOUT = 5
RBF_ERR_ILLCOND = 6

RBF_RENUMBER_MORTON = 0x1
RBF_NO_RESIDENT = 0x2
RBF_NO_PDL = 0x4
RBF_STREAM_LDG = 0x8
RBF_NO_CLUSTER = 0x10
RBF_NO_IDX16 = 0x20
RBF_NO_PAIR = 0x80
RBF_PAIR = 0x100
RBF_ACCEPT_ILLCOND = 0x200
RBF_NO_PERSIST = 0x400

RBF_MODE_FIXED = 0
RBF_MODE_STEADY = 1

# every symbol include/rbffd_b200.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "rbf_plan_create",
    "rbf_set_forcing",
    "rbf_set_field",
    "rbf_get_field",
    "rbf_run",
    "rbf_step",
    "rbf_step_kernel",
    "rbf_plan_get_info",
    "rbf_time_step_kernel",
    "rbf_plan_destroy",
    "rbf_last_error",
    "rbf_version",
    "rbf_nccl_unique_id",
    "rbf_plan_set_halo",
    "rbf_group_create",
    "rbf_group_run",
    "rbf_group_destroy",
    "rbf_assemble_weights",
    "rbf_plan_create_assembled",
    "rbf_plan_weight_row_sum_max",
    "rbf_plan_save",
    "rbf_plan_load",
    "rbf_knn",
    "rbf_generate_unit_disk_nodes",
    "rbf_free_host",
    "rbf_group_push_local",
    "rbf_group_push_export",
    "rbf_group_push_import",
    "rbf_group_push_mode",
    "rbf_group_fused",
    "rbf_group_push_off",
    "rbf_error_norms",
    "rbf_host_alloc",
    "rbf_host_free_pinned",
    "rbf_group_set_step_barrier",
    "rbf_knn_subset",
)


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("N", ctypes.c_int64),
        ("N_i", ctypes.c_int64),
        ("n", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("resident", ctypes.c_int32),
        ("renumbered", ctypes.c_int32),
        ("kernel_n", ctypes.c_int32),
        ("grid", ctypes.c_int32),
        ("block", ctypes.c_int32),
        ("variant", ctypes.c_int32),
        ("index_bits", ctypes.c_int32),
        ("device_bytes", ctypes.c_int64),
        ("bytes_per_step", ctypes.c_int64),
        ("launches", ctypes.c_int64),
        ("stream_bytes_per_step", ctypes.c_int64),
        ("pair", ctypes.c_int32),
        ("pair_tiles", ctypes.c_int32),
        ("pair_halo_rows", ctypes.c_int64),
        ("persist", ctypes.c_int32),
        ("persist_grid", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None


def load(path: os.PathLike | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library.  Raises OSError if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    if path is None and os.environ.get("RBFFD_LIB"):  # experiments: an alternative build
        path = os.environ["RBFFD_LIB"]
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise OSError(
            f"{p} not found: the CUDA library is not built "
            "(run `make -C paper_2107_03632_b200/csrc` or __graft_entry__.build())"
        )
    if "RBFFD_NCCL_LIB" not in os.environ:  # the torch-bundled NCCL, loaded lazily by the library
        try:
            import nvidia.nccl as _nccl  # type: ignore

            cand = Path(list(_nccl.__path__)[0]) / "lib" / "libnccl.so.2"
            if cand.exists():
                os.environ["RBFFD_NCCL_LIB"] = str(cand)
        except Exception:
            pass
    lib = ctypes.CDLL(str(p))
    vp, i64, i32, u32, dbl = (
        ctypes.c_void_p,
        ctypes.c_int64,
        ctypes.c_int32,
        ctypes.c_uint32,
        ctypes.c_double,
    )
    pi64 = ctypes.POINTER(ctypes.c_int64)
    pi32 = ctypes.POINTER(ctypes.c_int32)
    pdbl = ctypes.POINTER(ctypes.c_double)
    sig = {
        "rbf_plan_create": ([ctypes.POINTER(vp), i64, i64, i32, vp, vp, vp, vp, vp, i32, u32], i32),
        "rbf_set_forcing": ([vp, vp], i32),
        "rbf_set_field": ([vp, vp], i32),
        "rbf_get_field": ([vp, vp], i32),
        "rbf_run": ([vp, dbl, i64, i32, dbl, i64, i32, pi64, pdbl, pi32, pi64, pdbl], i32),
        "rbf_step": ([vp, dbl], i32),
        "rbf_step_kernel": ([vp, vp, i64, vp, vp, vp, vp, i64, i32, dbl, i64, vp, i32], i32),
        "rbf_plan_get_info": ([vp, ctypes.POINTER(PlanInfo)], i32),
        "rbf_time_step_kernel": ([vp, dbl, i32, pdbl], i32),
        "rbf_plan_destroy": ([vp], None),
        "rbf_last_error": ([], ctypes.c_char_p),
        "rbf_version": ([], i32),
        "rbf_nccl_unique_id": ([ctypes.c_char_p], i32),
        "rbf_plan_set_halo": ([vp, i32, vp, vp, vp, vp, vp], i32),
        "rbf_group_create": ([ctypes.POINTER(vp), i32, vp, vp, ctypes.c_char_p, i32, i32], i32),
        "rbf_group_run": ([vp, dbl, i64, i32, dbl, i64, pi64, pdbl, pi32, pi64, pdbl], i32),
        "rbf_group_destroy": ([vp], None),
        "rbf_assemble_weights": ([vp, i64, vp, i64, i32, i32, vp, pi64, vp, i32], i32),
        "rbf_plan_create_assembled": ([ctypes.POINTER(vp), i64, i64, i32, i32, vp, vp, vp, vp, i32, u32, vp], i32),
        "rbf_plan_weight_row_sum_max": ([vp, pdbl], i32),
        "rbf_plan_save": ([vp, ctypes.c_char_p], i32),
        "rbf_plan_load": ([ctypes.POINTER(vp), ctypes.c_char_p, i32, u32], i32),
        "rbf_knn": ([vp, i64, i32, vp, i32], i32),
        "rbf_generate_unit_disk_nodes": ([ctypes.c_double, vp, i32, vp, vp, vp], i32),
        "rbf_free_host": ([vp], None),
        "rbf_group_push_local": ([vp], i32),
        "rbf_group_push_export": ([vp, vp, i64, vp], i32),
        "rbf_group_push_import": ([vp, i32, vp, i64], i32),
        "rbf_group_push_mode": ([vp], i32),
        "rbf_group_fused": ([vp], i32),
        "rbf_group_push_off": ([vp], i32),
        "rbf_error_norms": ([vp, vp, pdbl, pdbl], i32),
        "rbf_host_alloc": ([i64, ctypes.POINTER(vp)], i32),
        "rbf_host_free_pinned": ([vp], None),
        "rbf_group_set_step_barrier": ([vp, vp, vp], i32),
        "rbf_knn_subset": ([vp, i64, i32, vp, i64, vp, i32], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if path is None or os.environ.get("RBFFD_LIB") == str(path):
        _lib = lib
    return lib


def last_error(lib: ctypes.CDLL | None = None) -> str:
    lib = lib or load()
    msg = lib.rbf_last_error()
    return msg.decode() if msg else ""
