"""ctypes binding of libsnop_cuda.so (the C-ABI declared in include/snop_cuda.h).

The product path has no CPU fallback: if the in-tree shared library is missing or no B200 is
visible, every call raises. ``load()`` only needs the .so (used by CPU tests that check the
exported symbols); ``Context()`` needs a GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from ._types import STATUS_NAMES, SnopCtxOptions, SnopDatasetInfo, SnopGrfSpec, SnopGrid, SnopModelInfo, SnopSolverConfig
from .errors import raise_for_status

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["SNOP_LIB"]) if os.environ.get("SNOP_LIB") else PKG / "libsnop_cuda.so"

# Every entry point include/snop_cuda.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = [
    "snop_abi_version", "snop_last_error", "snop_ctx_create", "snop_ctx_destroy", "snop_ctx_synchronize",
    "snop_ctx_launch_count", "snop_ctx_stream", "snop_gauss_legendre", "snop_source_iteration_batched",
    "snop_power_iteration_batched", "snop_recast_source", "snop_deeponet_create", "snop_fno_create",
    "snop_exact_operator_create", "snop_op_destroy", "snop_op_predict", "snop_recast_fixed_point",
    "snop_precondition_fixed_source", "snop_sp_eigen_batched", "snop_cp_eigen_batched",
    "snop_op_save", "snop_op_load", "snop_model_write_deeponet", "snop_model_write_fno", "snop_model_inspect",
    "snop_grf_sample", "snop_normalize_source", "snop_generate_dataset", "snop_dataset_write", "snop_dataset_read",
    "snop_source_iteration_leakage_batched", "snop_balance_report", "snop_ctx_set_options", "snop_ctx_get_options",
    "snop_sweep_batched", "snop_power_iteration_operator_batched",
]

_lib = None

vp = C.c_void_p
i32 = C.c_int32
dbl = C.c_double


def load():
    """Load the in-tree libsnop_cuda.so (raises ImportError loudly when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} not found: build the CUDA extension first (python -c 'import __graft_entry__ as g; g.build()'"
            " or make -C paper_2509_01416_b200/csrc). There is no CPU fallback.")
    lib = C.CDLL(str(LIB_PATH))
    lib.snop_abi_version.restype = i32
    lib.snop_last_error.restype = C.c_char_p
    lib.snop_ctx_create.argtypes = [i32, C.POINTER(vp)]
    lib.snop_ctx_destroy.argtypes = [vp]
    lib.snop_ctx_synchronize.argtypes = [vp]
    lib.snop_ctx_launch_count.argtypes = [vp]
    lib.snop_ctx_launch_count.restype = C.c_int64
    lib.snop_ctx_stream.argtypes = [vp]
    lib.snop_ctx_stream.restype = vp
    lib.snop_ctx_set_options.argtypes = [vp, C.POINTER(SnopCtxOptions)]
    lib.snop_ctx_get_options.argtypes = [vp, C.POINTER(SnopCtxOptions)]
    lib.snop_gauss_legendre.argtypes = [i32, vp, vp]
    lib.snop_source_iteration_batched.argtypes = [
        vp, i32, C.POINTER(SnopGrid), i32, i32, vp, vp, vp, vp, C.POINTER(SnopSolverConfig), vp, vp, vp, vp, vp]
    lib.snop_power_iteration_batched.argtypes = [
        vp, i32, C.POINTER(SnopGrid), i32, i32, i32, vp, vp, vp, vp, vp, C.POINTER(SnopSolverConfig), vp, vp, vp,
        vp, vp, vp, vp]
    lib.snop_recast_source.argtypes = [vp, i32, i32, i32, vp, vp, vp, vp, dbl, dbl, vp]
    lib.snop_sweep_batched.argtypes = [vp, i32, C.POINTER(SnopGrid), i32, i32, vp, vp, i32, i32, vp, vp, vp]
    lib.snop_deeponet_create.argtypes = [vp, C.POINTER(SnopGrid), dbl, dbl, i32, i32, vp, vp, i32, vp, vp, i32,
                                         C.c_float, C.POINTER(vp)]
    lib.snop_fno_create.argtypes = [vp, C.POINTER(SnopGrid), dbl, dbl, i32, i32, i32, i32, i32, vp, C.POINTER(vp)]
    lib.snop_exact_operator_create.argtypes = [vp, C.POINTER(SnopGrid), i32, dbl, dbl, C.POINTER(SnopSolverConfig),
                                               C.POINTER(vp)]
    lib.snop_op_destroy.argtypes = [vp]
    lib.snop_op_predict.argtypes = [vp, vp, i32, i32, vp, vp]
    lib.snop_recast_fixed_point.argtypes = [vp, vp, i32, i32, vp, vp, vp, dbl, i32, i32, vp, vp, vp, vp]
    lib.snop_precondition_fixed_source.argtypes = [vp, vp, i32, i32, i32, vp, vp, vp, vp, dbl, i32,
                                                   C.POINTER(SnopSolverConfig), vp, vp, vp, vp, vp]
    lib.snop_power_iteration_operator_batched.argtypes = [
        vp, vp, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, C.POINTER(SnopSolverConfig), dbl, i32, vp, vp, vp, vp,
        vp, vp]
    for fn in ("snop_sp_eigen_batched", "snop_cp_eigen_batched"):
        getattr(lib, fn).argtypes = [vp, vp, i32, i32, i32, i32, vp, vp, vp, vp, vp, C.POINTER(SnopSolverConfig), dbl,
                                     i32, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    lib.snop_op_save.argtypes = [vp, C.c_char_p]
    lib.snop_op_load.argtypes = [vp, C.c_char_p, C.POINTER(vp)]
    lib.snop_model_write_deeponet.argtypes = [C.c_char_p, C.POINTER(SnopGrid), dbl, dbl, i32, i32, vp, vp, i32, vp,
                                              vp, i32, C.c_float]
    lib.snop_model_write_fno.argtypes = [C.c_char_p, C.POINTER(SnopGrid), dbl, dbl, i32, i32, i32, i32, i32, vp]
    lib.snop_model_inspect.argtypes = [C.c_char_p, C.POINTER(SnopModelInfo)]
    lib.snop_grf_sample.argtypes = [vp, i32, C.POINTER(SnopGrid), C.POINTER(SnopGrfSpec), C.c_int64, i32, vp, vp]
    lib.snop_normalize_source.argtypes = [vp, i32, C.POINTER(SnopGrid), i32, vp, vp]
    lib.snop_generate_dataset.argtypes = [vp, i32, C.POINTER(SnopGrid), i32, C.POINTER(SnopGrfSpec), i32, dbl, dbl,
                                          dbl, vp, vp, vp]
    lib.snop_dataset_write.argtypes = [C.c_char_p, C.POINTER(SnopDatasetInfo), vp, vp]
    lib.snop_dataset_read.argtypes = [C.c_char_p, C.POINTER(SnopDatasetInfo), vp, vp]
    lib.snop_source_iteration_leakage_batched.argtypes = [
        vp, i32, C.POINTER(SnopGrid), i32, i32, vp, vp, vp, vp, C.POINTER(SnopSolverConfig), vp, vp, vp, vp, vp, vp]
    lib.snop_balance_report.argtypes = [vp, i32, C.POINTER(SnopGrid), i32, vp, vp, vp, vp, vp, vp]
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != 0:
        raise_for_status(status, load().snop_last_error().decode(errors="replace"))


__all__ = ["load", "check", "LIB_PATH", "EXPORTS", "STATUS_NAMES"]
