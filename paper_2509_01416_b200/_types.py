"""ctypes mirrors of the plain-C structs in include/snop_cuda.h (shared by the product binding
and by the test-side oracle binding, which takes the same struct layout)."""
from __future__ import annotations

import ctypes as C


class SnopGrid(C.Structure):
    _fields_ = [("length_cm", C.c_double), ("n_cells", C.c_int32), ("reserved", C.c_int32)]


class SnopSolverConfig(C.Structure):
    _fields_ = [
        ("tolerance", C.c_double),
        ("tolerance_k", C.c_double),
        ("tolerance_phi", C.c_double),
        ("max_inner", C.c_int32),
        ("max_outer", C.c_int32),
        ("bc_left", C.c_int32),
        ("bc_right", C.c_int32),
        ("norm", C.c_int32),
        ("reserved", C.c_int32),
    ]


class SnopModelInfo(C.Structure):
    _fields_ = [
        ("arch", C.c_int32),
        ("grid", SnopGrid),
        ("sigma_t_star", C.c_double),
        ("sigma_s0_star", C.c_double),
        ("activation", C.c_int32),
        ("n_params", C.c_int64),
        ("n_branch", C.c_int32),
        ("n_trunk", C.c_int32),
        ("latent", C.c_int32),
        ("has_bias0", C.c_int32),
        ("bias0", C.c_float),
        ("width", C.c_int32),
        ("modes", C.c_int32),
        ("layers", C.c_int32),
        ("hidden", C.c_int32),
    ]


class SnopGrfSpec(C.Structure):
    _fields_ = [("mean", C.c_double), ("variance", C.c_double), ("length_scale_cm", C.c_double),
                ("jitter", C.c_double), ("seed", C.c_uint64)]


class SnopDatasetInfo(C.Structure):
    _fields_ = [("n_samples", C.c_int64), ("grid", SnopGrid), ("order", C.c_int32), ("reserved", C.c_int32),
                ("spec", SnopGrfSpec), ("sigma_t_star", C.c_double), ("sigma_s0_star", C.c_double),
                ("tolerance", C.c_double)]


class SnopCtxOptions(C.Structure):
    _fields_ = [("cell_cluster", C.c_int32), ("pair_split", C.c_int32), ("pi_tail_cap", C.c_int32),
                ("host_chunks", C.c_int32), ("gemm_engine", C.c_int32), ("fno_dft", C.c_int32),
                ("fno_mix", C.c_int32), ("reserved", C.c_int32 * 9)]


def make_grid(length: float, n_cells: int) -> SnopGrid:
    return SnopGrid(float(length), int(n_cells), 0)


def make_config(tolerance=1e-4, tolerance_k=None, tolerance_phi=None, max_inner=10000, max_outer=5000,
                bc_left=0, bc_right=0, norm=0) -> SnopSolverConfig:
    return SnopSolverConfig(float(tolerance), float(tolerance if tolerance_k is None else tolerance_k),
                            float(tolerance if tolerance_phi is None else tolerance_phi), int(max_inner),
                            int(max_outer), int(bc_left), int(bc_right), int(norm), 0)


STATUS_NAMES = {0: "OK", 1: "INVALID_ARGUMENT", 2: "NUMERICAL_ERROR", 3: "DEGENERATE_PROBLEM",
                4: "IO_ERROR", 5: "CONFIG_ERROR", 6: "CUDA_ERROR"}
