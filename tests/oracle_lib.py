"""ctypes binding of the CPU oracle (oracle/_build/libsnop_oracle.so). TEST INFRASTRUCTURE ONLY:
importable from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2509_01416_b200._types import SnopGrid, SnopSolverConfig, make_config, make_grid

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "oracle" / "_build" / "libsnop_oracle.so"

_lib = None

dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
bp = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-C", str(ROOT / "oracle")], check=True, capture_output=True)
        _lib = C.CDLL(str(LIB))
        _lib.oracle_last_error.restype = C.c_char_p
        _lib.oracle_deeponet_create.restype = C.c_void_p
        _lib.oracle_fno_create.restype = C.c_void_p
        _lib.oracle_exact_operator_create.restype = C.c_void_p
        _lib.oracle_hardware_threads.restype = C.c_uint
    return _lib


def _check(code):
    if code != 0:
        raise OracleError(code, lib().oracle_last_error().decode())


def _opt(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(C.c_void_p)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def hardware_threads() -> int:
    return int(lib().oracle_hardware_threads())


def gauss_legendre(order: int):
    mu = np.empty(order)
    w = np.empty(order)
    _check(lib().oracle_gauss_legendre(C.c_int32(order), _p(mu), _p(w)))
    return mu, w


def chunk_bounds(n_items: int, n_chunks: int):
    k = n_items if (n_chunks == 0 or n_chunks > n_items) else n_chunks
    b = np.empty(k + 1, dtype=np.uint64)
    lib().oracle_chunk_bounds(C.c_uint64(n_items), C.c_uint64(n_chunks), _p(b))
    return [(int(b[c]), int(b[c + 1])) for c in range(k)]


def rng_stream(seed: int, n: int):
    u = np.empty(n, dtype=np.uint64)
    f = np.empty(n)
    g = np.empty(n)
    lib().oracle_rng_stream(C.c_uint64(seed), C.c_int32(n), _p(u), C.c_int32(n), _p(f), C.c_int32(n), _p(g))
    return u, f, g


def sweep(length, n_cells, order, sigma_t, emission, bc_left=0, bc_right=0, n_threads=0):
    """Oracle sweep: emission [B][Nc][N] -> psi_avg [B][N][Nc], net outflows [B]."""
    st = np.ascontiguousarray(sigma_t, dtype=np.float64)
    em = np.ascontiguousarray(emission, dtype=np.float64)
    B = st.shape[0]
    psi = np.empty((B, order, n_cells))
    ol = np.empty(B)
    orr = np.empty(B)
    grid = make_grid(length, n_cells)
    _check(lib().oracle_sweep_batched(C.byref(grid), C.c_int32(order), C.c_int32(B), _p(st), _p(em),
                                      C.c_int32(bc_left), C.c_int32(bc_right), _p(psi), _p(ol), _p(orr),
                                      C.c_int32(n_threads)))
    return psi, ol, orr


def source_iteration(length, n_cells, order, sigma_t, sigma_s0, source, cfg: SnopSolverConfig,
                     sigma_s1=None, initial_phi=None, n_threads=0, want_current=False, want_leak=False):
    st = np.ascontiguousarray(sigma_t, dtype=np.float64)
    B = st.shape[0]
    phi = np.empty((B, n_cells))
    cur = np.empty((B, n_cells)) if want_current else None
    it = np.empty(B, dtype=np.int32)
    cv = np.empty(B, dtype=np.uint8)
    leak = np.empty((B, 2)) if want_leak else None
    grid = make_grid(length, n_cells)
    ss = np.ascontiguousarray(sigma_s0, dtype=np.float64)
    src = np.ascontiguousarray(source, dtype=np.float64)
    _check(lib().oracle_source_iteration_batched(
        C.byref(grid), C.c_int32(order), C.c_int32(B), _p(st), _p(ss), _opt(sigma_s1), _p(src), C.byref(cfg),
        _opt(initial_phi), _p(phi), None if cur is None else _p(cur), _p(it), _p(cv),
        None if leak is None else _p(leak), C.c_int32(n_threads)))
    out = {"phi": phi, "iterations": it, "converged": cv.astype(bool)}
    if want_current:
        out["current"] = cur
    if want_leak:
        out["leak"] = leak
    return out


def power_iteration(length, n_cells, order, n_groups, sigma_t, sigma_s0, nu_sigma_f, chi, cfg,
                    sigma_s1=None, initial_k=None, initial_phi=None, n_threads=0):
    st = np.ascontiguousarray(sigma_t, dtype=np.float64)
    B = st.shape[0]
    k = np.empty(B)
    phi = np.empty((B, n_groups, n_cells))
    outer = np.empty(B, dtype=np.int32)
    inner = np.empty(B, dtype=np.int64)
    cv = np.empty(B, dtype=np.uint8)
    grid = make_grid(length, n_cells)
    ss = np.ascontiguousarray(sigma_s0, dtype=np.float64)
    nsf = np.ascontiguousarray(nu_sigma_f, dtype=np.float64)
    ch = np.ascontiguousarray(chi, dtype=np.float64)
    _check(lib().oracle_power_iteration_batched(
        C.byref(grid), C.c_int32(order), C.c_int32(B), C.c_int32(n_groups), _p(st), _p(ss), _opt(sigma_s1),
        _p(nsf), _p(ch), C.byref(cfg), _opt(initial_k), _opt(initial_phi), _p(k), _p(phi), _p(outer), _p(inner),
        _p(cv), C.c_int32(n_threads)))
    return {"k": k, "phi": phi, "outer": outer, "inner": inner, "converged": cv.astype(bool)}


def infinite_medium_k(sigma_t, sigma_s0, nu_sigma_f, chi) -> float:
    G = len(sigma_t)
    k = C.c_double()
    _check(lib().oracle_infinite_medium_k(
        C.c_int32(G), _p(np.ascontiguousarray(sigma_t, dtype=np.float64)),
        _p(np.ascontiguousarray(sigma_s0, dtype=np.float64)), _p(np.ascontiguousarray(nu_sigma_f, dtype=np.float64)),
        _p(np.ascontiguousarray(chi, dtype=np.float64)), C.byref(k)))
    return k.value


def recast_source(S, phi, sigma_t, sigma_s0, tstar, sstar):
    S = np.ascontiguousarray(S, dtype=np.float64)
    out = np.empty_like(S)
    B, n = S.shape
    lib().oracle_recast_source(C.c_int32(B), C.c_int32(n), _p(S), _p(np.ascontiguousarray(phi, dtype=np.float64)),
                               _p(np.ascontiguousarray(sigma_t, dtype=np.float64)),
                               _p(np.ascontiguousarray(sigma_s0, dtype=np.float64)), C.c_double(tstar),
                               C.c_double(sstar), _p(out))
    return out


def balance_residual(length, n_cells, sigma_t, sigma_s0, source, phi, leak_left, leak_right):
    out = C.c_double()
    grid = make_grid(length, n_cells)
    _check(lib().oracle_balance_residual(C.byref(grid), _p(np.ascontiguousarray(sigma_t, dtype=np.float64)),
                                         _p(np.ascontiguousarray(sigma_s0, dtype=np.float64)),
                                         _p(np.ascontiguousarray(source, dtype=np.float64)),
                                         _p(np.ascontiguousarray(phi, dtype=np.float64)), C.c_double(leak_left),
                                         C.c_double(leak_right), C.byref(out)))
    return out.value


class OracleOperator:
    """Oracle SolutionOperator handle (DeepONet / FNO / exact model-based solve at p*)."""

    def __init__(self, handle, n_cells):
        self.h = C.c_void_p(handle)
        self.n_cells = n_cells

    def __del__(self):
        try:
            lib().oracle_op_destroy(self.h)
        except Exception:
            pass

    @classmethod
    def deeponet(cls, length, n_cells, ref_params, activation, branch_sizes, branch_params, trunk_sizes,
                 trunk_params, bias0=None):
        grid = make_grid(length, n_cells)
        bs = np.ascontiguousarray(branch_sizes, dtype=np.int32)
        ts = np.ascontiguousarray(trunk_sizes, dtype=np.int32)
        bpar = np.ascontiguousarray(branch_params, dtype=np.float32)
        tpar = np.ascontiguousarray(trunk_params, dtype=np.float32)
        h = lib().oracle_deeponet_create(C.byref(grid), C.c_double(ref_params[0]), C.c_double(ref_params[1]),
                                         C.c_int32(activation), C.c_int32(len(bs)), _p(bs), _p(bpar),
                                         C.c_int32(len(ts)), _p(ts), _p(tpar), C.c_int32(bias0 is not None),
                                         C.c_float(0.0 if bias0 is None else bias0))
        return cls(h, n_cells)

    @classmethod
    def fno(cls, length, n_cells, ref_params, activation, width, modes, layers, hidden, params):
        grid = make_grid(length, n_cells)
        p = np.ascontiguousarray(params, dtype=np.float32)
        h = lib().oracle_fno_create(C.byref(grid), C.c_double(ref_params[0]), C.c_double(ref_params[1]),
                                    C.c_int32(activation), C.c_int32(width), C.c_int32(modes), C.c_int32(layers),
                                    C.c_int32(hidden), _p(p))
        op = cls(h, n_cells)
        op._keep = p
        return op

    @classmethod
    def exact(cls, length, n_cells, order, ref_params, cfg):
        grid = make_grid(length, n_cells)
        h = lib().oracle_exact_operator_create(C.byref(grid), C.c_int32(order), C.c_double(ref_params[0]),
                                               C.c_double(ref_params[1]), C.byref(cfg))
        return cls(h, n_cells)

    def predict(self, source, n_threads=0):
        src = np.ascontiguousarray(source, dtype=np.float64)
        out = np.empty_like(src)
        _check(lib().oracle_op_predict(self.h, C.c_int32(src.shape[0]), _p(src), _p(out), C.c_int32(n_threads)))
        return out

    def recast_fixed_point(self, source, sigma_t, sigma_s0, tol=1e-4, max_it=50, norm=0, initial_phi=None,
                           n_threads=0):
        src = np.ascontiguousarray(source, dtype=np.float64)
        B = src.shape[0]
        phi = np.empty_like(src)
        it = np.empty(B, dtype=np.int32)
        st = np.empty(B, dtype=np.int32)
        _check(lib().oracle_recast_fixed_point(
            self.h, C.c_int32(B), _p(src), _p(np.ascontiguousarray(sigma_t, dtype=np.float64)),
            _p(np.ascontiguousarray(sigma_s0, dtype=np.float64)), C.c_double(tol), C.c_int32(max_it),
            C.c_int32(norm), _opt(initial_phi), _p(phi), _p(it), _p(st), C.c_int32(n_threads)))
        return {"phi": phi, "iterations": it, "status": st}

    def precondition_fixed_source(self, order, sigma_t, sigma_s0, source, cfg, rtol=1e-4, rmax=50,
                                  sigma_s1=None, n_threads=0):
        src = np.ascontiguousarray(source, dtype=np.float64)
        B = src.shape[0]
        phi = np.empty_like(src)
        pit = np.empty(B, dtype=np.int32)
        rst = np.empty(B, dtype=np.int32)
        rit = np.empty(B, dtype=np.int32)
        cv = np.empty(B, dtype=np.uint8)
        _check(lib().oracle_precondition_fixed_source(
            self.h, C.c_int32(order), C.c_int32(B), _p(np.ascontiguousarray(sigma_t, dtype=np.float64)),
            _p(np.ascontiguousarray(sigma_s0, dtype=np.float64)), _opt(sigma_s1), _p(src), C.c_double(rtol),
            C.c_int32(rmax), C.byref(cfg), _p(phi), _p(pit), _p(rst), _p(rit), _p(cv), C.c_int32(n_threads)))
        return {"phi": phi, "precond_iterations": pit, "recast_status": rst, "refine_iterations": rit,
                "converged": cv.astype(bool)}

    def hybrid_eigen(self, algorithm, order, sigma_t, sigma_s0, nu_sigma_f, chi, cfg, rtol=1e-4, rmax=50,
                     sigma_s1=None, n_threads=0):
        """SP (algorithm 0) / CP (1) eigen solve."""
        st = np.ascontiguousarray(sigma_t, dtype=np.float64)
        B, G, n = st.shape
        k = np.empty(B)
        phi = np.empty((B, G, n))
        k1 = np.empty(B)
        o1 = np.empty(B, dtype=np.int32)
        i1 = np.empty(B, dtype=np.int64)
        o2 = np.empty(B, dtype=np.int32)
        i2 = np.empty(B, dtype=np.int64)
        cv = np.empty(B, dtype=np.uint8)
        fb = np.empty(B, dtype=np.uint8)
        _check(lib().oracle_sp_cp_eigen_batched(
            self.h, C.c_int32(algorithm), C.c_int32(order), C.c_int32(B), C.c_int32(G), _p(st),
            _p(np.ascontiguousarray(sigma_s0, dtype=np.float64)), _opt(sigma_s1),
            _p(np.ascontiguousarray(nu_sigma_f, dtype=np.float64)), _p(np.ascontiguousarray(chi, dtype=np.float64)),
            C.byref(cfg), C.c_double(rtol), C.c_int32(rmax), _p(k), _p(phi), _p(k1), _p(o1), _p(i1), _p(o2),
            _p(i2), _p(cv), _p(fb), C.c_int32(n_threads)))
        return {"k": k, "phi": phi, "stage1_k": k1, "stage1_outer": o1, "stage1_inner": i1, "stage2_outer": o2,
                "stage2_inner": i2, "converged": cv.astype(bool), "fallback": fb.astype(bool)}


def grf_sample(length, n_cells, spec, n_samples, first=0):
    """spec: paper_2509_01416_b200.snop.GrfSpec (or anything with .c() -> SnopGrfSpec)."""
    g = make_grid(length, n_cells)
    sp = spec.c()
    out = np.empty((n_samples, n_cells))
    neg = np.empty(n_samples, dtype=np.int64)
    jit = C.c_double()
    _check(lib().oracle_grf_sample(C.byref(g), C.byref(sp), C.c_int64(first), C.c_int32(n_samples), _p(out),
                                   _p(neg), C.byref(jit)))
    return out, neg, jit.value


def normalize_source(length, n_cells, raw):
    raw = np.ascontiguousarray(raw, dtype=np.float64)
    out = np.empty_like(raw)
    g = make_grid(length, n_cells)
    _check(lib().oracle_normalize_source(C.byref(g), C.c_int32(raw.shape[0]), _p(raw), _p(out)))
    return out


def generate_dataset(length, n_cells, order, spec, n_samples, tstar, sstar, tol, n_threads=0):
    g = make_grid(length, n_cells)
    sp = spec.c()
    S = np.empty((n_samples, n_cells))
    phi = np.empty((n_samples, n_cells))
    it = np.empty(n_samples, dtype=np.int32)
    _check(lib().oracle_generate_dataset(C.byref(g), C.c_int32(order), C.byref(sp), C.c_int32(n_samples),
                                         C.c_double(tstar), C.c_double(sstar), C.c_double(tol), _p(S), _p(phi),
                                         _p(it), C.c_int32(n_threads)))
    return S, phi, it


__all__ = ["grf_sample", "normalize_source", "generate_dataset", "lib", "gauss_legendre", "source_iteration", "power_iteration", "infinite_medium_k", "recast_source",
           "OracleOperator", "make_config", "make_grid", "SnopSolverConfig", "SnopGrid", "balance_residual",
           "chunk_bounds", "rng_stream", "hardware_threads", "OracleError"]
