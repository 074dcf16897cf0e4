"""Host-side mirror of the reference's ``snop::`` solver API for the S_N hot path, batched.

Every function here is a thin shim over one C-ABI entry point of libsnop_cuda.so
(include/snop_cuda.h); the computation runs in the sm_100a kernels, never on the host and never
in PyTorch. Arrays may be numpy (host memory: the call stages H2D/D2H) or CUDA torch tensors
(device memory: enqueued on the context's stream). Reference contracts:

  gauss_legendre
  source_iteration          SPEC.md:125-134 (sweep :115-123)
  balance_report
  power_iteration           SPEC.md:179-189 (+ decisions :206-209)
  recast_source
  predict
  recast_fixed_point
  precondition_fixed_source SPEC.md:413-421
  sp_eigen / cp_eigen
  save_model / load_model
  sample_grf / normalize_source / generate_dataset / dataset file
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._types import SnopCtxOptions, SnopDatasetInfo, SnopGrfSpec, SnopGrid, SnopModelInfo, SnopSolverConfig, make_grid

VACUUM, REFLECTIVE = 0, 1
REL_LINF, REL_L2 = 0, 1
RELU, TANH, GELU = 0, 1, 2
RECAST_CONVERGED, RECAST_MAXED, RECAST_DIVERGED = 0, 1, 2


@dataclass(frozen=True)
class Grid1D:
    """SPEC.md:22-27"""
    length_cm: float
    n_cells: int

    @property
    def dx(self) -> float:
        return self.length_cm / self.n_cells

    @property
    def centers(self) -> np.ndarray:
        return (np.arange(self.n_cells) + 0.5) * self.dx

    def c(self) -> SnopGrid:
        return make_grid(self.length_cm, self.n_cells)


@dataclass(frozen=True)
class AngularQuadrature:
    """SPEC.md:29-35 (nodes ascending, symmetric)."""
    order: int
    mu: np.ndarray
    w: np.ndarray


def gauss_legendre(order: int) -> AngularQuadrature:
    mu = np.empty(order)
    w = np.empty(order)
    _capi.check(_capi.load().snop_gauss_legendre(order, mu.ctypes.data, w.ctypes.data))
    return AngularQuadrature(order, mu, w)


@dataclass
class SolverConfig:
    """SPEC.md:57-61; eigen tolerances split."""
    tolerance: float = 1e-4
    tolerance_k: float | None = None
    tolerance_phi: float | None = None
    max_inner_iterations: int = 10000
    max_outer_iterations: int = 5000
    boundary_left: int = VACUUM
    boundary_right: int = VACUUM
    convergence_norm: int = REL_LINF

    def c(self) -> SnopSolverConfig:
        t = self.tolerance
        return SnopSolverConfig(float(t), float(t if self.tolerance_k is None else self.tolerance_k),
                                float(t if self.tolerance_phi is None else self.tolerance_phi),
                                int(self.max_inner_iterations), int(self.max_outer_iterations),
                                int(self.boundary_left), int(self.boundary_right), int(self.convergence_norm), 0)


class Context:
    """One CUDA device + stream + workspace (snop_ctx)."""

    def __init__(self, device: int = 0):
        self._lib = _capi.load()
        h = C.c_void_p()
        _capi.check(self._lib.snop_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.device = device
        # torch tensors read or written by device calls still in flight on this context's stream
        # (inputs converted by the call, outputs it allocated); released by synchronize()
        self._pending: list = []

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self._lib.snop_ctx_synchronize(self.h)
            self._pending = []
            self._lib.snop_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        try:
            _capi.check(self._lib.snop_ctx_synchronize(self.h))
        finally:
            self._pending = []

    OPTION_NAMES = ("cell_cluster", "pair_split", "pi_tail_cap", "host_chunks", "gemm_engine", "fno_dft", "fno_mix")

    def options(self) -> dict:
        """Execution options of this context (snop_ctx_options, include/snop_cuda.h); 0 = automatic."""
        o = SnopCtxOptions()
        _capi.check(self._lib.snop_ctx_get_options(self.h, C.byref(o)))
        return {k: int(getattr(o, k)) for k in self.OPTION_NAMES}

    def set_options(self, **kw) -> dict:
        """Update execution options (unknown names raise); returns the previous options."""
        prev = self.options()
        bad = set(kw) - set(self.OPTION_NAMES)
        if bad:
            raise ValueError(f"unknown context options {sorted(bad)}")
        o = SnopCtxOptions(**{**prev, **{k: int(v) for k, v in kw.items()}})
        _capi.check(self._lib.snop_ctx_set_options(self.h, C.byref(o)))
        return prev

    @property
    def launch_count(self) -> int:
        return int(self._lib.snop_ctx_launch_count(self.h))

    @property
    def stream_ptr(self) -> int:
        return int(self._lib.snop_ctx_stream(self.h) or 0)


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ---- array plumbing -----------------------------------------------------------------------
def _is_dev(a) -> bool:
    return a is not None and hasattr(a, "is_cuda") and bool(a.is_cuda)


class _Args:
    """Collects pointers for one call; all arrays must be in the same memory space."""

    def __init__(self, *arrays):
        present = [a for a in arrays if a is not None]
        dev = [_is_dev(a) for a in present]
        if any(dev) and not all(dev):
            raise ValueError("mix of host (numpy) and device (torch CUDA) arrays in one call")
        self.device = bool(dev) and all(dev)
        self.keep = []
        self.outs = []

    def ready(self, ctx: "Context") -> None:
        """Device calls: order the context's stream after torch's current stream (the producers of
        the inputs, including the dtype/contiguity conversions made here), and keep every tensor of
        the call referenced by the context until its next synchronize(), so torch's caching
        allocator cannot hand their memory to other work while the kernels still read or write it.
        (No record_stream on the context's stream: the allocator would record events on that stream
        when the tensors die, possibly after the context destroyed it.)"""
        if not self.device:
            return
        import torch
        ext = torch.cuda.ExternalStream(ctx.stream_ptr)
        ext.wait_stream(torch.cuda.current_stream())
        if len(ctx._pending) > 4096:  # bound what many unsynchronised calls keep alive
            ctx.synchronize()
        ctx._pending.extend(self.keep)
        ctx._pending.extend(self.outs)

    @property
    def memspace(self) -> int:
        return 1 if self.device else 0

    def inp(self, a, dtype=np.float64, shape=None):
        if a is None:
            return None
        if self.device:
            import torch
            tdt = {np.float64: torch.float64, np.float32: torch.float32, np.int32: torch.int32}[dtype]
            if a.dtype != tdt or not a.is_contiguous():
                a = a.to(tdt).contiguous()
            if shape is not None and tuple(a.shape) != tuple(shape):
                a = a.reshape(shape)
            self.keep.append(a)
            return a.data_ptr()
        a = np.ascontiguousarray(a, dtype=dtype)
        if shape is not None and a.shape != tuple(shape):
            a = a.reshape(shape)
        self.keep.append(a)
        return a.ctypes.data

    def out(self, shape, dtype=np.float64, into=None):
        """A fresh output array, or the caller's ``into`` (checked: same memory space, dtype, shape,
        contiguous) so results can land directly in e.g. pinned host memory."""
        if into is not None:
            if self.device != _is_dev(into):
                raise ValueError("output array is in the wrong memory space")
            if self.device:
                import torch
                tdt = {np.float64: torch.float64, np.int32: torch.int32, np.uint8: torch.uint8}[dtype]
                ok = into.dtype == tdt and into.is_contiguous() and tuple(into.shape) == tuple(shape)
                ptr = into.data_ptr()
                self.outs.append(into)
            else:
                ok = into.dtype == dtype and into.flags.c_contiguous and into.shape == tuple(shape)
                ptr = into.ctypes.data
            if not ok:
                raise ValueError(f"output array must be contiguous {np.dtype(dtype).name} of shape {tuple(shape)}")
            return into, ptr
        if self.device:
            import torch
            tdt = {np.float64: torch.float64, np.float32: torch.float32, np.int32: torch.int32,
                   np.int64: torch.int64, np.uint8: torch.uint8}[dtype]
            t = torch.empty(shape, dtype=tdt, device="cuda")
            self.outs.append(t)
            return t, t.data_ptr()
        a = np.empty(shape, dtype=dtype)
        return a, a.ctypes.data


@dataclass
class FixedSourceResult:
    """(FluxField, iterations, converged) of SPEC.md:125, batched."""
    phi: object
    iterations: object
    converged: object
    current: object = None
    leakage: object = None  # [B][2] net outflow at x=0, x=L of the last sweep (want_leakage)


def source_iteration(grid: Grid1D, order: int, sigma_t, sigma_s0, source, config: SolverConfig | None = None,
                     initial_phi=None, sigma_s1=None, want_current: bool = False, want_leakage: bool = False,
                     ctx: Context | None = None, sync: bool = True, out=None) -> FixedSourceResult:
    """Batched single-group fixed-source solve. Arrays are [B][Nc].
    Device (torch CUDA) arrays: enqueued on ctx's stream; with sync=False the caller must call
    ctx.synchronize() (which also reports kernel-raised argument errors) before using results.
    ``out`` = optional (phi, iterations, converged) arrays to write into (e.g. pinned host memory)."""
    ctx = ctx or default_context()
    config = config or SolverConfig()
    a = _Args(sigma_t, sigma_s0, source, initial_phi, sigma_s1)
    o_phi, o_it, o_cv = out if out is not None else (None, None, None)
    B = int(sigma_t.shape[0])
    n = grid.n_cells
    st, ss, src = a.inp(sigma_t, shape=(B, n)), a.inp(sigma_s0, shape=(B, n)), a.inp(source, shape=(B, n))
    s1, p0 = a.inp(sigma_s1, shape=(B, n)), a.inp(initial_phi, shape=(B, n))
    phi, phi_p = a.out((B, n), into=o_phi)
    cur, cur_p = a.out((B, n)) if want_current else (None, None)
    it, it_p = a.out((B,), np.int32, into=o_it)
    cv, cv_p = a.out((B,), np.uint8, into=o_cv)
    g, cfg = grid.c(), config.c()
    a.ready(ctx)
    if want_leakage:
        lk, lk_p = a.out((B, 2))
        _capi.check(ctx._lib.snop_source_iteration_leakage_batched(
            ctx.h, a.memspace, C.byref(g), int(order), B, st, ss, s1, src, C.byref(cfg), p0, phi_p, cur_p, it_p, cv_p,
            lk_p))
    else:
        lk = None
        _capi.check(ctx._lib.snop_source_iteration_batched(ctx.h, a.memspace, C.byref(g), int(order), B, st, ss, s1,
                                                           src, C.byref(cfg), p0, phi_p, cur_p, it_p, cv_p))
    if a.device and sync:
        ctx.synchronize()
    return FixedSourceResult(phi, it, cv, cur, lk)


def sweep(grid: Grid1D, order: int, sigma_t, emission, boundary_left: int = 0, boundary_right: int = 0,
          ctx: Context | None = None, sync: bool = True):
    """sweep, batched: one diamond-difference sweep of all directions.
    sigma_t [B][Nc], emission [B][Nc][order] (direction index ascending in mu); returns
    (psi_avg [B][order][Nc], outflow_left [B], outflow_right [B]) with the net outgoing partial
    currents at the two faces. boundary_*: 0 vacuum, 1 reflective."""
    ctx = ctx or default_context()
    a = _Args(sigma_t, emission)
    B = int(sigma_t.shape[0])
    n, N = grid.n_cells, int(order)
    st, em = a.inp(sigma_t, shape=(B, n)), a.inp(emission, shape=(B, n, N))
    psi, psi_p = a.out((B, N, n))
    ol, ol_p = a.out((B,))
    orr, or_p = a.out((B,))
    g = grid.c()
    a.ready(ctx)
    _capi.check(ctx._lib.snop_sweep_batched(ctx.h, a.memspace, C.byref(g), N, B, st, em, int(boundary_left),
                                            int(boundary_right), psi_p, ol_p, or_p))
    if a.device and sync:
        ctx.synchronize()
    return psi, ol, orr


def balance_report(grid: Grid1D, sigma_t, sigma_s0_out, source, phi, leakage, ctx: Context | None = None):
    """balance_report, batched [B][Nc]; leakage [B][2] from source_iteration."""
    ctx = ctx or default_context()
    a = _Args(sigma_t, sigma_s0_out, source, phi, leakage)
    B = int(sigma_t.shape[0])
    n = grid.n_cells
    st, ss, S, p = (a.inp(x, shape=(B, n)) for x in (sigma_t, sigma_s0_out, source, phi))
    lk = a.inp(leakage, shape=(B, 2))
    res, res_p = a.out((B,))
    g = grid.c()
    a.ready(ctx)
    _capi.check(ctx._lib.snop_balance_report(ctx.h, a.memspace, C.byref(g), B, st, ss, S, p, lk, res_p))
    if a.device:
        ctx.synchronize()
    return res


@dataclass
class EigenSolution:
    """SPEC.md:172-176, batched."""
    k: object
    phi: object
    outer_iterations: object
    total_inner_iterations: object
    converged: object


def power_iteration(grid: Grid1D, order: int, sigma_t, sigma_s0, nu_sigma_f, chi,
                    config: SolverConfig | None = None, initial_k=None, initial_phi=None, sigma_s1=None,
                    ctx: Context | None = None, sync: bool = True) -> EigenSolution:
    """Batched k-eigenvalue power iteration. sigma_t/nu_sigma_f/sigma_s1:
    [B][G][Nc]; sigma_s0: [B][G][G][Nc] ([g'][g] = g'->g); chi: [B][G]. Device (torch CUDA) arrays:
    enqueued on ctx's stream; with sync=False the caller must call ctx.synchronize() before reading."""
    ctx = ctx or default_context()
    config = config or SolverConfig()
    a = _Args(sigma_t, sigma_s0, nu_sigma_f, chi, initial_k, initial_phi, sigma_s1)
    B, G, n = (int(x) for x in sigma_t.shape)
    if n != grid.n_cells:
        raise ValueError("sigma_t last dim must equal grid.n_cells")
    st = a.inp(sigma_t, shape=(B, G, n))
    ss = a.inp(sigma_s0, shape=(B, G, G, n))
    nsf = a.inp(nu_sigma_f, shape=(B, G, n))
    ch = a.inp(chi, shape=(B, G))
    s1 = a.inp(sigma_s1, shape=(B, G, n))
    k0 = a.inp(initial_k, shape=(B,))
    p0 = a.inp(initial_phi, shape=(B, G, n))
    k, k_p = a.out((B,))
    phi, phi_p = a.out((B, G, n))
    outer, o_p = a.out((B,), np.int32)
    inner, i_p = a.out((B,), np.int64)
    cv, cv_p = a.out((B,), np.uint8)
    g, cfg = grid.c(), config.c()
    a.ready(ctx)
    _capi.check(ctx._lib.snop_power_iteration_batched(ctx.h, a.memspace, C.byref(g), int(order), B, G, st, ss, s1,
                                                      nsf, ch, C.byref(cfg), k0, p0, k_p, phi_p, o_p, i_p, cv_p))
    if a.device and sync:
        ctx.synchronize()
    return EigenSolution(k, phi, outer, inner, cv)


def recast_source(source, phi, sigma_t, sigma_s0, reference_params=(1.0, 0.5), ctx: Context | None = None):
    """SPEC.md:393-401 (paper Eq. 24), batched [B][Nc]."""
    ctx = ctx or default_context()
    a = _Args(source, phi, sigma_t, sigma_s0)
    B, n = (int(x) for x in source.shape)
    s, p, st, ss = (a.inp(x, shape=(B, n)) for x in (source, phi, sigma_t, sigma_s0))
    out, out_p = a.out((B, n))
    a.ready(ctx)
    _capi.check(ctx._lib.snop_recast_source(ctx.h, a.memspace, B, n, s, p, st, ss, float(reference_params[0]),
                                            float(reference_params[1]), out_p))
    if a.device:
        ctx.synchronize()
    return out


# ---- SolutionOperators and the MD-PNOP drivers ---------------------------------------------
class SolutionOperator:
    """Device-resident SolutionOperator: DeepONet, FNO or the exact model-based
    solve at p*. ``reference_params`` = p* = (Sigma_t*, Sigma_s0*)."""

    def __init__(self, handle, grid: Grid1D, reference_params, ctx: Context, keep=()):
        self.h = handle
        self.grid = grid
        self.reference_params = tuple(reference_params)
        self.ctx = ctx
        self._keep = keep

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.ctx._lib.snop_op_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @classmethod
    def deeponet(cls, grid: Grid1D, params, reference_params=(1.0, 0.5), ctx: Context | None = None):
        ctx = ctx or default_context()
        bs = np.ascontiguousarray(params.branch.sizes, dtype=np.int32)
        ts = np.ascontiguousarray(params.trunk.sizes, dtype=np.int32)
        bp, tp = params.branch.packed(), params.trunk.packed()
        h = C.c_void_p()
        g = grid.c()
        _capi.check(ctx._lib.snop_deeponet_create(
            ctx.h, C.byref(g), float(reference_params[0]), float(reference_params[1]), int(params.activation),
            len(bs), bs.ctypes.data, bp.ctypes.data, len(ts), ts.ctypes.data, tp.ctypes.data,
            int(params.bias0 is not None), float(params.bias0 or 0.0), C.byref(h)))
        return cls(h, grid, reference_params, ctx)

    @classmethod
    def fno(cls, grid: Grid1D, params, reference_params=(1.0, 0.8), ctx: Context | None = None):
        ctx = ctx or default_context()
        p = params.packed()
        h = C.c_void_p()
        g = grid.c()
        _capi.check(ctx._lib.snop_fno_create(ctx.h, C.byref(g), float(reference_params[0]),
                                             float(reference_params[1]), int(params.activation), int(params.width),
                                             int(params.modes), int(params.layers), int(params.hidden),
                                             p.ctypes.data, C.byref(h)))
        return cls(h, grid, reference_params, ctx)

    @classmethod
    def exact(cls, grid: Grid1D, order: int, reference_params=(1.0, 0.5), config: SolverConfig | None = None,
              ctx: Context | None = None):
        ctx = ctx or default_context()
        cfg = (config or SolverConfig(tolerance=1e-10)).c()
        h = C.c_void_p()
        g = grid.c()
        _capi.check(ctx._lib.snop_exact_operator_create(ctx.h, C.byref(g), int(order), float(reference_params[0]),
                                                        float(reference_params[1]), C.byref(cfg), C.byref(h)))
        return cls(h, grid, reference_params, ctx)

    @classmethod
    def load(cls, path, ctx: Context | None = None):
        """load_model(path): DeepONet or FNO from a model file."""
        ctx = ctx or default_context()
        info = inspect_model(path)
        h = C.c_void_p()
        _capi.check(ctx._lib.snop_op_load(ctx.h, os.fsencode(path), C.byref(h)))
        grid = Grid1D(info.grid.length_cm, info.grid.n_cells)
        return cls(h, grid, (info.sigma_t_star, info.sigma_s0_star), ctx)

    def save(self, path) -> None:
        """save_model(model, path)."""
        _capi.check(self.ctx._lib.snop_op_save(self.h, os.fsencode(path)))

    def predict(self, source, sync: bool = True):
        """predict(model, source), batched [B][Nc]."""
        a = _Args(source)
        B = int(source.shape[0])
        n = self.grid.n_cells
        s = a.inp(source, shape=(B, n))
        out, out_p = a.out((B, n))
        a.ready(self.ctx)
        _capi.check(self.ctx._lib.snop_op_predict(self.ctx.h, self.h, a.memspace, B, s, out_p))
        if a.device and sync:
            self.ctx.synchronize()
        return out


@dataclass
class RecastResult:
    phi: object
    iterations: object
    status: object


def recast_fixed_point(op: SolutionOperator, source, sigma_t, sigma_s0, tolerance: float = 1e-4,
                       max_iterations: int = 50, norm: int = REL_LINF, initial_phi=None) -> RecastResult:
    """phi^{k+1} = op(recast(S, phi^k)); status 0 converged / 1 maxed / 2 diverged."""
    a = _Args(source, sigma_t, sigma_s0, initial_phi)
    B = int(source.shape[0])
    n = op.grid.n_cells
    S, st, ss = (a.inp(x, shape=(B, n)) for x in (source, sigma_t, sigma_s0))
    p0 = a.inp(initial_phi, shape=(B, n))
    phi, phi_p = a.out((B, n))
    it, it_p = a.out((B,), np.int32)
    stt, st_p = a.out((B,), np.int32)
    a.ready(op.ctx)
    _capi.check(op.ctx._lib.snop_recast_fixed_point(op.ctx.h, op.h, a.memspace, B, S, st, ss, float(tolerance),
                                                    int(max_iterations), int(norm), p0, phi_p, it_p, st_p))
    if a.device:
        op.ctx.synchronize()
    return RecastResult(phi, it, stt)


@dataclass
class PreconditionedResult:
    phi: object
    precond_iterations: object
    recast_status: object
    refine_iterations: object
    converged: object


def precondition_fixed_source(op: SolutionOperator, order: int, sigma_t, sigma_s0, source,
                              config: SolverConfig | None = None, recast_tolerance: float = 1e-4,
                              recast_max_iterations: int = 50, sigma_s1=None) -> PreconditionedResult:
    """SPEC.md:413-421 (paper Eq. 10): recast fixed point, then source iteration warm-started."""
    config = config or SolverConfig()
    a = _Args(sigma_t, sigma_s0, source, sigma_s1)
    B = int(source.shape[0])
    n = op.grid.n_cells
    st, ss, S = (a.inp(x, shape=(B, n)) for x in (sigma_t, sigma_s0, source))
    s1 = a.inp(sigma_s1, shape=(B, n))
    phi, phi_p = a.out((B, n))
    pit, pit_p = a.out((B,), np.int32)
    rst, rst_p = a.out((B,), np.int32)
    rit, rit_p = a.out((B,), np.int32)
    cv, cv_p = a.out((B,), np.uint8)
    cfg = config.c()
    a.ready(op.ctx)
    _capi.check(op.ctx._lib.snop_precondition_fixed_source(
        op.ctx.h, op.h, a.memspace, int(order), B, st, ss, s1, S, float(recast_tolerance), int(recast_max_iterations),
        C.byref(cfg), phi_p, pit_p, rst_p, rit_p, cv_p))
    if a.device:
        op.ctx.synchronize()
    return PreconditionedResult(phi, pit, rst, rit, cv)


@dataclass
class HybridEigenSolution:
    """EigenSolution + stage diagnostics."""
    k: object
    phi: object
    stage1_k: object
    stage1_outer: object
    stage1_inner: object
    stage2_outer: object
    stage2_inner: object
    converged: object
    fallback: object


def _hybrid_eigen(fn: str, op: SolutionOperator, order: int, sigma_t, sigma_s0, nu_sigma_f, chi,
                  config: SolverConfig | None, recast_tolerance: float, recast_max_iterations: int,
                  sigma_s1) -> HybridEigenSolution:
    config = config or SolverConfig()
    a = _Args(sigma_t, sigma_s0, nu_sigma_f, chi, sigma_s1)
    B, G, n = (int(x) for x in sigma_t.shape)
    if n != op.grid.n_cells:
        raise ValueError("sigma_t last dim must equal the operator grid's n_cells")
    st = a.inp(sigma_t, shape=(B, G, n))
    ss = a.inp(sigma_s0, shape=(B, G, G, n))
    nsf = a.inp(nu_sigma_f, shape=(B, G, n))
    ch = a.inp(chi, shape=(B, G))
    s1 = a.inp(sigma_s1, shape=(B, G, n))
    k, k_p = a.out((B,))
    phi, phi_p = a.out((B, G, n))
    k1, k1_p = a.out((B,))
    o1, o1_p = a.out((B,), np.int32)
    i1, i1_p = a.out((B,), np.int64)
    o2, o2_p = a.out((B,), np.int32)
    i2, i2_p = a.out((B,), np.int64)
    cv, cv_p = a.out((B,), np.uint8)
    fb, fb_p = a.out((B,), np.uint8)
    cfg = config.c()
    a.ready(op.ctx)
    _capi.check(getattr(op.ctx._lib, fn)(
        op.ctx.h, op.h, a.memspace, int(order), B, G, st, ss, s1, nsf, ch, C.byref(cfg), float(recast_tolerance),
        int(recast_max_iterations), k_p, phi_p, k1_p, o1_p, i1_p, o2_p, i2_p, cv_p, fb_p))
    if a.device:
        op.ctx.synchronize()
    return HybridEigenSolution(k, phi, k1, o1, i1, o2, i2, cv, fb)


INNER_RECAST_FIXED_POINT, INNER_PREDICT_REFINE = 0, 1


@dataclass
class OperatorEigenSolution:
    """EigenSolution of a power iteration whose inner solver is a SolutionOperator."""
    k: object
    phi: object
    outer_iterations: object
    total_inner_iterations: object
    converged: object
    diverged: object


def power_iteration_with_operator(op: SolutionOperator, order: int, sigma_t, sigma_s0, nu_sigma_f, chi,
                                  config: SolverConfig | None = None, inner_solver: int = INNER_RECAST_FIXED_POINT,
                                  recast_tolerance: float = 1e-4, recast_max_iterations: int = 50,
                                  sigma_s1=None) -> OperatorEigenSolution:
    """power_iteration(..., inner_solver = neural-operator-backed): the within-group
    solve is the operator's recast fixed point (INNER_RECAST_FIXED_POINT: stage 1 of SP) or that
    prediction refined by a model-based source iteration (INNER_PREDICT_REFINE: stage 1 of CP).
    Layouts as power_iteration; flat start, k = 1."""
    config = config or SolverConfig()
    a = _Args(sigma_t, sigma_s0, nu_sigma_f, chi, sigma_s1)
    B, G, n = (int(x) for x in sigma_t.shape)
    if n != op.grid.n_cells:
        raise ValueError("sigma_t last dim must equal the operator grid's n_cells")
    st = a.inp(sigma_t, shape=(B, G, n))
    ss = a.inp(sigma_s0, shape=(B, G, G, n))
    nsf = a.inp(nu_sigma_f, shape=(B, G, n))
    ch = a.inp(chi, shape=(B, G))
    s1 = a.inp(sigma_s1, shape=(B, G, n))
    k, k_p = a.out((B,))
    phi, phi_p = a.out((B, G, n))
    o1, o1_p = a.out((B,), np.int32)
    i1, i1_p = a.out((B,), np.int64)
    cv, cv_p = a.out((B,), np.uint8)
    dv, dv_p = a.out((B,), np.uint8)
    cfg = config.c()
    a.ready(op.ctx)
    _capi.check(op.ctx._lib.snop_power_iteration_operator_batched(
        op.ctx.h, op.h, int(inner_solver), a.memspace, int(order), B, G, st, ss, s1, nsf, ch, C.byref(cfg),
        float(recast_tolerance), int(recast_max_iterations), k_p, phi_p, o1_p, i1_p, cv_p, dv_p))
    if a.device:
        op.ctx.synchronize()
    return OperatorEigenSolution(k, phi, o1, i1, cv, dv)


def sp_eigen(op: SolutionOperator, order: int, sigma_t, sigma_s0, nu_sigma_f, chi, config: SolverConfig | None = None,
             recast_tolerance: float = 1e-4, recast_max_iterations: int = 50, sigma_s1=None) -> HybridEigenSolution:
    """SP eigen solve (paper Eq. A5-A6), batched; layouts as power_iteration."""
    return _hybrid_eigen("snop_sp_eigen_batched", op, order, sigma_t, sigma_s0, nu_sigma_f, chi, config,
                         recast_tolerance, recast_max_iterations, sigma_s1)


def cp_eigen(op: SolutionOperator, order: int, sigma_t, sigma_s0, nu_sigma_f, chi, config: SolverConfig | None = None,
             recast_tolerance: float = 1e-4, recast_max_iterations: int = 50, sigma_s1=None) -> HybridEigenSolution:
    """CP eigen solve (paper Eq. A7-A8), batched; layouts as power_iteration."""
    return _hybrid_eigen("snop_cp_eigen_batched", op, order, sigma_t, sigma_s0, nu_sigma_f, chi, config,
                         recast_tolerance, recast_max_iterations, sigma_s1)


# ---- model files (host-only; no GPU needed) -----------------------------------------------------
def write_deeponet_file(path, grid: Grid1D, params, reference_params=(1.0, 0.5)) -> None:
    """Write a DeepONet model file (record layout csrc/model_io.h)."""
    lib = _capi.load()
    bs = np.ascontiguousarray(params.branch.sizes, dtype=np.int32)
    ts = np.ascontiguousarray(params.trunk.sizes, dtype=np.int32)
    bp, tp = params.branch.packed(), params.trunk.packed()
    g = grid.c()
    _capi.check(lib.snop_model_write_deeponet(
        os.fsencode(path), C.byref(g), float(reference_params[0]), float(reference_params[1]), int(params.activation),
        len(bs), bs.ctypes.data, bp.ctypes.data, len(ts), ts.ctypes.data, tp.ctypes.data,
        int(params.bias0 is not None), float(params.bias0 or 0.0)))


def write_fno_file(path, grid: Grid1D, params, reference_params=(1.0, 0.8)) -> None:
    """Write an FNO model file (record layout csrc/model_io.h)."""
    lib = _capi.load()
    p = params.packed()
    g = grid.c()
    _capi.check(lib.snop_model_write_fno(os.fsencode(path), C.byref(g), float(reference_params[0]),
                                         float(reference_params[1]), int(params.activation), int(params.width),
                                         int(params.modes), int(params.layers), int(params.hidden), p.ctypes.data))


def inspect_model(path) -> SnopModelInfo:
    """Read and validate a model file (magic, version, record, FNV-1a-64 digest); header summary."""
    info = SnopModelInfo()
    _capi.check(_capi.load().snop_model_inspect(os.fsencode(path), C.byref(info)))
    return info


# ---- GRF sources and training datasets -----------------------------------------
@dataclass(frozen=True)
class GrfSpec:
    """SPEC.md:226-230 (paper Appendix A1 defaults)."""
    mean: float = 0.07
    variance: float = 3e-4
    length_scale_cm: float = 1.2
    jitter: float = 1e-10
    seed: int = 0

    def c(self) -> SnopGrfSpec:
        return SnopGrfSpec(float(self.mean), float(self.variance), float(self.length_scale_cm), float(self.jitter),
                           int(self.seed))


def sample_grf(grid: Grid1D, spec: GrfSpec, n_samples: int, first_sample: int = 0, with_negatives: bool = False,
               ctx: Context | None = None, device: bool = False):
    """sample_grf for samples first..first+n-1 -> [n][Nc] raw fields (numpy, or a CUDA tensor
    when device=True); optionally the per-sample count of negative entries."""
    ctx = ctx or default_context()
    g, sp = grid.c(), spec.c()
    n = int(n_samples)
    if device:
        import torch
        out = torch.empty((n, grid.n_cells), dtype=torch.float64, device=f"cuda:{ctx.device}")
        neg = torch.empty(n, dtype=torch.int64, device=out.device) if with_negatives else None
        torch.cuda.ExternalStream(ctx.stream_ptr).wait_stream(torch.cuda.current_stream())
        _capi.check(ctx._lib.snop_grf_sample(ctx.h, 1, C.byref(g), C.byref(sp), int(first_sample), n, out.data_ptr(),
                                             neg.data_ptr() if neg is not None else None))
        ctx.synchronize()
    else:
        out = np.empty((n, grid.n_cells))
        neg = np.empty(n, dtype=np.int64) if with_negatives else None
        _capi.check(ctx._lib.snop_grf_sample(ctx.h, 0, C.byref(g), C.byref(sp), int(first_sample), n,
                                             out.ctypes.data, neg.ctypes.data if neg is not None else None))
    return (out, neg) if with_negatives else out


def normalize_source(grid: Grid1D, raw, ctx: Context | None = None):
    """normalize_source: raw / integral, per row."""
    ctx = ctx or default_context()
    a = _Args(raw)
    n = int(raw.shape[0])
    r = a.inp(raw, shape=(n, grid.n_cells))
    out, out_p = a.out((n, grid.n_cells))
    g = grid.c()
    a.ready(ctx)
    _capi.check(ctx._lib.snop_normalize_source(ctx.h, a.memspace, C.byref(g), n, r, out_p))
    if a.device:
        ctx.synchronize()
    return out


@dataclass
class TrainingDataset:
    """SPEC.md:232-236."""
    sources: object
    fluxes: object
    iterations: object
    grid: Grid1D
    order: int
    spec: GrfSpec
    reference_params: tuple
    tolerance: float


def generate_dataset(n_samples: int, spec: GrfSpec, grid: Grid1D, order: int, reference_params=(1.0, 0.5),
                     tolerance: float = 1e-8, ctx: Context | None = None) -> TrainingDataset:
    """generate_dataset on the device; host numpy arrays out."""
    ctx = ctx or default_context()
    n = int(n_samples)
    S = np.empty((n, grid.n_cells))
    phi = np.empty((n, grid.n_cells))
    it = np.empty(n, dtype=np.int32)
    g, sp = grid.c(), spec.c()
    _capi.check(ctx._lib.snop_generate_dataset(ctx.h, 0, C.byref(g), int(order), C.byref(sp), n,
                                               float(reference_params[0]), float(reference_params[1]),
                                               float(tolerance), S.ctypes.data, phi.ctypes.data, it.ctypes.data))
    return TrainingDataset(S, phi, it, grid, int(order), spec, tuple(reference_params), float(tolerance))


def save_dataset(path, ds: TrainingDataset) -> None:
    """Dataset file + text manifest; host-only."""
    info = SnopDatasetInfo(int(ds.sources.shape[0]), ds.grid.c(), int(ds.order), 0, ds.spec.c(),
                           float(ds.reference_params[0]), float(ds.reference_params[1]), float(ds.tolerance))
    S = np.ascontiguousarray(ds.sources, dtype=np.float64)
    phi = np.ascontiguousarray(ds.fluxes, dtype=np.float64)
    _capi.check(_capi.load().snop_dataset_write(os.fsencode(path), C.byref(info), S.ctypes.data, phi.ctypes.data))


def load_dataset(path) -> TrainingDataset:
    lib = _capi.load()
    info = SnopDatasetInfo()
    _capi.check(lib.snop_dataset_read(os.fsencode(path), C.byref(info), None, None))
    n, nc = int(info.n_samples), int(info.grid.n_cells)
    S = np.empty((n, nc))
    phi = np.empty((n, nc))
    _capi.check(lib.snop_dataset_read(os.fsencode(path), C.byref(info), S.ctypes.data, phi.ctypes.data))
    sp = info.spec
    return TrainingDataset(S, phi, None, Grid1D(info.grid.length_cm, nc), int(info.order),
                           GrfSpec(sp.mean, sp.variance, sp.length_scale_cm, sp.jitter, int(sp.seed)),
                           (info.sigma_t_star, info.sigma_s0_star), info.tolerance)
