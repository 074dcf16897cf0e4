"""Experiment: per-sweep cycle split of the pair-split exchange for the slowest C3 instance (#491, CS = 8).
Needs a -DSNOP_PHASE_TIMING -DSNOP_PS_TIMING build loaded through SNOP_LIB (tools/build_variant.sh)."""
import ctypes as C, sys
import numpy as np, torch
from paper_2509_01416_b200 import snop, workloads as W, _capi
lib = _capi.load()
fs = [getattr(lib, n) for n in ("snop_internal_phase_cycles_eigen", "snop_internal_phase_cycles_eigen_ps", "snop_internal_phase_cycles_disp") if hasattr(lib, n)]
for g_ in fs: g_.argtypes = [C.c_void_p, C.c_int]
def grab(reset):
    tot = np.zeros(20, dtype=np.uint64)
    for g_ in fs:
        tmp = np.zeros(20, dtype=np.uint64); g_(tmp.ctypes.data, reset); tot += tmp
    return tot
p = W.config3(); q = p.subset([491])
cfg = snop.SolverConfig(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi, boundary_left=p.bc_left, boundary_right=p.bc_right)
g = snop.Grid1D(p.length, p.n_cells)
snop.default_context().set_options(pair_split=8, pi_tail_cap=-1)
args = [torch.from_numpy(a).cuda() for a in (q.sigma_t, q.sigma_s0, q.nu_sigma_f, q.chi)]
snop.power_iteration(g, p.order, *args, cfg); torch.cuda.synchronize(); grab(1)
r = snop.power_iteration(g, p.order, *args, cfg); torch.cuda.synchronize()
b = grab(1).astype(np.float64)
sw = int(r.total_inner_iterations[0]) * 8  # per CTA sweeps (8 CTAs; thread 0 of each)
names = ["wait replays", "push partials", "cluster barrier", "owner update+push", "norm reduce"]
print("cycles per sweep per CTA:", {n: round(b[i] / sw) for i, n in enumerate(names)}, "pairs", round(b[5] / sw), "phi", round(b[6] / sw))
# whole-loop accounting (slot 8 = the outer loop, 7 = inside si_solve calls, 9 = per-group source build + staging)
outers = int(r.outer_iterations[0])
print("outers", outers, "sweeps", int(r.total_inner_iterations[0]),
      "| cycles per outer per CTA: whole loop", round(b[8] / (8 * outers)), "in si_solve", round(b[7] / (8 * outers)),
      "source build + staging", round(b[9] / (8 * outers)),
      "| loop cycles per sweep", round(b[8] / sw), "si_solve cycles per sweep", round(b[7] / sw))
import time
t0 = time.perf_counter(); r = snop.power_iteration(g, p.order, *args, cfg); torch.cuda.synchronize()
print("wall ms", 1e3 * (time.perf_counter() - t0))
