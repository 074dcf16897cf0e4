"""Experiment: K2 phase split for the slowest C3 instance (needs a -DSNOP_PHASE_TIMING build via SNOP_LIB)."""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_01416_b200 import snop, workloads as W, _capi
lib = _capi.load()
fs = [getattr(lib, n) for n in ("snop_internal_phase_cycles_eigen", "snop_internal_phase_cycles_eigen_ps",
                                  "snop_internal_phase_cycles_disp") if hasattr(lib, n)]
for g_ in fs:
    g_.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(20, dtype=np.uint64)


def f(out, reset):  # the kernel copy the runtime launches may live in any of these modules
    tot = np.zeros(20, dtype=np.uint64)
    for g_ in fs:
        tmp = np.zeros(20, dtype=np.uint64)
        g_(tmp.ctypes.data, reset)
        tot += tmp
    buf[:] = tot
p = W.config3()
cfg = snop.SolverConfig(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi,
                        boundary_left=p.bc_left, boundary_right=p.bc_right)
g = snop.Grid1D(p.length, p.n_cells)
q = p.subset([int(sys.argv[1]) if len(sys.argv) > 1 else 491])
cs = int(sys.argv[2]) if len(sys.argv) > 2 else 8  # pair-split cluster size for the whole solve (-1: one CTA)
snop.default_context().set_options(pair_split=cs, pi_tail_cap=-1)
nctas = cs if cs > 1 else 1
args = [torch.from_numpy(a).cuda() for a in (q.sigma_t, q.sigma_s0, q.nu_sigma_f, q.chi)]
import time
snop.power_iteration(g, p.order, *args, cfg); torch.cuda.synchronize()
f(buf.ctypes.data, 1)
t0 = time.perf_counter()
r = snop.power_iteration(g, p.order, *args, cfg); torch.cuda.synchronize()
dt = time.perf_counter() - t0
f(buf.ctypes.data, 1)
print(f"single instance: {dt*1e3:.1f} ms, {dt*1e6/int(r.total_inner_iterations[0]):.2f} us per sweep")
sweeps = int(r.total_inner_iterations[0]); outer = int(r.outer_iterations[0])
row = buf[:10].astype(np.float64)
groups = sweeps * max(1, (p.order // 4) // nctas) * nctas  # pair groups summed over the CTAs
sweeps *= nctas  # per-sweep sums below: per CTA
print(f"pair_split {cs}; C3 inst: sweeps {sweeps // nctas} outer {outer}: cycles per pair group (per CTA) maps {row[0]/groups:.0f} bar1 {row[1]/groups:.0f} "
      f"scan {row[2]/groups:.0f} bar2 {row[3]/groups:.0f} replay {row[4]/groups:.0f} | per sweep pairs {row[5]/sweeps:.0f} "
      f"phi {row[6]/sweeps:.0f} | in solve per sweep {row[7]/sweeps:.0f} | loop per sweep {row[8]/sweeps:.0f}")
