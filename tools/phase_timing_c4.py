"""Experiment: K2 time split for the slowest C4 instance (needs a -DSNOP_PHASE_TIMING build via SNOP_LIB)."""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_01416_b200 import snop, workloads as W, _capi
lib = _capi.load()
fs = [getattr(lib, n) for n in ("snop_internal_phase_cycles_eigen", "snop_internal_phase_cycles_eigen_ps", "snop_internal_phase_cycles_disp", "snop_internal_phase_cycles_ecl") if hasattr(lib, n)]
for g_ in fs:
    g_.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(20, dtype=np.uint64)


def f(out, reset):  # the kernel copy the runtime launches may live in either module
    tot = np.zeros(20, dtype=np.uint64)
    for g_ in fs:
        tmp = np.zeros(20, dtype=np.uint64)
        g_(tmp.ctypes.data, reset)
        tot += tmp
    buf[:] = tot
p = W.config4()
cfg = snop.SolverConfig(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi)
g = snop.Grid1D(p.length, p.n_cells)
if len(sys.argv) > 1:
    idx = int(sys.argv[1])
else:  # the batch's slowest instance (most inner sweeps)
    full = [torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi)]
    idx = int(snop.power_iteration(g, p.order, *full, cfg).total_inner_iterations.argmax())
import time
q = p.subset([idx])
args = [torch.from_numpy(a).cuda() for a in (q.sigma_t, q.sigma_s0, q.nu_sigma_f, q.chi)]
snop.power_iteration(g, p.order, *args, cfg); torch.cuda.synchronize()
f(buf.ctypes.data, 1)
t0 = time.perf_counter()
r = snop.power_iteration(g, p.order, *args, cfg); torch.cuda.synchronize()
print(f"instance {idx} alone: {1e3*(time.perf_counter()-t0):.2f} ms")
f(buf.ctypes.data, 1)
sweeps = int(r.total_inner_iterations[0]); outer = int(r.outer_iterations[0])
row = buf[:10].astype(np.float64)
groups = sweeps * (p.order // 4)
print(f"sweeps {sweeps} outer {outer}: per pair group maps {row[0]/groups:.0f} bar1 {row[1]/groups:.0f} scan {row[2]/groups:.0f} "
      f"bar2 {row[3]/groups:.0f} replay {row[4]/groups:.0f} | per sweep pairs {row[5]/sweeps:.0f} phi {row[6]/sweeps:.0f} | "
      f"in solve calls per sweep {row[7]/sweeps:.0f} | whole loop per sweep {row[8]/sweeps:.0f} cycles | "
      f"group-source build per group solve {row[9]/(outer*p.n_groups):.0f} | outer-loop rest per outer "
      f"{(row[8]-row[7]-row[9])/outer:.0f}")
