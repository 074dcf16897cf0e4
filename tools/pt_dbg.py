import ctypes as C, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2509_01416_b200 import snop, workloads as W, _capi
lib = _capi.load(); print(_capi.LIB_PATH)
fe = lib.snop_internal_phase_cycles_eigen; fe.argtypes = [C.c_void_p, C.c_int]
ff = lib.snop_internal_phase_cycles; ff.argtypes = [C.c_void_p, C.c_int]
p = W.config4()
cfg = snop.SolverConfig(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi)
g = snop.Grid1D(p.length, p.n_cells)
q = p.subset([9])
args = [torch.from_numpy(a).cuda() for a in (q.sigma_t, q.sigma_s0, q.nu_sigma_f, q.chi)]
r = snop.power_iteration(g, p.order, *args, cfg); torch.cuda.synchronize()
for f in (fe, ff):
    buf = np.zeros(20, dtype=np.uint64)
    print("ret", f(buf.ctypes.data, 0), buf)
print(int(r.total_inner_iterations[0]), int(r.outer_iterations[0]))
