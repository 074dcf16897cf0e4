import ctypes as C, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2509_01416_b200 import snop, workloads as W, _capi
lib = _capi.load()
ff = lib.snop_internal_phase_cycles; ff.argtypes = [C.c_void_p, C.c_int]
fe = lib.snop_internal_phase_cycles_eigen; fe.argtypes = [C.c_void_p, C.c_int]
p = W.config2(batch=148)
g = snop.Grid1D(p.length, p.n_cells)
args = [torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.source)]
r = snop.source_iteration(g, p.order, *args, snop.SolverConfig(tolerance=p.tolerance)); torch.cuda.synchronize()
buf = np.zeros(20, dtype=np.uint64); print("K1 ret", ff(buf.ctypes.data, 0), buf[:10])
q = W.config4().subset([9]); p4 = W.config4()
cfg = snop.SolverConfig(tolerance=p4.tolerance_inner, tolerance_k=p4.tolerance_k, tolerance_phi=p4.tolerance_phi)
a4 = [torch.from_numpy(a).cuda() for a in (q.sigma_t, q.sigma_s0, q.nu_sigma_f, q.chi)]
r = snop.power_iteration(snop.Grid1D(p4.length, p4.n_cells), p4.order, *a4, cfg); torch.cuda.synchronize()
buf = np.zeros(20, dtype=np.uint64); print("K2 ret", fe(buf.ctypes.data, 0), buf[:10])
