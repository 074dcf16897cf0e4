import ctypes as C, sys, os
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2509_01416_b200 import snop, workloads as W, _capi
lib = _capi.load(); print(_capi.LIB_PATH)
f = lib.snop_internal_phase_cycles; f.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(16, dtype=np.uint64)
p = W.config2(batch=148)
g = snop.Grid1D(p.length, p.n_cells)
args = [torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.source)]
r = snop.source_iteration(g, p.order, *args, snop.SolverConfig(tolerance=p.tolerance))
torch.cuda.synchronize()
print("ret", f(buf.ctypes.data, 0), buf)
