import sys
sys.path.insert(0, '.')
import torch
from paper_2509_01416_b200 import snop, workloads as W
p4 = W.config4(); q = p4.subset([int(sys.argv[1]) if len(sys.argv) > 1 else 9])
cfg = snop.SolverConfig(tolerance=p4.tolerance_inner, tolerance_k=p4.tolerance_k, tolerance_phi=p4.tolerance_phi)
a4 = [torch.from_numpy(a).cuda() for a in (q.sigma_t, q.sigma_s0, q.nu_sigma_f, q.chi)]
r = snop.power_iteration(snop.Grid1D(p4.length, p4.n_cells), p4.order, *a4, cfg); torch.cuda.synchronize()
print(int(r.total_inner_iterations[0]))
