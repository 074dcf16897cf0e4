import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2509_01416_b200 import snop, workloads as W
p = W.config3()
g = snop.Grid1D(p.length, p.n_cells)
cfg = snop.SolverConfig(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi, boundary_left=p.bc_left, boundary_right=p.bc_right)
dev = [torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi)]
r = snop.power_iteration(g, p.order, *dev, cfg)
o = r.outer_iterations.cpu().numpy(); i = r.total_inner_iterations.cpu().numpy()
print("outer pct 50/75/90/95/99/max", np.percentile(o, [50, 75, 90, 95, 99, 100]))
for c in (24, 32, 48, 64, 96, 128, 200, 400):
    m = o > c
    print(f"cap {c}: {m.sum()} instances beyond, inner sweeps beyond cap (approx) {int((i[m] * (1 - c / o[m])).sum())} of {int(i.sum())}")
print("sweeps per outer mean", float(i.sum() / o.sum()))
