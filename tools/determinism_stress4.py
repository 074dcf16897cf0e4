"""Experiment: bit-reproducibility of the SP/CP hybrid eigen solves and the warm-started fixed-source
solve (DeepONet), with other kernels run in between."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2509_01416_b200 import snop, operators as OPS, workloads as W

p = W.config3(batch=4, n_cells=400)
g = snop.Grid1D(p.length, p.n_cells)
cfg = snop.SolverConfig(tolerance=1e-7, tolerance_k=1e-8, tolerance_phi=1e-7, boundary_left=p.bc_left,
                        boundary_right=p.bc_right)
don = snop.SolutionOperator.deeponet(g, OPS.deeponet_init(p.n_cells, width=64, seed=4), (1.0, 0.5))
q = W.config2(batch=8, n_cells=400)
other = [W.config3(batch=3, n_cells=1000), W.config3(batch=4, n_cells=777)]


def filler():
    for o in other:
        gg = snop.Grid1D(o.length, o.n_cells)
        snop.power_iteration(gg, o.order, o.sigma_t, o.sigma_s0, o.nu_sigma_f, o.chi,
                             snop.SolverConfig(tolerance=1e-300, tolerance_k=1e-300, tolerance_phi=1e-300,
                                               max_outer_iterations=3, max_inner_iterations=3))


def run():
    a = snop.sp_eigen(don, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg, recast_max_iterations=5)
    b = snop.cp_eigen(don, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg, recast_max_iterations=5)
    c = snop.precondition_fixed_source(don, q.order, q.sigma_t, q.sigma_s0, q.source,
                                       snop.SolverConfig(tolerance=q.tolerance), recast_max_iterations=5)
    return [a.k, a.phi, b.k, b.phi, c.phi]


ref = run()
bad = 0
for it in range(int(os.environ.get("REPS", "30"))):
    filler()
    r = run()
    m = [not np.array_equal(x, y) for x, y in zip(r, ref)]
    if any(m):
        bad += 1
        print("rep", it, "mismatch in [sp.k, sp.phi, cp.k, cp.phi, precond.phi]:", m, flush=True)
print(f"{bad} mismatching reps")
