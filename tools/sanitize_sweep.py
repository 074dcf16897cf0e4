"""compute-sanitizer exercise of the round-2 additions: the standalone sweep (both kernel paths, all
boundary combinations, ragged tiles), the rewritten K1/K2 scan at every CTA size, and the
operator-backed power iteration."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2509_01416_b200 import snop, workloads as W
r = np.random.default_rng(0)
for B, Nc, N in ((3, 50, 8), (2, 37, 6), (5, 130, 16), (2, 9, 2), (3, 64, 64)):
    st = r.uniform(0.2, 2.0, (B, Nc))
    em = r.uniform(0.0, 1.0, (B, Nc, N))
    for bc in ((0, 0), (1, 0), (0, 1), (1, 1)):
        snop.sweep(snop.Grid1D(10.0, Nc), N, st, em, *bc)
cfg = snop.SolverConfig(tolerance=1e-6, max_inner_iterations=30)
for Nc in (200, 500, 1000, 2000, 4000):  # NT = 32 ... 512
    p = W.config2(batch=2, n_cells=Nc)
    snop.source_iteration(snop.Grid1D(10.0, Nc), 8, p.sigma_t, p.sigma_s0, p.source, cfg)
e = W.three_group_table9()
ec = snop.SolverConfig(tolerance=1e-7, tolerance_k=1e-8, tolerance_phi=1e-7, max_outer_iterations=30)
ex = snop.SolutionOperator.exact(snop.Grid1D(e.length, e.n_cells), 8, (1.0, 0.5), snop.SolverConfig(tolerance=1e-7))
snop.power_iteration_with_operator(ex, 8, e.sigma_t, e.sigma_s0, e.nu_sigma_f, e.chi, ec, inner_solver=1)
print("sweep / scan sanitize cases done")
