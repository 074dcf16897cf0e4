"""Small end-to-end exercise of every entry point for compute-sanitizer runs."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2509_01416_b200 import snop, operators as OPS, workloads as W
g = snop.Grid1D(10.0, 300)
p = W.config2(batch=40, n_cells=300)
cfg = snop.SolverConfig(tolerance=1e-8)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
r = snop.source_iteration(g, 16, p.sigma_t, p.sigma_s0, p.source, cfg, want_leakage=True, want_current=True,
                          sigma_s1=0.1 * p.sigma_s0)
snop.balance_report(g, p.sigma_t, p.sigma_s0, p.source, r.phi, r.leakage)
outs = (pin(np.empty((40, 300))), pin(np.empty(40, dtype=np.int32)), pin(np.empty(40, dtype=np.uint8)))
snop.source_iteration(g, 16, pin(p.sigma_t), pin(p.sigma_s0), pin(p.source), cfg, out=outs)
e = W.three_group_table9()
snop.power_iteration(snop.Grid1D(e.length, e.n_cells), 8, e.sigma_t, e.sigma_s0, e.nu_sigma_f, e.chi,
                     snop.SolverConfig(tolerance=1e-7, tolerance_k=1e-8, tolerance_phi=1e-7))
don = snop.SolutionOperator.deeponet(g, OPS.deeponet_init(300, width=32), (1.0, 0.5))
snop.precondition_fixed_source(don, 16, p.sigma_t, p.sigma_s0, p.source, cfg)
fno = snop.SolutionOperator.fno(snop.Grid1D(10.0, 256), OPS.fno_init(16, 8, 2, 32), (1.0, 0.8))
fno.predict(np.random.default_rng(0).uniform(0, 1, (5, 256)))
ex = snop.SolutionOperator.exact(snop.Grid1D(e.length, e.n_cells), 8, (1.0, 0.5), snop.SolverConfig(tolerance=1e-7))
snop.cp_eigen(ex, 8, e.sigma_t, e.sigma_s0, e.nu_sigma_f, e.chi, snop.SolverConfig(tolerance=1e-7, tolerance_k=1e-8, tolerance_phi=1e-7, max_outer_iterations=50))
snop.generate_dataset(8, snop.GrfSpec(seed=1), snop.Grid1D(10.0, 100), 8)
print("sanitize cases done")
