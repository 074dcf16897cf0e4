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
# round-2 paths: streaming K1 / device-looped power iteration (forced), rate-routed two-stream tail
# split, tensor-core FNO (width 64: DFT, mixing, inverse+W, projection), recast fixed point loop
ctx = snop.default_context()
ctx.set_options(cell_cluster=-1)
q = W.config2(batch=3, n_cells=2100)
snop.source_iteration(snop.Grid1D(10.0, 2100), 8, q.sigma_t, q.sigma_s0, q.source, cfg, want_leakage=True)
m = W.config4(batch=2, n_cells=200)
snop.power_iteration(snop.Grid1D(m.length, m.n_cells), 8, m.sigma_t, m.sigma_s0, m.nu_sigma_f, m.chi,
                     snop.SolverConfig(tolerance=1e-6, tolerance_k=1e-7, tolerance_phi=1e-6, max_outer_iterations=20))
ctx.set_options(cell_cluster=0, pi_tail_cap=6)
c3 = W.config3(batch=12, n_cells=512)
snop.power_iteration(snop.Grid1D(c3.length, c3.n_cells), 16, c3.sigma_t, c3.sigma_s0, c3.nu_sigma_f, c3.chi,
                     snop.SolverConfig(tolerance=1e-7, tolerance_k=1e-8, tolerance_phi=1e-7, boundary_left=1))
ctx.set_options(pi_tail_cap=0)
f64 = snop.SolutionOperator.fno(snop.Grid1D(10.0, 512), OPS.fno_init(64, 16, 2, 128, OPS.GELU), (1.0, 0.8))
p5 = W.config5(batch=6, n_cells=512)
snop.recast_fixed_point(f64, p5.source, p5.sigma_t, p5.sigma_s0, 1e-4, 10)
print("round-2 sanitize cases done")
