"""Experiment: time the C2 DeepONet warm-start pieces (recast FP, refine solve) on the device."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_01416_b200 import snop, operators as OPS, workloads as W
p = W.config2()
g = snop.Grid1D(p.length, p.n_cells)
cfg = snop.SolverConfig(tolerance=p.tolerance)
st, ss, src = (torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.source))
ctx = snop.default_context()
don = snop.SolutionOperator.deeponet(g, OPS.deeponet_init(p.n_cells), p.ref_params, ctx=ctx)
def t(label, fn, reps=3):
    for r in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize()
        print(f"{label}: {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
    return out
t("zero-guess solve", lambda: snop.source_iteration(g, p.order, st, ss, src, cfg))
rf = t("recast FP (max 1)", lambda: snop.recast_fixed_point(don, src, st, ss, max_iterations=1))
t("warm solve from phi_NO", lambda: snop.source_iteration(g, p.order, st, ss, src, cfg, initial_phi=rf.phi))
t("precondition_fixed_source", lambda: snop.precondition_fixed_source(don, p.order, st, ss, src, cfg, recast_max_iterations=1))
# after a zero-copy host-API solve (as in bench.py's e2e arm)
pin = [torch.from_numpy(a).pin_memory() for a in (p.sigma_t, p.sigma_s0, p.source)]
host = [x.numpy() for x in pin]
outs = (torch.empty((p.batch, p.n_cells), dtype=torch.float64).pin_memory().numpy(),
        torch.empty(p.batch, dtype=torch.int32).pin_memory().numpy(),
        torch.empty(p.batch, dtype=torch.uint8).pin_memory().numpy())
t("host zero-copy solve", lambda: snop.source_iteration(g, p.order, *host, cfg, out=outs))
t("precondition_fixed_source after zero-copy", lambda: snop.precondition_fixed_source(don, p.order, st, ss, src, cfg, recast_max_iterations=1))
t("zero-guess solve after zero-copy", lambda: snop.source_iteration(g, p.order, st, ss, src, cfg))
