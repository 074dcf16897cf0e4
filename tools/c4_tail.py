"""Experiment: C4 per-instance inner-sweep counts and the single-instance latency of the slowest one."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_01416_b200 import workloads as W, snop
p = W.config4()
cfg = snop.SolverConfig(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi)
g = snop.Grid1D(p.length, p.n_cells)
r = snop.power_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)
inner = np.asarray(r.total_inner_iterations); outer = np.asarray(r.outer_iterations)
i = int(inner.argmax())
print("inner sweeps: mean", inner.mean(), "max", inner.max(), "at", i, "outer", outer[i], "| outer mean", outer.mean())
q = p.subset([i])
args = [torch.from_numpy(a).cuda() for a in (q.sigma_t, q.sigma_s0, q.nu_sigma_f, q.chi)]
snop.power_iteration(g, p.order, *args, cfg)
torch.cuda.synchronize(); t = time.perf_counter()
r1 = snop.power_iteration(g, p.order, *args, cfg)
torch.cuda.synchronize(); dt = time.perf_counter() - t
n1 = int(r1.total_inner_iterations[0])
print(f"slowest instance alone: {dt*1e3:.1f} ms, {n1} inner sweeps, {dt/n1*1e6:.2f} us per sweep")
allargs = [torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi)]
torch.cuda.synchronize(); t = time.perf_counter()
snop.power_iteration(g, p.order, *allargs, cfg)
torch.cuda.synchronize(); print(f"whole C4 batch: {(time.perf_counter()-t)*1e3:.1f} ms")
