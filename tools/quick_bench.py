"""Quick device-resident timing of the fused kernels (not the bench contract; see bench.py)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2509_01416_b200 import snop, workloads as W

print(torch.cuda.get_device_name(0), flush=True)
ctx = snop.default_context()


def time_si(p, reps=3):
    g = snop.Grid1D(p.length, p.n_cells)
    args = [torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.source)]
    cfg = snop.SolverConfig(tolerance=p.tolerance)
    for rep in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = snop.source_iteration(g, p.order, *args, cfg)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        it = r.iterations.cpu().numpy().astype(np.int64)
        upd = it.sum() * p.n_cells * p.order
        print(f"{p.name} B={p.batch} Nc={p.n_cells} S{p.order}: {dt*1e3:.2f} ms iters mean {it.mean():.1f} "
              f"max {it.max()} | {upd/dt:.3e} upd/s | alg {it.sum()*p.n_cells*40/dt/1e9:.0f} GB/s", flush=True)


def time_pi(p, reps=2):
    g = snop.Grid1D(p.length, p.n_cells)
    args = [torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi)]
    cfg = snop.SolverConfig(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi,
                            boundary_left=p.bc_left, boundary_right=p.bc_right)
    for rep in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = snop.power_iteration(g, p.order, *args, cfg)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        inner = r.total_inner_iterations.cpu().numpy()
        upd = inner.sum() * p.n_cells * p.order
        print(f"{p.name} B={p.batch} G={p.n_groups}: {dt*1e3:.2f} ms outer mean {r.outer_iterations.float().mean():.1f}"
              f" inner sum {inner.sum()} | {upd/dt:.3e} upd/s", flush=True)


which = sys.argv[1:] or ["c2", "c5", "c3", "c4"]
if "c2" in which: time_si(W.config2())
if "c5" in which: time_si(W.config5())
if "c3" in which: time_pi(W.config3())
if "c4" in which: time_pi(W.config4())
