"""Run one solve of a config on the GPU (for ncu / sanitizer captures)."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2509_01416_b200 import snop, workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("config", choices=["c2", "c3", "c4", "c5"])
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
if a.config in ("c2", "c5"):
    p = (W.config2 if a.config == "c2" else W.config5)(**({"batch": a.batch} if a.batch else {}))
    g = snop.Grid1D(p.length, p.n_cells)
    args = [torch.from_numpy(x).cuda() for x in (p.sigma_t, p.sigma_s0, p.source)]
    for _ in range(a.reps):
        r = snop.source_iteration(g, p.order, *args, snop.SolverConfig(tolerance=p.tolerance))
    print("iters", r.iterations.float().mean().item())
else:
    p = (W.config3 if a.config == "c3" else W.config4)(**({"batch": a.batch} if a.batch else {}))
    g = snop.Grid1D(p.length, p.n_cells)
    args = [torch.from_numpy(x).cuda() for x in (p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi)]
    cfg = snop.SolverConfig(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi,
                            boundary_left=p.bc_left, boundary_right=p.bc_right)
    for _ in range(a.reps):
        r = snop.power_iteration(g, p.order, *args, cfg)
    print("outer", r.outer_iterations.float().mean().item())
