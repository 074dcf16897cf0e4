"""Experiment: repeat a batched eigen solve and count bit-level mismatches (SNOP_PS / SNOP_PI_SPLIT
from the environment)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2509_01416_b200 import snop, workloads as W
p = W.config3(batch=int(os.environ.get("B", "6")), n_cells=int(os.environ.get("NC", "700")))
g = snop.Grid1D(p.length, p.n_cells)
cfg = snop.SolverConfig(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi,
                        boundary_left=p.bc_left, boundary_right=p.bc_right)
ref = snop.power_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)
bad = 0
for _ in range(int(os.environ.get("REPS", "20"))):
    r = snop.power_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)
    if not (np.array_equal(r.k, ref.k) and np.array_equal(r.phi, ref.phi)):
        bad += 1
        print("mismatch: k maxrel", float(np.max(np.abs(r.k - ref.k) / ref.k)), "phi maxrel",
              float(np.max(np.abs(r.phi - ref.phi)) / np.max(np.abs(ref.phi))),
              "outer", r.outer_iterations.tolist(), ref.outer_iterations.tolist())
print(f"PS={os.environ.get('SNOP_PS')} SPLIT={os.environ.get('SNOP_PI_SPLIT')}: {bad} mismatches")
