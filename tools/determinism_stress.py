"""Experiment: look for run-to-run differences of the tail-split / pair-split eigen solve, with
differently sized solves interleaved (workspace reuse) as in the test sequence."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2509_01416_b200 import snop, workloads as W


def solve(p, ps, split):
    os.environ["SNOP_PS"] = ps
    os.environ["SNOP_PI_SPLIT"] = split
    g = snop.Grid1D(p.length, p.n_cells)
    cfg = snop.SolverConfig(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi,
                            boundary_left=p.bc_left, boundary_right=p.bc_right)
    return snop.power_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)


main = W.config3(batch=6, n_cells=700)
other = [W.config3(batch=3, n_cells=1000), W.config3(batch=4, n_cells=777)]
MPS, MSPLIT = os.environ.get("MPS", "8"), os.environ.get("MSPLIT", "4")
ref = solve(main, MPS, MSPLIT)
bad = 0
N = int(os.environ.get("REPS", "100"))
for it in range(N):
    if os.environ.get("INTERLEAVE", "1") == "1":
        for q, ps in zip(other, ("2", "4")):
            solve(q, ps, "0")
    r = solve(main, MPS, MSPLIT)
    if not (np.array_equal(r.k, ref.k) and np.array_equal(r.phi, ref.phi)):
        bad += 1
        dk = np.abs(r.k - ref.k) / ref.k
        print(f"rep {it}: k rel diff per instance {dk.tolist()} outer {r.outer_iterations.tolist()} "
              f"inner {r.total_inner_iterations.tolist()} vs {ref.total_inner_iterations.tolist()}", flush=True)
print(f"MPS={MPS} MSPLIT={MSPLIT} interleave={os.environ.get('INTERLEAVE', '1')}: {bad} mismatches in {N}")
