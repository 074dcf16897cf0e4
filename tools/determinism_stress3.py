"""Experiment: bit-reproducibility of ONE K1 sweep (fixed source) on C3-like instances with other
kernels run in between; varies the boundary condition to localise the difference."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2509_01416_b200 import snop, workloads as W

p3 = W.config3(batch=6, n_cells=700)
st, ss = p3.sigma_t[:, 0], p3.sigma_s0[:, 0, 0]
src = np.ones_like(st)
g = snop.Grid1D(p3.length, p3.n_cells)
other = [W.config3(batch=3, n_cells=1000), W.config3(batch=4, n_cells=777)]


def filler():
    for q in other:
        os.environ["SNOP_PS"] = "0"
        gg = snop.Grid1D(q.length, q.n_cells)
        snop.power_iteration(gg, q.order, q.sigma_t, q.sigma_s0, q.nu_sigma_f, q.chi,
                             snop.SolverConfig(tolerance=1e-300, tolerance_k=1e-300, tolerance_phi=1e-300,
                                               max_outer_iterations=3, max_inner_iterations=3))


for bl, br, its in ((1, 0, 1), (0, 0, 1), (0, 1, 1), (1, 0, 5)):
    cfg = snop.SolverConfig(tolerance=1e-300, max_inner_iterations=its, boundary_left=bl, boundary_right=br)
    ref = snop.source_iteration(g, 32, st, ss, src, cfg).phi
    bad = []
    for it in range(60):
        filler()
        r = snop.source_iteration(g, 32, st, ss, src, cfg).phi
        if not np.array_equal(r, ref):
            d = np.abs(r - ref)
            bad.append((it, [int(x) for x in np.nonzero(d.max(axis=1))[0]], int(np.argmax(d.max(axis=0))),
                        float(d.max() / np.abs(ref).max())))
    print(f"bc {bl}{br} its {its}: {len(bad)} mismatches {bad[:3]}", flush=True)
