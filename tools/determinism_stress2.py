"""Experiment: is the single-CTA eigen kernel bit-reproducible when other kernels ran on the SMs in
between? Fixed (tiny) iteration counts so a difference can be localised."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2509_01416_b200 import snop, workloads as W

os.environ["SNOP_PI_SPLIT"] = "0"


def solve(p, ps, outer, inner):
    os.environ["SNOP_PS"] = ps
    g = snop.Grid1D(p.length, p.n_cells)
    cfg = snop.SolverConfig(tolerance=1e-300, tolerance_k=1e-300, tolerance_phi=1e-300, max_outer_iterations=outer,
                            max_inner_iterations=inner, boundary_left=p.bc_left, boundary_right=p.bc_right)
    return snop.power_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)


main = W.config3(batch=6, n_cells=700)
other = [W.config3(batch=3, n_cells=1000), W.config3(batch=4, n_cells=777)]
for outer, inner in ((1, 1), (1, 3), (3, 3), (8, 8)):
    ref = solve(main, "0", outer, inner)
    bad = []
    for it in range(60):
        for q, ps in zip(other, (os.environ.get("OPS", "2"), os.environ.get("OPS2", "4"))):
            solve(q, ps, 3, 3)
        r = solve(main, "0", outer, inner)
        if not np.array_equal(r.phi, ref.phi):
            d = np.abs(r.phi - ref.phi)
            bad.append((it, [int(x) for x in np.nonzero(d.reshape(6, -1).max(axis=1))[0]],
                        int(np.argmax(d.reshape(6, -1).max(axis=0)))))
    print(f"outer {outer} inner {inner}: {len(bad)} mismatches {bad[:4]}", flush=True)
