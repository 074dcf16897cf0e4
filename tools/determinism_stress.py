"""Probe: bit-reproducibility of repeated solves with differently sized solves interleaved (so
shared memory and workspaces hold other data between repeats).

  python tools/determinism_stress.py eigen  [--pair-split 8] [--tail-cap 4] [--reps 100]
  python tools/determinism_stress.py hybrid [--reps 30]     # SP / CP eigen + warm-started fixed source
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2509_01416_b200 import operators as OPS, snop, workloads as W  # noqa: E402


def eigen(p, ctx, **opt):
    ctx.set_options(**opt)
    cfg = snop.SolverConfig(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi,
                            boundary_left=p.bc_left, boundary_right=p.bc_right)
    r = snop.power_iteration(snop.Grid1D(p.length, p.n_cells), p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi,
                             cfg, ctx=ctx)
    return [r.k, r.phi]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["eigen", "hybrid"])
    ap.add_argument("--pair-split", type=int, default=8)
    ap.add_argument("--tail-cap", type=int, default=4)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--no-interleave", action="store_true")
    a = ap.parse_args()
    ctx = snop.Context(0)
    main_p = W.config3(batch=6, n_cells=700)
    other = [W.config3(batch=3, n_cells=1000), W.config3(batch=4, n_cells=777)]
    if a.mode == "eigen":
        run = lambda: eigen(main_p, ctx, pair_split=a.pair_split, pi_tail_cap=a.tail_cap)  # noqa: E731
        filler = lambda: [eigen(q, ctx, pair_split=ps, pi_tail_cap=-1) for q, ps in zip(other, (2, 4))]  # noqa: E731
    else:
        p = W.config3(batch=4, n_cells=400)
        g = snop.Grid1D(p.length, p.n_cells)
        cfg = snop.SolverConfig(tolerance=1e-7, tolerance_k=1e-8, tolerance_phi=1e-7, boundary_left=p.bc_left,
                                boundary_right=p.bc_right)
        don = snop.SolutionOperator.deeponet(g, OPS.deeponet_init(p.n_cells, width=64, seed=4), (1.0, 0.5), ctx=ctx)
        q = W.config2(batch=8, n_cells=400)

        def run():
            x = snop.sp_eigen(don, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg, recast_max_iterations=5)
            y = snop.cp_eigen(don, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg, recast_max_iterations=5)
            z = snop.precondition_fixed_source(don, q.order, q.sigma_t, q.sigma_s0, q.source,
                                               snop.SolverConfig(tolerance=q.tolerance), recast_max_iterations=5)
            return [x.k, x.phi, y.k, y.phi, z.phi]

        filler = lambda: [eigen(o, ctx, pair_split=0, pi_tail_cap=0) for o in other]  # noqa: E731
    ref = run()
    bad = 0
    for it in range(a.reps):
        if not a.no_interleave:
            filler()
        r = run()
        m = [not np.array_equal(x, y) for x, y in zip(r, ref)]
        if any(m):
            bad += 1
            print(f"rep {it}: mismatching outputs {m}", flush=True)
    print(f"{a.mode}: {bad} mismatching reps of {a.reps}")


if __name__ == "__main__":
    main()
