"""Probe: MD-PNOP warm-start arms on the BASELINE configs (device timing, CUDA events).

C5: zero guess vs FNO (single shot / full recast fixed point) vs the exact operator (single shot
/ full fixed point), plus Delta p = 0 with the exact operator. C3: SP / CP hybrid eigen solves with
the exact operator and with the random-init FNO against the cold power iteration.
Usage: PYTHONPATH=. python tools/md_pnop_probe.py [c5] [c3]"""
import sys
import time

import numpy as np
import torch

from paper_2509_01416_b200 import operators as OPS, snop, workloads as W


def timed(ctx, fn, reps=2):
    stream = torch.cuda.ExternalStream(ctx.stream_ptr)
    out = fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = fn()
        e1.record(stream)
        ctx.synchronize()
        ts.append(e0.elapsed_time(e1))
    return out, min(ts)


def c5(ctx):
    p = W.config5()
    g = snop.Grid1D(p.length, p.n_cells)
    cfg = snop.SolverConfig(tolerance=p.tolerance)
    st, ss, src = (torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.source))
    fno = snop.SolutionOperator.fno(g, OPS.fno_init(64, 16, 4, 128, OPS.GELU), p.ref_params, ctx=ctx)
    exact = snop.SolutionOperator.exact(g, p.order, p.ref_params, snop.SolverConfig(tolerance=1e-8), ctx=ctx)
    cold, t = timed(ctx, lambda: snop.source_iteration(g, p.order, st, ss, src, cfg, ctx=ctx, sync=False))
    print(f"C5 zero guess: {t:.2f} ms, iterations mean {cold.iterations.float().mean().item():.2f}")
    for name, op, rmax in (("fno 1", fno, 1), ("fno 50", fno, 50), ("exact 1", exact, 1), ("exact 50", exact, 50)):
        r, t = timed(ctx, lambda: snop.precondition_fixed_source(op, p.order, st, ss, src, cfg, recast_max_iterations=rmax))
        print(f"C5 {name}: {t:.2f} ms, recast it mean {r.precond_iterations.float().mean().item():.2f} max "
              f"{r.precond_iterations.max().item()}, status {np.bincount(r.recast_status.cpu().numpy(), minlength=3)}, "
              f"refine mean {r.refine_iterations.float().mean().item():.2f} max {r.refine_iterations.max().item()}")
    one = torch.ones_like(st)
    r, t = timed(ctx, lambda: snop.precondition_fixed_source(exact, p.order, one, 0.8 * one, src, cfg))
    print(f"C5 dp=0 exact: {t:.2f} ms, recast it max {r.precond_iterations.max().item()}, refine max "
          f"{r.refine_iterations.max().item()}")


def c3(ctx):
    p = W.config3()
    g = snop.Grid1D(p.length, p.n_cells)
    cfg = snop.SolverConfig(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi,
                            boundary_left=p.bc_left, boundary_right=p.bc_right)
    dev = [torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi)]
    cold, t = timed(ctx, lambda: snop.power_iteration(g, p.order, *dev, cfg, ctx=ctx, sync=False), reps=1)
    print(f"C3 cold: {t:.1f} ms, outer mean {cold.outer_iterations.float().mean().item():.1f}, inner total "
          f"{cold.total_inner_iterations.sum().item()}")
    exact = snop.SolutionOperator.exact(g, p.order, (1.0, 0.5), snop.SolverConfig(tolerance=1e-7,
                                        boundary_left=p.bc_left, boundary_right=p.bc_right), ctx=ctx)
    fno = snop.SolutionOperator.fno(g, OPS.fno_init(64, 16, 4, 128, OPS.GELU), (1.0, 0.5), ctx=ctx)
    for opname, op in (("exact", exact), ("fno", fno)):
        for alg in ("sp", "cp"):
            fn = getattr(snop, f"{alg}_eigen")
            t0 = time.perf_counter()
            r, t = timed(ctx, lambda: fn(op, p.order, *dev, cfg), reps=1)
            print(f"C3 {alg.upper()} {opname}: {t:.1f} ms (wall {1e3 * (time.perf_counter() - t0):.0f}), "
                  f"stage1 outer mean {r.stage1_outer.float().mean().item():.1f}, stage2 outer mean "
                  f"{r.stage2_outer.float().mean().item():.1f}, stage2 inner total {int(r.stage2_inner.sum().item())}, "
                  f"k err vs cold {(r.k - cold.k).abs().div(cold.k).max().item():.1e}")


if __name__ == "__main__":
    ctx = snop.Context(0)
    which = sys.argv[1:] or ["c5", "c3"]
    if "c5" in which:
        c5(ctx)
    if "c3" in which:
        c3(ctx)
