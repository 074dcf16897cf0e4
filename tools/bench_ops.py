"""Device timing of the neural-operator forwards and the MD-PNOP warm start (C2 DeepONet, C5 FNO)."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2509_01416_b200 import operators as OPS, snop, workloads as W

ctx = snop.default_context()


def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    return min(ts)


p2 = W.config2()
g2 = snop.Grid1D(10.0, 2000)
don = snop.SolutionOperator.deeponet(g2, OPS.deeponet_init(2000), (1.0, 0.5))
src2 = torch.from_numpy(p2.source).cuda()
t = timeit(lambda: don.predict(src2))
fl = 2 * 2048 * (2000 * 128 + 3 * 128 * 128) + 2 * 2048 * 2000 * 128
print(f"DeepONet C2 predict: {t*1e3:.3f} ms  {fl/t/1e12:.2f} TFLOP/s (fp32-equivalent)")
p5 = W.config5()
g5 = snop.Grid1D(10.0, 1024)
fno = snop.SolutionOperator.fno(g5, OPS.fno_init(), (1.0, 0.8))
src5 = torch.from_numpy(p5.source).cuda()
t = timeit(lambda: fno.predict(src5), reps=3)
fl = 86.5e6 * 4096
print(f"FNO C5 predict: {t*1e3:.3f} ms  {fl/t/1e12:.2f} TFLOP/s (fp32-equivalent)")
st5, ss5 = (torch.from_numpy(x).cuda() for x in (p5.sigma_t, p5.sigma_s0))
for name, op, p, st, ss, S in (("C2/DeepONet", don, p2, None, None, src2), ("C5/FNO", fno, p5, st5, ss5, src5)):
    if st is None:
        st, ss = (torch.from_numpy(x).cuda() for x in (p.sigma_t, p.sigma_s0))
    cfg = snop.SolverConfig(tolerance=1e-8)
    t0 = timeit(lambda: snop.source_iteration(snop.Grid1D(10.0, p.n_cells), p.order, st, ss, S, cfg), reps=2)
    r0 = snop.source_iteration(snop.Grid1D(10.0, p.n_cells), p.order, st, ss, S, cfg)
    for rmax in (0, 1, 50):
        tw = timeit(lambda: snop.precondition_fixed_source(op, p.order, st, ss, S, cfg, recast_max_iterations=rmax), reps=2)
        rw = snop.precondition_fixed_source(op, p.order, st, ss, S, cfg, recast_max_iterations=rmax)
        print(f"{name}: zero-guess {t0*1e3:.2f} ms ({r0.iterations.float().mean():.1f} it) | warm rmax={rmax}: {tw*1e3:.2f} ms "
              f"refine {rw.refine_iterations.float().mean():.1f} it, recast it {rw.precond_iterations.float().mean():.1f}, "
              f"status {np.bincount(rw.recast_status.cpu().numpy(), minlength=3)}")
