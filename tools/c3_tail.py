import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_01416_b200 import workloads as W, snop
p = W.config3()
cfg = snop.SolverConfig(tolerance=1e-7, tolerance_k=1e-8, tolerance_phi=1e-7, boundary_left=1)
g = snop.Grid1D(10., 4096)
idx = [int(sys.argv[1])] if len(sys.argv) > 1 else None
if idx is None:
    r = snop.power_iteration(g, 32, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)
    i = np.asarray(r.total_inner_iterations); print("argmax", int(i.argmax()), i.max()); sys.exit()
q = p.subset(idx)
cs = int(sys.argv[2]) if len(sys.argv) > 2 else 0
snop.default_context().set_options(pair_split=cs)
args = [torch.from_numpy(a).cuda() for a in (q.sigma_t, q.sigma_s0, q.nu_sigma_f, q.chi)]
snop.power_iteration(g, 32, *args, cfg)
torch.cuda.synchronize(); t = time.perf_counter()
r = snop.power_iteration(g, 32, *args, cfg)
torch.cuda.synchronize(); dt = time.perf_counter() - t
inner = int(r.total_inner_iterations[0])
print(f"pair_split={cs} inst {idx[0]}: {dt*1e3:.1f} ms, inner {inner}, {dt/inner*1e6:.1f} us/inner sweep, k={float(r.k[0]):.8f}")
