"""One warm K1 launch on a BASELINE config (profiling target: ncu -k regex:si_fixed -s 2 -c 1).
Usage: PYTHONPATH=. python tools/k1_once.py c2|c5"""
import sys

import torch

from paper_2509_01416_b200 import snop, workloads as W

p = W.config2() if sys.argv[1] == "c2" else W.config5()
g = snop.Grid1D(p.length, p.n_cells)
args = [torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.source)]
cfg = snop.SolverConfig(tolerance=p.tolerance)
for _ in range(3):
    r = snop.source_iteration(g, p.order, *args, cfg)
torch.cuda.synchronize()
print(sys.argv[1], "cell-pairs", int(r.iterations.to(torch.int64).sum()) * p.n_cells * p.order // 2)
