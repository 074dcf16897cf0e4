"""Experiment: where does the host-API (e2e) time of C2 go? H2D/D2H bandwidth and host-path timings."""
import os, subprocess, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_01416_b200 import snop, workloads as W

p = W.config2()
g = snop.Grid1D(p.length, p.n_cells)
cfg = snop.SolverConfig(tolerance=p.tolerance)
pin = [torch.from_numpy(a).pin_memory() for a in (p.sigma_t, p.sigma_s0, p.source)]
dev = [torch.empty_like(x, device="cuda") for x in pin]
torch.cuda.synchronize()
for rep in range(2):
    t = time.perf_counter()
    for d, h in zip(dev, pin):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"H2D 3 arrays {3 * pin[0].numel() * 8 / 1e6:.0f} MB: {dt * 1e3:.2f} ms ({3 * pin[0].numel() * 8 / dt / 1e9:.1f} GB/s)")
out = (torch.empty((p.batch, p.n_cells), dtype=torch.float64).pin_memory().numpy(),
       torch.empty(p.batch, dtype=torch.int32).pin_memory().numpy(),
       torch.empty(p.batch, dtype=torch.uint8).pin_memory().numpy())
host = [x.numpy() for x in pin]
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    snop.source_iteration(g, p.order, *dev, cfg)
    torch.cuda.synchronize()
    print(f"device path: {(time.perf_counter() - t) * 1e3:.2f} ms")
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    snop.source_iteration(g, p.order, *host, cfg, out=out)
    print(f"host path (host_chunks={snop.default_context().options()['host_chunks']}): {(time.perf_counter() - t) * 1e3:.2f} ms")
