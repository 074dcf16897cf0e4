"""Experiment: per-phase cycle breakdown of K1 (needs a -DSNOP_PHASE_TIMING build via SNOP_LIB).
Usage: SNOP_LIB=tmp_exp/timing.so python tools/phase_timing.py [c2|c5 ...] [batch ...]"""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_01416_b200 import snop, workloads as W, _capi
lib = _capi.load()
f = lib.snop_internal_phase_cycles
f.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(20, dtype=np.uint64)
labels = ["A maps", "bar1", "B scan", "bar2", "C replay", "pairs total", "phi+norm"]
cfgs = [a for a in sys.argv[1:] if not a.isdigit()] or ["c2"]
for batch in [int(a) for a in sys.argv[1:] if a.isdigit()] or [0]:
    for name, p in [(c.upper(), (W.config2(batch=batch) if batch else W.config2()) if c == "c2" else
                     (W.config5(batch=batch) if batch else W.config5())) for c in cfgs]:
        g = snop.Grid1D(p.length, p.n_cells)
        args = [torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.source)]
        snop.source_iteration(g, p.order, *args, snop.SolverConfig(tolerance=p.tolerance))
        torch.cuda.synchronize()
        f(buf.ctypes.data, 1)
        r = snop.source_iteration(g, p.order, *args, snop.SolverConfig(tolerance=p.tolerance))
        torch.cuda.synchronize()
        rc = f(buf.ctypes.data, 1)
        assert rc == 0, f"snop_internal_phase_cycles -> cudaError {rc}"
        it = int(np.asarray(r.iterations.cpu() if hasattr(r.iterations, "cpu") else r.iterations).astype(np.int64).sum())
        ngroups = it * (p.order // 2 // 2)
        for w in range(2):
            row = buf[w * 10: w * 10 + 10].astype(np.float64)
            print(name, "B", p.batch, "warp", w, " | ".join(f"{labels[k]} {row[k] / (ngroups if k < 5 else it):7.0f}"
                                                         for k in range(7)), "(cycles per group / per iteration)")
