"""Randomised differential run of the fused solvers and the sweep against the CPU oracle: random
cell counts around every CTA-size boundary, orders, boundary conditions, norms, P1 moments, thin and
thick cells, group counts with upscatter. Fixed iteration counts (tolerance -> 0), so fluxes / k must
agree at 1e-10. Usage: python tools/fuzz_parity.py [n_cases] [seed]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2509_01416_b200 import snop
from tests import oracle_lib as O

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
edges = [1, 2, 7, 8, 9, 255, 256, 257, 511, 512, 513, 1023, 1024, 1025, 2047, 2048, 2049, 4095, 4096, 4097, 5000]
worst = {"si": 0.0, "pi_k": 0.0, "pi_phi": 0.0, "sweep": 0.0}
for case in range(n_cases):
    kind = rng.choice(["si", "si", "pi", "sweep"])
    Nc = int(rng.choice(edges)) if rng.random() < 0.6 else int(rng.integers(1, 3000))
    N = int(rng.choice([2, 4, 6, 8, 16, 32, 64]))
    L = float(rng.uniform(0.5, 40.0))
    bl, br = int(rng.integers(0, 2)), int(rng.integers(0, 2))
    lo = 10.0 ** rng.uniform(-5, -0.5) if rng.random() < 0.3 else 0.2
    B = int(rng.integers(1, 5))
    if kind == "sweep":
        st = rng.uniform(lo, 3.0, (B, Nc)); em = rng.uniform(0, 2.0, (B, Nc, N))
        psi, ol, orr = snop.sweep(snop.Grid1D(L, Nc), N, st, em, bl, br)
        o_psi, o_ol, o_or = O.sweep(L, Nc, N, st, em, bl, br)
        e = np.max(np.abs(psi - o_psi)) / max(np.max(np.abs(o_psi)), 1e-300)
        sc = max(np.max(np.abs(o_ol)), np.max(np.abs(o_or)), 1e-300)
        e = max(e, np.max(np.abs(ol - o_ol)) / sc, np.max(np.abs(orr - o_or)) / sc)
        worst["sweep"] = max(worst["sweep"], e)
    elif kind == "si":
        st = rng.uniform(lo, 3.0, (B, Nc)); c = rng.uniform(0.0, 0.98, (B, 1)); ss = c * st
        src = rng.uniform(0.0, 2.0, (B, Nc))
        s1 = (rng.uniform(0.0, 0.3, (B, Nc)) * ss) if rng.random() < 0.3 else None
        norm = int(rng.integers(0, 2)); nit = int(rng.integers(1, 9))
        phi0 = rng.uniform(0.0, 1.0, (B, Nc)) if rng.random() < 0.3 else None
        cfg = snop.SolverConfig(tolerance=1e-300, max_inner_iterations=nit, boundary_left=bl, boundary_right=br,
                                convergence_norm=norm)
        r = snop.source_iteration(snop.Grid1D(L, Nc), N, st, ss, src, cfg, initial_phi=phi0, sigma_s1=s1,
                                  want_current=True)
        o = O.source_iteration(L, Nc, N, st, ss, src, cfg.c(), sigma_s1=s1, initial_phi=phi0, want_current=True)
        e = np.max(np.abs(r.phi - o["phi"])) / max(np.max(np.abs(o["phi"])), 1e-300)
        worst["si"] = max(worst["si"], e)
    else:
        G = int(rng.choice([1, 1, 2, 3, 7])); Nc = min(Nc, 2100)
        st = rng.uniform(max(lo, 0.05), 2.0, (B, G, Nc))
        ssm = rng.uniform(0.0, 1.0, (B, G, G, Nc))
        ssm *= (0.7 * st[:, :, None, :] / ssm.sum(axis=2, keepdims=True).clip(1e-30))  # row sums < Sigma_t
        nsf = rng.uniform(0.0, 0.4, (B, G, Nc)); nsf[:, 0, : max(1, Nc // 2)] += 0.05
        chi = rng.uniform(0.0, 1.0, (B, G)); chi /= chi.sum(axis=1, keepdims=True)
        cfg = snop.SolverConfig(tolerance=1e-300, tolerance_k=1e-300, tolerance_phi=1e-300,
                                max_inner_iterations=int(rng.integers(1, 4)),
                                max_outer_iterations=int(rng.integers(1, 6)), boundary_left=bl, boundary_right=br)
        r = snop.power_iteration(snop.Grid1D(L, Nc), N, st, ssm, nsf, chi, cfg)
        o = O.power_iteration(L, Nc, N, G, st, ssm, nsf, chi, cfg.c())
        worst["pi_k"] = max(worst["pi_k"], float(np.max(np.abs(r.k - o["k"]) / np.abs(o["k"]))))
        worst["pi_phi"] = max(worst["pi_phi"], float(np.max(np.abs(r.phi - o["phi"])) / np.max(np.abs(o["phi"]))))
    bad = {k: v for k, v in worst.items() if not (v < 1e-10)}
    if bad:
        print("FAIL at case", case, kind, dict(Nc=Nc, N=N, L=L, bl=bl, br=br, lo=lo, B=B), worst, flush=True)
        sys.exit(1)
print(f"{n_cases} cases ok; worst relative differences {worst}")
