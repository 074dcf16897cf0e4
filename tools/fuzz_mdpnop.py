"""Randomised differential run of the MD-PNOP drivers with the exact operator (fp64 on both sides, so
statuses, counts and fields must agree): recast_fixed_point (per-instance freeze / divergence guard /
max-iteration status), precondition_fixed_source (recast fixed point -> warm-started source
iteration) and power_iteration_with_operator / cp_eigen on small random single- and multigroup
problems, against the CPU oracle. Usage: python tools/fuzz_mdpnop.py [n_cases] [seed]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2509_01416_b200 import snop
from tests import oracle_lib as O

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
fails = 0
worst = {"recast_phi": 0.0, "precond_phi": 0.0, "cp_k": 0.0}
for case in range(n_cases):
    Nc = int(rng.choice([5, 16, 40, 100, 257, 600])); N = int(rng.choice([4, 8, 16])); L = float(rng.uniform(2.0, 20.0))
    B = int(rng.integers(1, 7))
    tstar = float(rng.uniform(0.6, 1.5)); sstar = float(rng.uniform(0.1, 0.8)) * tstar
    tol = 10.0 ** rng.uniform(-9, -6)
    bl, br = int(rng.integers(0, 2)), int(rng.integers(0, 2))
    ocfg = O.make_config(tol, bc_left=bl, bc_right=br)
    dcfg = snop.SolverConfig(tolerance=tol, boundary_left=bl, boundary_right=br)
    g = snop.Grid1D(L, Nc)
    op = snop.SolutionOperator.exact(g, N, (tstar, sstar), dcfg)
    oo = O.OracleOperator.exact(L, Nc, N, (tstar, sstar), ocfg)
    kind = rng.choice(["recast", "precond", "cp"])
    # deviations from p*: small (converges), large scattering excess (may diverge -> status 2)
    dev = float(rng.choice([0.0, 0.05, 0.3, 1.5]))
    st = tstar * (1.0 + dev * rng.uniform(-0.3, 0.3, (B, Nc)))
    ss = np.minimum(sstar * (1.0 + dev * rng.uniform(-0.5, 0.9, (B, Nc))), 0.97 * st)
    S = rng.uniform(0.1, 1.0, (B, Nc))
    desc = dict(kind=str(kind), Nc=Nc, N=N, B=B, dev=dev, bl=bl, br=br, tol=tol)
    try:
        if kind == "recast":
            rmax = int(rng.choice([1, 3, 50])); rtol = 10.0 ** rng.uniform(-6, -3)
            r = snop.recast_fixed_point(op, S, st, ss, rtol, rmax)
            o = oo.recast_fixed_point(S, st, ss, rtol, rmax)
            ok = np.array_equal(r.status, o["status"]) and np.all(np.abs(r.iterations - o["iterations"]) <= 1)
            same = r.iterations == o["iterations"]
            e = float(np.max(np.abs(r.phi[same] - o["phi"][same])) / max(np.max(np.abs(o["phi"])), 1e-300)) if same.any() else 0.0
            worst["recast_phi"] = max(worst["recast_phi"], e)
            ok = ok and e < 1e-8
        elif kind == "precond":
            r = snop.precondition_fixed_source(op, N, st, ss, S, dcfg, 1e-4, 50)
            o = oo.precondition_fixed_source(N, st, ss, S, ocfg, 1e-4, 50)
            ok = np.array_equal(r.recast_status, o["recast_status"]) and np.all(np.abs(r.refine_iterations - o["refine_iterations"]) <= 1) \
                and np.array_equal(np.asarray(r.converged, bool), o["converged"])
            e = float(np.max(np.abs(r.phi - o["phi"])) / max(np.max(np.abs(o["phi"])), 1e-300))
            worst["precond_phi"] = max(worst["precond_phi"], e)
            ok = ok and e < 100 * tol  # converged fields agree to the solver tolerance
        else:
            G = int(rng.choice([1, 2, 3])); Nc2 = min(Nc, 100)
            g2 = snop.Grid1D(L, Nc2)
            ecfg_o = O.make_config(1e-7, 1e-8, 1e-7, bc_left=bl, bc_right=br)
            ecfg_d = snop.SolverConfig(tolerance=1e-7, tolerance_k=1e-8, tolerance_phi=1e-7, boundary_left=bl, boundary_right=br)
            op.close()
            op = snop.SolutionOperator.exact(g2, N, (tstar, sstar), ecfg_d)
            oo = O.OracleOperator.exact(L, Nc2, N, (tstar, sstar), ecfg_o)
            stg = tstar * (1.0 + 0.1 * rng.uniform(-1, 1, (B, G, Nc2)))
            ssm = rng.uniform(0.0, 1.0, (B, G, G, Nc2)); ssm *= (0.6 * stg[:, :, None, :] / ssm.sum(axis=2, keepdims=True))
            nsf = rng.uniform(0.05, 0.5, (B, G, Nc2)); chi = rng.uniform(0.1, 1.0, (B, G)); chi /= chi.sum(axis=1, keepdims=True)
            r = snop.cp_eigen(op, N, stg, ssm, nsf, chi, ecfg_d)
            o = oo.hybrid_eigen(1, N, stg, ssm, nsf, chi, ecfg_o)
            e = float(np.max(np.abs(r.k - o["k"]) / np.abs(o["k"])))
            worst["cp_k"] = max(worst["cp_k"], e)
            ok = e < 1e-6 and np.array_equal(np.asarray(r.fallback, bool), o["fallback"]) and \
                np.all(np.abs(r.stage1_outer - o["stage1_outer"]) <= 1)
            desc["G"] = G
    finally:
        op.close()
    if not ok:
        fails += 1
        print("MISMATCH at case", case, desc, flush=True)
print(f"{n_cases} cases, {fails} mismatches; worst {worst}")
sys.exit(1 if fails else 0)
