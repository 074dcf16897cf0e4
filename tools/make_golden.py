"""Generates tests/golden/oracle_cases.npz: small seeded cases solved by the CPU oracle (the
restated reference solver). The oracle itself is pinned by tests/test_oracle_pins.py against the
reference-compiled RNG/partition goldens and SPEC/paper known answers. TEST INFRASTRUCTURE ONLY."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2509_01416_b200 import operators as OPS, workloads as W  # noqa: E402
from tests import oracle_lib as O  # noqa: E402


def main():
    out = {}
    # fixed source: C2 subset at reduced cells, fixed 5 iterations and converged 1e-8
    p = W.config2(batch=6, n_cells=400)
    for tag, cfg in (("fix5", O.make_config(1e-300, max_inner=5)), ("conv", O.make_config(1e-8))):
        r = O.source_iteration(p.length, p.n_cells, p.order, p.sigma_t, p.sigma_s0, p.source, cfg)
        out[f"si_{tag}_phi"] = r["phi"]
        out[f"si_{tag}_it"] = r["iterations"]
    out["si_sigma_t"], out["si_sigma_s0"], out["si_source"] = p.sigma_t, p.sigma_s0, p.source
    # reflective-left, P1
    cfg = O.make_config(1e-300, max_inner=6, bc_left=1)
    r = O.source_iteration(p.length, p.n_cells, 16, p.sigma_t, p.sigma_s0, p.source, cfg, sigma_s1=0.3 * p.sigma_s0)
    out["si_p1_refl_phi"] = r["phi"]
    # eigen: Table 9 and a C4 subset
    t9 = W.three_group_table9()
    r = O.power_iteration(t9.length, t9.n_cells, t9.order, 3, t9.sigma_t, t9.sigma_s0, t9.nu_sigma_f, t9.chi,
                          O.make_config(1e-7, tolerance_k=1e-8, tolerance_phi=1e-7))
    out["t9_k"], out["t9_outer"], out["t9_phi"] = r["k"], r["outer"], r["phi"]
    c4 = W.config4(batch=2, n_cells=200)
    r = O.power_iteration(c4.length, c4.n_cells, c4.order, 7, c4.sigma_t, c4.sigma_s0, c4.nu_sigma_f, c4.chi,
                          O.make_config(1e-7, tolerance_k=1e-8, tolerance_phi=1e-7))
    out["c4_k"], out["c4_outer"] = r["k"], r["outer"]
    # operators
    prm = OPS.deeponet_init(100, width=32, activation=OPS.TANH, seed=3)
    oo = O.OracleOperator.deeponet(10.0, 100, (1.0, 0.5), OPS.TANH, prm.branch.sizes, prm.branch.packed(),
                                   prm.trunk.sizes, prm.trunk.packed())
    s = np.random.default_rng(0).uniform(0, 1, (3, 100))
    out["don_in"], out["don_out"] = s, oo.predict(s)
    fp = OPS.fno_init(16, 8, 2, 32, OPS.GELU, seed=5)
    fo = O.OracleOperator.fno(10.0, 64, (1.0, 0.8), OPS.GELU, 16, 8, 2, 32, fp.packed())
    s = np.random.default_rng(1).uniform(0, 1, (3, 64))
    out["fno_in"], out["fno_out"] = s, fo.predict(s)
    np.savez_compressed(ROOT / "tests" / "golden" / "oracle_cases.npz", **out)
    print("wrote tests/golden/oracle_cases.npz", {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
