"""GPU path vs the committed golden fixtures (tests/golden/oracle_cases.npz, made by
tools/make_golden.py from the pinned oracle) — no oracle execution needed on the box."""
from pathlib import Path

import numpy as np
import pytest

from paper_2509_01416_b200 import operators as OPS, snop, workloads as W

pytestmark = pytest.mark.gpu
G = np.load(Path(__file__).resolve().parent / "golden" / "oracle_cases.npz")


def _rel(a, b):
    return np.max(np.abs(np.asarray(a) - b)) / np.max(np.abs(b))


def test_si_fixed_iterations_golden():
    g = snop.Grid1D(10.0, 400)
    r = snop.source_iteration(g, 32, G["si_sigma_t"], G["si_sigma_s0"], G["si_source"],
                              snop.SolverConfig(tolerance=1e-300, max_inner_iterations=5))
    assert _rel(r.phi, G["si_fix5_phi"]) < 1e-10


def test_si_converged_golden():
    g = snop.Grid1D(10.0, 400)
    r = snop.source_iteration(g, 32, G["si_sigma_t"], G["si_sigma_s0"], G["si_source"], snop.SolverConfig(tolerance=1e-8))
    assert np.all(np.abs(r.iterations - G["si_conv_it"]) <= 1)


def test_si_p1_reflective_golden():
    g = snop.Grid1D(10.0, 400)
    r = snop.source_iteration(g, 16, G["si_sigma_t"], G["si_sigma_s0"], G["si_source"],
                              snop.SolverConfig(tolerance=1e-300, max_inner_iterations=6, boundary_left=1),
                              sigma_s1=0.3 * G["si_sigma_s0"])
    assert _rel(r.phi, G["si_p1_refl_phi"]) < 1e-10


def test_table9_golden():
    t9 = W.three_group_table9()
    e = snop.power_iteration(snop.Grid1D(10.0, 100), 32, t9.sigma_t, t9.sigma_s0, t9.nu_sigma_f, t9.chi,
                             snop.SolverConfig(tolerance=1e-7, tolerance_k=1e-8, tolerance_phi=1e-7))
    assert abs(e.outer_iterations[0] - G["t9_outer"][0]) <= 1
    tol = 1e-10 if e.outer_iterations[0] == G["t9_outer"][0] else 1e-8
    assert abs(e.k[0] - G["t9_k"][0]) / G["t9_k"][0] < tol


def test_operator_goldens():
    prm = OPS.deeponet_init(100, width=32, activation=OPS.TANH, seed=3)
    op = snop.SolutionOperator.deeponet(snop.Grid1D(10.0, 100), prm)
    assert _rel(op.predict(G["don_in"]), G["don_out"]) < 1e-5
    fp = OPS.fno_init(16, 8, 2, 32, OPS.GELU, seed=5)
    fo = snop.SolutionOperator.fno(snop.Grid1D(10.0, 64), fp)
    assert _rel(fo.predict(G["fno_in"]), G["fno_out"]) < 1e-5
