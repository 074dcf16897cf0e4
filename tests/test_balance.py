"""Balance diagnostic: net face leakages from the last sweep of the fused
source iteration (K1) and the batched balance report, against the oracle and the SPEC examples."""
import numpy as np
import pytest

from paper_2509_01416_b200 import snop, workloads as W
from paper_2509_01416_b200.errors import NumericalError
from tests import oracle_lib as O


def _case1(B=4, n=100, seed=0):
    """Case-1-like: Sigma_t = 1, Sigma_s0 = 0.5, positive smooth sources, vacuum."""
    rng = np.random.default_rng(seed)
    x = (np.arange(n) + 0.5) * (10.0 / n)
    S = 0.1 + 0.05 * np.sin(2 * np.pi * rng.uniform(1, 3, (B, 1)) * x / 10.0)
    return np.ones((B, n)), np.full((B, n), 0.5), S


# ---------------------------------------------------------------- oracle (CPU) ----------------------
def test_oracle_reflective_infinite_medium_balance():
    n = 50
    st, ss, S = np.full((1, n), 0.5), np.zeros((1, n)), np.full((1, n), 0.1)
    r = O.source_iteration(10.0, n, 8, st, ss, S, O.make_config(1e-12, bc_left=1, bc_right=1), want_leak=True)
    assert O.balance_residual(10.0, n, st[0], ss[0], S[0], r["phi"][0], *r["leak"][0]) < 1e-10


def test_oracle_case1_balance_and_unconverged():
    st, ss, S = _case1()
    r = O.source_iteration(10.0, 100, 16, st, ss, S, O.make_config(1e-10), want_leak=True)
    for b in range(len(S)):
        assert O.balance_residual(10.0, 100, st[b], ss[b], S[b], r["phi"][b], *r["leak"][b]) < 1e-8
    r1 = O.source_iteration(10.0, 100, 16, st, ss, S, O.make_config(1e-10, max_inner=1), want_leak=True)
    assert O.balance_residual(10.0, 100, st[0], ss[0], S[0], r1["phi"][0], *r1["leak"][0]) > 1e-3


# ---------------------------------------------------------------- device -----------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("bcl,bcr,aniso", [(0, 0, False), (1, 0, False), (0, 1, False), (1, 1, False),
                                           (0, 0, True)])
def test_gpu_leakage_matches_oracle(bcl, bcr, aniso):
    st, ss, S = _case1(B=6, n=300, seed=bcl + 2 * bcr)
    s1 = np.full_like(st, 0.3) if aniso else None
    cfg = snop.SolverConfig(tolerance=1e-10, boundary_left=bcl, boundary_right=bcr)
    g = snop.Grid1D(10.0, 300)
    r = snop.source_iteration(g, 16, st, ss, S, cfg, sigma_s1=s1, want_leakage=True)
    o = O.source_iteration(10.0, 300, 16, st, ss, S, cfg.c(), sigma_s1=s1, want_leak=True)
    same = r.iterations == o["iterations"]
    assert same.all()
    prod = S.sum(axis=1) * g.dx
    assert np.max(np.abs(r.leakage - o["leak"]) / prod[:, None]) < 1e-10
    if bcl:
        assert np.all(np.abs(r.leakage[:, 0]) < 1e-14 * prod)


@pytest.mark.gpu
def test_gpu_balance_report_examples():
    g = snop.Grid1D(10.0, 100)
    st, ss, S = _case1(B=8)
    r = snop.source_iteration(g, 16, st, ss, S, snop.SolverConfig(tolerance=1e-10), want_leakage=True)
    res = snop.balance_report(g, st, ss, S, r.phi, r.leakage)
    assert np.all(res < 1e-8)
    for b in range(8):  # the oracle's report on the device's own outputs
        assert abs(res[b] - O.balance_residual(10.0, 100, st[b], ss[b], S[b], r.phi[b], *r.leakage[b])) < 1e-14
    r1 = snop.source_iteration(g, 16, st, ss, S, snop.SolverConfig(tolerance=1e-10, max_inner_iterations=1),
                               want_leakage=True)
    assert np.all(snop.balance_report(g, st, ss, S, r1.phi, r1.leakage) > 1e-3)
    # reflective infinite medium converged to 1e-12 -> exact balance
    n = 50
    gi = snop.Grid1D(10.0, n)
    sti, ssi, Si = np.full((1, n), 0.5), np.zeros((1, n)), np.full((1, n), 0.1)
    ri = snop.source_iteration(gi, 8, sti, ssi, Si, snop.SolverConfig(tolerance=1e-12, boundary_left=1,
                                                                      boundary_right=1), want_leakage=True)
    assert snop.balance_report(gi, sti, ssi, Si, ri.phi, ri.leakage)[0] < 1e-10
    with pytest.raises(NumericalError):
        snop.balance_report(g, st, ss, np.zeros_like(S), r.phi, r.leakage)


@pytest.mark.gpu
def test_gpu_c2_subset_balance():
    p = W.config2(batch=64)
    g = snop.Grid1D(p.length, p.n_cells)
    r = snop.source_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.source, snop.SolverConfig(tolerance=1e-10),
                              want_leakage=True)
    res = snop.balance_report(g, p.sigma_t, p.sigma_s0, p.source, r.phi, r.leakage)
    assert r.converged.all() and np.all(res < 1e-8)
