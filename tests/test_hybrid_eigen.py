"""SP / CP hybrid eigenvalue solves (paper Appendix A2 Eqs. A5-A8).

CPU tests pin the oracle's SP/CP restatement against the SPEC's examples (exact operator:
infinite-medium k at stage 1, Delta p = 0 SP == CP, hybrid fidelity on the Tables 7-8 problem,
divergence fallback). GPU tests compare snop_sp_eigen_batched / snop_cp_eigen_batched with the
oracle on the same inputs, and the hybrid result with the cold-start model-based power iteration.
"""
import numpy as np
import pytest

from paper_2509_01416_b200 import operators as OPS, workloads as W
from tests import oracle_lib as O

SP, CP = 0, 1


def _homogeneous(n, st, ss, nsf, B=1):
    return (np.full((B, 1, n), st), np.full((B, 1, 1, n), ss), np.full((B, 1, n), nsf), np.ones((B, 1)))


def _c3_like(batch, n_cells, seed=3000):
    p = W.config3(batch=batch, n_cells=n_cells, seed=seed)
    return p


# ---------------------------------------------------------------- oracle (CPU) -----------------
@pytest.mark.parametrize("alg", [SP, CP])
def test_oracle_infinite_medium_exact_operator(alg):
    # single-group reflective infinite medium with the exact operator -> k_inf at stage 1
    n, order = 20, 8
    cfg = O.make_config(1e-10, 1e-10, 1e-9, bc_left=1, bc_right=1)
    op = O.OracleOperator.exact(10.0, n, order, (1.0, 0.5), cfg)
    st, ss, nsf, chi = _homogeneous(n, 1.0, 0.6, 0.5)  # Delta Sigma_s only: recast is exact
    r = op.hybrid_eigen(alg, order, st, ss, nsf, chi, cfg, rtol=1e-11, rmax=200)
    kinf = 0.5 / (1.0 - 0.6)
    assert abs(r["stage1_k"][0] - kinf) < 1e-6
    assert abs(r["k"][0] - kinf) < 1e-6
    assert not r["fallback"][0] and r["converged"][0]


def test_oracle_delta_p_zero_sp_equals_cp():
    # Delta p = 0 with the exact operator -> SP and CP produce identical k within 1e-10
    n, order = 40, 8
    cfg = O.make_config(1e-12, 1e-12, 1e-11)
    op = O.OracleOperator.exact(10.0, n, order, (1.0, 0.5), cfg)
    st, ss, nsf, chi = _homogeneous(n, 1.0, 0.5, 0.6)
    a = op.hybrid_eigen(SP, order, st, ss, nsf, chi, cfg, rtol=1e-12, rmax=50)
    b = op.hybrid_eigen(CP, order, st, ss, nsf, chi, cfg, rtol=1e-12, rmax=50)
    assert abs(a["k"][0] - b["k"][0]) < 1e-10
    assert abs(a["stage1_k"][0] - b["stage1_k"][0]) < 1e-10


@pytest.mark.parametrize("alg", [SP, CP])
def test_oracle_table9_hybrid_fidelity(alg):
    # SPEC.md:429 + Invariants "Hybrid fidelity": final k equals the cold-start k within tolerance
    p = W.three_group_table9()
    order = 8
    cfg = O.make_config(1e-7, 1e-8, 1e-7)
    cold = O.power_iteration(p.length, p.n_cells, order, 3, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)
    op = O.OracleOperator.exact(p.length, p.n_cells, order, (1.0, 0.5), cfg)
    r = op.hybrid_eigen(alg, order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)
    assert r["converged"][0]
    assert abs(r["k"][0] - cold["k"][0]) < 5e-7
    phi_h = r["phi"][0] / np.linalg.norm(r["phi"][0])
    phi_c = cold["phi"][0] / np.linalg.norm(cold["phi"][0])
    assert np.max(np.abs(phi_h - phi_c)) / np.max(np.abs(phi_c)) < 2e-6
    if alg == CP:  # CP stage 1 already sits at the model-based fixed point
        assert abs(r["stage1_k"][0] - cold["k"][0]) < 1e-6
        assert r["stage2_outer"][0] < cold["outer"][0]


def test_oracle_divergence_falls_back_to_cold_start():
    # stage-1 divergence -> cold-start model-based solve, flagged
    n, order = 20, 8
    cfg = O.make_config(1e-9, 1e-9, 1e-8)
    op = O.OracleOperator.exact(10.0, n, order, (1.0, 0.9), cfg)  # recast ratio |dSs|/(St*-Ss*) = 4
    st, ss, nsf, chi = _homogeneous(n, 1.0, 0.5, 0.6)
    r = op.hybrid_eigen(SP, order, st, ss, nsf, chi, cfg, rtol=1e-6, rmax=50)
    cold = O.power_iteration(10.0, n, order, 1, st, ss, nsf, chi, cfg)
    assert r["fallback"][0]
    assert abs(r["k"][0] - cold["k"][0]) < 1e-12
    assert r["stage2_outer"][0] == cold["outer"][0]


# ---------------------------------------------------------------- device (GPU) -----------------
def _dev():
    from paper_2509_01416_b200 import snop
    return snop


def _dev_cfg(snop, cfg):
    return snop.SolverConfig(tolerance=cfg.tolerance, tolerance_k=cfg.tolerance_k, tolerance_phi=cfg.tolerance_phi,
                             max_inner_iterations=cfg.max_inner, max_outer_iterations=cfg.max_outer,
                             boundary_left=cfg.bc_left, boundary_right=cfg.bc_right)


def _run_dev(snop, op, alg, order, st, ss, nsf, chi, cfg, **kw):
    fn = snop.sp_eigen if alg == SP else snop.cp_eigen
    return fn(op, order, st, ss, nsf, chi, _dev_cfg(snop, cfg), **kw)


@pytest.mark.gpu
@pytest.mark.parametrize("alg", [SP, CP])
def test_gpu_infinite_medium_exact_operator(alg):
    snop = _dev()
    n, order = 20, 8
    cfg = O.make_config(1e-10, 1e-10, 1e-9, bc_left=1, bc_right=1)
    op = snop.SolutionOperator.exact(snop.Grid1D(10.0, n), order, (1.0, 0.5), _dev_cfg(snop, cfg))
    st, ss, nsf, chi = _homogeneous(n, 1.0, 0.6, 0.5, B=3)
    r = _run_dev(snop, op, alg, order, st, ss, nsf, chi, cfg, recast_tolerance=1e-11, recast_max_iterations=200)
    kinf = 0.5 / 0.4
    assert np.all(np.abs(r.stage1_k - kinf) < 1e-6)
    assert np.all(np.abs(r.k - kinf) < 1e-6)
    assert not r.fallback.any() and r.converged.all()


@pytest.mark.gpu
@pytest.mark.parametrize("alg", [SP, CP])
def test_gpu_table9_exact_operator_parity(alg):
    snop = _dev()
    p = W.three_group_table9()
    order = 8
    cfg = O.make_config(1e-7, 1e-8, 1e-7)
    o = O.OracleOperator.exact(p.length, p.n_cells, order, (1.0, 0.5), cfg).hybrid_eigen(
        alg, order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)
    op = snop.SolutionOperator.exact(snop.Grid1D(p.length, p.n_cells), order, (1.0, 0.5), _dev_cfg(snop, cfg))
    r = _run_dev(snop, op, alg, order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)
    assert bool(r.fallback[0]) == bool(o["fallback"][0])
    assert abs(int(r.stage1_outer[0]) - int(o["stage1_outer"][0])) <= 1
    assert abs(r.stage1_k[0] - o["stage1_k"][0]) / o["stage1_k"][0] < 1e-7
    assert abs(r.k[0] - o["k"][0]) / o["k"][0] < 1e-7
    assert abs(int(r.stage2_outer[0]) - int(o["stage2_outer"][0])) <= 1
    assert r.converged[0]


@pytest.mark.gpu
@pytest.mark.parametrize("alg", [SP, CP])
def test_gpu_deeponet_hybrid_matches_cold_start(alg):
    # Hybrid fidelity with an (untrained, random-init) DeepONet: stage 2 repairs any stage-1 error.
    snop = _dev()
    p = _c3_like(6, 128)
    order = 8
    cfg = O.make_config(1e-8, 1e-9, 1e-8, bc_left=p.bc_left, bc_right=p.bc_right, max_outer=400)
    prm = OPS.deeponet_init(p.n_cells, width=32, activation=OPS.TANH, seed=3)
    op = snop.SolutionOperator.deeponet(snop.Grid1D(p.length, p.n_cells), prm, (1.0, 0.5))
    r = _run_dev(snop, op, alg, order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg, recast_max_iterations=20)
    cold = snop.power_iteration(snop.Grid1D(p.length, p.n_cells), order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi,
                                _dev_cfg(snop, cfg))
    assert r.converged.all()
    assert np.max(np.abs(r.k - cold.k) / cold.k) < 1e-7
    oo = O.OracleOperator.deeponet(p.length, p.n_cells, (1.0, 0.5), OPS.TANH, prm.branch.sizes, prm.branch.packed(),
                                   prm.trunk.sizes, prm.trunk.packed())
    o = oo.hybrid_eigen(alg, order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg, rmax=20)
    assert np.array_equal(r.fallback.astype(bool), o["fallback"])
    assert np.max(np.abs(r.k - o["k"]) / o["k"]) < 1e-7


@pytest.mark.gpu
def test_gpu_divergence_fallback_and_device_memspace():
    import torch
    snop = _dev()
    n, order = 20, 8
    cfg = O.make_config(1e-9, 1e-9, 1e-8)
    op = snop.SolutionOperator.exact(snop.Grid1D(10.0, n), order, (1.0, 0.9), _dev_cfg(snop, cfg))
    st, ss, nsf, chi = _homogeneous(n, 1.0, 0.5, 0.6, B=2)
    r = _run_dev(snop, op, SP, order, st, ss, nsf, chi, cfg, recast_tolerance=1e-6)
    cold = snop.power_iteration(snop.Grid1D(10.0, n), order, st, ss, nsf, chi, _dev_cfg(snop, cfg))
    assert r.fallback.all()
    assert np.max(np.abs(r.k - cold.k)) < 1e-12
    d = [torch.from_numpy(x).cuda() for x in (st, ss, nsf, chi)]
    rd = _run_dev(snop, op, SP, order, *d, cfg, recast_tolerance=1e-6)
    assert np.array_equal(rd.k.cpu().numpy(), r.k)
    assert np.array_equal(rd.phi.cpu().numpy(), r.phi)


@pytest.mark.gpu
@pytest.mark.parametrize("alg", [SP, CP])
def test_gpu_power_iteration_with_operator_inner_solver(alg):
    """power_iteration with a neural-operator-backed inner_solver = stage 1 of
    SP / CP on its own: against the oracle's stage 1 (Table 9, exact operator), bit-identical to the
    stage-1 diagnostics of the two-stage entry points, and k-infinity for the reflective medium."""
    snop = _dev()
    p = W.three_group_table9()
    order = 8
    cfg = O.make_config(1e-7, 1e-8, 1e-7)
    o = O.OracleOperator.exact(p.length, p.n_cells, order, (1.0, 0.5), cfg).hybrid_eigen(
        alg, order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)
    op = snop.SolutionOperator.exact(snop.Grid1D(p.length, p.n_cells), order, (1.0, 0.5), _dev_cfg(snop, cfg))
    r = snop.power_iteration_with_operator(op, order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, _dev_cfg(snop, cfg),
                                           inner_solver=alg)
    assert r.converged[0] and not r.diverged[0]
    assert abs(int(r.outer_iterations[0]) - int(o["stage1_outer"][0])) <= 1
    assert abs(r.k[0] - o["stage1_k"][0]) / o["stage1_k"][0] < 1e-7
    two = _run_dev(snop, op, alg, order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)
    assert r.k[0] == two.stage1_k[0] and int(r.outer_iterations[0]) == int(two.stage1_outer[0])
    assert int(r.total_inner_iterations[0]) == int(two.stage1_inner[0])
    # the stage-1 flux is normalised to a unit fission integral; with a Sigma_t deviation it is
    # the recast model's eigenmode (isotropic approximation, paper Eq. 23), not the transport one
    dx = p.length / p.n_cells
    assert abs(dx * float(np.sum(p.nu_sigma_f[0] * r.phi[0])) - 1.0) < 1e-12
    # reflective infinite medium: k = nu Sigma_f / Sigma_a at stage 1
    n = 20
    cfg2 = O.make_config(1e-10, 1e-10, 1e-9, bc_left=1, bc_right=1)
    op2 = snop.SolutionOperator.exact(snop.Grid1D(10.0, n), order, (1.0, 0.5), _dev_cfg(snop, cfg2))
    st, ss, nsf, chi = _homogeneous(n, 1.0, 0.6, 0.5, B=3)
    r2 = snop.power_iteration_with_operator(op2, order, st, ss, nsf, chi, _dev_cfg(snop, cfg2), inner_solver=alg,
                                            recast_tolerance=1e-11, recast_max_iterations=200)
    assert np.all(np.abs(r2.k - 0.5 / 0.4) < 1e-6) and r2.converged.all()
    with pytest.raises(Exception):
        snop.power_iteration_with_operator(op2, order, st, ss, nsf, chi, _dev_cfg(snop, cfg2), inner_solver=7)
