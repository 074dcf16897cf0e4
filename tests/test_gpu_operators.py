"""Parity of the device SolutionOperators and MD-PNOP drivers against the CPU oracle:
predict, recast_source (:393-401), recast_fixed_point (:403-411),
precondition_fixed_source (:413-421). fp32 operator outputs within 1e-5 (north_star)."""
import numpy as np
import pytest

from paper_2509_01416_b200 import operators as OPS, snop, workloads as W
from tests import oracle_lib as O

pytestmark = pytest.mark.gpu

OP_RTOL = 1e-5  # north_star: fp32 operator outputs within 1e-5


def _rel(a, b):
    return np.max(np.abs(np.asarray(a) - b)) / max(np.max(np.abs(b)), 1e-300)


def _deeponet(n_cells, width=32, act=OPS.TANH, bias0=None):
    prm = OPS.deeponet_init(n_cells, width=width, activation=act, seed=3)
    prm.bias0 = bias0
    g = snop.Grid1D(10.0, n_cells)
    op = snop.SolutionOperator.deeponet(g, prm, (1.0, 0.5))
    oo = O.OracleOperator.deeponet(10.0, n_cells, (1.0, 0.5), act, prm.branch.sizes, prm.branch.packed(),
                                   prm.trunk.sizes, prm.trunk.packed(), bias0)
    return op, oo


def _fno(n_cells, width=16, modes=8, layers=2, hidden=32, act=OPS.GELU):
    prm = OPS.fno_init(width, modes, layers, hidden, act, seed=5)
    g = snop.Grid1D(10.0, n_cells)
    op = snop.SolutionOperator.fno(g, prm, (1.0, 0.8))
    oo = O.OracleOperator.fno(10.0, n_cells, (1.0, 0.8), act, width, modes, layers, hidden, prm.packed())
    return op, oo


@pytest.mark.parametrize("act", [OPS.RELU, OPS.TANH, OPS.GELU])
def test_deeponet_predict(act):
    op, oo = _deeponet(200, act=act, bias0=0.25 if act == OPS.RELU else None)
    s = np.random.default_rng(0).uniform(0, 1, (7, 200))
    assert _rel(op.predict(s), oo.predict(s)) < OP_RTOL


def test_deeponet_c2_shape():
    prm = OPS.deeponet_init(2000, width=128, activation=OPS.TANH)
    g = snop.Grid1D(10.0, 2000)
    op = snop.SolutionOperator.deeponet(g, prm)
    oo = O.OracleOperator.deeponet(10.0, 2000, (1.0, 0.5), OPS.TANH, prm.branch.sizes, prm.branch.packed(),
                                   prm.trunk.sizes, prm.trunk.packed())
    s = W.config2(batch=16).source * np.random.default_rng(1).uniform(0.5, 1.5, (16, 1))
    assert _rel(op.predict(s), oo.predict(s)) < OP_RTOL


@pytest.mark.parametrize("n_cells,modes", [(64, 8), (100, 16), (1024, 16), (32, 17)])
def test_fno_predict(n_cells, modes):
    op, oo = _fno(n_cells, modes=modes)
    s = np.random.default_rng(2).uniform(0, 1, (5, n_cells))
    assert _rel(op.predict(s), oo.predict(s)) < OP_RTOL


def test_fno_c5_architecture():
    prm = OPS.fno_init()
    g = snop.Grid1D(10.0, 1024)
    op = snop.SolutionOperator.fno(g, prm, (1.0, 0.8))
    oo = O.OracleOperator.fno(10.0, 1024, (1.0, 0.8), OPS.GELU, 64, 16, 4, 128, prm.packed())
    s = W.config5(batch=6).source
    assert _rel(op.predict(s), oo.predict(s)) < OP_RTOL


def test_zero_weights_zero_output():
    # SPEC.md:325
    prm = OPS.deeponet_init(50, width=8)
    for w in prm.branch.weights + prm.trunk.weights:
        w[:] = 0
    op = snop.SolutionOperator.deeponet(snop.Grid1D(10.0, 50), prm)
    assert np.all(op.predict(np.ones((2, 50))) == 0)


@pytest.mark.parametrize("c", [2.0, 0.37])
def test_deeponet_branch_linearity(c):
    """scaling the branch's final layer by c scales predictions by c. c = 2 is exact in
    floating point (the 3xTF32 split of 2x is 2 x the split of x), so the device result is
    bit-identical; other c within the fp32 operator tolerance."""
    n = 300
    prm = OPS.deeponet_init(n, width=64, activation=OPS.TANH, seed=6)
    prm.branch.biases[-1][:] = np.random.default_rng(3).uniform(-0.1, 0.1, prm.branch.biases[-1].shape)
    g = snop.Grid1D(10.0, n)
    s = np.random.default_rng(4).uniform(0, 1, (9, n))
    base = snop.SolutionOperator.deeponet(g, prm).predict(s)
    prm.branch.weights[-1] *= np.float32(c)
    prm.branch.biases[-1] *= np.float32(c)
    scaled = snop.SolutionOperator.deeponet(g, prm).predict(s)
    if c == 2.0:
        assert np.array_equal(scaled, 2.0 * base)
    else:
        assert _rel(scaled, c * base) < OP_RTOL


def test_fno_identity_spectral_layer_is_lowpass():
    # W = 0, b = 0, R = identity on retained modes -> DFT truncation low-pass
    n, C, M = 64, 4, 6
    prm = OPS.fno_init(C, M, 1, 4, OPS.RELU, seed=1)
    prm.W[0][:] = 0
    prm.R_re[0][:] = 0
    prm.R_im[0][:] = 0
    for m in range(M):
        prm.R_re[0][m] = np.eye(C, dtype=np.float32)
    prm.lift_W[:] = 0
    prm.lift_W[:, 0] = 1.0   # channel c = S
    prm.activation = 3 if False else OPS.RELU
    prm.P1_W[:] = 0
    prm.P1_W[0, 0] = 1.0
    prm.P2_W[:] = 0
    prm.P2_W[0] = 1.0
    s = 1.0 + 0.5 * np.sin(2 * np.pi * 3 * np.arange(n) / n) + 0.2 * np.cos(2 * np.pi * 20 * np.arange(n) / n)
    s = s[None, :]
    op = snop.SolutionOperator.fno(snop.Grid1D(10.0, n), prm)
    got = op.predict(s)[0]
    X = np.fft.rfft(s[0])
    X[M:] = 0
    want = np.maximum(np.fft.irfft(X, n), 0.0)
    assert np.max(np.abs(got - want)) < 1e-5


def test_recast_source_examples():
    n = 10
    g = snop.recast_source(np.zeros((1, n)), np.ones((1, n)), np.full((1, n), 1.2), np.full((1, n), 0.8), (1.0, 0.5))
    assert np.allclose(g, 0.1, rtol=1e-14)
    S = np.random.default_rng(0).uniform(0, 1, (3, n))
    assert np.array_equal(snop.recast_source(S, np.zeros((3, n)), np.full((3, n), 2.0), np.full((3, n), 1.0)), S)
    assert np.array_equal(snop.recast_source(S, np.ones((3, n)), np.full((3, n), 1.0), np.full((3, n), 0.5)), S)
    rng = np.random.default_rng(4)
    a = [rng.uniform(0.5, 2, (4, 777)) for _ in range(4)]
    want = O.recast_source(a[0], a[1], a[2], a[3], 1.0, 0.5)
    assert _rel(snop.recast_source(a[0], a[1], a[2], a[3], (1.0, 0.5)), want) < 1e-15


def test_exact_operator_recast_equivalence():
    # SPEC.md:409 / acceptance 1, exact operator at p* = (1, 0.5). With a Sigma_s0-only deviation the
    # recast (Eq. 24) is exact and the fixed point equals the direct solve at p'. With a Sigma_t
    # deviation Eq. 24 folds the angular absorption term into phi (the isotropic approximation,
    # paper Eq. 23), so the fixed point differs from the direct solve by O(1e-2) in the oracle as
    # well -- SPEC's (1.2, 0.8) example is not attainable as written ("Oracle pins").
    n, order = 100, 32
    g = snop.Grid1D(10.0, n)
    cfg = snop.SolverConfig(tolerance=1e-12)
    op = snop.SolutionOperator.exact(g, order, (1.0, 0.5), cfg)
    oo = O.OracleOperator.exact(10.0, n, order, (1.0, 0.5), cfg.c())
    S = np.random.default_rng(9).uniform(0.05, 0.1, (2, n))
    for t, s_, bound in [(1.0, 0.8, 1e-6), (1.2, 0.8, None)]:
        st, ss = np.full((2, n), t), np.full((2, n), s_)
        r = snop.recast_fixed_point(op, S, st, ss, tolerance=1e-10, max_iterations=300)
        direct = snop.source_iteration(g, order, st, ss, S, cfg)
        assert (r.status == 0).all()
        l2 = np.linalg.norm(r.phi - direct.phi, axis=1) / np.linalg.norm(direct.phi, axis=1)
        if bound is not None:
            assert l2.max() < bound
        else:  # same approximation error as the oracle's restatement of Eq. 24
            o = oo.recast_fixed_point(S, st, ss, tol=1e-10, max_it=300)
            lo = np.linalg.norm(o["phi"] - direct.phi, axis=1) / np.linalg.norm(direct.phi, axis=1)
            assert np.allclose(l2, lo, rtol=1e-6)


def test_recast_fixed_point_parity_exact():
    n, order = 100, 16
    cfg = snop.SolverConfig(tolerance=1e-12)
    op = snop.SolutionOperator.exact(snop.Grid1D(10.0, n), order, (1.0, 0.5), cfg)
    oo = O.OracleOperator.exact(10.0, n, order, (1.0, 0.5), cfg.c())
    rng = np.random.default_rng(3)
    S = rng.uniform(0, 1, (4, n))
    st = rng.uniform(0.9, 1.3, (4, n))
    ss = st * rng.uniform(0.4, 0.7, (4, 1))
    r = snop.recast_fixed_point(op, S, st, ss, tolerance=1e-8, max_iterations=100)
    o = oo.recast_fixed_point(S, st, ss, tol=1e-8, max_it=100)
    assert np.all(np.abs(r.iterations - o["iterations"]) <= 1)
    assert np.array_equal(r.status, o["status"])
    assert _rel(r.phi, o["phi"]) < 1e-8


def test_recast_delta_p_zero_converges_immediately():
    # dp = 0 -> converges in <= 2 iterations to op(S)
    op, oo = _deeponet(64)
    S = np.random.default_rng(0).uniform(0, 1, (3, 64))
    r = snop.recast_fixed_point(op, S, np.full((3, 64), 1.0), np.full((3, 64), 0.5))
    assert (r.iterations <= 2).all() and (r.status == 0).all()
    assert _rel(r.phi, op.predict(S)) < 1e-12


def test_recast_divergence_guard():
    # a large parameter deviation with a random operator: status diverged or maxed, finite output
    op, oo = _deeponet(64, width=16)
    S = np.random.default_rng(0).uniform(0, 1, (3, 64))
    st, ss = np.full((3, 64), 3.0), np.full((3, 64), 0.1)
    r = snop.recast_fixed_point(op, S, st, ss, max_iterations=50)
    o = oo.recast_fixed_point(S, st, ss, tol=1e-4, max_it=50)
    assert np.array_equal(r.status, o["status"])
    assert np.isfinite(r.phi).all()


def test_recast_device_loop_cache_and_launch_accounting():
    """The recast fixed point iterates on the device (a CUDA graph with a WHILE conditional node,
    cached on the context by its buffers and scalars): repeated calls on the same device buffers
    relaunch the cached graph and give bit-identical results; a different iteration cap or
    tolerance is a different graph; the context's launch counter counts every iteration's kernels."""
    import torch
    op, oo = _deeponet(64, width=16)
    rng = np.random.default_rng(4)
    S, st = rng.uniform(0, 1, (5, 64)), rng.uniform(0.8, 1.4, (5, 64))
    ss = st * 0.6
    dS, dst, dss = (torch.from_numpy(a).cuda() for a in (S, st, ss))
    ctx = op.ctx
    runs = []
    for max_it in (50, 50, 3, 50):
        n0 = ctx.launch_count
        r = snop.recast_fixed_point(op, dS, dst, dss, tolerance=1e-6, max_iterations=max_it)
        runs.append((r.phi.cpu().numpy(), r.iterations.cpu().numpy(), r.status.cpu().numpy(), ctx.launch_count - n0))
    assert np.array_equal(runs[0][0], runs[1][0]) and np.array_equal(runs[0][0], runs[3][0])
    assert runs[0][3] == runs[1][3] == runs[3][3]
    assert runs[2][1].max() <= 3 and runs[2][3] < runs[0][3]
    o = oo.recast_fixed_point(S, st, ss, tol=1e-6, max_it=50)
    assert np.array_equal(runs[0][2], o["status"])
    assert np.all(np.abs(runs[0][1] - o["iterations"]) <= 1)


def test_precondition_fixed_source_exact_operator():
    # exact operator, dp = 0 -> refinement converges in <= 2 iterations
    n, order = 200, 16
    g = snop.Grid1D(10.0, n)
    op = snop.SolutionOperator.exact(g, order, (1.0, 0.5), snop.SolverConfig(tolerance=1e-12))
    S = np.random.default_rng(1).uniform(0, 1, (3, n))
    st, ss = np.full((3, n), 1.0), np.full((3, n), 0.5)
    r = snop.precondition_fixed_source(op, order, st, ss, S, snop.SolverConfig(tolerance=1e-8))
    assert (r.refine_iterations <= 2).all() and r.converged.all()


def test_precondition_fixed_source_deeponet_parity():
    p = W.config2(batch=4, n_cells=2000)
    prm = OPS.deeponet_init(2000, width=128, activation=OPS.TANH)
    g = snop.Grid1D(p.length, p.n_cells)
    op = snop.SolutionOperator.deeponet(g, prm)
    oo = O.OracleOperator.deeponet(10.0, 2000, (1.0, 0.5), OPS.TANH, prm.branch.sizes, prm.branch.packed(),
                                   prm.trunk.sizes, prm.trunk.packed())
    cfg = snop.SolverConfig(tolerance=1e-8)
    r = snop.precondition_fixed_source(op, p.order, p.sigma_t, p.sigma_s0, p.source, cfg, recast_max_iterations=5)
    o = oo.precondition_fixed_source(p.order, p.sigma_t, p.sigma_s0, p.source, cfg.c(), rmax=5)
    assert np.array_equal(r.recast_status, o["recast_status"])
    assert np.all(np.abs(r.refine_iterations - o["refine_iterations"]) <= 1)
    assert r.converged.all()
    same = r.refine_iterations == o["refine_iterations"]
    assert _rel(r.phi[same], o["phi"][same]) < 1e-8


@pytest.mark.parametrize("opts", [{}, {"fno_mix": 1}, {"fno_dft": 1}, {"gemm_engine": 1}, {"gemm_engine": 2}])
def test_fno_width64_kernel_paths(opts, ctx_options):
    """The C5-width FNO runs on dedicated paths (tensor-core forward DFT, register-tiled mixing,
    TMA-store epilogue, resident pre-split weights); each against the oracle, with the other paths
    selectable through the context options (FFMA forward DFT, tcgen05 engine v1 only, FFMA engine)."""
    ctx_options(**opts)
    prm = OPS.fno_init(64, 16, 2, 128, OPS.GELU, seed=11)
    g = snop.Grid1D(10.0, 512)
    op = snop.SolutionOperator.fno(g, prm, (1.0, 0.8))
    oo = O.OracleOperator.fno(10.0, 512, (1.0, 0.8), OPS.GELU, 64, 16, 2, 128, prm.packed())
    s = np.random.default_rng(7).uniform(0, 1, (13, 512))  # 13: ragged against the 8-sample DFT blocks
    assert _rel(op.predict(s), oo.predict(s)) < OP_RTOL


def test_fno_predict_deterministic():
    prm = OPS.fno_init(64, 16, 2, 128, OPS.GELU, seed=12)
    op = snop.SolutionOperator.fno(snop.Grid1D(10.0, 256), prm, (1.0, 0.8))
    s = np.random.default_rng(9).uniform(0, 1, (11, 256))
    assert np.array_equal(op.predict(s), op.predict(s))


def test_fno_width64_persistent_wrap():
    """More sample pairs / tiles than CTAs (151 pairs, 604 inverse+W tiles on 148 SMs): the
    persistent kernels' ring phases, the double-buffered TMA-store staging and the multiply-high
    tile decomposition cross tile boundaries; an odd batch leaves a one-sample last pair."""
    prm = OPS.fno_init(64, 16, 2, 128, OPS.GELU, seed=13)
    g = snop.Grid1D(10.0, 512)
    op = snop.SolutionOperator.fno(g, prm, (1.0, 0.8))
    oo = O.OracleOperator.fno(10.0, 512, (1.0, 0.8), OPS.GELU, 64, 16, 2, 128, prm.packed())
    s = np.random.default_rng(17).uniform(0, 1, (301, 512))
    got = op.predict(s)
    idx = np.r_[0:8, 140:160, 290:301]  # oracle on a subset (CPU time); first, wrapped and last pairs
    assert _rel(got[idx], oo.predict(s[idx])) < OP_RTOL
    assert _rel(got[idx], op.predict(s[idx])) < 1e-6  # a sample's result does not depend on its batch
