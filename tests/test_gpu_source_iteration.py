"""Parity of the fused sm_100a source-iteration kernel (K1) against the CPU oracle
(SPEC.md:115-134). Strict 1e-10 parity at equal iteration counts (fixed-iteration mode), and
converged iteration counts within +-1 (BASELINE.md parity gate)."""
import numpy as np
import pytest

from paper_2509_01416_b200 import snop, workloads as W
from paper_2509_01416_b200.errors import InvalidArgument
from tests import oracle_lib as O

pytestmark = pytest.mark.gpu

FLUX_RTOL = 1e-10  # north_star: scalar flux within 1e-10 relative in fp64 at equal iteration counts


def _rel(a, b):
    return np.max(np.abs(np.asarray(a) - b)) / max(np.max(np.abs(b)), 1e-300)


def _run_both(p, cfg_kw, sigma_s1=None, initial_phi=None):
    cfg = snop.SolverConfig(**cfg_kw)
    g = snop.Grid1D(p.length, p.n_cells)
    r = snop.source_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.source, cfg, initial_phi=initial_phi,
                              sigma_s1=sigma_s1, want_current=True)
    o = O.source_iteration(p.length, p.n_cells, p.order, p.sigma_t, p.sigma_s0, p.source, cfg.c(),
                           sigma_s1=sigma_s1, initial_phi=initial_phi, want_current=True)
    return r, o


@pytest.mark.parametrize("n_iter", [1, 2, 7])
def test_fixed_iterations_parity_c2(n_iter):
    p = W.config2(batch=16, n_cells=2000)
    r, o = _run_both(p, dict(tolerance=1e-300, max_inner_iterations=n_iter))
    assert (r.iterations == n_iter).all() and (o["iterations"] == n_iter).all()
    assert _rel(r.phi, o["phi"]) < FLUX_RTOL


def test_c1_known_answer():
    p = W.config1()
    r, o = _run_both(p, dict(tolerance=1e-8))
    assert abs(int(r.iterations[0]) - int(o["iterations"][0])) <= 1
    assert int(o["iterations"][0]) == 26
    assert _rel(r.phi, o["phi"]) < FLUX_RTOL


def test_c2_converged_counts_and_flux():
    p = W.config2(batch=64, n_cells=2000)
    r, o = _run_both(p, dict(tolerance=1e-8))
    d = np.abs(r.iterations.astype(int) - o["iterations"].astype(int))
    assert d.max() <= 1
    same = d == 0
    assert same.sum() >= 0.9 * len(d)
    assert _rel(r.phi[same], o["phi"][same]) < FLUX_RTOL
    assert r.converged.all()


@pytest.mark.parametrize("n_cells", [1, 7, 31, 100, 257, 1000, 4096])
def test_ragged_sizes(n_cells):
    rng = np.random.default_rng(n_cells)
    B = 3
    st = rng.uniform(0.5, 2.0, (B, n_cells))
    ss = st * rng.uniform(0.2, 0.9, (B, 1))
    q = rng.uniform(0.0, 1.0, (B, n_cells))
    p = W.FixedSourceProblem("r", 10.0, n_cells, 16, st, ss, q)
    r, o = _run_both(p, dict(tolerance=1e-300, max_inner_iterations=5))
    assert _rel(r.phi, o["phi"]) < FLUX_RTOL
    # current is O(phi) or exactly 0 by symmetry: compare against the flux scale
    assert np.max(np.abs(r.current - o["current"])) < 1e-10 * np.max(np.abs(o["phi"]))


@pytest.mark.parametrize("bc", [(1, 0), (0, 1), (1, 1)])
def test_reflective_boundaries(bc):
    p = W.config2(batch=4, n_cells=500)
    p.order = 16
    r, o = _run_both(p, dict(tolerance=1e-300, max_inner_iterations=6, boundary_left=bc[0], boundary_right=bc[1]))
    assert _rel(r.phi, o["phi"]) < FLUX_RTOL


def test_reflective_infinite_medium_spec_example():
    # reflective both sides, St=0.5, Ss0=0, S=0.1 -> phi = S/Sa = 0.2
    n = 100
    p = W.FixedSourceProblem("inf", 10.0, n, 16, np.full((1, n), 0.5), np.zeros((1, n)), np.full((1, n), 0.1))
    r, o = _run_both(p, dict(tolerance=1e-12, boundary_left=1, boundary_right=1))
    assert np.allclose(r.phi, 0.2, rtol=1e-10)


def test_no_scatter_two_iterations():
    # Sigma_s0 = 0 -> exactly 2 iterations
    n = 300
    p = W.FixedSourceProblem("ns", 10.0, n, 16, np.full((2, n), 1.3), np.zeros((2, n)),
                             np.random.default_rng(0).uniform(0, 1, (2, n)))
    r, _ = _run_both(p, dict(tolerance=1e-8))
    assert (r.iterations == 2).all()


def test_zero_source_zero_flux():
    n = 64
    p = W.FixedSourceProblem("z", 10.0, n, 8, np.ones((1, n)), np.full((1, n), 0.5), np.zeros((1, n)))
    r, _ = _run_both(p, dict(tolerance=1e-8))
    assert (r.phi == 0).all() and r.converged.all()


def test_warm_start_from_converged():
    # initial_phi = converged solution -> <= 2 iterations
    p = W.config2(batch=8, n_cells=2000)
    cfg = dict(tolerance=1e-8)
    r, _ = _run_both(p, cfg)
    r2, _ = _run_both(p, cfg, initial_phi=np.asarray(r.phi))
    assert (r2.iterations <= 2).all()


def test_anisotropic_p1():
    p = W.config2(batch=4, n_cells=400)
    s1 = 0.3 * p.sigma_s0
    r, o = _run_both(p, dict(tolerance=1e-300, max_inner_iterations=8), sigma_s1=s1)
    assert _rel(r.phi, o["phi"]) < FLUX_RTOL


def test_l2_norm_counts():
    p = W.config2(batch=16, n_cells=1000)
    r, o = _run_both(p, dict(tolerance=1e-8, convergence_norm=1))
    assert np.abs(r.iterations.astype(int) - o["iterations"].astype(int)).max() <= 1


def test_nonpositive_sigma_t_is_invalid_argument():
    n = 50
    st = np.ones((2, n))
    st[1, 7] = 0.0
    with pytest.raises(InvalidArgument):
        snop.source_iteration(snop.Grid1D(10.0, n), 8, st, np.zeros((2, n)), np.ones((2, n)))


@pytest.mark.parametrize("n_cells", [2000, 4096])
@pytest.mark.parametrize("order", [16, 32])
@pytest.mark.parametrize("bc", [(0, 0), (1, 0), (1, 1)])
@pytest.mark.parametrize("sigma_scale", [1e-6, 1e-4, 1e-2, 1.0])
def test_thin_cell_flux_parity(sigma_scale, bc, order, n_cells):
    """Optically thin and near-void cells (SPEC.md:119 allows any Sigma_t > 0): phi = sum w psi_avg
     at 1e-10 against the oracle, fixed iteration count, all BC combinations."""
    rng = np.random.default_rng(int(sigma_scale * 1e6) + n_cells + order)
    B, L = 2, 10.0
    x = (np.arange(n_cells) + 0.5) * (L / n_cells)
    st = sigma_scale * (1.0 + 0.5 * np.sin(2 * np.pi * rng.integers(1, 5, (B, 1)) * x / L))
    ss = rng.uniform(0.3, 0.9, (B, 1)) * st
    src = rng.uniform(0.5, 1.5, (B, n_cells))
    cfg = snop.SolverConfig(tolerance=1e-300, max_inner_iterations=4, boundary_left=bc[0], boundary_right=bc[1])
    r = snop.source_iteration(snop.Grid1D(L, n_cells), order, st, ss, src, cfg)
    o = O.source_iteration(L, n_cells, order, st, ss, src, cfg.c())
    assert (r.iterations == 4).all()
    assert _rel(r.phi, o["phi"]) < FLUX_RTOL


def test_grid_limits_are_invalid_argument():
    # n_cells must be positive; the C ABI's upper bound is 2^26 cells per instance (the
    # streaming path has no smaller limit: 16385+ cells are solved, test_long_slab_parity)
    for n in (0, 2**26 + 1):
        with pytest.raises(InvalidArgument):
            snop.source_iteration(snop.Grid1D(10.0, n), 8, np.ones((0, n)), np.zeros((0, n)), np.ones((0, n)))


def test_empty_batch():
    r = snop.source_iteration(snop.Grid1D(10.0, 10), 8, np.zeros((0, 10)), np.zeros((0, 10)), np.zeros((0, 10)))
    assert r.phi.shape == (0, 10)


def test_device_memspace_matches_host():
    import torch
    p = W.config2(batch=8, n_cells=2000)
    cfg = snop.SolverConfig(tolerance=1e-8)
    g = snop.Grid1D(p.length, p.n_cells)
    h = snop.source_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.source, cfg)
    d = snop.source_iteration(g, p.order, torch.from_numpy(p.sigma_t).cuda(), torch.from_numpy(p.sigma_s0).cuda(),
                              torch.from_numpy(p.source).cuda(), cfg)
    assert np.array_equal(h.phi, d.phi.cpu().numpy())
    assert np.array_equal(h.iterations, d.iterations.cpu().numpy())


@pytest.mark.parametrize("aniso", [False, True])
def test_host_pipelined_path_matches_device(aniso):
    """batch >= 4 x SMs takes the chunked H2D / solve / D2H pipeline on the host path (4 streams);
    every output must equal the single-launch device-memspace result bit for bit."""
    import torch
    B, n = 700, 300
    p = W.config2(batch=B, n_cells=n)
    rng = np.random.default_rng(3)
    s1 = 0.2 * p.sigma_s0 if aniso else None
    phi0 = rng.uniform(0.0, 1.0, (B, n))
    cfg = snop.SolverConfig(tolerance=1e-9)
    g = snop.Grid1D(p.length, n)
    pinned = (torch.empty((B, n), dtype=torch.float64).pin_memory().numpy(),
              torch.empty(B, dtype=torch.int32).pin_memory().numpy(),
              torch.empty(B, dtype=torch.uint8).pin_memory().numpy())
    h = snop.source_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.source, cfg, initial_phi=phi0, sigma_s1=s1,
                              want_current=True, want_leakage=True, out=pinned)
    dv = [torch.from_numpy(x).cuda() for x in (p.sigma_t, p.sigma_s0, p.source, phi0)]
    d = snop.source_iteration(g, p.order, dv[0], dv[1], dv[2], cfg, initial_phi=dv[3],
                              sigma_s1=None if s1 is None else torch.from_numpy(s1).cuda(), want_current=True,
                              want_leakage=True)
    assert h.phi is pinned[0]
    assert np.array_equal(h.phi, d.phi.cpu().numpy())
    assert np.array_equal(h.current, d.current.cpu().numpy())
    assert np.array_equal(h.iterations, d.iterations.cpu().numpy())
    assert np.array_equal(h.converged, d.converged.cpu().numpy())
    assert np.array_equal(h.leakage, d.leakage.cpu().numpy())


@pytest.mark.parametrize("B,aniso,warm", [(37, False, False), (700, False, True), (64, True, True)])
def test_host_zero_copy_path_matches_device(B, aniso, warm):
    """All host arrays pinned -> the kernel reads inputs / writes results over the bus itself
    (device staging workspace for the per-iteration operands); must equal the device path bit for bit."""
    import torch
    n = 300
    p = W.config2(batch=B, n_cells=n)
    rng = np.random.default_rng(4)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    st, ss, src = pin(p.sigma_t), pin(p.sigma_s0), pin(p.source)
    s1 = pin(0.2 * p.sigma_s0) if aniso else None
    phi0 = pin(rng.uniform(0.0, 1.0, (B, n))) if warm else None
    cfg = snop.SolverConfig(tolerance=1e-9)
    g = snop.Grid1D(p.length, n)
    outs = (pin(np.empty((B, n))), pin(np.empty(B, dtype=np.int32)), pin(np.empty(B, dtype=np.uint8)))
    # leakage output is allocated by the wrapper (pageable) -> zero-copy needs it pinned too, so
    # exercise both: without leakage (zero-copy) and with it (staged path)
    h = snop.source_iteration(g, p.order, st, ss, src, cfg, initial_phi=phi0, sigma_s1=s1, out=outs)
    dv = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
    d = snop.source_iteration(g, p.order, dv(st), dv(ss), dv(src), cfg, initial_phi=dv(phi0), sigma_s1=dv(s1))
    assert np.array_equal(h.phi, d.phi.cpu().numpy())
    assert np.array_equal(h.iterations, d.iterations.cpu().numpy())
    assert np.array_equal(h.converged, d.converged.cpu().numpy())
    bad = st.copy()
    bad[B // 2, 5] = 0.0
    with pytest.raises(InvalidArgument):
        snop.source_iteration(g, p.order, pin(bad), ss, src, cfg, out=outs)


def test_deterministic_repeat():
    p = W.config2(batch=8, n_cells=2000)
    cfg = snop.SolverConfig(tolerance=1e-8)
    g = snop.Grid1D(p.length, p.n_cells)
    a = snop.source_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.source, cfg)
    b = snop.source_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.source, cfg)
    assert np.array_equal(a.phi, b.phi)


@pytest.mark.parametrize("cs", [2, 4, 8])
def test_cluster_mode_parity(cs):
    """The thread-block-cluster variant (instance split across CTAs, DSMEM scan), forced through the
    context's execution options, must match the oracle like the one-CTA path."""
    ctx = snop.Context(0)
    try:
        ctx.set_options(cell_cluster=cs)
        assert ctx.options()["cell_cluster"] == cs
        p = W.config2(batch=6, n_cells=2000)
        for bc in ((0, 0), (1, 0), (1, 1)):
            cfg = snop.SolverConfig(tolerance=1e-300, max_inner_iterations=6, boundary_left=bc[0], boundary_right=bc[1])
            r = snop.source_iteration(snop.Grid1D(10.0, 2000), 32, p.sigma_t, p.sigma_s0, p.source, cfg, ctx=ctx)
            o = O.source_iteration(10.0, 2000, 32, p.sigma_t, p.sigma_s0, p.source, cfg.c())
            e = np.max(np.abs(r.phi - o["phi"])) / np.max(np.abs(o["phi"]))
            assert e < 1e-10, (bc, e)
        q = W.config4(batch=2, n_cells=500)
        cfg = snop.SolverConfig(tolerance=1e-7, tolerance_k=1e-8, tolerance_phi=1e-7)
        k = snop.power_iteration(snop.Grid1D(10.0, 500), 16, q.sigma_t, q.sigma_s0, q.nu_sigma_f, q.chi, cfg,
                                 ctx=ctx).k
        ko = O.power_iteration(10.0, 500, 16, 7, q.sigma_t, q.sigma_s0, q.nu_sigma_f, q.chi, cfg.c())["k"]
        assert np.max(np.abs(k - ko) / ko) < 1e-10
    finally:
        ctx.close()


def test_context_options_validation():
    ctx = snop.Context(0)
    try:
        with pytest.raises(InvalidArgument):
            ctx.set_options(cell_cluster=3)
        with pytest.raises(ValueError):
            ctx.set_options(no_such_option=1)
        assert ctx.options()["cell_cluster"] == 0
    finally:
        ctx.close()


# ---- slabs of any length: cluster path (4097..16384 cells) and streaming path (beyond) -------
def _slab(B, n, order, seed, ratio=(0.3, 0.9)):
    rng = np.random.default_rng(seed)
    x = (np.arange(n) + 0.5) * (10.0 / n)
    st = rng.uniform(0.5, 1.5, (B, 1)) * (1.0 + 0.5 * np.sin(2 * np.pi * rng.integers(1, 5, (B, 1)) * x / 10.0))
    ss = st * rng.uniform(*ratio, (B, 1))
    return W.FixedSourceProblem("slab", 10.0, n, order, st, ss, rng.uniform(0.5, 1.5, (B, n)))


@pytest.mark.parametrize("n_cells", [5000, 12000, 20000])
def test_long_slab_parity(n_cells):
    """SPEC.md:23 (n_cells: any positive integer): 5000 and 12000 cells run on thread-block
    clusters, 20000 on the streaming kernel; fixed iterations at 1e-10 for every BC combination and
    converged counts +-1 against the oracle."""
    p = _slab(3, n_cells, 16, n_cells)
    for bc in ((0, 0), (1, 0), (1, 1)):
        r, o = _run_both(p, dict(tolerance=1e-300, max_inner_iterations=5, boundary_left=bc[0], boundary_right=bc[1]))
        assert (r.iterations == 5).all()
        assert _rel(r.phi, o["phi"]) < FLUX_RTOL, bc
        assert np.max(np.abs(r.current - o["current"])) < 1e-10 * np.max(np.abs(o["phi"]))
    r, o = _run_both(p, dict(tolerance=1e-8))
    d = np.abs(r.iterations.astype(int) - o["iterations"].astype(int))
    assert d.max() <= 1
    assert _rel(r.phi[d == 0], o["phi"][d == 0]) < FLUX_RTOL


@pytest.mark.parametrize("n_cells", [1, 7, 100, 2047, 2048, 2049, 4500])
@pytest.mark.parametrize("order", [8, 16, 32])
def test_streaming_path_forced(n_cells, order, ctx_options):
    """The streaming kernel (ctx option cell_cluster = -1) on small slabs against the oracle: tile
    edges (2048-cell tiles), ragged last tiles, all BC combinations, P1 and the face leakages."""
    ctx_options(cell_cluster=-1)
    p = _slab(2, n_cells, order, 100 + n_cells + order)
    for bc in ((0, 0), (1, 0), (0, 1), (1, 1)):
        r, o = _run_both(p, dict(tolerance=1e-300, max_inner_iterations=4, boundary_left=bc[0], boundary_right=bc[1]))
        assert _rel(r.phi, o["phi"]) < FLUX_RTOL, bc
        assert np.max(np.abs(r.current - o["current"])) < 1e-10 * np.max(np.abs(o["phi"])), bc
    r, o = _run_both(p, dict(tolerance=1e-300, max_inner_iterations=4), sigma_s1=0.2 * p.sigma_s0)
    assert _rel(r.phi, o["phi"]) < FLUX_RTOL
    cfg = snop.SolverConfig(tolerance=1e-10)
    g = snop.Grid1D(p.length, p.n_cells)
    lk = snop.source_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.source, cfg, want_leakage=True)
    ol = O.source_iteration(p.length, p.n_cells, p.order, p.sigma_t, p.sigma_s0, p.source, cfg.c(), want_leak=True)
    same = lk.iterations == ol["iterations"]
    assert np.max(np.abs(lk.leakage[same] - ol["leak"][same])) < 1e-10 * np.max(np.abs(ol["phi"]))
