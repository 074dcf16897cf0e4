"""Parity of the fused power-iteration kernel (K2) against the CPU oracle."""
import numpy as np
import pytest

from paper_2509_01416_b200 import snop, workloads as W
from paper_2509_01416_b200.errors import DegenerateProblem
from tests import oracle_lib as O

pytestmark = pytest.mark.gpu

K_RTOL = 1e-10  # north_star: k_eff within 1e-10 relative


def _cfg(p, **kw):
    d = dict(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi,
             boundary_left=p.bc_left, boundary_right=p.bc_right)
    d.update(kw)
    return snop.SolverConfig(**d)


def _both(p, cfg, **kw):
    g = snop.Grid1D(p.length, p.n_cells)
    r = snop.power_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg, **kw)
    o = O.power_iteration(p.length, p.n_cells, p.order, p.n_groups, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi,
                          cfg.c(), **kw)
    return r, o


def test_table9_three_group_k():
    # PAPER.md:379 model-based k = 1.30621 (vacuum, N=32, dx=0.1, L=10)
    p = W.three_group_table9()
    r, o = _both(p, _cfg(p))
    assert abs(r.k[0] - 1.30621) < 5e-5
    assert abs(int(r.outer_iterations[0]) - int(o["outer"][0])) <= 1
    if r.outer_iterations[0] == o["outer"][0]:
        assert abs(r.k[0] - o["k"][0]) / o["k"][0] < K_RTOL


def test_reflective_three_group_equals_dense():
    p = W.three_group_table9(bc=1)
    r, _ = _both(p, _cfg(p, tolerance=1e-10, tolerance_k=1e-11, tolerance_phi=1e-10))
    kinf = O.infinite_medium_k(p.sigma_t[0, :, 0], p.sigma_s0[0, :, :, 0], p.nu_sigma_f[0, :, 0], p.chi[0])
    assert abs(r.k[0] - kinf) < 1e-6


def test_single_group_kinf():
    # reflective, St=1, Ss0=0.5, nuSf=0.9 -> k = 1.8
    n = 50
    p = W.EigenProblem("k", 10.0, n, 8, 1, np.ones((1, 1, n)), np.full((1, 1, 1, n), 0.5), np.full((1, 1, n), 0.9),
                       np.ones((1, 1)), bc_left=1, bc_right=1, tolerance_k=1e-8, tolerance_phi=1e-6,
                       tolerance_inner=1e-6)
    r, _ = _both(p, _cfg(p))
    assert abs(r.k[0] - 1.8) < 1e-4


def _converged_parity(r, o):
    """Outer counts +-1; identical (outer, total inner) counts -> k and phi at 1e-10; otherwise the
    extra sweep moves k by less than its tolerance."""
    do = np.abs(r.outer_iterations.astype(int) - o["outer"].astype(int))
    assert do.max() <= 1
    same = (do == 0) & (r.total_inner_iterations == o["inner"])
    dk = np.abs(r.k - o["k"]) / o["k"]
    assert same.any()
    assert dk[same].max() < K_RTOL
    assert np.max(np.abs(r.phi[same] - o["phi"][same])) / np.max(np.abs(o["phi"][same])) < K_RTOL
    if (~same).any():
        assert dk[~same].max() < 1e-8


def test_c3_subset_parity():
    p = W.config3(batch=6, n_cells=1024)
    r, o = _both(p, _cfg(p))
    _converged_parity(r, o)


def test_c4_subset_parity():
    p = W.config4(batch=3, n_cells=500)
    r, o = _both(p, _cfg(p))
    _converged_parity(r, o)


def test_fixed_outer_flux_parity():
    p = W.config4(batch=2, n_cells=300)
    cfg = _cfg(p, tolerance_k=1e-300, tolerance_phi=1e-300, max_outer_iterations=3, max_inner_iterations=4,
               tolerance=1e-300)
    r, o = _both(p, cfg)
    assert (r.outer_iterations == 3).all()
    assert (r.total_inner_iterations == o["inner"]).all()
    assert np.max(np.abs(r.phi - o["phi"])) / np.max(np.abs(o["phi"])) < K_RTOL
    assert np.max(np.abs(r.k - o["k"]) / o["k"]) < K_RTOL


def test_scale_invariance_initial_guess():
    # SPEC.md:201
    p = W.three_group_table9()
    cfg = _cfg(p)
    g = snop.Grid1D(p.length, p.n_cells)
    a = snop.power_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg,
                             initial_phi=np.full((1, 3, p.n_cells), 1.0))
    b = snop.power_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg,
                             initial_phi=np.full((1, 3, p.n_cells), 7.5))
    assert abs(a.k[0] - b.k[0]) < 1e-10


def test_zero_fission_is_degenerate():
    n = 20
    p = W.EigenProblem("d", 10.0, n, 8, 1, np.ones((1, 1, n)), np.full((1, 1, 1, n), 0.5), np.zeros((1, 1, n)),
                       np.ones((1, 1)))
    with pytest.raises(DegenerateProblem):
        snop.power_iteration(snop.Grid1D(10.0, n), 8, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, _cfg(p))


@pytest.mark.parametrize("cs", ["0", "2", "4", "8"])
def test_pair_split_cluster_parity(cs, ctx_options):
    """Pair-split clusters (si_solve PS, single-group eigen): each CTA sweeps a range of pair groups
    and the partial edge currents are exchanged through DSMEM. Fixed iteration counts: flux and k
    against the oracle at 1e-10; cs = 0 is the one-CTA kernel. C3 shapes (reflective left)."""
    ctx_options(pair_split=int(cs) if cs != "0" else -1)
    p = W.config3(batch=3, n_cells=1000)
    cfg = _cfg(p, tolerance_k=1e-300, tolerance_phi=1e-300, max_outer_iterations=4, max_inner_iterations=5,
               tolerance=1e-300)
    r, o = _both(p, cfg)
    assert (r.total_inner_iterations == o["inner"]).all()
    assert np.max(np.abs(r.phi - o["phi"])) / np.max(np.abs(o["phi"])) < K_RTOL
    assert np.max(np.abs(r.k - o["k"]) / o["k"]) < K_RTOL


def test_pair_split_converged_matches_single_cta(ctx_options):
    p = W.config3(batch=4, n_cells=777)  # ragged cell count (padding cells in the last chunk)
    g = snop.Grid1D(p.length, p.n_cells)
    out = {}
    for cs in ("0", "4"):
        ctx_options(pair_split=int(cs) if cs != "0" else -1, pi_tail_cap=-1)
        out[cs] = snop.power_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, _cfg(p))
    a, b = out["0"], out["4"]
    assert np.all(np.abs(a.outer_iterations.astype(int) - b.outer_iterations.astype(int)) <= 1)
    assert np.max(np.abs(a.k - b.k) / a.k) < 1e-10


def test_tail_split_resume_parity(ctx_options):
    """Tail split: phase 1 (one CTA, outer <= cap) then phase 2 (pair-split clusters) resuming from
    (k, phi, counts) for the unconverged instances. cap = 3 forces every instance through both
    phases; converged k against the oracle and against the unsplit single-CTA solve."""
    p = W.config3(batch=5, n_cells=640)
    g = snop.Grid1D(p.length, p.n_cells)
    ctx_options(pi_tail_cap=3)
    r, o = _both(p, _cfg(p))
    _converged_parity(r, o)
    ctx_options(pi_tail_cap=-1, pair_split=-1)
    a = snop.power_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, _cfg(p))
    assert np.all(np.abs(a.outer_iterations.astype(int) - r.outer_iterations.astype(int)) <= 1)
    assert np.all(np.abs(a.total_inner_iterations - r.total_inner_iterations) <= 2 * a.total_inner_iterations // 100 + 5)
    assert np.max(np.abs(a.k - r.k) / a.k) < 1e-10


def test_tail_split_fixed_iterations(ctx_options):
    """Fixed iteration counts across the phase boundary (cap 2 of 5 outers): flux and k at 1e-10."""
    ctx_options(pi_tail_cap=2)
    p = W.config3(batch=3, n_cells=512)
    cfg = _cfg(p, tolerance_k=1e-300, tolerance_phi=1e-300, max_outer_iterations=5, max_inner_iterations=4,
               tolerance=1e-300)
    r, o = _both(p, cfg)
    assert (r.outer_iterations == 5).all()
    assert (r.total_inner_iterations == o["inner"]).all()
    assert np.max(np.abs(r.phi - o["phi"])) / np.max(np.abs(o["phi"])) < K_RTOL
    assert np.max(np.abs(r.k - o["k"]) / o["k"]) < K_RTOL


def test_tail_split_deterministic_and_batch_independent(ctx_options):
    """Repeated tail-split solves are bit-identical, and an instance's result does not depend on the
    batch it is solved in (the schedule depends on (G, order) and its own outer count only)."""
    ctx_options(pi_tail_cap=4)
    p = W.config3(batch=6, n_cells=700)
    g = snop.Grid1D(p.length, p.n_cells)
    cfg = _cfg(p)
    a = snop.power_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)
    b = snop.power_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)
    assert np.array_equal(a.k, b.k) and np.array_equal(a.phi, b.phi)
    q = p.subset([4, 1])
    c = snop.power_iteration(g, q.order, q.sigma_t, q.sigma_s0, q.nu_sigma_f, q.chi, cfg)
    assert np.array_equal(c.k, a.k[[4, 1]]) and np.array_equal(c.phi, a.phi[[4, 1]])
    assert np.array_equal(c.outer_iterations, a.outer_iterations[[4, 1]])


@pytest.mark.parametrize("order", [10, 14])
def test_pair_split_odd_pair_count(order, ctx_options):
    """S10 / S14: an odd number of +/-mu pairs (the tail pair goes to the last rank of the cluster)."""
    ctx_options(pair_split=2)
    base = W.config3(batch=2, n_cells=300)
    p = W.EigenProblem("odd", base.length, base.n_cells, order, 1, base.sigma_t, base.sigma_s0, base.nu_sigma_f,
                       base.chi, None, base.bc_left, base.bc_right)
    cfg = _cfg(p, tolerance_k=1e-300, tolerance_phi=1e-300, max_outer_iterations=3, max_inner_iterations=4,
               tolerance=1e-300)
    r, o = _both(p, cfg)
    assert (r.total_inner_iterations == o["inner"]).all()
    assert np.max(np.abs(r.phi - o["phi"])) / np.max(np.abs(o["phi"])) < K_RTOL
    assert np.max(np.abs(r.k - o["k"]) / o["k"]) < K_RTOL


@pytest.mark.parametrize("forced", [True, False])
def test_streaming_power_iteration(forced, ctx_options):
    """Power iteration beyond the resident kernels: the device-looped outer iteration around the
    streaming K1 (forced on a C4-like multigroup problem, and automatic at 20000 cells single-group),
    fixed counts at 1e-10 and converged k against the oracle."""
    if forced:
        ctx_options(cell_cluster=-1)
        p = W.config4(batch=2, n_cells=300)
    else:
        p = W.config3(batch=2, n_cells=20000)
    cfg = _cfg(p, tolerance_k=1e-300, tolerance_phi=1e-300, max_outer_iterations=3, max_inner_iterations=4,
               tolerance=1e-300)
    r, o = _both(p, cfg)
    assert (r.outer_iterations == 3).all() and (r.total_inner_iterations == o["inner"]).all()
    assert np.max(np.abs(r.phi - o["phi"])) / np.max(np.abs(o["phi"])) < K_RTOL
    assert np.max(np.abs(r.k - o["k"]) / o["k"]) < K_RTOL
    r, o = _both(p, _cfg(p))
    _converged_parity(r, o)
