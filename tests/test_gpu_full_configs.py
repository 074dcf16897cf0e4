"""BASELINE configurations at their FULL sizes against the CPU oracle (repo BASELINE.json configs;
SURVEY §8a). The reduced-size suites elsewhere pin the kernels' arithmetic; these pin the
production schedules that only appear at full size: the tail split of the single-group eigen
solve (phase 1 on one CTA per instance, phase 2 on 8-CTA pair-split clusters for the instances
still iterating after 12 outers: predicted-long ones on clusters at once, the rest after up to 32 more single-CTA outers), the longest-first dispatch of the 2048-instance fixed-source
batch, and the C5 MD-PNOP pipeline (FNO -> recast fixed point -> warm-started K1).

Tolerances (north_star): outer/inner iteration counts within +-1; k and scalar flux within
1e-10 relative at equal iteration counts; fp32 operator outputs within 1e-5 of the output max.
Reference contracts: power_iteration SPEC.md:179-189, source_iteration :125-134, predict
:319-322, recast_fixed_point :403-411, precondition_fixed_source :413-421."""
import numpy as np
import pytest

from paper_2509_01416_b200 import operators as OPS, snop, workloads as W
from tests import oracle_lib as O

pytestmark = pytest.mark.gpu

RTOL = 1e-10     # k_eff and scalar flux, fp64, equal iteration counts
OP_RTOL = 1e-5   # fp32 operator outputs
TH = O.hardware_threads()


def _rel(a, b):
    return np.max(np.abs(np.asarray(a) - b)) / max(np.max(np.abs(b)), 1e-300)


def _rel_rows(a, b):
    a, b = np.asarray(a).reshape(len(a), -1), np.asarray(b).reshape(len(b), -1)
    return np.max(np.abs(a - b), axis=1) / np.maximum(np.max(np.abs(b), axis=1), 1e-300)


def _eig_cfg(p, **kw):
    d = dict(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi,
             boundary_left=p.bc_left, boundary_right=p.bc_right)
    d.update(kw)
    return snop.SolverConfig(**d)


def _oracle_eig(q, cfg):
    return O.power_iteration(q.length, q.n_cells, q.order, q.n_groups, q.sigma_t, q.sigma_s0, q.nu_sigma_f, q.chi,
                             cfg.c(), n_threads=TH)


def _gpu_eig(p, cfg):
    g = snop.Grid1D(p.length, p.n_cells)
    return snop.power_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi, cfg)


def _check_converged_eigen(r, o, idx):
    """Converged power iterations: outer counts +-1; where outer AND total inner counts agree, the
    two runs performed the same operations, so k and phi agree to rounding (1e-10)."""
    do = np.abs(r.outer_iterations[idx].astype(int) - o["outer"].astype(int))
    assert do.max() <= 1, f"outer counts differ by {do.max()}"
    assert r.converged[idx].all() and o["converged"].all()
    same = (do == 0) & (r.total_inner_iterations[idx] == o["inner"])
    assert same.mean() >= 0.75, f"only {same.sum()} of {len(idx)} instances with identical counts"
    dk = np.abs(r.k[idx] - o["k"]) / np.abs(o["k"])
    assert dk[same].max() < RTOL, f"k {dk[same].max():.2e}"
    assert _rel_rows(r.phi[idx][same], o["phi"][same]).max() < RTOL
    # differing counts: one extra inner/outer sweep moves k by less than the k tolerance
    if (~same).any():
        assert dk[~same].max() < 1e-8
    return same


# ---- C3: 512 x 4096 x S32, single-group eigen, reflective left / vacuum right ----------------

@pytest.fixture(scope="module")
def c3():
    p = W.config3()
    cfg = _eig_cfg(p)
    return p, cfg, _gpu_eig(p, cfg)


def test_c3_full_tail_and_random_instances(c3):
    """The 32 instances with the most outer iterations (all of them finish in phase 2 of the tail
    split, on pair-split clusters; the slowest needs >1000 outers) plus 32 random others, against
    the oracle, from one production-size batch."""
    p, cfg, r = c3
    longest = np.argsort(-r.outer_iterations.astype(int), kind="stable")[:32]
    rest = np.setdiff1d(np.arange(p.batch), longest)
    idx = np.concatenate([longest, np.random.default_rng(3).choice(rest, 32, replace=False)])
    assert (r.outer_iterations[longest] > 32).all()  # phase 2 exercised at full size
    o = _oracle_eig(p.subset(idx), cfg)
    _check_converged_eigen(r, o, idx)


def test_c3_full_fixed_iterations_across_phase_boundary():
    """Fixed counts (52 outers x 2 inner sweeps, tolerances 0): every instance crosses the tail-split
    boundaries (12 and 44 outers); flux and k at 1e-10 on 16 instances of the full 512-instance batch."""
    p = W.config3()
    cfg = _eig_cfg(p, tolerance=1e-300, tolerance_k=1e-300, tolerance_phi=1e-300, max_outer_iterations=52,
                   max_inner_iterations=2)
    r = _gpu_eig(p, cfg)
    # a fast-converging instance can reach a bit-exact fixed point (an inner sweep or an outer
    # iteration that changes nothing: 0 < 1e-300) and stop early; its flux is then compared against
    # the oracle's 52-outer flux like the others
    early = np.nonzero(r.converged)[0]
    assert (r.outer_iterations[early] > 30).all()
    run = ~r.converged
    assert (r.outer_iterations[run] == 52).all() and (r.total_inner_iterations[run] == 104).all()
    idx = np.union1d(np.random.default_rng(5).choice(p.batch, 16, replace=False), early)
    o = _oracle_eig(p.subset(idx), cfg)
    assert _rel_rows(r.phi[idx], o["phi"]).max() < RTOL
    assert (np.abs(r.k[idx] - o["k"]) / o["k"]).max() < RTOL


# ---- C4: 128 x 2000 x S16 x G7, Gauss-Seidel with upscatter -----------------------------------

def test_c4_full_all_instances():
    p = W.config4()
    cfg = _eig_cfg(p)
    r = _gpu_eig(p, cfg)
    o = _oracle_eig(p, cfg)
    _check_converged_eigen(r, o, np.arange(p.batch))


def test_c4_full_fixed_iterations():
    p = W.config4()
    cfg = _eig_cfg(p, tolerance=1e-300, tolerance_k=1e-300, tolerance_phi=1e-300, max_outer_iterations=3,
                   max_inner_iterations=3)
    r = _gpu_eig(p, cfg)
    idx = np.arange(0, p.batch, 8)
    o = _oracle_eig(p.subset(idx), cfg)
    assert (r.total_inner_iterations[idx] == o["inner"]).all()
    assert _rel_rows(r.phi[idx], o["phi"]).max() < RTOL
    assert (np.abs(r.k[idx] - o["k"]) / o["k"]).max() < RTOL


# ---- C2: 2048 x 2000 x S32 fixed source (longest-first dispatch) ------------------------------

def test_c2_full_batch():
    p = W.config2()
    cfg = snop.SolverConfig(tolerance=p.tolerance)
    r = snop.source_iteration(snop.Grid1D(p.length, p.n_cells), p.order, p.sigma_t, p.sigma_s0, p.source, cfg)
    o = O.source_iteration(p.length, p.n_cells, p.order, p.sigma_t, p.sigma_s0, p.source, cfg.c(), n_threads=TH)
    d = np.abs(r.iterations.astype(int) - o["iterations"].astype(int))
    assert d.max() <= 1
    same = d == 0
    assert same.mean() >= 0.9
    assert _rel_rows(r.phi[same], o["phi"][same]).max() < RTOL
    assert r.converged.all() and o["converged"].all()


# ---- C5: FNO -> recast fixed point -> warm-started K1 (MD-PNOP pipeline) ------------------------

@pytest.fixture(scope="module")
def c5():
    p = W.config5()
    prm = OPS.fno_init(64, 16, 4, 128, OPS.GELU)
    g = snop.Grid1D(p.length, p.n_cells)
    op = snop.SolutionOperator.fno(g, prm, p.ref_params)
    oo = O.OracleOperator.fno(p.length, p.n_cells, p.ref_params, OPS.GELU, 64, 16, 4, 128, prm.packed())
    return p, op, oo


def test_c5_fno_all_samples(c5):
    """phi0 = op(S) (Eq. 9 with a zero initial guess) for all 4096 recast-source fields."""
    p, op, oo = c5
    y = op.predict(p.source)
    yo = oo.predict(p.source, n_threads=TH)
    assert _rel(y, yo) < OP_RTOL


def test_c5_recast_fixed_point_subset(c5):
    """Full recast fixed point (tol 1e-4, max 50) on 256 of the 4096 fields: statuses and counts
    equal, iterates within the fp32 operator tolerance."""
    p, op, oo = c5
    idx = np.arange(0, p.batch, 16)
    q = p.subset(idx)
    r = snop.recast_fixed_point(op, q.source, q.sigma_t, q.sigma_s0, 1e-4, 50)
    o = oo.recast_fixed_point(q.source, q.sigma_t, q.sigma_s0, tol=1e-4, max_it=50, n_threads=TH)
    assert np.array_equal(r.status, o["status"])
    assert np.all(np.abs(r.iterations - o["iterations"]) <= 1)
    same = r.iterations == o["iterations"]
    assert _rel(r.phi[same], o["phi"][same]) < OP_RTOL


def test_c5_pipeline_warm_start_full(c5):
    """The pipeline at full size: the device recast fixed point gives phi_NO; K1 warm-started from
    phi_NO against the oracle's source iteration from the SAME phi_NO (iterations +-1, flux 1e-10);
    and the fused precondition_fixed_source call equals that composition bit for bit."""
    p, op, oo = c5
    cfg = snop.SolverConfig(tolerance=p.tolerance)
    g = snop.Grid1D(p.length, p.n_cells)
    rf = snop.recast_fixed_point(op, p.source, p.sigma_t, p.sigma_s0, 1e-4, 50)
    assert (rf.status != 2).all()
    phi_no = np.asarray(rf.phi)
    r = snop.source_iteration(g, p.order, p.sigma_t, p.sigma_s0, p.source, cfg, initial_phi=phi_no)
    o = O.source_iteration(p.length, p.n_cells, p.order, p.sigma_t, p.sigma_s0, p.source, cfg.c(),
                           initial_phi=phi_no, n_threads=TH)
    d = np.abs(r.iterations.astype(int) - o["iterations"].astype(int))
    assert d.max() <= 1
    same = d == 0
    assert same.mean() >= 0.9
    assert _rel_rows(r.phi[same], o["phi"][same]).max() < RTOL
    fused = snop.precondition_fixed_source(op, p.order, p.sigma_t, p.sigma_s0, p.source, cfg,
                                           recast_tolerance=1e-4, recast_max_iterations=50)
    assert np.array_equal(fused.precond_iterations, rf.iterations)
    assert np.array_equal(fused.recast_status, rf.status)
    assert np.array_equal(fused.refine_iterations, r.iterations)
    assert np.array_equal(fused.phi, r.phi)
