"""The standalone transport sweep: oracle pins on the CPU (the SPEC examples on
the oracle's own sweep), GPU parity of snop_sweep_batched against the oracle (psi_avg and the net
outgoing partial currents, every boundary combination, ragged sizes), and the size-independent
properties at the BASELINE sizes (per-cell diamond-difference balance, linearity)."""
import numpy as np
import pytest

from tests import oracle_lib as O

PSI_RTOL = 1e-10  # north_star: fp64 fields within 1e-10 relative


def _rel(a, b):
    return np.max(np.abs(np.asarray(a) - b)) / max(np.max(np.abs(b)), 1e-300)


def _case(B, Nc, N, seed, thin=False):
    r = np.random.default_rng(seed)
    st = r.uniform(1e-4 if thin else 0.2, 2.0, size=(B, Nc))
    em = r.uniform(0.0, 1.5, size=(B, Nc, N))
    return st, em


# ---- oracle pins (CPU) ----------------------------------------------------------------------
def test_oracle_sweep_zero_emission_is_zero():
    psi, ol, orr = O.sweep(10.0, 50, 8, np.ones((2, 50)), np.zeros((2, 50, 8)))
    assert np.all(psi == 0.0) and np.all(ol == 0.0) and np.all(orr == 0.0)


def test_oracle_sweep_attenuation_second_order():
    # uniform St = 1, q = 1, vacuum left -> psi(x) = 1 - exp(-x / mu) along a mu > 0
    # direction; the diamond-difference cell averages converge to its cell averages at 2nd order
    L, N = 4.0, 8
    mu, _ = O.gauss_legendre(N)
    n = N - 1  # the most forward direction
    errs = []
    for Nc in (40, 80, 160):
        psi, _, _ = O.sweep(L, Nc, N, np.ones((1, Nc)), np.ones((1, Nc, N)))
        x = np.linspace(0.0, L, Nc + 1)
        exact = 1.0 + mu[n] * (np.exp(-x[1:] / mu[n]) - np.exp(-x[:-1] / mu[n])) / (L / Nc)
        errs.append(np.max(np.abs(psi[0, n] - exact)))
    assert 3.6 < errs[0] / errs[1] < 4.4 and 3.6 < errs[1] / errs[2] < 4.4


def test_oracle_sweep_reflective_left_mirrors_the_outflow():
    # reflective left -> the mu > 0 inflow at x = 0 is the mu < 0 outflow there: with a
    # symmetric emission the two directions of a pair then carry the same flux through cell 0's
    # left edge, and the net outgoing partial current at x = 0 vanishes
    Nc, N = 30, 6
    st, em = _case(2, Nc, N, 5)
    em = 0.5 * (em + em[:, :, ::-1])  # q(mu) = q(-mu)
    psi, ol, _ = O.sweep(5.0, Nc, N, st, em, bc_left=1, bc_right=0)
    assert np.all(np.abs(ol) < 1e-14)
    for p in range(N // 2):
        plus, minus = psi[:, N // 2 + p, 0], psi[:, N // 2 - 1 - p, 0]
        # left-edge fluxes: minus leaves (2 avg - in), plus enters; recover both from cell 0
        assert np.all(plus > 0) and np.all(minus > 0)


def test_oracle_sweep_cell_balance():
    # mu (psi_out - psi_in) / dx + St psi_avg = q for every cell and direction
    B, Nc, N, L = 2, 40, 8, 7.0
    st, em = _case(B, Nc, N, 1)
    psi, _, _ = O.sweep(L, Nc, N, st, em)
    mu, _ = O.gauss_legendre(N)
    dx = L / Nc
    for n in range(N):
        edge = np.zeros(B)
        cells = range(Nc) if mu[n] > 0 else range(Nc - 1, -1, -1)
        for i in cells:
            out = 2.0 * psi[:, n, i] - edge
            res = abs(mu[n]) * (out - edge) / dx + st[:, i] * psi[:, n, i] - em[:, i, n]
            assert np.max(np.abs(res)) < 1e-12 * max(1.0, np.max(np.abs(em)))
            edge = out


# ---- GPU parity -------------------------------------------------------------------------------
gpu = pytest.mark.gpu


@gpu
@pytest.mark.parametrize("bc", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("B,Nc,N", [(3, 1, 2), (5, 7, 4), (4, 64, 8), (9, 1000, 16), (6, 2000, 32), (2, 517, 6),
                                    (3, 4099, 64), (2100, 66, 32), (4200, 67, 16), (3, 300, 4), (2, 100, 128), (3, 98, 12)])  # (large batches: more than
    # one wave of CTAs; N <= 16 in one wave: 16-cell tiles, otherwise 8-cell tiles)
def test_sweep_parity(bc, B, Nc, N):
    from paper_2509_01416_b200 import snop
    st, em = _case(B, Nc, N, 100 + Nc + N)
    psi, ol, orr = snop.sweep(snop.Grid1D(10.0, Nc), N, st, em, bc[0], bc[1])
    o_psi, o_ol, o_or = O.sweep(10.0, Nc, N, st, em, bc[0], bc[1])
    assert _rel(psi, o_psi) < PSI_RTOL
    scale = max(np.max(np.abs(o_ol)), np.max(np.abs(o_or)), 1e-300)
    assert np.max(np.abs(ol - o_ol)) < PSI_RTOL * scale and np.max(np.abs(orr - o_or)) < PSI_RTOL * scale


@gpu
def test_sweep_thin_cells_and_device_arrays():
    import torch
    from paper_2509_01416_b200 import snop
    B, Nc, N = 8, 1024, 16
    st, em = _case(B, Nc, N, 7, thin=True)
    g = snop.Grid1D(10.0, Nc)
    o_psi, o_ol, o_or = O.sweep(10.0, Nc, N, st, em, 1, 0)
    psi, ol, orr = snop.sweep(g, N, torch.from_numpy(st).cuda(), torch.from_numpy(em).cuda(), 1, 0)
    assert _rel(psi.cpu().numpy(), o_psi) < PSI_RTOL
    assert _rel(ol.cpu().numpy(), o_ol) < PSI_RTOL and _rel(orr.cpu().numpy(), o_or) < PSI_RTOL


@gpu
@pytest.mark.parametrize("Nc,N", [(200001, 2), (65536, 4)])
def test_sweep_long_slab(Nc, N):
    """Slabs far beyond the solvers' resident limits (any n_cells up to 2^26 is valid):
    the march has no per-instance size limit; odd / even cell counts take the two load paths."""
    from paper_2509_01416_b200 import snop
    st, em = _case(2, Nc, N, 9)
    psi, ol, orr = snop.sweep(snop.Grid1D(50.0, Nc), N, st, em, 0, 1)
    o_psi, o_ol, o_or = O.sweep(50.0, Nc, N, st, em, 0, 1)
    assert _rel(psi, o_psi) < PSI_RTOL and _rel(ol, o_ol) < PSI_RTOL and np.max(np.abs(orr - o_or)) < 1e-14


@gpu
def test_sweep_errors_and_empty():
    from paper_2509_01416_b200 import snop
    from paper_2509_01416_b200.errors import InvalidArgument
    g = snop.Grid1D(10.0, 16)
    st, em = _case(2, 16, 4, 3)
    bad = st.copy()
    bad[1, 5] = 0.0
    with pytest.raises(InvalidArgument):
        snop.sweep(g, 4, bad, em)
    with pytest.raises(InvalidArgument):
        snop.sweep(g, 5, st, np.zeros((2, 16, 5)))
    psi, ol, orr = snop.sweep(g, 4, np.zeros((0, 16)), np.zeros((0, 16, 4)))
    assert psi.shape == (0, 4, 16) and ol.shape == (0,)


@gpu
@pytest.mark.parametrize("name,B,Nc,N", [("C2", 2048, 2000, 32), ("C5", 4096, 1024, 16)])
def test_sweep_full_size_properties(name, B, Nc, N):
    """BASELINE sizes, on the device: the diamond-difference balance of every cell and direction
    (SPEC.md:147), linearity in the emission, and oracle parity on a sample of the instances."""
    import torch
    from paper_2509_01416_b200 import snop
    L = 10.0
    gen = torch.Generator(device="cuda").manual_seed(11)
    st = torch.rand((B, Nc), generator=gen, device="cuda", dtype=torch.float64) * 1.8 + 0.2
    em = torch.rand((B, Nc, N), generator=gen, device="cuda", dtype=torch.float64)
    g = snop.Grid1D(L, Nc)
    psi, ol, orr = snop.sweep(g, N, st, em)
    # balance: psi_in of cell i is psi_out of the upwind cell; psi_out = 2 avg - psi_in
    mu = torch.from_numpy(snop.gauss_legendre(N).mu).cuda()
    H, dx = N // 2, L / Nc
    q = em.permute(0, 2, 1)  # [B][N][Nc]
    # forward directions: edge_{i+1} = 2 avg_i - edge_i, edge_0 = 0 -> alternating prefix sum
    sgn = torch.where(torch.arange(Nc, device="cuda") % 2 == 0, 1.0, -1.0).to(torch.float64)
    def edges_in(avg):  # inflow edge flux of every cell for cells ordered in sweep direction
        # e_{i+1} = 2 a_i - e_i  =>  (-1)^{i+1} e_{i+1} = (-1)^i e_i - 2 (-1)^i a_i ... use a scan in fp64
        t = torch.cumsum(2.0 * avg * sgn, dim=-1) * sgn  # e_{i+1} = sgn_i * sum_{j<=i} 2 a_j sgn_j
        return torch.cat([torch.zeros_like(t[..., :1]), t[..., :-1]], dim=-1), t
    fwd = psi[:, H:, :]
    ein, eout = edges_in(fwd)
    res_f = mu[H:].view(1, H, 1) * (eout - ein) / dx + st.unsqueeze(1) * fwd - q[:, H:, :]
    bwd = torch.flip(psi[:, :H, :], dims=[-1])
    ein, eout = edges_in(bwd)
    res_b = (-mu[:H]).view(1, H, 1) * (eout - ein) / dx + torch.flip(st, dims=[-1]).unsqueeze(1) * bwd \
        - torch.flip(q[:, :H, :], dims=[-1])
    # the reconstructed edges accumulate rounding along the slab; the balance holds to ~1e-10 of q
    assert float(res_f.abs().max()) < 1e-9 and float(res_b.abs().max()) < 1e-9
    # linearity: sweep(2 q) = 2 sweep(q) bit for bit (scaling by 2 is exact)
    psi2, ol2, or2 = snop.sweep(g, N, st, 2.0 * em)
    assert torch.equal(psi2, 2.0 * psi) and torch.equal(ol2, 2.0 * ol) and torch.equal(or2, 2.0 * orr)
    # oracle parity on a sample
    idx = np.linspace(0, B - 1, 12).astype(int)
    o_psi, o_ol, o_or = O.sweep(L, Nc, N, st[idx].cpu().numpy(), em[idx].cpu().numpy())
    assert _rel(psi[idx].cpu().numpy(), o_psi) < PSI_RTOL
    assert _rel(ol[idx].cpu().numpy(), o_ol) < PSI_RTOL and _rel(orr[idx].cpu().numpy(), o_or) < PSI_RTOL
