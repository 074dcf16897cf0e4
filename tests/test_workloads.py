"""Seeded synthetic inputs (BASELINE configs C1-C5) are deterministic and respect the ranges
SURVEY §8d / §9 pin."""
import numpy as np

from paper_2509_01416_b200 import operators as OPS, workloads as W


def test_c2_ranges_and_determinism():
    a = W.config2(batch=64)
    b = W.config2(batch=64)
    assert np.array_equal(a.sigma_t, b.sigma_t) and np.array_equal(a.sigma_s0, b.sigma_s0)
    c = a.sigma_s0[:, 0] / a.sigma_t[:, 0]
    assert (c >= 0.5).all() and (c < 0.95).all()
    assert a.sigma_t.min() > 0.8 * 0.5 - 1e-12 and a.sigma_t.max() < 1.5 * 1.5 + 1e-12
    assert a.order == 32 and a.sigma_t.shape == (64, 2000)


def test_c3_has_fissile_region_and_reflective_left():
    p = W.config3(batch=32, n_cells=512)
    assert (p.nu_sigma_f.max(axis=(1, 2)) > 0).all()
    assert p.bc_left == 1 and p.bc_right == 0 and p.order == 32
    c = p.sigma_s0[:, 0, 0] / p.sigma_t[:, 0]
    assert (c >= 0.3 - 1e-12).all() and (c < 0.9).all()


def test_c4_scattering_rows_below_total_and_upscatter_only_thermal():
    p = W.config4(batch=8, n_cells=50)
    S = p.sigma_s0[:, :, :, 0]          # [b][g'][g] = g' -> g
    rows = S.sum(axis=2)                # total scattering out of g'
    assert (rows < p.sigma_t[:, :, 0]).all()
    for g_src in range(7):
        for g_dst in range(g_src):
            up = S[:, g_src, g_dst]
            if not (g_src in W.THERMAL and g_dst in W.THERMAL):
                assert (up == 0).all()
    assert np.allclose(p.chi.sum(axis=1), 1.0) and (p.chi[:, 3:] == 0).all()


def test_c5_mix_of_profiles():
    p = W.config5(batch=8)
    assert np.allclose(p.sigma_s0, 0.8 * p.sigma_t)
    assert len(np.unique(p.sigma_t[1])) <= 5  # step profile
    assert len(np.unique(p.sigma_t[0])) > 5   # sinusoid


def test_operator_init_deterministic():
    a = OPS.fno_init().packed()
    b = OPS.fno_init().packed()
    assert np.array_equal(a, b) and a.dtype == np.float32
    d = OPS.deeponet_init(2000)
    assert d.branch.sizes == [2000, 128, 128, 128, 128] and d.trunk.sizes == [1, 128, 128, 128, 128]
    lim = np.sqrt(6.0 / (2000 + 128))
    assert np.abs(d.branch.weights[0]).max() <= lim
