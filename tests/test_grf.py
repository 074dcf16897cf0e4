"""GRF sources and training datasets (paper Appendix A1).

CPU: the oracle's sample_grf / normalize_source / generate_dataset against the SPEC examples
(degenerate variance, empirical mean and lag-l correlation, normalisation identities, balance of
every generated pair, determinism) and against an independent numpy restatement driven by the
pinned Python Rng; the product's host-only dataset file writer/reader (round trip, manifest,
corruption). GPU: device sampling / normalisation / dataset generation against the oracle.
"""
import math

import numpy as np
import pytest

from paper_2509_01416_b200 import snop
from paper_2509_01416_b200.errors import InvalidArgument, IoError
from paper_2509_01416_b200.rng import Rng
from tests import oracle_lib as O

PAPER = snop.GrfSpec(0.07, 3e-4, 1.2, 1e-10, 2024)


def _numpy_field(n, L, spec, sample):
    """Independent restatement: SE covariance + jitter, numpy Cholesky, normals from the pinned Rng."""
    dx = L / n
    x = (np.arange(n) + 0.5) * dx
    C = spec.variance * np.exp(-(x[:, None] - x[None, :]) ** 2 / (2 * spec.length_scale_cm ** 2))
    r = Rng(spec.seed + sample)
    z = np.array([r.normal() for _ in range(n)])
    jitter = spec.jitter
    while True:
        try:
            Lc = np.linalg.cholesky(C + jitter * spec.variance * np.eye(n))
            break
        except np.linalg.LinAlgError:
            jitter *= 10
            assert jitter <= 1e-6 * (1 + 1e-12)
    return spec.mean + Lc @ z, jitter


# ---------------------------------------------------------------- oracle / host (CPU) -------------
def test_oracle_matches_numpy_restatement():
    n = 100
    f, neg, jit = O.grf_sample(10.0, n, PAPER, 3, first=5)
    for k in range(3):
        ref, jit_np = _numpy_field(n, 10.0, PAPER, 5 + k)
        assert jit == pytest.approx(jit_np)
        # the SE covariance is numerically singular (jitter-regularised), so factors computed with a
        # different elimination order (LAPACK blocked vs row-by-row) agree only to ~1e-7 relative
        assert np.max(np.abs(f[k] - ref)) < 1e-6 * 0.07
        assert neg[k] == int(np.sum(f[k] < 0))


def test_degenerate_variance_is_constant():
    f, _, _ = O.grf_sample(10.0, 100, snop.GrfSpec(0.07, 1e-18, 1.2, 1e-10, 1), 4)
    assert np.max(np.abs(f - 0.07)) < 1e-8


def test_empirical_mean_and_lag_correlation():
    n = 100
    f, neg, _ = O.grf_sample(10.0, n, PAPER, 1000)
    assert abs(f.mean() - 0.07) < 0.005
    lag = int(round(1.2 / 0.1))
    a, b = f[:, :-lag] - f.mean(axis=0)[:-lag], f[:, lag:] - f.mean(axis=0)[lag:]
    corr = np.mean(a * b) / math.sqrt(np.mean(a * a) * np.mean(b * b))
    assert abs(corr - math.exp(-0.5)) < 0.05
    assert neg.sum() < 1e-4 * f.size + 1                     # SPEC.md:265 (negativity negligible)


def test_normalize_identities():
    raw = np.full((1, 100), 0.07)
    np.testing.assert_allclose(O.normalize_source(10.0, 100, raw), 0.1, rtol=1e-14)
    f, _, _ = O.grf_sample(10.0, 100, PAPER, 8)
    s = O.normalize_source(10.0, 100, f)
    np.testing.assert_allclose(s.sum(axis=1) * 0.1, 1.0, atol=1e-12)
    np.testing.assert_allclose(O.normalize_source(10.0, 100, 5.0 * f), s, rtol=1e-15)
    with pytest.raises(O.OracleError):
        O.normalize_source(10.0, 100, -f)


def test_oracle_dataset_balance_and_determinism():
    n, order = 100, 8
    S, phi, it = O.generate_dataset(10.0, n, order, PAPER, 40, 1.0, 0.5, 1e-10)
    S2, phi2, it2 = O.generate_dataset(10.0, n, order, PAPER, 40, 1.0, 0.5, 1e-10, n_threads=3)
    assert np.array_equal(S, S2) and np.array_equal(phi, phi2) and np.array_equal(it, it2)
    cfg = O.make_config(1e-10)
    st, ss = np.full((40, n), 1.0), np.full((40, n), 0.5)
    r = O.source_iteration(10.0, n, order, st, ss, S, cfg, initial_phi=phi, want_leak=True)
    for b in range(40):
        res = O.balance_residual(10.0, n, st[b], ss[b], S[b], r["phi"][b], *r["leak"][b])
        assert res < 1e-8


def test_degenerate_dataset_is_uniform_solve():
    sp = snop.GrfSpec(0.07, 1e-18, 1.2, 1e-10, 9)
    S, phi, _ = O.generate_dataset(10.0, 50, 8, sp, 1, 1.0, 0.5, 1e-10)
    cfg = O.make_config(1e-10)
    r = O.source_iteration(10.0, 50, 8, np.ones((1, 50)), np.full((1, 50), 0.5), np.full((1, 50), 0.1), cfg)
    assert np.max(np.abs(phi - r["phi"])) / np.max(r["phi"]) < 1e-7


def test_dataset_file_roundtrip(tmp_path):
    n = 64
    S, phi, it = O.generate_dataset(10.0, n, 8, PAPER, 5, 1.0, 0.5, 1e-8)
    ds = snop.TrainingDataset(S, phi, it, snop.Grid1D(10.0, n), 8, PAPER, (1.0, 0.5), 1e-8)
    p = tmp_path / "ds.bin"
    snop.save_dataset(p, ds)
    back = snop.load_dataset(p)
    assert np.array_equal(back.sources, S) and np.array_equal(back.fluxes, phi)
    assert back.grid == ds.grid and back.spec == PAPER and back.reference_params == (1.0, 0.5)
    assert back.order == 8 and back.tolerance == 1e-8
    manifest = (tmp_path / "ds.bin.txt").read_text()
    assert "n_samples = 5" in manifest and "grf_seed = 2024" in manifest
    raw = p.read_bytes()
    assert len(raw) == 4 + 12 + 4 + 8 + 8 + 8 + 4 + 8 * 4 + 8 + 8 * 3 + 2 * 8 * 5 * n + 8
    for bad in (raw[:-1], raw[: len(raw) // 2], raw[:100] + bytes([raw[100] ^ 1]) + raw[101:]):
        p.write_bytes(bad)
        with pytest.raises(IoError):
            snop.load_dataset(p)


# ---------------------------------------------------------------- device --------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("n,count,first", [(100, 64, 0), (2000, 9, 77), (33, 5, 3)])
def test_gpu_grf_sample_parity(n, count, first):
    f, neg = snop.sample_grf(snop.Grid1D(10.0, n), PAPER, count, first, with_negatives=True)
    o, oneg, _ = O.grf_sample(10.0, n, PAPER, count, first)
    assert np.max(np.abs(f - o)) < 1e-13
    assert np.array_equal(neg, oneg)
    d = snop.sample_grf(snop.Grid1D(10.0, n), PAPER, count, first, device=True)
    assert np.array_equal(d.cpu().numpy(), f)


@pytest.mark.gpu
def test_gpu_normalize_parity_and_error():
    o, _, _ = O.grf_sample(10.0, 100, PAPER, 16)
    s = snop.normalize_source(snop.Grid1D(10.0, 100), o)
    assert np.max(np.abs(s - O.normalize_source(10.0, 100, o))) < 1e-14
    bad = o.copy()
    bad[3] *= -1.0
    with pytest.raises(InvalidArgument, match="sample 3"):
        snop.normalize_source(snop.Grid1D(10.0, 100), bad)


@pytest.mark.gpu
def test_gpu_generate_dataset_parity():
    n, order, count = 100, 16, 96
    ds = snop.generate_dataset(count, PAPER, snop.Grid1D(10.0, n), order, (1.0, 0.5), 1e-8)
    S, phi, it = O.generate_dataset(10.0, n, order, PAPER, count, 1.0, 0.5, 1e-8)
    assert np.max(np.abs(ds.sources - S)) / np.max(S) < 1e-13
    assert np.max(np.abs(ds.iterations - it)) <= 1
    same = ds.iterations == it
    assert same.mean() > 0.9
    assert np.max(np.abs(ds.fluxes[same] - phi[same])) / np.max(phi) < 1e-10
