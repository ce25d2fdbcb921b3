"""The reference's per-step functions (fastfca.hpp:28-53) through the Python
mirror of the C-ABI (csrc/steps.cu), checked against closed forms written out
in numpy (the checker) -- the same identities test_fastfca.cpp:84-209 uses.
The C++ port of those tests, with the oracle side by side, is
tests/cpp/test_steps_gpu.cpp."""
import numpy as np
import pytest

from paper_2101_08563_b200 import api

pytestmark = pytest.mark.gpu


def crandn(rng, shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2.0)


def positive(rng, shape, lo=0.2, hi=2.0):
    return np.exp(rng.uniform(np.log(lo), np.log(hi), shape))


def covs_of(x):
    return api.sample_covs(api.Spectrogram(x))


def test_weighted_cov_matches_the_definition(gpu):
    rng = np.random.default_rng(1)
    for M, T in [(1, 50), (3, 60), (8, 700)]:
        x = crandn(rng, (2, M, T))
        covs = covs_of(x)
        sig = positive(rng, T)
        q = api.weighted_cov(covs, 1, sig)
        ref = (x[1] / sig) @ x[1].conj().T / T
        assert np.linalg.norm(q - ref) <= 1e-13 * np.linalg.norm(ref)
        assert np.array_equal(q, q.conj().T)
    # block covariances (fastfca.cpp:29-32)
    mats = crandn(rng, (1, 9, 3, 3))
    mats = mats @ np.swapaxes(mats.conj(), -1, -2)
    cb = api.SampleCovSet(mats=mats, block_size=4, frames=36)
    sig = positive(rng, 9)
    q = api.weighted_cov(cb, 0, sig)
    ref = (mats[0] / sig[:, None, None]).sum(0) / 9
    assert np.linalg.norm(q - ref) <= 1e-13 * np.linalg.norm(ref)


def test_ip_update_w_normalises_each_column(gpu):
    """w_m^H Q_m w_m = 1 and (W^H Q_m) w_m = e_m after a sweep (fastfca.cpp:47-60)."""
    rng = np.random.default_rng(2)
    for M, N, T in [(1, 1, 50), (2, 3, 80), (4, 2, 120), (8, 12, 900)]:
        x = crandn(rng, (3, M, T))
        covs = covs_of(x)
        W0 = np.eye(M) + 0.5 * crandn(rng, (M, M))
        L, H = positive(rng, (M, N), 0.3, 3.0), positive(rng, (N, T), 0.3, 3.0)
        W = api.ip_update_w(covs, 2, W0, L, H)
        eps = max(1e-8 * covs.power(2), 1e-300)
        sig = L @ H + eps
        Wseq = W0.copy()
        for m in range(M):
            q = api.weighted_cov(covs, 2, sig[m])
            a = Wseq.conj().T @ q
            e = np.zeros(M); e[m] = 1.0
            wm = np.linalg.solve(a, e)
            wm = wm / np.sqrt((wm.conj() @ q @ wm).real)
            Wseq[:, m] = wm
            assert abs((W[:, m].conj() @ q @ W[:, m]).real - 1.0) <= 1e-10
        assert np.linalg.norm(W - Wseq) <= 1e-9 * np.linalg.norm(Wseq)


def test_ip_update_w_singular_raises(gpu):
    x = np.zeros((1, 2, 20), np.complex128)
    covs = api.SampleCovSet(snapshots=x, power_scale=np.zeros(1))
    with pytest.raises(api.NumericalError, match="ip_update_w: singular system for column 0"):
        api.ip_update_w(covs, 0, np.eye(2), np.ones((2, 1)), np.ones((1, 20)))


def test_source_gains_partition_to_one(gpu):
    rng = np.random.default_rng(3)
    L, H = positive(rng, (4, 3)), positive(rng, (3, 9))
    tot = sum(api.source_gain(L, H, n) for n in range(3))
    assert np.abs(tot - 1.0).max() < 1e-12
    g1 = api.source_gain(L, H, 1)
    assert np.allclose(g1, np.outer(L[:, 1], H[1]) / (L @ H), rtol=1e-13)


def test_em_update_lh_closed_forms(gpu):
    L, H = api.em_update_lh(np.array([[3.4]]), np.array([[0.7]]), np.array([[1.9]]))
    assert abs(L[0, 0] - 3.4 / 1.9) <= 1e-12 and abs(H[0, 0] - 1.9) <= 1e-12
    rng = np.random.default_rng(4)
    L0, H0 = positive(rng, (3, 1)), positive(rng, (1, 7))
    u = L0 @ H0
    L, H = api.em_update_lh(u, L0, H0)
    assert np.abs(L @ H - u).max() < 1e-10 * u.max()
    # one sweep of the sequential update written out (fastfca.cpp:84-98)
    M, N, T = 4, 3, 50
    u, L0, H0 = positive(rng, (M, T), 0.05, 20.0), positive(rng, (M, N)), positive(rng, (N, T))
    Lr, Hr = L0.copy(), H0.copy()
    for n in range(N):
        lh = Lr @ Hr + 1e-3
        ln = np.outer(Lr[:, n], Hr[n])
        g = ln / lh
        phi = g * g * u + (1 - g) * ln
        Lr[:, n] = np.maximum((phi / Hr[n]).sum(1) / T, 1e-300)
        Hr[n] = np.maximum((phi / Lr[:, n][:, None]).sum(0) / M, 1e-300)
    L, H = api.em_update_lh(u, L0, H0, True, 1e-3)
    assert np.allclose(L, Lr, rtol=1e-12) and np.allclose(H, Hr, rtol=1e-12)
    L, H = api.em_update_lh(u, L0, H0, False, 1e-3)
    assert np.array_equal(L, L0)


def test_mm_update_lh_fixed_point_and_recurrence(gpu):
    rng = np.random.default_rng(5)
    L0, H0 = positive(rng, (3, 2)), positive(rng, (2, 8))
    L, H = api.mm_update_lh(L0 @ H0, L0, H0)
    assert np.abs(L - L0).max() < 1e-12 * L0.max() and np.abs(H - H0).max() < 1e-12 * H0.max()
    u, L, H = np.array([[2.0]]), np.array([[0.4]]), np.array([[1.1]])
    l, h = 0.4, 1.1
    for _ in range(4):
        L, H = api.mm_update_lh(u, L, H)
        l = l * np.sqrt(2.0 / (l * h))
        h = h * np.sqrt(2.0 / (l * h))
        assert abs(L[0, 0] - l) <= 1e-12 and abs(H[0, 0] - h) <= 1e-12


def test_log_abs_det2(gpu):
    rng = np.random.default_rng(6)
    for M in (1, 2, 5, 8):
        W = np.eye(M) + 0.5 * crandn(rng, (M, M))
        assert abs(api.log_abs_det2(W) - 2.0 * np.linalg.slogdet(W)[1]) <= 1e-12
    with pytest.raises(api.NumericalError, match="singular decorrelation matrix"):
        api.log_abs_det2(np.zeros((3, 3)))
