"""Determined ICA mode (ica_mode_fit, fastfca.cpp:241-264) and
decorrelated_powers (sigmodel.cpp:93-107) on the GPU against the fp64 oracle.

ICA mode is FastFCA with N = M, L fixed at the identity (one-hot loadings with
exact zeros) and H initialised to the floored decorrelated powers of W_init
(pinned by test_fastfca.cpp:452-502, whose first case is
ported in oracle/kat_tests.cpp)."""
import numpy as np
import pytest

import oracle
from paper_2101_08563_b200 import api
from paper_2101_08563_b200._lib import InvalidArgument

pytestmark = pytest.mark.gpu

NLL_TOL = {"fp32": 1e-5, "fp64": 1e-10}


def determined_mixture(M, F, T, seed, rho=0.97, scale=1.5):
    """Instantaneous M x M mixture of M sources with smooth AR(1) log-powers
    (the variance diversity the determined-mode likelihood needs)."""
    rng = np.random.default_rng(seed)
    A = np.eye(M) + 0.6 * (rng.standard_normal((F, M, M)) + 1j * rng.standard_normal((F, M, M))) / np.sqrt(2)
    x = np.empty((F, M, T), np.complex128)
    for f in range(F):
        logh = np.empty((M, T))
        state = rng.standard_normal(M)
        for t in range(T):
            state = rho * state + np.sqrt(1 - rho * rho) * rng.standard_normal(M)
            logh[:, t] = scale * state
        z = (rng.standard_normal((M, T)) + 1j * rng.standard_normal((M, T))) / np.sqrt(2)
        x[f] = A[f] @ (np.exp(0.5 * logh) * z)
    return x.astype(np.complex64).astype(np.complex128), A


def leak(W, A):
    tot = 0.0
    for f in range(W.shape[0]):
        e = np.abs(W[f].conj().T @ A[f]) ** 2
        M = e.shape[0]
        if M == 2:
            direct = max(e[0, 0] + e[1, 1], e[0, 1] + e[1, 0])
        else:  # best assignment by greedy row maxima (good enough for a bound)
            direct = sum(e[r].max() for r in range(M))
        tot += 1.0 - direct / e.sum()
    return tot / W.shape[0]


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("floor", [None, 1e-12, 1e-3])
def test_decorrelated_powers_matches_oracle(gpu, precision, floor):
    x, _ = determined_mixture(3, 5, 300, seed=1)
    rng = np.random.default_rng(2)
    W = np.eye(3) + 0.3 * (rng.standard_normal((5, 3, 3)) + 1j * rng.standard_normal((5, 3, 3)))
    covs = api.sample_covs(api.Spectrogram(x))
    got = api.decorrelated_powers(covs, W, floor_rel=floor, precision=precision)
    want = oracle.decorrelated_powers(x, W, floor_rel=floor)
    tol = 1e-12 if precision == "fp64" else 2e-5
    np.testing.assert_allclose(got, want, rtol=tol, atol=tol * want.max())


# precision="fp32" is accepted but the mode always runs the fp64 kernels
# (ffca.h: the determined-mode fixed point amplifies fp32 cancellation), so
# both requests must match the oracle at the fp64 tolerance.
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("M,F,T,iters", [(2, 4, 600, 80), (3, 3, 500, 30)])
def test_ica_mode_fit_matches_oracle(gpu, precision, M, F, T, iters):
    x, A = determined_mixture(M, F, T, seed=10 + M)
    covs = api.sample_covs(api.Spectrogram(x))
    w_init = np.tile(np.eye(M, dtype=np.complex128), (F, 1, 1))
    r = api.ica_mode_fit(covs, M, iters, w_init, precision=precision)
    Wo, Lo, Ho, nll_o = oracle.ica_fit(x, w_init, iters)
    nll_g = np.asarray(r.nll)
    rel = np.abs(nll_g - nll_o) / np.abs(nll_o)
    assert rel.max() <= NLL_TOL["fp64"], (rel.max(), int(rel.argmax()))
    # fastfca.cpp:257: the loadings stay the identity, exact zeros included.
    assert np.array_equal(r.params.loading, np.tile(np.eye(M), (F, 1, 1)))
    assert (np.diff(nll_g) <= 1e-6 * np.abs(nll_g[:-1])).all()
    if M == 2:  # test_fastfca.cpp:484-491: the mixture is unmixed
        assert leak(r.params.decorr, A) <= 0.05


def test_ica_mode_zero_iterations_returns_floored_powers(gpu):
    x, _ = determined_mixture(2, 3, 200, seed=5)
    covs = api.sample_covs(api.Spectrogram(x))
    w_init = np.tile(np.eye(2, dtype=np.complex128), (3, 1, 1))
    r = api.ica_mode_fit(covs, 2, 0, w_init, precision="fp64")
    _, _, Ho, nll_o = oracle.ica_fit(x, w_init, 0)
    np.testing.assert_allclose(r.params.act, Ho, rtol=1e-12)
    assert np.array_equal(r.params.decorr, w_init)
    assert len(r.nll) == 1 and abs(r.nll[0] - nll_o[0]) <= 1e-10 * abs(nll_o[0])


def test_ica_mode_separation_with_zero_gains(gpu):
    # One-hot loadings give exactly-zero Wiener gains for the other channels
    # (SURVEY §8(f) #2); the images still partition the mixture.
    x, _ = determined_mixture(2, 4, 400, seed=8)
    covs = api.sample_covs(api.Spectrogram(x))
    w_init = np.tile(np.eye(2, dtype=np.complex128), (4, 1, 1))
    r = api.ica_mode_fit(covs, 2, 20, w_init, precision="fp64")
    imgs = api.fastfca_separate(api.Spectrogram(x), r.params, precision="fp64")
    want = oracle.separate(x, r.params.decorr, r.params.loading, r.params.act)
    for n in range(2):
        np.testing.assert_allclose(imgs[n].f, want[n], rtol=1e-10, atol=1e-12)
    # Sum of gains is LH / max(LH, 1e-12 mean LH) (floor_positive): 1 except
    # where some H(m, t) falls under the floor, which ICA mode's H = |w^H x|^2
    # fixed point does reach -- so the partition holds to that level only.
    total = sum(img.f for img in imgs)
    assert np.linalg.norm(total - x) <= 1e-7 * np.linalg.norm(x)


def test_ica_mode_rejects_source_count(gpu):
    # fastfca.cpp:244-246 (test_fastfca.cpp:493-494)
    x, _ = determined_mixture(2, 2, 50, seed=3)
    covs = api.sample_covs(api.Spectrogram(x))
    w_init = np.tile(np.eye(2, dtype=np.complex128), (2, 1, 1))
    with pytest.raises(InvalidArgument):
        api.ica_mode_fit(covs, 3, 1, w_init)
    with pytest.raises(InvalidArgument):
        api.ica_mode_fit(covs, 2, 1, w_init[:1])
