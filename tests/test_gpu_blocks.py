"""Block-stationary input (SampleCovSet with block_size B > 1) on the GPU
against the fp64 oracle: sample_covs / piecewise_prepare (sigmodel.cpp:17-48),
the mats branches of weighted_cov and decorrelated_powers (fastfca.cpp:29-32,
sigmodel.cpp:97-105) inside fastfca_fit / ica_mode_fit, fastfca_nll, and
expand_block_params + fastfca_separate (sigmodel.cpp:164-196).

Tolerances as tests/test_gpu_parity.py: fp32 NLL trace 1e-5 relative, fp64
1e-10; block covariances 1e-12 (fp64 arithmetic on both sides).
"""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_2101_08563_b200 import _lib, api, synth

pytestmark = pytest.mark.gpu

NLL_TOL = {"fp32": 1e-5, "fp64": 1e-10}


def make_case(M, N, F, T, B, seed=0, kind="jd"):
    cfg = synth.small(M, N, F, T, seed=seed, kind=kind)
    x = synth.mixture(cfg).astype(np.complex128)
    W, L, _ = synth.init_params(cfg)
    J = -(-T // B)
    H = np.random.default_rng(seed + 1).lognormal(0.0, 1.0, (F, N, J))
    return x, W, L, H


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - b) / np.abs(b)))


@pytest.mark.parametrize("B,T", [(4, 11), (3, 12), (12, 12), (7, 626), (1, 40)])
def test_sample_covs_blocks_match_oracle(gpu, B, T):
    x, _, _, _ = make_case(3, 2, 5, T, B, seed=B)
    covs = api.sample_covs(api.Spectrogram(x), B)
    mats_o, pow_o = oracle.block_covs(x, B)
    assert covs.blocks == -(-T // B) and covs.frames == T and covs.block_size == B
    np.testing.assert_allclose(covs.power_scale, pow_o, rtol=1e-13)
    if B == 1:
        assert covs.has_snapshots()
        return
    assert not covs.has_snapshots()
    err = np.abs(covs.mats - mats_o).max() / np.abs(mats_o).max()
    assert err < 1e-12
    # every block is Hermitian (the ragged tail averages over its own width)
    assert np.abs(covs.mats - np.conj(np.swapaxes(covs.mats, -1, -2))).max() == 0.0


CASES = [  # M, N, F, T, B, iters, flavor, kind
    (2, 3, 8, 626, 4, 40, 0, "jd"),
    (2, 2, 6, 1250, 10, 50, 0, "jd"),
    (3, 4, 6, 626, 3, 30, 0, "jd"),
    (4, 6, 4, 2000, 8, 20, 0, "fullrank"),
    (2, 3, 6, 400, 4, 25, 1, "jd"),
    (1, 2, 4, 300, 5, 15, 0, "jd"),
    (5, 3, 3, 500, 5, 10, 0, "jd"),
    (8, 12, 2, 960, 8, 6, 0, "jd"),
]


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: "M{}N{}T{}B{}fl{}".format(c[0], c[1], c[3],
                                                                               c[4], c[6]))
def test_block_fit_nll_trace_matches_oracle(gpu, case, precision):
    M, N, F, T, B, iters, flavor, kind = case
    x, W, L, H = make_case(M, N, F, T, B, seed=10 * M + N, kind=kind)
    covs = api.sample_covs(api.Spectrogram(x), B)
    r = api.fastfca_fit(covs, api.FastFcaParams(W, L, H), flavor, iters, precision=precision)
    mats_o, pow_o = oracle.block_covs(x, B)
    Wo, Lo, Ho, nll_o, _ = oracle.fit_covs(mats_o, W, L, H, iters, flavor=flavor, power=pow_o)
    assert rel(r.nll, nll_o) <= NLL_TOL[precision]
    assert (r.bin_status == 0).all()
    if precision == "fp64":
        assert rel(r.params.loading, Lo) < 1e-8
        np.testing.assert_allclose(r.params.decorr, Wo, rtol=0, atol=1e-8 * np.abs(Wo).max())


def diagonal_covset(dim, frames, rng):
    """test_fastfca.cpp:63-78: one bin of diagonal block covariances, no power_scale."""
    d = 0.2 + np.abs(rng.standard_normal((frames, dim)))
    mats = np.zeros((1, frames, dim, dim), np.complex128)
    for k in range(dim):
        mats[0, :, k, k] = d[:, k]
    return api.SampleCovSet(None, None, dim, mats, frames=frames)


def test_caller_built_set_without_power_scale(gpu):
    rng = np.random.default_rng(63)
    covs = diagonal_covset(3, 40, rng)
    W = np.eye(3, dtype=np.complex128)[None] + 0.05 * rng.standard_normal((1, 3, 3))
    L = rng.uniform(0.5, 2.0, (1, 3, 2))
    H = rng.uniform(0.5, 2.0, (1, 2, 40))
    r = api.fastfca_fit(covs, api.FastFcaParams(W, L, H), api.LhFlavor.em, 12, precision="fp64")
    Wo, Lo, Ho, nll_o, _ = oracle.fit_covs(covs.mats, W, L, H, 12, power=None)
    assert rel(r.nll, nll_o) <= 1e-10
    assert abs(covs.power(0) - np.trace(covs.mats[0], axis1=-2, axis2=-1).real.mean() / 3) < 1e-15


def test_ica_mode_keeps_diagonal_blocks(gpu):
    # test_fastfca.cpp:493-502 on the GPU.
    covs = diagonal_covset(2, 30, np.random.default_rng(78))
    r = api.ica_mode_fit(covs, 2, 10, np.eye(2, dtype=np.complex128)[None])
    w = r.params.decorr[0]
    assert abs(w[0, 1]) < 1e-12 and abs(w[1, 0]) < 1e-12
    Wo, Lo, Ho, nll_o = oracle.ica_fit_covs(covs.mats, np.eye(2, dtype=np.complex128)[None], 10)
    assert rel(r.nll, nll_o) <= 1e-10
    np.testing.assert_allclose(r.params.act, Ho, rtol=1e-10)


def test_ica_mode_on_blocks_matches_oracle(gpu):
    x, _, _, _ = make_case(3, 3, 4, 600, 6, seed=5)
    covs = api.sample_covs(api.Spectrogram(x), 6)
    w0 = np.tile(np.eye(3, dtype=np.complex128), (4, 1, 1))
    r = api.ica_mode_fit(covs, 3, 20, w0)
    Wo, Lo, Ho, nll_o = oracle.ica_fit_covs(covs.mats, w0, 20, power=covs.power_scale)
    assert rel(r.nll, nll_o) <= 1e-10


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_block_nll_and_powers_match_oracle(gpu, precision):
    x, W, L, H = make_case(4, 3, 5, 240, 4, seed=3)
    covs = api.sample_covs(api.Spectrogram(x), 4)
    p = api.FastFcaParams(W, L, H)
    nb = api.fastfca_nll_bins(covs, p, precision=precision)
    assert rel(nb, oracle.nll_bins_covs(covs.mats, W, L, H)) <= NLL_TOL[precision]
    u = api.decorrelated_powers(covs, W, precision="fp64")
    uo = oracle.decorrelated_powers_covs(covs.mats, W, floor_rel=None)
    assert np.abs(u - uo).max() <= 1e-12 * np.abs(uo).max()


def test_rank_one_blocks_reproduce_snapshot_fit(gpu):
    # B = 1 block covariances x x^H carry the same statistics as the
    # snapshots: the two GPU paths agree to fp64 rounding.
    x, W, L, H = make_case(2, 3, 4, 300, 1, seed=9)
    snap = api.sample_covs(api.Spectrogram(x))
    mats = np.einsum("fmt,fnt->ftmn", x, np.conj(x))
    blk = api.SampleCovSet(None, snap.power_scale, 1, mats, frames=300)
    p = api.FastFcaParams(W, L, H)
    a = api.fastfca_fit(snap, p, api.LhFlavor.em, 20, precision="fp64")
    b = api.fastfca_fit(blk, p, api.LhFlavor.em, 20, precision="fp64")
    assert rel(b.nll, np.asarray(a.nll)) <= 1e-10


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_expand_block_params_then_separate(gpu, precision):
    M, N, F, T, B = 2, 3, 6, 500, 5
    x, W, L, H = make_case(M, N, F, T, B, seed=4)
    covs = api.sample_covs(api.Spectrogram(x), B)
    r = api.fastfca_fit(covs, api.FastFcaParams(W, L, H), api.LhFlavor.em, 20, precision=precision)
    full = api.expand_block_params(r.params, B, T)
    assert full.frames == T
    assert np.array_equal(full.act[:, :, 7], r.params.act[:, :, 1])
    img = api.fastfca_separate(api.Spectrogram(x), full, precision=precision)
    Wo, Lo, Ho, _, _ = oracle.fit_covs(covs.mats, W, L, H, 20, power=covs.power_scale)
    Ho_full = Ho[:, :, np.minimum(np.arange(T) // B, Ho.shape[2] - 1)]
    img_o = oracle.separate(x, Wo, Lo, Ho_full)
    tol = 1e-3 if precision == "fp32" else 1e-9
    for n in range(N):
        e = np.linalg.norm(img[n].f - img_o[n]) / np.linalg.norm(img_o[n])
        assert e <= tol


def test_device_block_path_matches_host_path(gpu):
    """ffca_block_covs_device + ffca_fit_covs_device (device-resident inputs)
    give the host path's results bit for bit on complex64-exact inputs."""
    import torch
    M, N, F, T, B, iters = 3, 4, 6, 626, 4, 25
    x, W, L, H = make_case(M, N, F, T, B, seed=2)
    covs = api.sample_covs(api.Spectrogram(x), B)
    host = api.fastfca_fit(covs, api.FastFcaParams(W, L, H), api.LhFlavor.em, iters)
    J = covs.blocks
    dev = torch.device("cuda", 0)
    xd = torch.from_numpy(np.ascontiguousarray(np.swapaxes(x, -1, -2))).to(dev, torch.complex64)
    rec = torch.empty((F, J, M * M), dtype=torch.float32, device=dev)
    pw = torch.empty(F, dtype=torch.float64, device=dev)
    Wd = torch.from_numpy(np.ascontiguousarray(np.swapaxes(W, -1, -2))).to(dev)
    Ld = torch.from_numpy(np.ascontiguousarray(np.swapaxes(L, -1, -2))).to(dev)
    Hd = torch.from_numpy(np.ascontiguousarray(np.swapaxes(H, -1, -2))).to(dev, torch.float32)
    slots = torch.zeros((iters + 1, F), dtype=torch.float64, device=dev)
    st = torch.zeros(F, dtype=torch.int32, device=dev)
    ctx = _lib.context(0)
    Lb = _lib.lib()
    _lib.check(Lb.ffca_block_covs_device(ctx.handle, F, M, T, B, _lib.PREC_FP32, _lib.ptr(xd),
                                         _lib.ptr(rec), _lib.ptr(pw), None))
    o = _lib.FitOpts(_lib.FLAVOR_EM, iters, 1, 0, 1, 0, _lib.PREC_FP32)
    _lib.check(Lb.ffca_fit_covs_device(ctx.handle, F, F, 0, M, N, J, o, _lib.ptr(rec),
                                       _lib.ptr(pw), _lib.ptr(Wd), _lib.ptr(Ld), _lib.ptr(Hd),
                                       _lib.ptr(slots), _lib.ptr(st), None))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(pw.cpu().numpy(), covs.power_scale)
    nll_dev = slots.cpu().numpy().sum(axis=1)
    assert rel(nll_dev, np.asarray(host.nll)) <= 1e-12
    np.testing.assert_array_equal(np.swapaxes(Ld.cpu().numpy(), -1, -2), host.params.loading)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_block_fit_streaming_bin_matches_oracle(gpu, precision):
    # 2000 blocks of M = 4 records (240 KB per bin) exceed one CTA's shared
    # memory: the block path streams its records from global memory.
    M, N, F, T, B, iters = 4, 6, 2, 4000, 2, 5
    x, W, L, H = make_case(M, N, F, T, B, seed=31, kind="fullrank")
    covs = api.sample_covs(api.Spectrogram(x), B)
    assert covs.blocks == 2000
    r = api.fastfca_fit(covs, api.FastFcaParams(W, L, H), api.LhFlavor.em, iters,
                        precision=precision)
    Wo, Lo, Ho, nll_o, _ = oracle.fit_covs(covs.mats, W, L, H, iters, power=covs.power_scale)
    assert rel(r.nll, nll_o) <= NLL_TOL[precision]
