"""GPU parity against the fp64 oracle (the CUDA path through the C-ABI).

Tolerances (BASELINE.json north_star):
  fp32 path : per-iteration NLL within 1e-5 relative; separated STFTs within
              1e-3 relative L2 after the configured iterations.
  fp64 mode : 1e-10 for both.
Inputs are seeded synthetic mixtures rounded to complex64; the oracle sees the
same values promoted to double.
"""
import numpy as np
import pytest

import oracle
from paper_2101_08563_b200 import api, synth
from paper_2101_08563_b200._lib import InvalidArgument, NumericalError

pytestmark = pytest.mark.gpu

NLL_TOL = {"fp32": 1e-5, "fp64": 1e-10}
SEP_TOL = {"fp32": 1e-3, "fp64": 1e-10}


def make_case(M, N, F, T, seed=0, kind="jd", sigma_v=1.5):
    cfg = synth.small(M, N, F, T, seed=seed, kind=kind, sigma_v=sigma_v)
    x = synth.mixture(cfg).astype(np.complex128)
    W, L, H = synth.init_params(cfg)
    return x, W, L, H


def gpu_fit(x, W, L, H, iters, precision, flavor=0, **kw):
    covs = api.sample_covs(api.Spectrogram(x))
    init = api.FastFcaParams(W, L, H)
    fo = api.FitOptions(record_trace=kw.pop("record_trace", True), seed=kw.pop("seed", 0))
    oo = api.FastFcaOptions(**kw)
    return api.fastfca_fit(covs, init, flavor, iters, fo, oo, precision=precision)


def rel_l2(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


CASES = [
    # M, N, F, T, iters, kind
    (2, 3, 16, 626, 50, "jd"),      # config 0 shape, fewer bins
    (2, 2, 8, 1250, 100, "jd"),     # config 1 shape
    (3, 4, 8, 626, 50, "jd"),       # config 4 mixture shape
    (4, 6, 6, 2000, 30, "fullrank"),  # config 2 shape (silent frames)
    (1, 2, 5, 300, 20, "jd"),
    (5, 3, 3, 500, 10, "jd"),
    (8, 12, 2, 1200, 8, "jd"),      # config 3 channel/source counts, fewer frames
]


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: "M{}N{}F{}T{}".format(*c[:4]))
def test_fit_nll_trace_matches_oracle(gpu, case, precision):
    M, N, F, T, iters, kind = case
    x, W, L, H = make_case(M, N, F, T, seed=M * 100 + N, kind=kind)
    r = gpu_fit(x, W, L, H, iters, precision)
    Wo, Lo, Ho, nll_o, _, _ = oracle.fit(x, W, L, H, iters)
    nll_g = np.asarray(r.nll)
    assert nll_g.shape == nll_o.shape
    rel = np.abs(nll_g - nll_o) / np.abs(nll_o)
    assert rel.max() <= NLL_TOL[precision], (rel.max(), int(rel.argmax()))
    assert (r.bin_status == 0).all()


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_fit_then_separate_matches_oracle(gpu, precision):
    M, N, F, T, iters = 2, 3, 12, 626, 50
    x, W, L, H = make_case(M, N, F, T, seed=7)
    r = gpu_fit(x, W, L, H, iters, precision)
    Wo, Lo, Ho, _, _, _ = oracle.fit(x, W, L, H, iters)
    img_g = api.fastfca_separate(api.Spectrogram(x), r.params, precision=precision)
    img_o = oracle.separate(x, Wo, Lo, Ho)
    for n in range(N):
        assert rel_l2(img_g[n].f, img_o[n]) <= SEP_TOL[precision]


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("M,N", [(1, 1), (2, 3), (3, 4), (4, 6), (8, 12)])
def test_separate_matches_oracle_same_params(gpu, precision, M, N):
    x, W, L, H = make_case(M, N, 4, 300, seed=11)
    rng = np.random.default_rng(5)
    W = W + 0.3 * (rng.standard_normal(W.shape) + 1j * rng.standard_normal(W.shape))
    L = np.exp(rng.standard_normal(L.shape))
    img_g = api.fastfca_separate(api.Spectrogram(x), api.FastFcaParams(W, L, H),
                                 precision=precision)
    img_o = oracle.separate(x, W, L, H)
    for n in range(N):
        assert rel_l2(img_g[n].f, img_o[n]) <= SEP_TOL[precision]
    # test_fastfca.cpp:342-359: the images partition the mixture.
    total = sum(img.f for img in img_g)
    assert rel_l2(total, x) <= (1e-5 if precision == "fp32" else 1e-12)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_nll_bins_matches_oracle(gpu, precision):
    x, W, L, H = make_case(3, 2, 6, 400, seed=3)
    covs = api.sample_covs(api.Spectrogram(x))
    got = api.fastfca_nll_bins(covs, api.FastFcaParams(W, L, H), precision=precision)
    want = oracle.nll_bins(x, W, L, H)
    assert np.max(np.abs(got - want) / np.abs(want)) <= NLL_TOL[precision]


def test_power_scale_matches_oracle(gpu):
    x, *_ = make_case(3, 2, 6, 400, seed=3)
    covs = api.sample_covs(api.Spectrogram(x))
    np.testing.assert_allclose(covs.power_scale, oracle.power_scale(x), rtol=1e-13)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_mm_flavor_matches_oracle(gpu, precision):
    x, W, L, H = make_case(3, 3, 6, 500, seed=21)
    r = gpu_fit(x, W, L, H, 30, precision, flavor=1)
    _, _, _, nll_o, _, _ = oracle.fit(x, W, L, H, 30, flavor=1)
    rel = np.abs(np.asarray(r.nll) - nll_o) / np.abs(nll_o)
    assert rel.max() <= NLL_TOL[precision]


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_fix_loadings_and_no_normalize(gpu, precision):
    x, W, L, H = make_case(2, 2, 4, 600, seed=4)
    for kw in ({"fix_loadings": True}, {"normalize_scales": False}):
        r = gpu_fit(x, W, L, H, 15, precision, **kw)
        _, _, _, nll_o, _, _ = oracle.fit(x, W, L, H, 15,
                                          normalize_scales=kw.get("normalize_scales", True),
                                          fix_loadings=kw.get("fix_loadings", False))
        rel = np.abs(np.asarray(r.nll) - nll_o) / np.abs(nll_o)
        assert rel.max() <= NLL_TOL[precision], kw


def test_zero_iterations_returns_init_bit_exactly(gpu):
    # test_fastfca.cpp:273-284
    x, W, L, H = make_case(2, 2, 2, 10, seed=71)
    r = gpu_fit(x, W, L, H, 0, "fp32")
    assert len(r.nll) == 1
    assert np.array_equal(r.params.decorr, W)
    assert np.array_equal(r.params.act, H)
    assert np.array_equal(r.params.loading, L)


def test_silent_band_keeps_init(gpu):
    # fastfca.cpp:165-170: power(i) <= 0 -> parameters stay at the init.
    x, W, L, H = make_case(2, 3, 4, 200, seed=9)
    x[2] = 0.0
    r = gpu_fit(x, W, L, H, 10, "fp32")
    assert r.bin_status[2] == 1
    assert np.array_equal(r.params.act[2], H[2])
    assert np.array_equal(r.params.decorr[2], W[2])
    Wo, Lo, Ho, nll_o, _, _ = oracle.fit(x, W, L, H, 10)
    rel = np.abs(np.asarray(r.nll) - nll_o) / np.abs(nll_o)
    assert rel.max() <= 1e-5


def test_record_trace_off_same_params(gpu):
    x, W, L, H = make_case(2, 2, 4, 300, seed=5)
    a = gpu_fit(x, W, L, H, 10, "fp64")
    b = gpu_fit(x, W, L, H, 10, "fp64", record_trace=False)
    assert b.nll == []
    np.testing.assert_array_equal(a.params.act, b.params.act)
    np.testing.assert_array_equal(a.params.decorr, b.params.decorr)


def test_returned_params_reproduce_last_trace_entry(gpu):
    # test_fastfca.cpp:245-246: fastfca_nll(returned params) == nll.back()
    x, W, L, H = make_case(3, 3, 4, 120, seed=69)
    r = gpu_fit(x, W, L, H, 50, "fp64")
    assert abs(oracle.nll_bins(x, r.params.decorr, r.params.loading, r.params.act).sum()
               - r.nll[-1]) <= 1e-10 * abs(r.nll[-1])


def test_trace_monotone(gpu):
    x, W, L, H = make_case(2, 3, 8, 626, seed=1)
    r = gpu_fit(x, W, L, H, 50, "fp32")
    nll = np.asarray(r.nll)
    assert (nll[1:] <= nll[:-1] + 1e-6 * np.abs(nll[:-1])).all()


def test_shape_errors_raise_invalid_argument(gpu):
    x, W, L, H = make_case(2, 2, 3, 50)
    covs = api.sample_covs(api.Spectrogram(x))
    with pytest.raises(InvalidArgument):
        api.fastfca_fit(covs, api.FastFcaParams(W[:2], L[:2], H[:2]), 0, 3)
    with pytest.raises(InvalidArgument):
        api.fastfca_separate(api.Spectrogram(x[:, :, :40]), api.FastFcaParams(W, L, H))
    with pytest.raises(InvalidArgument):
        api.sample_covs(api.Spectrogram(x), block_size=0)


def test_singular_init_raises_numerical_error(gpu):
    x, W, L, H = make_case(2, 2, 3, 50)
    W[1] = 0.0  # log_abs_det2 throws on a singular W (sigmodel.cpp:124-125)
    with pytest.raises(NumericalError):
        gpu_fit(x, W, L, H, 3, "fp32")


# Bins too large for one CTA's shared memory: frames split over a thread-block
# cluster (DSMEM reductions); config 3's M, N, T.
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("M,N,T,iters", [(8, 12, 8000, 3), (2, 3, 14000, 5), (4, 6, 6000, 4)])
def test_cluster_split_bins_match_oracle(gpu, precision, M, N, T, iters):
    x, W, L, H = make_case(M, N, 2, T, seed=17)
    r = gpu_fit(x, W, L, H, iters, precision)
    Wo, Lo, Ho, nll_o, _, _ = oracle.fit(x, W, L, H, iters)
    rel = np.abs(np.asarray(r.nll) - nll_o) / np.abs(nll_o)
    assert rel.max() <= NLL_TOL[precision], rel.max()
    img_g = api.fastfca_separate(api.Spectrogram(x), r.params, precision=precision)
    img_o = oracle.separate(x, Wo, Lo, Ho)
    for n in range(N):
        assert rel_l2(img_g[n].f, img_o[n]) <= SEP_TOL[precision]


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_pipelined_host_fit_matches_single_launch(gpu, precision, monkeypatch):
    # ffca_fit splits >= 256 bins into chunks on separate streams (transfers
    # overlap the fit); every bin's result must be bit-identical to one launch.
    x, W, L, H = make_case(2, 3, 300, 200, seed=5)
    monkeypatch.setenv("FFCA_FIT_CHUNKS", "1")
    a = gpu_fit(x, W, L, H, 8, precision)
    monkeypatch.setenv("FFCA_FIT_CHUNKS", "3")
    b = gpu_fit(x, W, L, H, 8, precision)
    assert np.array_equal(np.asarray(a.nll), np.asarray(b.nll))
    assert np.array_equal(a.params.act, b.params.act)
    assert np.array_equal(a.params.loading, b.params.loading)
    assert np.array_equal(a.params.decorr, b.params.decorr)
    Wo, Lo, Ho, nll_o, _, _ = oracle.fit(x, W, L, H, 8)
    assert (np.abs(np.asarray(b.nll) - nll_o) / np.abs(nll_o)).max() <= NLL_TOL[precision]


# A bin beyond a 16-CTA cluster's shared memory streams its records from
# global memory (the !RES variant).  M = 8 with N = 10 sources (N = 12 belongs
# to the large-bin kernel, tests/test_gpu_big.py) and T = 24000 frames.
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_streaming_bin_matches_oracle(gpu, precision):
    x, W, L, H = make_case(8, 10, 1, 24000, seed=23)
    r = gpu_fit(x, W, L, H, 2, precision)
    Wo, Lo, Ho, nll_o, _, _ = oracle.fit(x, W, L, H, 2)
    rel = np.abs(np.asarray(r.nll) - nll_o) / np.abs(nll_o)
    assert rel.max() <= NLL_TOL[precision], rel.max()


# Streaming bins through the pipelined host fit (FFCA_FIT_CHUNKS = 3 chunks
# on 3 streams): the chunks' kernels run concurrently, so each must work in
# its own rows of the one U/Phi scratch allocation.  Uneven chunks (7 bins).
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_streaming_bins_chunked_match_oracle(gpu, precision, monkeypatch):
    x, W, L, H = make_case(8, 10, 7, 24000, seed=29)
    monkeypatch.setenv("FFCA_FIT_CHUNKS", "3")
    r = gpu_fit(x, W, L, H, 2, precision)
    monkeypatch.delenv("FFCA_FIT_CHUNKS")
    r1 = gpu_fit(x[:1], W[:1], L[:1], H[:1], 2, precision)
    Wo, Lo, Ho, nll_o, slots_o, _ = oracle.fit(x, W, L, H, 2)
    rel = np.abs(np.asarray(r.nll) - nll_o) / np.abs(nll_o)
    assert rel.max() <= NLL_TOL[precision], rel.max()
    tol = 1e-9 if precision == "fp64" else 2e-3
    for f in range(7):
        e = np.linalg.norm(np.asarray(r.params.act[f]) - Ho[f]) / np.linalg.norm(Ho[f])
        assert e <= tol, (f, e)
    # a chunked bin equals the same bin fitted alone, bit for bit
    assert np.array_equal(np.asarray(r.params.act[0]), np.asarray(r1.params.act[0]))


# ffca_fit_bins: the fit on per-bin host buffers (the reference's containers),
# gathered into pinned staging on host threads and pipelined over bin chunks --
# the same bits as ffca_fit on the contiguous buffers.
@pytest.mark.parametrize("shape", [(2, 3, 9, 300), (8, 12, 6, 2500)])
def test_fit_bins_matches_contiguous_fit(gpu, shape):
    import ctypes as C
    from paper_2101_08563_b200 import _lib
    M, N, F, T = shape
    x, W, L, H = make_case(M, N, F, T, seed=61)
    x[1] = 0.0  # a silent bin keeps its init
    iters = 4
    r = gpu_fit(x, W, L, H, iters, "fp32")
    xb = [np.ascontiguousarray(x[f].T, np.complex128) for f in range(F)]          # [T][M]
    Wb = [np.ascontiguousarray(W[f].T, np.complex128) for f in range(F)]          # col-major
    Lb = [np.ascontiguousarray(L[f].T, np.float64) for f in range(F)]
    Hb = [np.ascontiguousarray(H[f].T, np.float64) for f in range(F)]            # [T][N]
    power = np.array([np.mean(np.abs(x[f]) ** 2) for f in range(F)])

    def ptrs(arrs):
        return (C.c_void_p * F)(*[a.ctypes.data for a in arrs])
    nll = np.zeros(iters + 1)
    status = np.zeros(F, np.int32)
    d = _lib.Dims(1, F, M, N, T)
    o = _lib.FitOpts(_lib.FLAVOR_EM, iters, 1, 0, 1, 0, _lib.PREC_FP32)
    pw, pl, ph = ptrs(Wb), ptrs(Lb), ptrs(Hb)
    _lib.check(_lib.lib().ffca_fit_bins(gpu.handle, d, o, ptrs(xb), None, pw, pl, ph, pw, pl, ph,
                                        _lib.ptr(nll), None, _lib.ptr(status), 3))
    assert np.array_equal(nll, np.asarray(r.nll))
    assert np.array_equal(status, r.bin_status)
    for f in range(F):
        assert np.array_equal(Hb[f].T, np.asarray(r.params.act[f])), f
        assert np.array_equal(Wb[f].T, np.asarray(r.params.decorr[f])), f
        assert np.array_equal(Lb[f].T, np.asarray(r.params.loading[f])), f
    del power
