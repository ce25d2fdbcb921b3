"""GPU parity of the large-bin fit kernel (csrc/fit_big.cuh: M = 8, N = 12,
BASELINE config 3's channel/source counts, and M = 4, N = 6, config 2's, in
fp32) against the fp64 oracle, through the C-ABI.  Frame counts are chosen so
the bin runs on one CTA and on clusters (M = 8: 4096 frames per CTA in fp32,
1792 in fp64; M = 4: 2048).

Tolerances (BASELINE.json north_star): fp32 NLL 1e-5 relative per iteration
and separated STFTs 1e-3 relative L2; fp64 check mode 1e-10 for both.
"""
import os

import numpy as np
import pytest

import oracle
from paper_2101_08563_b200 import api, synth

pytestmark = pytest.mark.gpu

NLL_TOL = {"fp32": 1e-5, "fp64": 1e-10}
SEP_TOL = {"fp32": 1e-3, "fp64": 1e-10}


def make_case(F, T, seed, sigma_v=2.0, M=8, N=12, kind="jd"):
    cfg = synth.small(M, N, F, T, seed=seed, sigma_v=sigma_v, kind=kind)
    x = synth.mixture(cfg).astype(np.complex128)
    W, L, H = synth.init_params(cfg)
    return x, W, L, H


def fit(x, W, L, H, iters, precision, **kw):
    covs = api.sample_covs(api.Spectrogram(x))
    fo = api.FitOptions(record_trace=kw.pop("record_trace", True), seed=kw.pop("seed", 0))
    oo = api.FastFcaOptions(**kw)
    return api.fastfca_fit(covs, api.FastFcaParams(W, L, H), api.LhFlavor.em, iters, fo, oo,
                           precision=precision)


def rel_l2(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("T", [700, 3000, 8000])
def test_big_fit_trace_and_separation(gpu, precision, T):
    iters = 5 if T == 8000 else 8
    x, W, L, H = make_case(2, T, seed=T)
    r = fit(x, W, L, H, iters, precision)
    Wo, Lo, Ho, nll_o, _, _ = oracle.fit(x, W, L, H, iters)
    rel = np.abs(np.asarray(r.nll) - nll_o) / np.abs(nll_o)
    assert rel.max() <= NLL_TOL[precision], (rel.max(), int(rel.argmax()))
    assert (r.bin_status == 0).all()
    img_g = api.fastfca_separate(api.Spectrogram(x), r.params, precision=precision)
    img_o = oracle.separate(x, Wo, Lo, Ho)
    for n in range(12):
        assert rel_l2(img_g[n].f, img_o[n]) <= SEP_TOL[precision], n


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_big_fit_options(gpu, precision):
    """normalize_scales off, record_trace off, iters = 0 (fastfca.cpp:146-191)."""
    x, W, L, H = make_case(2, 3000, seed=5)
    r = fit(x, W, L, H, 4, precision, normalize_scales=False)
    _, _, _, nll_o, _, _ = oracle.fit(x, W, L, H, 4, normalize_scales=False)
    rel = np.abs(np.asarray(r.nll) - nll_o) / np.abs(nll_o)
    assert rel.max() <= NLL_TOL[precision]
    r2 = fit(x, W, L, H, 4, precision, record_trace=False)
    assert len(r2.nll) == 0
    r1 = fit(x, W, L, H, 4, precision)
    for a, b in zip(r2.params.act, r1.params.act):
        assert np.array_equal(a, b)  # the trace does not change the fit
    r0 = fit(x, W, L, H, 0, precision)
    assert len(r0.nll) == 1
    for a, b in zip(r0.params.act, [h for h in H]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_big_silent_bin_untouched(gpu, precision):
    x, W, L, H = make_case(3, 3000, seed=9)
    x[1] = 0.0
    r = fit(x, W, L, H, 3, precision)
    _, _, _, nll_o, _, _ = oracle.fit(x, W, L, H, 3)
    rel = np.abs(np.asarray(r.nll) - nll_o) / np.abs(nll_o)
    assert rel.max() <= NLL_TOL[precision]
    assert np.array_equal(r.params.act[1], H[1])
    assert np.array_equal(r.params.decorr[1], W[1])


def test_big_matches_cluster_kernel(gpu, monkeypatch):
    """The large-bin kernel and the round-1 cluster kernel (FFCA_NO_BIG) run the
    same algorithm: their fp32 traces agree to the parity tolerance."""
    x, W, L, H = make_case(3, 6000, seed=13)
    r_big = fit(x, W, L, H, 6, "fp32")
    monkeypatch.setenv("FFCA_NO_BIG", "1")
    r_old = fit(x, W, L, H, 6, "fp32")
    a, b = np.asarray(r_big.nll), np.asarray(r_old.nll)
    assert np.max(np.abs(a - b) / np.abs(b)) <= 1e-5


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_big_ip_restart_matches_oracle(gpu, precision):
    """A zero first column of W makes W^H Q_0 singular: the reference's first
    solve fails, the column restarts from its seeded perturbation and the
    retry succeeds (fastfca.cpp:51-70).  The fast IP detects the singular W
    and reruns the sweep the reference's way; W, L, H must match the oracle."""
    x, W, L, H = make_case(2, 3000, seed=21)
    W = W.copy()
    W[1, :, 0] = 0.0
    r = fit(x, W, L, H, 3, precision, record_trace=False, seed=7)
    Wo, Lo, Ho, _, _, _ = oracle.fit(x, W, L, H, 3, record_trace=False, seed=7)
    tol = 1e-9 if precision == "fp64" else 2e-3
    assert (r.bin_status == 0).all()
    for f in range(2):
        assert rel_l2(np.asarray(r.params.decorr[f]), Wo[f]) <= tol, f
        assert rel_l2(np.asarray(r.params.act[f]), Ho[f]) <= tol, f


# ---- M = 4, N = 6 (BASELINE config 2's shape): the same kernel with 256
# threads x 8 frame slots per CTA, three CTAs per SM.  T = 700 and 2000 run on
# one CTA (T = 700 with empty frame slots skipped), 5000 on a 3-CTA cluster.
@pytest.mark.parametrize("kind", ["jd", "fullrank"])
@pytest.mark.parametrize("T", [700, 2000, 5000])
def test_big_m4_fit_trace_and_separation(gpu, T, kind):
    iters = 8
    x, W, L, H = make_case(3, T, seed=T + 1, sigma_v=1.5, M=4, N=6, kind=kind)
    r = fit(x, W, L, H, iters, "fp32")
    Wo, Lo, Ho, nll_o, _, _ = oracle.fit(x, W, L, H, iters)
    rel = np.abs(np.asarray(r.nll) - nll_o) / np.abs(nll_o)
    assert rel.max() <= NLL_TOL["fp32"], (rel.max(), int(rel.argmax()))
    assert (r.bin_status == 0).all()
    img_g = api.fastfca_separate(api.Spectrogram(x), r.params, precision="fp32")
    img_o = oracle.separate(x, Wo, Lo, Ho)
    for n in range(6):
        assert rel_l2(img_g[n].f, img_o[n]) <= SEP_TOL["fp32"], n


def test_big_m4_options_and_silent_bin(gpu, monkeypatch):
    x, W, L, H = make_case(3, 2000, seed=31, sigma_v=1.5, M=4, N=6, kind="fullrank")
    x[1] = 0.0  # a silent bin keeps its init (fastfca.cpp:165-170)
    r = fit(x, W, L, H, 5, "fp32", normalize_scales=False)
    _, _, _, nll_o, _, _ = oracle.fit(x, W, L, H, 5, normalize_scales=False)
    rel = np.abs(np.asarray(r.nll) - nll_o) / np.abs(nll_o)
    assert rel.max() <= NLL_TOL["fp32"]
    assert np.array_equal(r.params.act[1], H[1]) and np.array_equal(r.params.decorr[1], W[1])
    r2 = fit(x, W, L, H, 5, "fp32", record_trace=False, normalize_scales=False)
    assert len(r2.nll) == 0
    for a, b in zip(r2.params.act, r.params.act):
        assert np.array_equal(a, b)
    # the round-1 kernel (FFCA_NO_BIG) runs the same algorithm
    r_big = fit(x, W, L, H, 6, "fp32")
    monkeypatch.setenv("FFCA_NO_BIG", "1")
    r_old = fit(x, W, L, H, 6, "fp32")
    a, b = np.asarray(r_big.nll), np.asarray(r_old.nll)
    assert np.max(np.abs(a - b) / np.abs(b)) <= 1e-5


def test_big_m4_ip_restart_matches_oracle(gpu):
    x, W, L, H = make_case(2, 2000, seed=37, sigma_v=1.5, M=4, N=6)
    W = W.copy()
    W[1, :, 0] = 0.0
    r = fit(x, W, L, H, 3, "fp32", record_trace=False, seed=7)
    Wo, Lo, Ho, _, _, _ = oracle.fit(x, W, L, H, 3, record_trace=False, seed=7)
    assert (r.bin_status == 0).all()
    for f in range(2):
        assert rel_l2(np.asarray(r.params.decorr[f]), Wo[f]) <= 2e-3, f
        assert rel_l2(np.asarray(r.params.act[f]), Ho[f]) <= 2e-3, f


# ---- M = 3, N = 4 (BASELINE config 4's shape): 96 threads x 7 frame slots per
# bin, eight bins per SM; odd M exercises the padded tensor-memory records, the
# idle fourth lane of the covariance pass and the reference-order IP.
@pytest.mark.parametrize("T", [200, 626, 672])
def test_big_m3_fit_trace_and_separation(gpu, T):
    iters = 10
    x, W, L, H = make_case(5, T, seed=T + 2, sigma_v=1.5, M=3, N=4)
    r = fit(x, W, L, H, iters, "fp32")
    Wo, Lo, Ho, nll_o, _, _ = oracle.fit(x, W, L, H, iters)
    rel = np.abs(np.asarray(r.nll) - nll_o) / np.abs(nll_o)
    assert rel.max() <= NLL_TOL["fp32"], (rel.max(), int(rel.argmax()))
    assert (r.bin_status == 0).all()
    img_g = api.fastfca_separate(api.Spectrogram(x), r.params, precision="fp32")
    img_o = oracle.separate(x, Wo, Lo, Ho)
    for n in range(4):
        assert rel_l2(img_g[n].f, img_o[n]) <= SEP_TOL["fp32"], n


def test_big_m3_options_silent_bin_and_old_kernel(gpu, monkeypatch):
    x, W, L, H = make_case(4, 626, seed=41, sigma_v=1.5, M=3, N=4)
    x[2] = 0.0
    r = fit(x, W, L, H, 6, "fp32", normalize_scales=False)
    _, _, _, nll_o, _, _ = oracle.fit(x, W, L, H, 6, normalize_scales=False)
    rel = np.abs(np.asarray(r.nll) - nll_o) / np.abs(nll_o)
    assert rel.max() <= NLL_TOL["fp32"]
    assert np.array_equal(r.params.act[2], H[2]) and np.array_equal(r.params.decorr[2], W[2])
    r2 = fit(x, W, L, H, 6, "fp32", record_trace=False, normalize_scales=False)
    assert len(r2.nll) == 0
    for a, b in zip(r2.params.act, r.params.act):
        assert np.array_equal(a, b)
    r_big = fit(x, W, L, H, 6, "fp32")
    monkeypatch.setenv("FFCA_NO_BIG", "1")
    r_old = fit(x, W, L, H, 6, "fp32")
    a, b = np.asarray(r_big.nll), np.asarray(r_old.nll)
    assert np.max(np.abs(a - b) / np.abs(b)) <= 1e-5


def test_big_m3_ip_restart_matches_oracle(gpu):
    x, W, L, H = make_case(2, 626, seed=43, sigma_v=1.5, M=3, N=4)
    W = W.copy()
    W[1, :, 0] = 0.0
    r = fit(x, W, L, H, 3, "fp32", record_trace=False, seed=7)
    Wo, Lo, Ho, _, _, _ = oracle.fit(x, W, L, H, 3, record_trace=False, seed=7)
    assert (r.bin_status == 0).all()
    for f in range(2):
        assert rel_l2(np.asarray(r.params.decorr[f]), Wo[f]) <= 2e-3, f
        assert rel_l2(np.asarray(r.params.act[f]), Ho[f]) <= 2e-3, f


# The pipelined host fit (bin chunks on their own streams, concurrently) with
# the large-bin kernel: each chunk works in its own rows of the U scratch and
# of the cold-path scratch, so chunked and single-launch fits agree bit for bit.
@pytest.mark.parametrize("shape", [(8, 12, 3000), (4, 6, 2000), (3, 4, 626)])
def test_big_chunked_host_fit_is_bit_equal(gpu, monkeypatch, shape):
    M, N, T = shape
    x, W, L, H = make_case(7, T, seed=51 + M, sigma_v=1.5, M=M, N=N)
    monkeypatch.setenv("FFCA_FIT_CHUNKS", "1")
    r1 = fit(x, W, L, H, 4, "fp32")
    monkeypatch.setenv("FFCA_FIT_CHUNKS", "3")
    r3 = fit(x, W, L, H, 4, "fp32")
    assert np.array_equal(np.asarray(r1.nll), np.asarray(r3.nll))
    for a, b in zip(r1.params.act, r3.params.act):
        assert np.array_equal(a, b)
    for a, b in zip(r1.params.decorr, r3.params.decorr):
        assert np.array_equal(a, b)


def test_big_exact_variances_switch(gpu, monkeypatch):
    """FFCA_EXACT_VARIANCES=1 selects the c3 kernel that sums the mixture
    variances afresh in every EM sweep; the default (incremental within an
    iteration, rebuilt exactly by the variance pass) stays within the fp32
    parity tolerance of it and of the oracle."""
    x, W, L, H = make_case(2, 5000, seed=71)
    r_incr = fit(x, W, L, H, 10, "fp32")
    monkeypatch.setenv("FFCA_EXACT_VARIANCES", "1")
    r_exact = fit(x, W, L, H, 10, "fp32")
    _, _, _, nll_o, _, _ = oracle.fit(x, W, L, H, 10)
    for r in (r_incr, r_exact):
        rel = np.abs(np.asarray(r.nll) - nll_o) / np.abs(nll_o)
        assert rel.max() <= NLL_TOL["fp32"], rel.max()
    a, b = np.asarray(r_incr.nll), np.asarray(r_exact.nll)
    assert np.max(np.abs(a - b) / np.abs(b)) <= 1e-5  # both within parity tolerance of each other
