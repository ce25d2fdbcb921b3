"""Committed golden fixtures (tests/golden/*.npz, made by make_golden.py).

CPU part: the oracle, pinned by the reference's ported KATs, still reproduces
the frozen vectors (guards the checker against drift).
GPU part: the CUDA path, called through the C-ABI via the reference-shaped
API, against the stored vectors -- no oracle run needed on the GPU box.
Tolerances are BASELINE.json north_star's: per-iteration NLL 1e-5 relative
(fp32 path) / 1e-10 (fp64 mode); separated STFTs 1e-3 / 1e-10 relative L2.
fp64 mode also checks the fitted W, L, H at 1e-7 relative L2 (the NLL is the
stable quantity; parameters inherit the conditioning of the per-bin solves).
"""
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"
FIT_FILES = sorted(p.name for p in GOLD.glob("fit_*.npz"))
BLOCK_FILES = sorted(p.name for p in GOLD.glob("block_*.npz"))
STFT_FILES = sorted(p.name for p in GOLD.glob("stft_*.npz"))
NLL_TOL = {"fp32": 1e-5, "fp64": 1e-10}
SEP_TOL = {"fp32": 1e-3, "fp64": 1e-10}


def load(name):
    with np.load(GOLD / name) as z:
        return {k: z[k] for k in z.files}


def rel_l2(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def max_rel(a, b):
    return float((np.abs(a - b) / np.abs(b)).max())


def test_fixture_set_complete():
    assert len(FIT_FILES) >= 8 and len(BLOCK_FILES) >= 2 and len(STFT_FILES) >= 2 and (GOLD / "ica_m2.npz").exists()
    g = load("fit_m2n3_em.npz")
    assert g["nll"].shape == (int(g["iters"]) + 1,) and "images" in g


# ------------------------------------------------------------------ CPU --
@pytest.mark.parametrize("name", FIT_FILES)
def test_oracle_reproduces_golden_fit(built, name):
    import oracle
    g = load(name)
    x = g["x"].astype(np.complex128)
    Wo, Lo, Ho, nll, _, _ = oracle.fit(x, g["W0"], g["L0"], g["H0"], int(g["iters"]),
                                       flavor=int(g["flavor"]),
                                       normalize_scales=bool(g["normalize_scales"]),
                                       fix_loadings=bool(g["fix_loadings"]))
    assert max_rel(nll, g["nll"]) <= 1e-12
    for got, want in ((Wo, g["W"]), (Lo, g["L"]), (Ho, g["H"])):
        assert rel_l2(got, want) <= 1e-10
    if "images" in g:
        assert rel_l2(oracle.separate(x, Wo, Lo, Ho), g["images"]) <= 1e-10


def test_oracle_reproduces_golden_ica(built):
    import oracle
    g = load("ica_m2.npz")
    Wo, Lo, Ho, nll = oracle.ica_fit(g["x"].astype(np.complex128), g["W0"], int(g["iters"]))
    assert max_rel(nll, g["nll"]) <= 1e-12
    assert rel_l2(Wo, g["W"]) <= 1e-10 and rel_l2(Ho, g["H"]) <= 1e-10


# ------------------------------------------------------------------ GPU --
@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("name", FIT_FILES)
def test_gpu_fit_matches_golden(gpu, name, precision):
    from paper_2101_08563_b200 import api
    g = load(name)
    covs = api.sample_covs(api.Spectrogram(g["x"].astype(np.complex128)))
    init = api.FastFcaParams(g["W0"], g["L0"], g["H0"])
    oo = api.FastFcaOptions(fix_loadings=bool(g["fix_loadings"]),
                            normalize_scales=bool(g["normalize_scales"]))
    r = api.fastfca_fit(covs, init, int(g["flavor"]), int(g["iters"]), api.FitOptions(), oo,
                        precision=precision)
    nll = np.asarray(r.nll)
    assert nll.shape == g["nll"].shape
    assert max_rel(nll, g["nll"]) <= NLL_TOL[precision]
    assert (r.bin_status == 0).all()
    if precision == "fp64":
        assert rel_l2(r.params.decorr, g["W"]) <= 1e-7
        assert rel_l2(r.params.loading, g["L"]) <= 1e-7
        assert rel_l2(r.params.act, g["H"]) <= 1e-7
    if "images" in g:
        imgs = api.fastfca_separate(api.Spectrogram(g["x"].astype(np.complex128)), r.params,
                                    precision=precision)
        for n in range(g["images"].shape[0]):
            assert rel_l2(imgs[n].f, g["images"][n]) <= SEP_TOL[precision]


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_gpu_ica_matches_golden(gpu, precision):
    from paper_2101_08563_b200 import api
    g = load("ica_m2.npz")
    covs = api.sample_covs(api.Spectrogram(g["x"].astype(np.complex128)))
    M = g["W0"].shape[-1]
    r = api.ica_mode_fit(covs, M, int(g["iters"]), g["W0"], precision=precision)
    assert max_rel(np.asarray(r.nll), g["nll"]) <= NLL_TOL[precision]
    assert np.array_equal(r.params.loading, np.tile(np.eye(M), (g["x"].shape[0], 1, 1)))
    if precision == "fp64":
        assert rel_l2(r.params.decorr, g["W"]) <= 1e-7


# --------------------------------------------- block-stationary fixtures --
@pytest.mark.parametrize("name", BLOCK_FILES)
def test_oracle_reproduces_golden_block_fit(built, name):
    import oracle
    g = load(name)
    mats, power = oracle.block_covs(g["x"].astype(np.complex128), int(g["block_size"]))
    assert rel_l2(mats, g["mats"]) <= 1e-14 and max_rel(power, g["power"]) <= 1e-14
    Wo, Lo, Ho, nll, _ = oracle.fit_covs(mats, g["W0"], g["L0"], g["H0"], int(g["iters"]),
                                         flavor=int(g["flavor"]), power=power)
    assert max_rel(nll, g["nll"]) <= 1e-12
    for got, want in ((Wo, g["W"]), (Lo, g["L"]), (Ho, g["H"])):
        assert rel_l2(got, want) <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("name", BLOCK_FILES)
def test_gpu_block_fit_matches_golden(gpu, name, precision):
    from paper_2101_08563_b200 import api
    g = load(name)
    covs = api.sample_covs(api.Spectrogram(g["x"].astype(np.complex128)), int(g["block_size"]))
    assert rel_l2(covs.mats, g["mats"]) <= 1e-12  # block covariances are fp64 on the GPU
    assert max_rel(covs.power_scale, g["power"]) <= 1e-12
    r = api.fastfca_fit(covs, api.FastFcaParams(g["W0"], g["L0"], g["H0"]), int(g["flavor"]),
                        int(g["iters"]), precision=precision)
    assert max_rel(np.asarray(r.nll), g["nll"]) <= NLL_TOL[precision]
    assert (r.bin_status == 0).all()
    if precision == "fp64":
        assert rel_l2(r.params.loading, g["L"]) <= 1e-7
        assert rel_l2(r.params.decorr, g["W"]) <= 1e-7


# ------------------------------------------------- STFT / iSTFT fixtures --
@pytest.mark.parametrize("name", STFT_FILES)
def test_oracle_reproduces_golden_stft(name):
    import stft_oracle
    g = load(name)
    fl, sh, pad = int(g["frame_len"]), int(g["shift"]), int(g["pad"])
    spec = stft_oracle.stft(g["wave"], fl, sh, pad)
    assert np.abs(spec - g["spec"]).max() <= 1e-12 * np.abs(g["spec"]).max()
    back = stft_oracle.istft(g["spec"], fl, sh, g["wave"].shape[1], pad)
    assert np.abs(back - g["back"]).max() <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name", STFT_FILES)
def test_gpu_stft_istft_match_golden(gpu, name):
    from paper_2101_08563_b200 import api
    g = load(name)
    fl, sh, pad = int(g["frame_len"]), int(g["shift"]), int(g["pad"])
    n = g["wave"].shape[1]
    spec = api.stft(api.MultichannelWave(g["wave"], 16000.0), fl, sh, pad)
    assert spec.f.shape == g["spec"].shape
    # fp64 FFTs on both sides: error grows like eps * log2(frame_len) * scale
    assert np.abs(spec.f - g["spec"]).max() <= 1e-13 * np.abs(g["spec"]).max() * np.log2(fl)
    back = api.istft(api.Spectrogram(g["spec"]), fl, sh, n, 16000.0, pad)
    np.testing.assert_allclose(back.samples, g["back"], atol=1e-12)


# ------------------------------------------------ batch (config-4 family) --
def test_oracle_reproduces_golden_batch(built):
    import oracle
    g = load("batch3_m3n4_em.npz")
    Wo, Lo, Ho, nll, _, _ = oracle.fit(g["x"].astype(np.complex128), g["W0"], g["L0"], g["H0"],
                                       int(g["iters"]))
    assert max_rel(nll, g["nll"]) <= 1e-12
    assert rel_l2(Ho, g["H"]) <= 1e-10 and rel_l2(Wo, g["W"]) <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_gpu_fit_batch_matches_golden(gpu, precision):
    """fastfca_fit_batch: one batched C-ABI call equals the per-mixture loop."""
    from paper_2101_08563_b200 import api
    g = load("batch3_m3n4_em.npz")
    x = g["x"].astype(np.complex128)
    covs = [api.sample_covs(api.Spectrogram(xb)) for xb in x]
    init = [api.FastFcaParams(g["W0"][b], g["L0"][b], g["H0"][b]) for b in range(x.shape[0])]
    rs = api.fastfca_fit_batch(covs, init, api.LhFlavor.em, int(g["iters"]), precision=precision)
    assert len(rs) == x.shape[0]
    for b, r in enumerate(rs):
        assert max_rel(np.asarray(r.nll), g["nll"][b]) <= NLL_TOL[precision]
        assert (r.bin_status == 0).all()
        if precision == "fp64":
            assert rel_l2(r.params.act, g["H"][b]) <= 1e-7
    # the batch equals the loop of single fits
    one = api.fastfca_fit(covs[1], init[1], api.LhFlavor.em, int(g["iters"]), precision=precision)
    assert np.array_equal(np.asarray(one.nll), np.asarray(rs[1].nll))
    with pytest.raises(api.InvalidArgument):
        api.fastfca_fit_batch(covs, init[:2], api.LhFlavor.em, 3)
