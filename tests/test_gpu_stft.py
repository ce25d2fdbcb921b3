"""STFT front end / iSTFT back end on the GPU against
the numpy restatement (oracle/stft_oracle.py) and the reference's own known
answers (tests/test_stft.cpp:68-187), plus the device path that feeds the fit
kernel its x layout directly."""
import numpy as np
import pytest
import torch

import stft_oracle as so
from paper_2101_08563_b200 import _lib, api
from paper_2101_08563_b200._lib import InvalidArgument

pytestmark = pytest.mark.gpu


def rwave(C, n, seed, dtype=np.float64):
    return np.random.default_rng(seed).uniform(-0.5, 0.5, (C, n)).astype(dtype).astype(np.float64)


def wave(x):
    return api.MultichannelWave(x, 16000.0)


@pytest.mark.parametrize("n", [64, 256, 512, 1024, 4096])
@pytest.mark.parametrize("pad", [so.CENTERED, so.FULL_FRAMES])
def test_stft_matches_oracle(gpu, n, pad):
    x = rwave(3, 5 * n + 77, seed=n + pad)
    got = api.stft(wave(x), n, n // 2, pad).f
    want = so.stft(x, n, n // 2, pad)
    assert got.shape == want.shape
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= 1e-13 * scale * np.log2(n)


def test_zero_signal_and_validation(gpu):  # test_stft.cpp:78-93
    assert np.abs(api.stft(wave(np.zeros((2, 4000))), 512, 256).f).max() == 0.0
    w = wave(rwave(1, 4000, 21))
    for args in ((1000, 500), (1024, 256)):
        with pytest.raises(InvalidArgument):
            api.stft(w, *args)
    with pytest.raises(InvalidArgument):
        api.stft(wave(rwave(1, 100, 22)), 1024, 512)


def test_bin_centered_sinusoid(gpu):  # test_stft.cpp:95-123
    n, shift, b = 1024, 512, 100
    t = np.arange(8 * n)
    x = np.cos(2 * np.pi * b * t / n + 0.3)[None]
    f = api.stft(wave(x), n, shift, api.StftPadding.full_frames).f
    j = 4
    frame = x[0, j * shift:j * shift + n] * api.sqrt_hann_window(n)
    k = np.arange(n)
    direct = np.array([np.sum(frame * np.exp(-2j * np.pi * bb * k / n)) for bb in range(n // 2 + 1)])
    assert np.abs(f[:, 0, j] - direct).max() < 1e-8 * np.linalg.norm(direct)
    e = np.abs(f[:, 0, j]) ** 2
    total = (e[0] + e[-1] + 2 * e[1:-1].sum()) / n
    center = 2 * e[b] / n
    main = center + 2 * (e[b - 1] + e[b + 1]) / n
    assert 0.81 < center / total < 0.82 and main / total > 0.99


def test_frame_counts(gpu):  # test_stft.cpp:125-132
    n = 8 * 16000
    assert api.stft_frame_count(n, 1024, 512, api.StftPadding.full_frames) == 249
    assert api.stft_frame_count(n, 1024, 512, api.StftPadding.centered) == 251
    with pytest.raises(InvalidArgument):
        api.stft_frame_count(100, 1024, 512, api.StftPadding.full_frames)


def test_parseval(gpu):  # test_stft.cpp:134-149
    n, shift = 256, 128
    x = rwave(2, 3000, 23)
    f = api.stft(wave(x), n, shift, api.StftPadding.full_frames).f
    w = api.sqrt_hann_window(n)
    for j in range(0, f.shape[2], 3):
        for ch in range(2):
            te = np.sum((x[ch, j * shift:j * shift + n] * w) ** 2)
            e = np.abs(f[:, ch, j]) ** 2
            assert abs((e[0] + e[-1] + 2 * e[1:-1].sum()) / n - te) <= 1e-9 * te


@pytest.mark.parametrize("length", [4000, 4097])
def test_round_trip_centered(gpu, length):  # test_stft.cpp:151-160
    x = rwave(2, length, 24)
    s = api.stft(wave(x), 512, 256)
    back = api.istft(s, 512, 256, length, 16000.0).samples
    assert np.abs(back - x).max() < 1e-10
    np.testing.assert_allclose(back, so.istft(s.f, 512, 256, length), atol=1e-13)


def test_round_trip_cases(gpu):  # test_stft.cpp:161-187
    z = api.istft(api.Spectrogram.zero(1, 257, 9), 512, 256, 2048, 16000.0).samples
    assert np.abs(z).max() == 0.0
    rng = np.random.default_rng(25)
    x = rng.uniform(-0.5, 0.5, (2, 16000))
    for ch in range(2):  # one-pole lowpass + slow AM, a speech-shaped signal
        st = 0.0
        for t in range(16000):
            st = 0.95 * st + 0.05 * x[ch, t]
            x[ch, t] = st * (0.6 + 0.4 * np.sin(2 * np.pi * 3.0 * t / 16000))
    back = api.istft(api.stft(wave(x), 1024, 512), 1024, 512, 16000, 16000.0).samples
    assert np.linalg.norm(back - x) / np.linalg.norm(x) < 1e-9
    y = rwave(1, 4096, 26)
    fs = api.stft(wave(y), 512, 256, api.StftPadding.full_frames)
    back = api.istft(fs, 512, 256, 4096, 16000.0, api.StftPadding.full_frames).samples
    hi = (fs.frames - 1) * 256 + 512 - 256
    assert np.abs(back[0, 256:hi] - y[0, 256:hi]).max() < 1e-10
    s = api.stft(wave(rwave(1, 4000, 27)), 512, 256)
    with pytest.raises(InvalidArgument):
        api.istft(s, 1024, 512, 4000, 16000.0)
    with pytest.raises(InvalidArgument):
        api.istft(s, 512, 256, 9999, 16000.0)


def test_istft_of_filtered_spectrum_matches_oracle(gpu):
    # Non-Hermitian DC / Nyquist (as separated images have): the imaginary
    # parts drop out exactly as in the reference's real inverse FFT.
    rng = np.random.default_rng(28)
    f = rng.standard_normal((257, 2, 20)) + 1j * rng.standard_normal((257, 2, 20))
    out_len = (20 - 1) * 256 - 255
    got = api.istft(api.Spectrogram(f), 512, 256, out_len, 16000.0).samples
    np.testing.assert_allclose(got, so.istft(f, 512, 256, out_len), atol=1e-12)


def test_device_stft_writes_the_fit_layout(gpu):
    """ffca_stft_device writes the fit's x layout [bins][frames][channels] in
    complex64, bit-identical to the host STFT rounded once (so a fit on it is
    the host-path fit on the same spectrogram)."""
    C, n, shift, length = 2, 512, 256, 256 * 120
    x = rwave(C, length, 30, dtype=np.float32)  # fp32-representable samples
    dev = torch.device("cuda", 0)
    ctx = _lib.context(0)
    L = _lib.lib()
    frames = api.stft_frame_count(length, n, shift)
    bins = n // 2 + 1
    s_dev = torch.from_numpy(np.ascontiguousarray(x.T.astype(np.float32))).to(dev)
    x_dev = torch.empty((bins, frames, C), dtype=torch.complex64, device=dev)
    _lib.check(L.ffca_stft_device(ctx.handle, C, length, n, shift, 0, _lib.PREC_FP32,
                                  _lib.ptr(s_dev), _lib.ptr(x_dev), None))
    torch.cuda.synchronize()
    host = api.stft(wave(x), n, shift).f  # [bins, C, frames] complex128
    got = x_dev.cpu().numpy()
    np.testing.assert_array_equal(got, np.swapaxes(host, 1, 2).astype(np.complex64))
    # The device path back: istft of the complex64 spectrum.
    back = torch.empty((length, C), dtype=torch.float32, device=dev)
    _lib.check(L.ffca_istft_device(ctx.handle, C, frames, n, shift, 0, length, _lib.PREC_FP32,
                                   _lib.ptr(x_dev), _lib.ptr(back), None))
    torch.cuda.synchronize()
    assert np.abs(back.cpu().numpy().T - x).max() < 1e-5


def test_waveform_pipeline_partitions_the_mixture(gpu):
    """wave -> GPU STFT -> fit -> decomposed MWF -> GPU iSTFT per source: the
    source images add back to the mixture (test_fastfca.cpp:342-359 carried
    through the STFT round trip)."""
    from paper_2101_08563_b200 import synth
    C, n, length = 2, 256, 128 * 80
    rng = np.random.default_rng(31)
    x = rng.standard_normal((C, length)) * np.linspace(0.2, 1.0, length)
    spec = api.stft(wave(x), n, n // 2)
    covs = api.sample_covs(spec)
    cfg = synth.small(C, 2, spec.bins, spec.frames, seed=3)
    W, Lw, H = synth.init_params(cfg)
    r = api.fastfca_fit(covs, api.FastFcaParams(W, Lw, H), 0, 10, precision="fp64")
    imgs = api.fastfca_separate(spec, r.params, precision="fp64")
    waves = [api.istft(im, n, n // 2, length, 16000.0).samples for im in imgs]
    assert np.linalg.norm(sum(waves) - x) <= 1e-9 * np.linalg.norm(x)
