"""The numpy STFT restatement (oracle/stft_oracle.py) pinned by the reference's
own known answers (tests/test_stft.cpp:68-187; random inputs are drawn here
with numpy, the properties hold for any input)."""
import numpy as np
import pytest

import stft_oracle as so


def rwave(C, n, seed):
    return np.random.default_rng(seed).uniform(-0.5, 0.5, (C, n))


def one_sided_energy(f, ch, j, n):  # test_stft.cpp:61-65
    e = abs(f[0, ch, j]) ** 2 + abs(f[-1, ch, j]) ** 2
    e += 2.0 * np.sum(np.abs(f[1:-1, ch, j]) ** 2)
    return e / n


@pytest.mark.parametrize("n", [64, 256, 1024])
def test_cola(n):  # test_stft.cpp:68-76
    w = so.sqrt_hann_window(n)
    s = n // 2
    np.testing.assert_allclose(w[:s] ** 2 + w[s:] ** 2, 1.0, rtol=1e-12)


def test_zero_signal_and_validation():  # test_stft.cpp:78-93
    assert np.abs(so.stft(np.zeros((2, 4000)), 512, 256)).max() == 0.0
    w = rwave(1, 4000, 21)
    for args in ((1000, 500), (1024, 256)):
        with pytest.raises(ValueError):
            so.stft(w, *args)
    with pytest.raises(ValueError):
        so.stft(rwave(1, 100, 22), 1024, 512)


def test_bin_centered_sinusoid():  # test_stft.cpp:95-123
    n, shift, b = 1024, 512, 100
    t = np.arange(8 * n)
    x = np.cos(2 * np.pi * b * t / n + 0.3)[None]
    f = so.stft(x, n, shift, so.FULL_FRAMES)
    j = 4
    frame = x[0, j * shift:j * shift + n] * so.sqrt_hann_window(n)
    k = np.arange(n)
    direct = np.array([np.sum(frame * np.exp(-2j * np.pi * bb * k / n)) for bb in range(n // 2 + 1)])
    assert np.abs(f[:, 0, j] - direct).max() < 1e-8 * np.linalg.norm(direct)
    total = one_sided_energy(f, 0, j, n)
    center = 2 * abs(f[b, 0, j]) ** 2 / n
    main = center + 2 * (abs(f[b - 1, 0, j]) ** 2 + abs(f[b + 1, 0, j]) ** 2) / n
    assert 0.81 < center / total < 0.82 and main / total > 0.99


def test_frame_counts():  # test_stft.cpp:125-132
    n = 8 * 16000
    assert so.stft_frame_count(n, 1024, 512, so.FULL_FRAMES) == 249
    assert 513 * so.stft_frame_count(n, 1024, 512, so.FULL_FRAMES) == 127737
    assert so.stft_frame_count(n, 1024, 512, so.CENTERED) == 251


def test_parseval():  # test_stft.cpp:134-149
    n, shift = 256, 128
    x = rwave(2, 3000, 23)
    f = so.stft(x, n, shift, so.FULL_FRAMES)
    w = so.sqrt_hann_window(n)
    for j in range(0, f.shape[2], 3):
        for ch in range(2):
            te = np.sum((x[ch, j * shift:j * shift + n] * w) ** 2)
            assert abs(one_sided_energy(f, ch, j, n) - te) <= 1e-9 * te


@pytest.mark.parametrize("length", [4000, 4097])
def test_round_trip(length):  # test_stft.cpp:151-187
    x = rwave(2, length, 24)
    back = so.istft(so.stft(x, 512, 256), 512, 256, length)
    assert np.abs(back - x).max() < 1e-10
    assert np.abs(so.istft(np.zeros((257, 1, 9), complex), 512, 256, 2048)).max() == 0.0
    y = rwave(1, 4096, 25)
    fs = so.stft(y, 512, 256, so.FULL_FRAMES)
    back = so.istft(fs, 512, 256, 4096, so.FULL_FRAMES)
    hi = (fs.shape[2] - 1) * 256 + 512 - 256
    assert np.abs(back[0, 256:hi] - y[0, 256:hi]).max() < 1e-10
    with pytest.raises(ValueError):
        so.istft(so.stft(x, 512, 256), 1024, 512, length)
    with pytest.raises(ValueError):
        so.istft(so.stft(x, 512, 256), 512, 256, 9999)
