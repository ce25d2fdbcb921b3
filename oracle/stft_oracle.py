"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference STFT front
end / iSTFT back end (reference proj/src/stft.cpp), the checker for the GPU
kernels in paper_2101_08563_b200/csrc/stft_kernels.cuh.  Only tests/ may use
it.  It is pinned by the reference's own known answers (tests/test_stft.cpp,
ported in tests/test_stft_oracle.py).

Layouts follow the reference containers: samples [channels, length] (numpy,
row = channel), spectrogram f [bins, channels, frames]."""
import numpy as np

CENTERED, FULL_FRAMES = 0, 1


def sqrt_hann_window(frame_len: int) -> np.ndarray:
    """stft.cpp:33-39 (periodic Hann, square-rooted)."""
    k = np.arange(frame_len)
    return np.sqrt(0.5 - 0.5 * np.cos(2.0 * np.pi * k / frame_len))


def _validate(frame_len: int, shift: int) -> None:
    """stft.cpp:14-19."""
    if frame_len <= 0 or frame_len & (frame_len - 1):
        raise ValueError("stft: frame length must be a power of two")
    if shift * 2 != frame_len:
        raise ValueError("stft: shift must be frame_len/2")


def stft_frame_count(length: int, frame_len: int, shift: int, pad: int = CENTERED) -> int:
    """stft.cpp:41-49."""
    if pad == CENTERED:
        return (length + shift - 1) // shift + 1
    if length < frame_len:
        raise ValueError("stft: signal shorter than one frame")
    return (length - frame_len) // shift + 1


def stft(samples: np.ndarray, frame_len: int, shift: int, pad: int = CENTERED) -> np.ndarray:
    """stft.cpp:51-83: frame j covers [j*shift - offset, +frame_len), zero
    outside the signal, times the window; bins 0..frame_len/2 of its DFT."""
    _validate(frame_len, shift)
    C, n = samples.shape
    if n < frame_len:
        raise ValueError("stft: signal shorter than one frame")
    frames = stft_frame_count(n, frame_len, shift, pad)
    offset = shift if pad == CENTERED else 0
    w = sqrt_hann_window(frame_len)
    padded = np.zeros((C, offset + (frames - 1) * shift + frame_len + frame_len))
    padded[:, offset:offset + n] = samples
    idx = np.arange(frames)[:, None] * shift + np.arange(frame_len)[None, :]
    fr = padded[:, idx] * w  # [C, frames, frame_len]
    spec = np.fft.rfft(fr, axis=-1)  # [C, frames, bins]
    return np.ascontiguousarray(np.transpose(spec, (2, 0, 1)))  # [bins, C, frames]


def istft(spec: np.ndarray, frame_len: int, shift: int, out_len: int,
          pad: int = CENTERED) -> np.ndarray:
    """stft.cpp:85-128: real inverse FFT per frame (DC / Nyquist imaginary
    parts drop out), windowed overlap-add divided by max(sum w^2, 1e-12)."""
    _validate(frame_len, shift)
    bins, C, frames = spec.shape
    if bins != frame_len // 2 + 1:
        raise ValueError("istft: bin count does not match frame_len")
    if frames != stft_frame_count(out_len, frame_len, shift, pad):
        raise ValueError("istft: frame count inconsistent with out_len and padding")
    offset = shift if pad == CENTERED else 0
    buf_len = (frames - 1) * shift + frame_len
    w = sqrt_hann_window(frame_len)
    wsum = np.zeros(buf_len)
    acc = np.zeros((C, buf_len))
    fr = np.fft.irfft(np.transpose(spec, (1, 2, 0)), n=frame_len, axis=-1)  # [C, frames, n]
    for j in range(frames):
        wsum[j * shift:j * shift + frame_len] += w * w
        acc[:, j * shift:j * shift + frame_len] += w * fr[:, j]
    out = np.zeros((C, out_len))
    p = np.arange(out_len) + offset
    ok = p < buf_len
    out[:, ok] = acc[:, p[ok]] / np.maximum(wsum[p[ok]], 1e-12)
    return out
