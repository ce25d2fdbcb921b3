"""Python mirror of the reference FastFCA API for the hot path.

Same names, argument meaning and error behaviour as the reference C++ API
(proj/include/fastfca/fastfca.hpp:16-66, sigmodel.hpp:34-111, stft.hpp:21-29),
so parity tests read like the reference's own tests.  Arrays use natural
numpy indexing (row index first); they are converted to the reference's
Eigen column-major buffers at the C-ABI boundary (include/ffca.h).  All
compute runs in libffca.so on the GPU.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import InvalidArgument, NumericalError  # noqa: F401  (re-exported)


class LhFlavor:  # fastfca.hpp:16
    em = _lib.FLAVOR_EM
    mm = _lib.FLAVOR_MM


@dataclass
class FitOptions:  # sigmodel.hpp:34-38
    workers: int = 1            # host threads (unused by the GPU path; kept for the API)
    record_trace: bool = True
    seed: int = 0


@dataclass
class FastFcaOptions:  # fastfca.hpp:18-21
    fix_loadings: bool = False
    normalize_scales: bool = True


@dataclass
class Spectrogram:  # stft.hpp:21-29; f[i] is channels x frames
    f: np.ndarray  # complex [bins, channels, frames]

    @property
    def bins(self) -> int:
        return self.f.shape[0]

    @property
    def channels(self) -> int:
        return self.f.shape[1]

    @property
    def frames(self) -> int:
        return self.f.shape[2]

    @staticmethod
    def zero(channels: int, bins: int, frames: int) -> "Spectrogram":
        return Spectrogram(np.zeros((bins, channels, frames), np.complex128))


@dataclass
class MultichannelWave:  # stft.hpp:12-17
    samples: np.ndarray  # float [channels, length]
    sample_rate: float = 0.0

    @property
    def channels(self) -> int:
        return self.samples.shape[0]

    @property
    def length(self) -> int:
        return self.samples.shape[1]


class StftPadding:  # stft.hpp:30-37
    centered = 0
    full_frames = 1


class SampleCovSet:  # sigmodel.hpp:48-56
    """Observation statistics.  block_size == 1: the snapshots (the hot path
    reads them; the rank-one `mats` are not materialised).
    block_size B > 1: mats [bins, blocks, dim, dim] complex, the B-frame block
    covariances (sigmodel.cpp:34-41).  power_scale may be None for a
    caller-built set: power(i) then falls back to the block traces
    (sigmodel.cpp:50-55), computed on the GPU by the fit."""

    def __init__(self, snapshots=None, power_scale=None, block_size: int = 1, mats=None,
                 frames: int | None = None):
        self.snapshots = None if snapshots is None else np.asarray(snapshots)
        self.power_scale = None if power_scale is None else np.asarray(power_scale, np.float64)
        self.block_size = int(block_size)
        self.mats = None if mats is None else np.asarray(mats)
        if self.snapshots is None and self.mats is None:
            raise InvalidArgument("SampleCovSet: snapshots or mats required")
        self._frames = frames

    def has_snapshots(self) -> bool:
        return self.snapshots is not None

    @property
    def dim(self) -> int:
        return (self.snapshots if self.has_snapshots() else self.mats).shape[-2]

    @property
    def bins(self) -> int:
        return (self.snapshots if self.has_snapshots() else self.mats).shape[0]

    @property
    def blocks(self) -> int:
        return self.snapshots.shape[2] if self.has_snapshots() else self.mats.shape[1]

    @property
    def frames(self) -> int:
        return self._frames if self._frames is not None else self.blocks * (
            1 if self.has_snapshots() else self.block_size)

    def power(self, i: int) -> float:
        if self.power_scale is not None and i < len(self.power_scale):
            return float(self.power_scale[i])
        tr = np.trace(self.mats[i], axis1=-2, axis2=-1).real.sum()
        return float(tr / (self.blocks * self.dim))


@dataclass
class FastFcaParams:  # sigmodel.hpp:72-78
    decorr: np.ndarray   # complex [bins, dim, dim]    W_i
    loading: np.ndarray  # [bins, dim, sources]        L_i
    act: np.ndarray      # [bins, sources, frames]     H_i

    @property
    def dim(self) -> int:
        return self.decorr.shape[1]

    @property
    def bins(self) -> int:
        return self.decorr.shape[0]

    @property
    def sources(self) -> int:
        return self.loading.shape[2]

    @property
    def frames(self) -> int:
        return self.act.shape[2]

    def copy(self) -> "FastFcaParams":
        return FastFcaParams(self.decorr.copy(), self.loading.copy(), self.act.copy())


@dataclass
class FastFcaFitResult:  # fastfca.hpp:23-26
    params: FastFcaParams
    nll: list = field(default_factory=list)
    bin_status: np.ndarray | None = None


# ------------------------------------------------------------ layout glue --
def _x_ref(snapshots: np.ndarray) -> np.ndarray:
    """[..., bins, dim, frames] -> reference [..., bins, frames, dim] complex128."""
    return np.ascontiguousarray(np.swapaxes(snapshots, -1, -2), dtype=np.complex128)


def _params_ref(p: FastFcaParams):
    # Always copies: with a size-1 axis swapaxes is already contiguous, and a
    # view would let the in/out C buffers alias the caller's arrays (the
    # reference copies init, fastfca.cpp:153-154).
    W = np.array(np.swapaxes(p.decorr, -1, -2), dtype=np.complex128, order="C", copy=True)
    L = np.array(np.swapaxes(p.loading, -1, -2), dtype=np.float64, order="C", copy=True)
    H = np.array(np.swapaxes(p.act, -1, -2), dtype=np.float64, order="C", copy=True)
    return W, L, H


def _params_from_ref(W, L, H) -> FastFcaParams:
    return FastFcaParams(np.ascontiguousarray(np.swapaxes(W, -1, -2)),
                         np.ascontiguousarray(np.swapaxes(L, -1, -2)),
                         np.ascontiguousarray(np.swapaxes(H, -1, -2)))


def _mats_ref(mats: np.ndarray) -> np.ndarray:
    """[..., blocks, dim, dim] -> reference per-block Eigen col-major complex128."""
    return np.ascontiguousarray(np.swapaxes(mats, -1, -2), dtype=np.complex128)


def _covs_input(covs: SampleCovSet):
    """(buffer, power or None, snapshot?) for the C-ABI fit entry points."""
    pw = None if covs.power_scale is None else np.ascontiguousarray(covs.power_scale, np.float64)
    if covs.has_snapshots():
        if pw is None:
            raise InvalidArgument("SampleCovSet: snapshots need power_scale")
        return _x_ref(covs.snapshots), pw, True
    return _mats_ref(covs.mats), pw, False


def _prec(precision: str) -> int:
    if precision not in ("fp32", "fp64"):
        raise InvalidArgument(f"precision must be 'fp32' or 'fp64', not {precision!r}")
    return _lib.PREC_FP64 if precision == "fp64" else _lib.PREC_FP32


# ------------------------------------------------------------------- API --
def sample_covs(spec: Spectrogram, block_size: int = 1, *, device: int | None = None) -> SampleCovSet:
    """sigmodel.cpp:17-48 on the GPU: block_size == 1 keeps the snapshots and
    computes power_scale; block_size B > 1 computes the block covariances
    (ceil(T/B) blocks, the last one ragged) and power_scale."""
    if spec.bins == 0 or spec.frames == 0 or spec.channels == 0:
        raise InvalidArgument("sample_covs: empty spectrogram")
    if block_size < 1:
        raise InvalidArgument("sample_covs: block size must be >= 1")
    x = _x_ref(spec.f)
    d = _lib.Dims(1, spec.bins, spec.channels, 1, spec.frames)
    out = np.empty(spec.bins)
    ctx = _lib.context(device)
    if block_size == 1:
        _lib.check(_lib.lib().ffca_power_scale(ctx.handle, d, _lib.ptr(x), _lib.ptr(out)))
        return SampleCovSet(np.asarray(spec.f, dtype=np.complex128), out)
    J = -(-spec.frames // block_size)
    M = spec.channels
    mats = np.empty((spec.bins, J, M, M), np.complex128)  # Eigen col-major per block
    _lib.check(_lib.lib().ffca_block_covs(ctx.handle, d, int(block_size), _lib.ptr(x),
                                          _lib.ptr(mats), _lib.ptr(out)))
    return SampleCovSet(None, out, block_size, np.swapaxes(mats, -1, -2), frames=spec.frames)


def piecewise_prepare(spec: Spectrogram, block_size: int, **kw) -> SampleCovSet:
    """fastfca.cpp:266-268."""
    return sample_covs(spec, block_size, **kw)


def expand_block_params(params: "FastFcaParams", block_size: int, frames: int) -> "FastFcaParams":
    """sigmodel.cpp:164-196: block-level H -> frame level (column j takes block
    min(j // B, blocks - 1)).  A host-side index copy."""
    if block_size == 1 and frames == params.frames:
        return params
    jb = np.minimum(np.arange(frames) // block_size, params.frames - 1)
    return FastFcaParams(params.decorr.copy(), params.loading.copy(),
                         np.ascontiguousarray(params.act[:, :, jb]))


def _check_shape(covs: SampleCovSet, init: FastFcaParams, what: str) -> None:
    if (init.dim != covs.dim or init.bins != covs.bins or init.frames != covs.blocks
            or init.loading.shape[:2] != (covs.bins, covs.dim)
            or init.act.shape[:2] != (covs.bins, init.sources)):
        raise InvalidArgument(f"{what}: init/covariance shape mismatch")



def fastfca_fit(covs: SampleCovSet, init: FastFcaParams, flavor: int, iters: int,
                fit: FitOptions | None = None, opts: FastFcaOptions | None = None, *,
                precision: str = "fp32", device: int | None = None) -> FastFcaFitResult:
    """fastfca.cpp:146-191 on the GPU (one CTA per frequency bin)."""
    fit = fit or FitOptions()
    opts = opts or FastFcaOptions()
    _check_shape(covs, init, "fastfca_fit")
    if iters < 0:
        raise InvalidArgument("fastfca_fit: negative iteration count")
    x, power, snap = _covs_input(covs)
    W, L, H = _params_ref(init)
    F = covs.bins
    d = _lib.Dims(1, F, covs.dim, init.sources, covs.blocks)
    o = _lib.FitOpts(int(flavor), int(iters), int(bool(fit.record_trace)), int(fit.seed),
                     int(bool(opts.normalize_scales)), int(bool(opts.fix_loadings)),
                     _prec(precision))
    nll = np.zeros(iters + 1) if fit.record_trace else None
    status = np.zeros(F, np.int32)
    ctx = _lib.context(device)
    fn = _lib.lib().ffca_fit if snap else _lib.lib().ffca_fit_covs
    _lib.check(fn(ctx.handle, d, o, _lib.ptr(x), _lib.ptr(power), _lib.ptr(W),
                                   _lib.ptr(L), _lib.ptr(H), _lib.ptr(nll), None,
                                   _lib.ptr(status)))
    return FastFcaFitResult(_params_from_ref(W, L, H), list(nll) if nll is not None else [],
                            status)


def fastfca_fit_batch(covs: list[SampleCovSet], init: list[FastFcaParams], flavor: int,
                      iters: int, fit: FitOptions | None = None,
                      opts: FastFcaOptions | None = None, *, precision: str = "fp32",
                      device: int | None = None) -> list[FastFcaFitResult]:
    """Batch entry (config 4): equal to the loop of fastfca_fit
    over the mixtures, run as ONE C-ABI call with dims.batch = len(covs) (the
    C++ shim's fastfca_fit_batch on one device).  All mixtures share one shape."""
    fit = fit or FitOptions()
    opts = opts or FastFcaOptions()
    if len(covs) != len(init):
        raise InvalidArgument("fastfca_fit_batch: covariance/init count mismatch")
    if not covs:
        return []
    c0, i0 = covs[0], init[0]
    for c, p in zip(covs, init):
        _check_shape(c, p, "fastfca_fit")
        if (c.dim, c.bins, c.blocks, p.sources, c.has_snapshots(), c.power_scale is None) != \
                (c0.dim, c0.bins, c0.blocks, i0.sources, c0.has_snapshots(), c0.power_scale is None):
            raise InvalidArgument("fastfca_fit_batch: mixtures must share one shape")
    if iters < 0:
        raise InvalidArgument("fastfca_fit: negative iteration count")
    B, F = len(covs), c0.bins
    ins = [_covs_input(c) for c in covs]
    x = np.ascontiguousarray(np.stack([t[0] for t in ins]))
    power = None if ins[0][1] is None else np.ascontiguousarray(np.stack([t[1] for t in ins]))
    refs = [_params_ref(p) for p in init]
    W, L, H = (np.ascontiguousarray(np.stack([r[k] for r in refs])) for k in range(3))
    d = _lib.Dims(B, F, c0.dim, i0.sources, c0.blocks)
    o = _lib.FitOpts(int(flavor), int(iters), int(bool(fit.record_trace)), int(fit.seed),
                     int(bool(opts.normalize_scales)), int(bool(opts.fix_loadings)),
                     _prec(precision))
    nll = np.zeros((B, iters + 1)) if fit.record_trace else None
    status = np.zeros(B * F, np.int32)
    ctx = _lib.context(device)
    fn = _lib.lib().ffca_fit if ins[0][2] else _lib.lib().ffca_fit_covs
    _lib.check(fn(ctx.handle, d, o, _lib.ptr(x), _lib.ptr(power), _lib.ptr(W), _lib.ptr(L),
                  _lib.ptr(H), _lib.ptr(nll), None, _lib.ptr(status)))
    return [FastFcaFitResult(_params_from_ref(W[b], L[b], H[b]),
                             list(nll[b]) if nll is not None else [], status[b * F:(b + 1) * F])
            for b in range(B)]


def ica_mode_fit(covs: SampleCovSet, sources: int, iters: int, w_init: np.ndarray,
                 fit: FitOptions | None = None, *, precision: str = "fp32",
                 device: int | None = None) -> FastFcaFitResult:
    """fastfca.cpp:241-264 on the GPU: determined ICA mode (L = identity, H =
    floored decorrelated powers of w_init, IP+MM with the loadings fixed).
    `precision` is accepted for symmetry with fastfca_fit, but this mode always
    computes in fp64 (ffca.h, ffca_ica_fit: at its fixed point H tracks
    |w^H x|^2 and the 1/H weights amplify fp32 cancellation)."""
    fit = fit or FitOptions()
    if sources != covs.dim:
        raise InvalidArgument("ica_mode_fit: requires as many sources as channels")
    w_init = np.asarray(w_init)
    if w_init.shape[0] != covs.bins:
        raise InvalidArgument("ica_mode_fit: one W per frequency required")
    if iters < 0:
        raise InvalidArgument("fastfca_fit: negative iteration count")
    F, M, T = covs.bins, covs.dim, covs.blocks
    x, power, snap = _covs_input(covs)
    W = np.array(np.swapaxes(w_init, -1, -2), dtype=np.complex128, order="C", copy=True)
    L = np.zeros((F, M, M))
    H = np.zeros((F, T, M))
    d = _lib.Dims(1, F, M, M, T)
    o = _lib.FitOpts(_lib.FLAVOR_MM, int(iters), int(bool(fit.record_trace)), int(fit.seed), 1, 1,
                     _prec(precision))
    nll = np.zeros(iters + 1) if fit.record_trace else None
    status = np.zeros(F, np.int32)
    ctx = _lib.context(device)
    fn = _lib.lib().ffca_ica_fit if snap else _lib.lib().ffca_ica_fit_covs
    _lib.check(fn(ctx.handle, d, o, _lib.ptr(x), _lib.ptr(power),
                                       _lib.ptr(W), _lib.ptr(L), _lib.ptr(H), _lib.ptr(nll), None,
                                       _lib.ptr(status)))
    return FastFcaFitResult(_params_from_ref(W, L, H), list(nll) if nll is not None else [],
                            status)


def decorrelated_powers(covs: SampleCovSet, w: np.ndarray, *, floor_rel: float | None = None,
                        precision: str = "fp64", device: int | None = None) -> np.ndarray:
    """|W^H x|^2 for every bin (sigmodel.cpp:93-107), w [bins, dim, dim];
    floor_positive(u, floor_rel) (sigmodel.cpp:10-15) when floor_rel is given.
    Returns [bins, dim, frames]."""
    F, M, T = covs.bins, covs.dim, covs.blocks
    x = _x_ref(covs.snapshots) if covs.has_snapshots() else _mats_ref(covs.mats)
    W = np.array(np.swapaxes(w, -1, -2), dtype=np.complex128, order="C", copy=True)
    out = np.empty((F, T, M))
    d = _lib.Dims(1, F, M, M, T)
    ctx = _lib.context(device)
    fn = (_lib.lib().ffca_decorrelated_powers if covs.has_snapshots()
          else _lib.lib().ffca_decorrelated_powers_covs)
    _lib.check(fn(
        ctx.handle, d, _prec(precision), _lib.ptr(x), _lib.ptr(W),
        -1.0 if floor_rel is None else float(floor_rel), _lib.ptr(out)))
    return np.ascontiguousarray(np.swapaxes(out, -1, -2))


# ----------------------------------------------------- per-step functions --
# fastfca.hpp:28-53: each a single-bin fp64 launch (csrc/steps.cu).  Arrays are
# the natural layouts (x [dim, frames], w [dim, dim], loading [dim, sources],
# act [sources, frames], u [dim, frames]); results are new arrays.
def _bin_stats(covs: SampleCovSet, i: int):
    if not 0 <= i < covs.bins:
        raise InvalidArgument("bin out of range")
    if covs.has_snapshots():
        return np.ascontiguousarray(covs.snapshots[i].T, np.complex128), 0
    return np.ascontiguousarray(np.swapaxes(covs.mats[i], -1, -2), np.complex128), 1


def _colmajor(a, dtype=np.float64) -> np.ndarray:
    return np.array(np.asarray(a).T, dtype=dtype, order="C", copy=True)


def weighted_cov(covs: SampleCovSet, i: int, sigma2_row, *, device: int | None = None) -> np.ndarray:
    """Q = symmetrize((1/J) sum_j X_j / sigma2_row[j]) (fastfca.cpp:22-34)."""
    x, blk = _bin_stats(covs, i)
    sig = np.ascontiguousarray(np.asarray(sigma2_row, np.float64).ravel())
    if sig.size != covs.blocks:
        raise InvalidArgument("weighted_cov: variance row length mismatch")
    M = covs.dim
    q = np.empty((M, M), np.complex128)
    _lib.check(_lib.lib().ffca_weighted_cov(_lib.context(device).handle, M, covs.blocks, blk,
                                            _lib.ptr(x), _lib.ptr(sig), _lib.ptr(q)))
    return np.ascontiguousarray(q.T)


def ip_update_w(covs: SampleCovSet, i: int, w, loading, act, restart_seed: int = 0, *,
                device: int | None = None) -> np.ndarray:
    """One IP sweep over the columns of w at bin i (fastfca.cpp:36-72); returns the new w."""
    x, blk = _bin_stats(covs, i)
    M = covs.dim
    loading, act = np.asarray(loading), np.asarray(act)
    if np.shape(w) != (M, M) or loading.shape[0] != M or act.shape != (loading.shape[1], covs.blocks):
        raise InvalidArgument("ip_update_w: shape mismatch")
    W, L, H = _colmajor(w, np.complex128), _colmajor(loading), _colmajor(act)
    _lib.check(_lib.lib().ffca_ip_update_w(_lib.context(device).handle, M, loading.shape[1],
                                           covs.blocks, blk, _lib.ptr(x), float(covs.power(i)),
                                           _lib.ptr(W), _lib.ptr(L), _lib.ptr(H),
                                           int(restart_seed), int(i)))
    return np.ascontiguousarray(W.T)


def source_gain(loading, act, n: int, *, device: int | None = None) -> np.ndarray:
    """G_n = L_n H_n / floor_positive(L H) (fastfca.cpp:74-78), [dim, frames]."""
    loading, act = np.asarray(loading), np.asarray(act)
    if act.shape[0] != loading.shape[1]:
        raise InvalidArgument("source_gain: shape mismatch")
    M, N, T = loading.shape[0], loading.shape[1], act.shape[1]
    g = np.empty((T, M))
    L, H = _colmajor(loading), _colmajor(act)
    _lib.check(_lib.lib().ffca_source_gain(_lib.context(device).handle, M, N, T, _lib.ptr(L),
                                           _lib.ptr(H), int(n), _lib.ptr(g)))
    return np.ascontiguousarray(g.T)


def _lh_update(fn, u, loading, act, update_loading, eps, device):
    u, loading, act = np.asarray(u), np.asarray(loading), np.asarray(act)
    M, T = u.shape
    N = loading.shape[1]
    if loading.shape[0] != M or act.shape != (N, T):
        raise InvalidArgument("lh update: shape mismatch")
    U, L, H = _colmajor(u), _colmajor(loading), _colmajor(act)
    _lib.check(fn(_lib.context(device).handle, M, N, T, _lib.ptr(U), _lib.ptr(L), _lib.ptr(H),
                  1 if update_loading else 0, float(eps)))
    return np.ascontiguousarray(L.T), np.ascontiguousarray(H.T)


def em_update_lh(u, loading, act, update_loading: bool = True, eps: float = 0.0, *,
                 device: int | None = None):
    """em_update_lh (fastfca.cpp:80-99); returns the new (loading, act)."""
    return _lh_update(_lib.lib().ffca_em_update_lh, u, loading, act, update_loading, eps, device)


def mm_update_lh(u, loading, act, update_loading: bool = True, eps: float = 0.0, *,
                 device: int | None = None):
    """mm_update_lh (fastfca.cpp:101-117); returns the new (loading, act)."""
    return _lh_update(_lib.lib().ffca_mm_update_lh, u, loading, act, update_loading, eps, device)


def log_abs_det2(w, *, device: int | None = None) -> float:
    """ln|det w|^2 (sigmodel.cpp:118-129); NumericalError when singular."""
    W = _colmajor(w, np.complex128)
    out = np.zeros(1)
    _lib.check(_lib.lib().ffca_log_abs_det2(_lib.context(device).handle, W.shape[0], _lib.ptr(W),
                                            _lib.ptr(out)))
    return float(out[0])


# ------------------------------------------------------------------- stft --
def sqrt_hann_window(frame_len: int) -> np.ndarray:
    """stft.cpp:33-39 (a constant table)."""
    k = np.arange(frame_len)
    return np.sqrt(0.5 - 0.5 * np.cos(2.0 * np.pi * k / frame_len))


def stft_frame_count(length: int, frame_len: int, shift: int,
                     pad: int = StftPadding.centered) -> int:
    """stft.cpp:41-49."""
    n = _lib.lib().ffca_stft_frame_count(int(length), int(frame_len), int(shift), int(pad))
    if n < 0:
        raise InvalidArgument(_lib.lib().ffca_last_error().decode())
    return int(n)


def stft(wave: MultichannelWave, frame_len: int, shift: int, pad: int = StftPadding.centered,
         *, device: int | None = None) -> Spectrogram:
    """stft.cpp:51-83 on the GPU (fp64 FFTs)."""
    C, n = wave.samples.shape
    s = np.ascontiguousarray(np.asarray(wave.samples, np.float64).T)  # [length][channels]
    if frame_len > 0 and not (frame_len & (frame_len - 1)) and shift * 2 == frame_len and n >= frame_len:
        frames = stft_frame_count(n, frame_len, shift, pad)
    else:
        frames = 1  # the library raises the reference's error
    out = np.empty((frame_len // 2 + 1 if frame_len > 0 else 1, frames, C), np.complex128)
    ctx = _lib.context(device)
    _lib.check(_lib.lib().ffca_stft(ctx.handle, C, n, int(frame_len), int(shift), int(pad),
                                    _lib.ptr(s), _lib.ptr(out)))
    return Spectrogram(np.ascontiguousarray(np.swapaxes(out, 1, 2)))


def istft(spec: Spectrogram, frame_len: int, shift: int, out_len: int, sample_rate: float,
          pad: int = StftPadding.centered, *, device: int | None = None) -> MultichannelWave:
    """stft.cpp:85-128 on the GPU."""
    x = np.ascontiguousarray(np.swapaxes(spec.f, 1, 2), dtype=np.complex128)  # [bins][frames][C]
    out = np.zeros((out_len, spec.channels))
    ctx = _lib.context(device)
    _lib.check(_lib.lib().ffca_istft(ctx.handle, spec.channels, spec.bins, spec.frames,
                                     int(frame_len), int(shift), int(pad), int(out_len),
                                     _lib.ptr(x), _lib.ptr(out)))
    return MultichannelWave(np.ascontiguousarray(out.T), sample_rate)


def fastfca_separate(spec: Spectrogram, params: FastFcaParams, *, precision: str = "fp32",
                     device: int | None = None) -> list[Spectrogram]:
    """fastfca.cpp:205-223: decorrelate, per-channel Wiener gains, project back."""
    if spec.channels != params.dim or spec.bins != params.bins or spec.frames != params.frames:
        raise InvalidArgument("fastfca_separate: shape mismatch")
    x = _x_ref(spec.f)
    W, L, H = _params_ref(params)
    N, F, T, M = params.sources, spec.bins, spec.frames, spec.channels
    out = np.empty((N, F, T, M), np.complex128)
    d = _lib.Dims(1, F, M, N, T)
    ctx = _lib.context(device)
    _lib.check(_lib.lib().ffca_separate(ctx.handle, d, _prec(precision), _lib.ptr(x),
                                        _lib.ptr(W), _lib.ptr(L), _lib.ptr(H), _lib.ptr(out)))
    return [Spectrogram(np.ascontiguousarray(np.swapaxes(out[n], -1, -2))) for n in range(N)]


def fastfca_nll_bins(covs: SampleCovSet, params: FastFcaParams, *, precision: str = "fp32",
                     device: int | None = None) -> np.ndarray:
    """fastfca_nll_freq for every bin (sigmodel.cpp:155-162)."""
    _check_shape(covs, params, "nll")
    snap = covs.has_snapshots()
    x = _x_ref(covs.snapshots) if snap else _mats_ref(covs.mats)
    W, L, H = _params_ref(params)
    out = np.empty(covs.bins)
    d = _lib.Dims(1, covs.bins, covs.dim, params.sources, covs.blocks)
    ctx = _lib.context(device)
    fn = _lib.lib().ffca_nll_bins if snap else _lib.lib().ffca_nll_bins_covs
    _lib.check(fn(ctx.handle, d, _prec(precision), _lib.ptr(x),
                                        _lib.ptr(W), _lib.ptr(L), _lib.ptr(H), _lib.ptr(out)))
    return out


def fastfca_nll(covs: SampleCovSet, params: FastFcaParams, **kw) -> float:
    """sigmodel.cpp:215-222 (bin-order sum)."""
    return float(sum(fastfca_nll_bins(covs, params, **kw)))
