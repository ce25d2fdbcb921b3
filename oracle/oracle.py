"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of liboracle.so, the fp64 CPU
restatement of the reference FastFCA path (oracle.cpp; citations there).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this module, and only as the checker or the
timed CPU baseline.  Arrays use the same natural numpy layout as
paper_2101_08563_b200.api (x [bins, dim, frames], W [bins, dim, dim],
L [bins, dim, sources], H [bins, sources, frames]).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-s", "-C", str(HERE), "liboracle.so"], check=True)
        L = C.CDLL(str(LIB))
        P, i, d, u64 = C.c_void_p, C.c_int, C.c_double, C.c_uint64
        L.oracle_default_workers.restype = i
        L.oracle_power_scale.argtypes = [i, i, i, P, P, P, i]
        L.oracle_fit.argtypes = [i, i, i, i, i, P, P, P, P, i, i, i, u64, i, i, i, P, P, P, P, i]
        L.oracle_nll_bins.argtypes = [i, i, i, i, P, P, P, P, P, P, i]
        L.oracle_fca_nll_jd.argtypes = [i, i, i, i, P, P, P, P, P, P, i]
        L.oracle_separate.argtypes = [i, i, i, i, P, P, P, P, P, P, i]
        L.oracle_ip_update_w.argtypes = [i, i, i, P, P, P, P, u64, P, i]
        L.oracle_lh_update.argtypes = [i, i, i, i, P, P, P, i, d, P, i]
        L.oracle_source_gain.argtypes = [i, i, i, P, P, i, P, P, i]
        L.oracle_ica_fit.argtypes = [i, i, i, i, P, P, P, P, i, i, u64, i, P, P, i]
        L.oracle_decorrelated_powers.argtypes = [i, i, i, P, P, d, P, P, i]
        L.oracle_block_covs.argtypes = [i, i, i, i, P, P, P, P, i]
        L.oracle_fit_covs.argtypes = [i, i, i, i, P, P, P, P, P, i, i, i, u64, i, i, i, i, P, P,
                                      P, i]
        L.oracle_nll_bins_covs.argtypes = [i, i, i, i, P, P, P, P, P, P, i]
        L.oracle_decorrelated_powers_covs.argtypes = [i, i, i, P, P, d, P, P, i]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _call(fn, *args):
    err = C.create_string_buffer(512)
    rc = fn(*args, err, 512)
    if rc != 0:
        raise OracleError(rc, err.value.decode())


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def _xref(x: np.ndarray) -> np.ndarray:
    return np.array(np.swapaxes(x, -1, -2), dtype=np.complex128, order="C", copy=True)


def _pref(W, L, H):
    # Always copies: for size-1 axes swapaxes is already contiguous and a view
    # would let the in/out buffers alias the caller's arrays.
    return (np.array(np.swapaxes(W, -1, -2), dtype=np.complex128, order="C", copy=True),
            np.array(np.swapaxes(L, -1, -2), dtype=np.float64, order="C", copy=True),
            np.array(np.swapaxes(H, -1, -2), dtype=np.float64, order="C", copy=True))


def default_workers() -> int:
    return lib().oracle_default_workers()


def power_scale(x: np.ndarray) -> np.ndarray:
    F, M, T = x.shape
    out = np.empty(F)
    xr = _xref(x)  # keep the buffer alive across the call
    _call(lib().oracle_power_scale, F, M, T, _p(xr), _p(out))
    return out


def fit(x, W, L, H, iters, flavor=0, record_trace=True, seed=0, normalize_scales=True,
        fix_loadings=False, workers=1, slots=False):
    """fastfca_fit on one mixture (x [F,M,T]) or a batch (x [B,F,M,T]).
    Returns (W, L, H, nll [B][iters+1] or [iters+1], slots or None, fit_seconds)."""
    batched = x.ndim == 4
    if not batched:
        x, W, L, H = x[None], W[None], L[None], H[None]
    B, F, M, T = x.shape
    N = L.shape[-1]
    xr = _xref(x)
    Wr, Lr, Hr = _pref(W, L, H)
    nll = np.zeros((B, iters + 1))
    sl = np.zeros((B, iters + 1, F)) if slots else None
    secs = C.c_double(0.0)
    _call(lib().oracle_fit, B, F, M, N, T, _p(xr), _p(Wr), _p(Lr), _p(Hr), int(flavor),
          int(iters), int(record_trace), int(seed), int(normalize_scales), int(fix_loadings),
          int(workers), _p(nll), _p(sl), C.addressof(secs))
    Wo = np.swapaxes(Wr, -1, -2)
    Lo = np.swapaxes(Lr, -1, -2)
    Ho = np.swapaxes(Hr, -1, -2)
    if not batched:
        return Wo[0], Lo[0], Ho[0], nll[0], (sl[0] if slots else None), secs.value
    return Wo, Lo, Ho, nll, sl, secs.value


def ica_fit(x, W_init, iters, record_trace=True, seed=0, workers=1):
    """ica_mode_fit (fastfca.cpp:241-264) on one mixture x [F,M,T] from W_init
    [F,M,M].  Returns (W, L, H, nll)."""
    F, M, T = x.shape
    xr = _xref(x)
    Wr = np.array(np.swapaxes(W_init, -1, -2), dtype=np.complex128, order="C", copy=True)
    Lr = np.zeros((F, M, M))
    Hr = np.zeros((F, T, M))
    nll = np.zeros(iters + 1)
    _call(lib().oracle_ica_fit, F, M, M, T, _p(xr), _p(Wr), _p(Lr), _p(Hr), int(iters),
          int(record_trace), int(seed), int(workers), _p(nll))
    return (np.swapaxes(Wr, -1, -2), np.swapaxes(Lr, -1, -2), np.swapaxes(Hr, -1, -2), nll)


def decorrelated_powers(x, W, floor_rel=1e-12):
    """|W^H x|^2 per bin (sigmodel.cpp:93-107), floored as floor_positive
    (sigmodel.cpp:10-15) unless floor_rel is None.  Returns [F,M,T]."""
    F, M, T = x.shape
    xr = _xref(x)
    Wr = np.array(np.swapaxes(W, -1, -2), dtype=np.complex128, order="C", copy=True)
    out = np.zeros((F, T, M))
    _call(lib().oracle_decorrelated_powers, F, M, T, _p(xr), _p(Wr),
          -1.0 if floor_rel is None else float(floor_rel), _p(out))
    return np.swapaxes(out, -1, -2)


def nll_bins(x, W, L, H) -> np.ndarray:
    F, M, T = x.shape
    N = L.shape[-1]
    Wr, Lr, Hr = _pref(W, L, H)
    out = np.empty(F)
    xr = _xref(x)
    _call(lib().oracle_nll_bins, F, M, N, T, _p(xr), _p(Wr), _p(Lr), _p(Hr), _p(out))
    return out


def fca_nll_jd(x, W, L, H) -> float:
    F, M, T = x.shape
    N = L.shape[-1]
    Wr, Lr, Hr = _pref(W, L, H)
    out = np.zeros(1)
    xr = _xref(x)
    _call(lib().oracle_fca_nll_jd, F, M, N, T, _p(xr), _p(Wr), _p(Lr), _p(Hr), _p(out))
    return float(out[0])


def separate(x, W, L, H) -> np.ndarray:
    """Images, natural layout [N, F, M, T] complex128."""
    F, M, T = x.shape
    N = L.shape[-1]
    Wr, Lr, Hr = _pref(W, L, H)
    out = np.empty((N, F, T, M), np.complex128)
    xr = _xref(x)
    _call(lib().oracle_separate, F, M, N, T, _p(xr), _p(Wr), _p(Lr), _p(Hr), _p(out))
    return np.swapaxes(out, -1, -2)


# ------------------------------------------------ block-stationary input --
def _mref(mats):
    """[F, J, M, M] natural -> per-block Eigen col-major complex128."""
    return np.array(np.swapaxes(mats, -1, -2), dtype=np.complex128, order="C", copy=True)


def block_covs(x, block_size):
    """sample_covs(spec, block_size) (sigmodel.cpp:17-48) on x [F,M,T]:
    (mats [F, J, M, M] natural layout, power_scale [F])."""
    F, M, T = x.shape
    J = -(-T // block_size)
    mats = np.zeros((F, J, M, M), np.complex128)
    power = np.zeros(F)
    xr = _xref(x)
    _call(lib().oracle_block_covs, F, M, T, int(block_size), _p(xr), _p(mats), _p(power))
    return np.swapaxes(mats, -1, -2), power


def fit_covs(mats, W, L, H, iters, flavor=0, power=None, record_trace=True, seed=0,
             normalize_scales=True, fix_loadings=False, workers=1, slots=False):
    """fastfca_fit on block covariances mats [F, J, M, M] (H [F, N, J]).
    Returns (W, L, H, nll, slots or None)."""
    F, J, M, _ = mats.shape
    N = L.shape[-1]
    mr = _mref(mats)
    Wr, Lr, Hr = _pref(W, L, H)
    nll = np.zeros(iters + 1)
    sl = np.zeros((iters + 1, F)) if slots else None
    pw = None if power is None else np.ascontiguousarray(power, np.float64)
    _call(lib().oracle_fit_covs, F, M, N, J, _p(mr), _p(pw), _p(Wr), _p(Lr), _p(Hr), int(flavor),
          int(iters), int(record_trace), int(seed), int(normalize_scales), int(fix_loadings),
          int(workers), 0, _p(nll), _p(sl))
    return (np.swapaxes(Wr, -1, -2), np.swapaxes(Lr, -1, -2), np.swapaxes(Hr, -1, -2), nll, sl)


def ica_fit_covs(mats, W_init, iters, power=None, record_trace=True, seed=0, workers=1):
    """ica_mode_fit on block covariances.  Returns (W, L, H, nll)."""
    F, J, M, _ = mats.shape
    mr = _mref(mats)
    Wr = np.array(np.swapaxes(W_init, -1, -2), dtype=np.complex128, order="C", copy=True)
    Lr = np.zeros((F, M, M))
    Hr = np.zeros((F, J, M))
    nll = np.zeros(iters + 1)
    pw = None if power is None else np.ascontiguousarray(power, np.float64)
    _call(lib().oracle_fit_covs, F, M, M, J, _p(mr), _p(pw), _p(Wr), _p(Lr), _p(Hr), 1,
          int(iters), int(record_trace), int(seed), 1, 1, int(workers), 1, _p(nll), None)
    return (np.swapaxes(Wr, -1, -2), np.swapaxes(Lr, -1, -2), np.swapaxes(Hr, -1, -2), nll)


def nll_bins_covs(mats, W, L, H) -> np.ndarray:
    F, J, M, _ = mats.shape
    N = L.shape[-1]
    mr = _mref(mats)
    Wr, Lr, Hr = _pref(W, L, H)
    out = np.empty(F)
    _call(lib().oracle_nll_bins_covs, F, M, N, J, _p(mr), _p(Wr), _p(Lr), _p(Hr), _p(out))
    return out


def decorrelated_powers_covs(mats, W, floor_rel=1e-12):
    F, J, M, _ = mats.shape
    mr = _mref(mats)
    Wr = np.array(np.swapaxes(W, -1, -2), dtype=np.complex128, order="C", copy=True)
    out = np.zeros((F, J, M))
    _call(lib().oracle_decorrelated_powers_covs, F, M, J, _p(mr), _p(Wr),
          -1.0 if floor_rel is None else float(floor_rel), _p(out))
    return np.swapaxes(out, -1, -2)
