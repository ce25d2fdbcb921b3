"""ctypes binding of libffca.so (include/ffca.h).

The product path is the CUDA library; this module only marshals pointers.
Loading fails loudly if the library is missing, and every compute entry point
raises if no B200 is present -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

# FFCA_LIB selects a diagnostics build (e.g. libffca_timing.so); default is
# the production library.
LIB_PATH = Path(os.environ.get("FFCA_LIB", Path(__file__).resolve().parent / "libffca.so"))

OK, INVALID_ARGUMENT, NUMERICAL, CUDA_ERROR = 0, 1, 2, 3
FLAVOR_EM, FLAVOR_MM = 0, 1
PREC_FP32, PREC_FP64 = 0, 1
BIN_OK, BIN_SILENT, BIN_IP_SINGULAR, BIN_SINGULAR_W = 0, 1, 2, 3

# Every symbol include/ffca.h declares (checked by tests/test_capi_exports.py).
EXPORTS = (
    "ffca_version", "ffca_last_error", "ffca_device_count", "ffca_ctx_create",
    "ffca_ctx_destroy", "ffca_fit", "ffca_separate", "ffca_nll_bins", "ffca_power_scale",
    "ffca_fit_device", "ffca_separate_device", "ffca_power_scale_device",
    "ffca_last_launch_count", "ffca_debug_set_timing", "ffca_ica_fit", "ffca_decorrelated_powers",
    "ffca_stft_frame_count", "ffca_stft", "ffca_istft", "ffca_stft_device", "ffca_istft_device",
    "ffca_block_covs", "ffca_fit_covs", "ffca_ica_fit_covs", "ffca_nll_bins_covs",
    "ffca_decorrelated_powers_covs", "ffca_block_covs_device", "ffca_fit_covs_device",
    "ffca_weighted_cov", "ffca_ip_update_w", "ffca_source_gain", "ffca_em_update_lh",
    "ffca_mm_update_lh", "ffca_log_abs_det2", "ffca_debug_restart_draws",
    "ffca_pinned_buffer", "ffca_mwf", "ffca_reconstruct_scms", "ffca_ajd_cost",
    "ffca_fit_bins",
)
STFT_CENTERED, STFT_FULL_FRAMES = 0, 1


class FfcaError(RuntimeError):
    pass


class InvalidArgument(FfcaError, ValueError):
    """The reference's std::invalid_argument (shape / option errors)."""


class NumericalError(FfcaError):
    """The reference's fastfca::NumericalError (types.hpp:21-24)."""


class CudaError(FfcaError):
    pass


class Dims(C.Structure):
    _fields_ = [("batch", C.c_int), ("bins", C.c_int), ("dim", C.c_int),
                ("sources", C.c_int), ("frames", C.c_int), ("first_bin", C.c_int),
                ("mixture_bins", C.c_int)]


class FitOpts(C.Structure):
    _fields_ = [("flavor", C.c_int), ("iters", C.c_int), ("record_trace", C.c_int),
                ("seed", C.c_uint64), ("normalize_scales", C.c_int),
                ("fix_loadings", C.c_int), ("precision", C.c_int)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FfcaError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                            "(no CPU fallback exists)")
        L = C.CDLL(str(LIB_PATH))
        P = C.c_void_p
        dp = C.POINTER(C.c_double)
        L.ffca_version.restype = C.c_int
        L.ffca_last_error.restype = C.c_char_p
        L.ffca_device_count.restype = C.c_int
        L.ffca_ctx_create.argtypes = [C.c_int, C.POINTER(P)]
        L.ffca_ctx_destroy.argtypes = [P]
        L.ffca_ctx_destroy.restype = None
        L.ffca_fit.argtypes = [P, C.POINTER(Dims), C.POINTER(FitOpts), P, P, P, P, P, P, P, P]
        L.ffca_separate.argtypes = [P, C.POINTER(Dims), C.c_int, P, P, P, P, P]
        L.ffca_nll_bins.argtypes = [P, C.POINTER(Dims), C.c_int, P, P, P, P, P]
        L.ffca_power_scale.argtypes = [P, C.POINTER(Dims), P, P]
        L.ffca_ica_fit.argtypes = [P, C.POINTER(Dims), C.POINTER(FitOpts), P, P, P, P, P, P, P, P]
        L.ffca_decorrelated_powers.argtypes = [P, C.POINTER(Dims), C.c_int, P, P, C.c_double, P]
        L.ffca_block_covs.argtypes = [P, C.POINTER(Dims), C.c_int, P, P, P]
        L.ffca_fit_covs.argtypes = [P, C.POINTER(Dims), C.POINTER(FitOpts), P, P, P, P, P, P, P, P]
        L.ffca_ica_fit_covs.argtypes = [P, C.POINTER(Dims), C.POINTER(FitOpts), P, P, P, P, P, P,
                                        P, P]
        L.ffca_nll_bins_covs.argtypes = [P, C.POINTER(Dims), C.c_int, P, P, P, P, P]
        L.ffca_decorrelated_powers_covs.argtypes = [P, C.POINTER(Dims), C.c_int, P, P, C.c_double,
                                                    P]
        L.ffca_block_covs_device.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P, P,
                                             P, P]
        L.ffca_fit_covs_device.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_int, C.POINTER(FitOpts), P, P, P, P, P, P, P, P]
        i, ll = C.c_int, C.c_longlong
        L.ffca_stft_frame_count.argtypes = [ll, i, i, i]
        L.ffca_stft_frame_count.restype = ll
        L.ffca_stft.argtypes = [P, i, ll, i, i, i, P, P]
        L.ffca_istft.argtypes = [P, i, i, i, i, i, i, ll, P, P]
        L.ffca_stft_device.argtypes = [P, i, ll, i, i, i, i, P, P, P]
        L.ffca_istft_device.argtypes = [P, i, i, i, i, i, ll, i, P, P, P]
        L.ffca_fit_device.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(FitOpts), P, P, P, P, P, P, P, P]
        L.ffca_separate_device.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                           P, P, P, P, P, P]
        L.ffca_power_scale_device.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, P, P, P]
        L.ffca_last_launch_count.argtypes = [P]
        L.ffca_weighted_cov.argtypes = [P, i, i, i, P, P, P]
        L.ffca_ip_update_w.argtypes = [P, i, i, i, i, P, C.c_double, P, P, P, C.c_uint64, i]
        L.ffca_source_gain.argtypes = [P, i, i, i, P, P, i, P]
        L.ffca_em_update_lh.argtypes = [P, i, i, i, P, P, P, i, C.c_double]
        L.ffca_mm_update_lh.argtypes = [P, i, i, i, P, P, P, i, C.c_double]
        L.ffca_log_abs_det2.argtypes = [P, i, P, P]
        L.ffca_fit_bins.argtypes = [P, C.POINTER(Dims), C.POINTER(FitOpts)] + [P] * 11 + [i]
        L.ffca_mwf.argtypes = [P, i, i, P, P, P, i, P]
        L.ffca_reconstruct_scms.argtypes = [P, i, i, i, P, P, P]
        L.ffca_ajd_cost.argtypes = [P, i, i, P, P, P, P]
        L.ffca_pinned_buffer.argtypes = [P, i, C.c_size_t]
        L.ffca_pinned_buffer.restype = P
        L.ffca_debug_restart_draws.argtypes = [P, C.c_uint64, i, i, P, P, P]
        L.ffca_debug_set_timing.argtypes = [P, P]
        _ = dp
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().ffca_last_error().decode(errors="replace")
    raise {INVALID_ARGUMENT: InvalidArgument, NUMERICAL: NumericalError}.get(rc, CudaError)(msg)


def ptr(a) -> int | None:
    """Address of a contiguous numpy array or torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
        return a.ctypes.data
    return int(a.data_ptr())


class Context:
    """One device's stream + buffers (ffca_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().ffca_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device

    def close(self) -> None:
        if getattr(self, "handle", None):
            lib().ffca_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launches(self) -> int:
        return lib().ffca_last_launch_count(self.handle)


_ctx_cache: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    if device is None:
        device = int(os.environ.get("FFCA_DEVICE", "0"))
    c = _ctx_cache.get(device)
    if c is None:
        c = _ctx_cache[device] = Context(device)
    return c
