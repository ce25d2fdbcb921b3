"""Parity at BASELINE.json's full sizes.  The whole configuration is fitted and
separated on the GPU (device-resident path, as bench.py runs it); since
frequency bins are independent (fastfca.cpp:158-184), a few of its bins --
first, middle, last -- are refitted and separated by the fp64 oracle on their
own and compared: per-bin NLL slots per iteration (1e-5 relative in the fp32
path, 1e-10 in the fp64 check mode) and the separated source images after
the configured iterations (1e-3 / 1e-10 relative L2, BASELINE.json
north_star).  Over ALL bins and mixtures (c4: all 256): every bin converges
without a numerical error, the bin-order trace of every mixture is
non-increasing, and the separated images of the sampled bins sum to the
mixture (size-independent properties of the EM/IP majorisation and the
Wiener partition)."""
import concurrent.futures as cf
import os

import numpy as np
import pytest

import oracle
from paper_2101_08563_b200 import _lib, synth
from paper_2101_08563_b200.shard import bin_order_trace

pytestmark = pytest.mark.gpu

NLL_TOL = {"fp32": 1e-5, "fp64": 1e-10}
SEP_TOL = {"fp32": 1e-3, "fp64": 1e-10}


def _inputs(cfg):
    def one(b):
        x = synth.mixture(cfg, b)
        return (x,) + synth.init_params(cfg, b)
    if cfg.batch == 1:
        parts = [one(0)]
    else:  # c4: 256 independently seeded mixtures
        with cf.ThreadPoolExecutor(min(16, os.cpu_count() or 4)) as ex:
            parts = list(ex.map(one, range(cfg.batch)))
    return tuple(np.concatenate([p[k] for p in parts]) for k in range(4))


def _device_fit_separate(cfg, x, W0, L0, H0, precision, sample):
    """Fit and separate every problem on the device; returns the NLL slots,
    the status words and the separated images of the `sample` problems."""
    import torch
    dev = torch.device("cuda", 0)
    fp64 = precision == "fp64"
    prec = _lib.PREC_FP64 if fp64 else _lib.PREC_FP32
    cdt, rdt = (torch.complex128, torch.float64) if fp64 else (torch.complex64, torch.float32)
    P, M, N, T, iters = x.shape[0], cfg.M, cfg.N, cfg.T, cfg.iters
    xd = torch.from_numpy(np.ascontiguousarray(np.swapaxes(x, -1, -2))).to(dev, cdt)
    Hd = torch.from_numpy(np.ascontiguousarray(np.swapaxes(H0, -1, -2))).to(dev, rdt)
    Wd = torch.from_numpy(np.ascontiguousarray(np.swapaxes(W0, -1, -2))).to(dev)
    Ld = torch.from_numpy(np.ascontiguousarray(np.swapaxes(L0, -1, -2))).to(dev)
    power = torch.empty(P, dtype=torch.float64, device=dev)
    slots = torch.zeros((iters + 1, P), dtype=torch.float64, device=dev)
    status = torch.zeros(P, dtype=torch.int32, device=dev)
    img = torch.empty((N, P, T, M), dtype=cdt, device=dev)
    ctx = _lib.context(0)
    L_ = _lib.lib()
    st = torch.cuda.Stream(dev)
    with torch.cuda.stream(st):
        _lib.check(L_.ffca_power_scale_device(ctx.handle, P, M, T, prec, _lib.ptr(xd),
                                              _lib.ptr(power), st.cuda_stream))
        o = _lib.FitOpts(_lib.FLAVOR_EM, iters, 1, 0, 1, 0, prec)
        _lib.check(L_.ffca_fit_device(ctx.handle, P, cfg.F, 0, M, N, T, o, _lib.ptr(xd),
                                      _lib.ptr(power), _lib.ptr(Wd), _lib.ptr(Ld), _lib.ptr(Hd),
                                      _lib.ptr(slots), _lib.ptr(status), st.cuda_stream))
        _lib.check(L_.ffca_separate_device(ctx.handle, P, M, N, T, prec, _lib.ptr(xd),
                                           _lib.ptr(Wd), _lib.ptr(Ld), _lib.ptr(Hd),
                                           _lib.ptr(img), st.cuda_stream))
    torch.cuda.synchronize()
    images = {p: np.swapaxes(img[:, p].cpu().numpy(), -1, -2) for p in sample}  # [N, M, T]
    out = slots.cpu().numpy(), status.cpu().numpy(), images
    del img, xd, Hd
    torch.cuda.empty_cache()
    return out


def _check(cfg, precision):
    x, W0, L0, H0 = _inputs(cfg)
    P = x.shape[0]
    sample = sorted({0, P // 2, P - 1})
    slots, status, images = _device_fit_separate(cfg, x, W0, L0, H0, precision, sample)
    assert (status == 0).all(), np.unique(status)
    trace = bin_order_trace(slots, cfg.batch, cfg.F)  # [iters+1, batch]: every mixture
    assert trace.shape[1] == cfg.batch
    assert (trace[1:] <= trace[:-1] + 1e-5 * np.abs(trace[:-1])).all()
    for p in sample:
        xp = x[p:p + 1].astype(np.complex128)
        Wo, Lo, Ho, nll_o, _, _ = oracle.fit(xp, W0[p:p + 1], L0[p:p + 1], H0[p:p + 1], cfg.iters,
                                             workers=1)
        rel = np.abs(slots[:, p] - nll_o) / np.abs(nll_o)
        assert rel.max() <= NLL_TOL[precision], (p, rel.max())
        img_o = oracle.separate(xp, Wo, Lo, Ho)  # [N][1, M, T]
        for n in range(cfg.N):
            ref = np.asarray(img_o[n])[0]
            err = np.linalg.norm(images[p][n] - ref) / max(np.linalg.norm(ref), 1e-300)
            assert err <= SEP_TOL[precision], (p, n, err)
        part = np.linalg.norm(images[p].sum(0) - xp[0]) / np.linalg.norm(xp[0])
        assert part <= (1e-5 if precision == "fp32" else 1e-12), (p, part)


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3", "c4"])
def test_full_size_config(gpu, name):
    _check(synth.CONFIGS[name], "fp32")


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_full_size_config_fp64_check_mode(gpu, name):
    _check(synth.CONFIGS[name], "fp64")
