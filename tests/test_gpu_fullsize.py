"""Parity at BASELINE.json's full sizes.  The whole configuration is fitted on
the GPU (device-resident path, as bench.py runs it); since frequency bins are
independent (fastfca.cpp:158-184), a few of its bins -- first, middle, last
-- are refitted by the fp64 oracle on their own and their per-bin NLL slots
compared (1e-5 relative per iteration, the fp32 tolerance).  Over all bins:
every bin converges without a numerical error and the bin-order trace is
non-increasing (size-independent properties of the EM/IP majorisation).
c4 (256 mixtures) is represented by its first 8 mixtures."""
import dataclasses

import numpy as np
import pytest

import oracle
from paper_2101_08563_b200 import _lib, synth
from paper_2101_08563_b200.shard import bin_order_trace

pytestmark = pytest.mark.gpu


def _device_fit(cfg, x, W0, L0, H0):
    import torch
    dev = torch.device("cuda", 0)
    P, M, N, T, iters = x.shape[0], cfg.M, cfg.N, cfg.T, cfg.iters
    xd = torch.from_numpy(np.ascontiguousarray(np.swapaxes(x, -1, -2))).to(dev, torch.complex64)
    Hd = torch.from_numpy(np.ascontiguousarray(np.swapaxes(H0, -1, -2))).to(dev, torch.float32)
    Wd = torch.from_numpy(np.ascontiguousarray(np.swapaxes(W0, -1, -2))).to(dev)
    Ld = torch.from_numpy(np.ascontiguousarray(np.swapaxes(L0, -1, -2))).to(dev)
    power = torch.empty(P, dtype=torch.float64, device=dev)
    slots = torch.zeros((iters + 1, P), dtype=torch.float64, device=dev)
    status = torch.zeros(P, dtype=torch.int32, device=dev)
    ctx = _lib.context(0)
    L_ = _lib.lib()
    st = torch.cuda.Stream(dev)
    with torch.cuda.stream(st):
        _lib.check(L_.ffca_power_scale_device(ctx.handle, P, M, T, _lib.PREC_FP32, _lib.ptr(xd),
                                              _lib.ptr(power), st.cuda_stream))
        o = _lib.FitOpts(_lib.FLAVOR_EM, iters, 1, 0, 1, 0, _lib.PREC_FP32)
        _lib.check(L_.ffca_fit_device(ctx.handle, P, cfg.F, 0, M, N, T, o, _lib.ptr(xd),
                                      _lib.ptr(power), _lib.ptr(Wd), _lib.ptr(Ld), _lib.ptr(Hd),
                                      _lib.ptr(slots), _lib.ptr(status), st.cuda_stream))
    torch.cuda.synchronize()
    return slots.cpu().numpy(), status.cpu().numpy()


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3", "c4"])
def test_full_size_config(gpu, name):
    cfg = synth.CONFIGS[name]
    B = min(cfg.batch, 8)
    xs, Ws, Ls, Hs = [], [], [], []
    for b in range(B):
        xs.append(synth.mixture(cfg, b))
        W, L, H = synth.init_params(cfg, b)
        Ws.append(W); Ls.append(L); Hs.append(H)
    x, W0, L0, H0 = (np.concatenate(v) for v in (xs, Ws, Ls, Hs))
    slots, status = _device_fit(cfg, x, W0, L0, H0)
    assert (status == 0).all(), np.unique(status)
    trace = bin_order_trace(slots, B, cfg.F)
    assert (trace[1:] <= trace[:-1] + 1e-5 * np.abs(trace[:-1])).all()
    for p in sorted({0, x.shape[0] // 2, x.shape[0] - 1}):
        _, _, _, nll_o, _, _ = oracle.fit(x[p:p + 1].astype(np.complex128), W0[p:p + 1],
                                          L0[p:p + 1], H0[p:p + 1], cfg.iters, workers=1)
        rel = np.abs(slots[:, p] - nll_o) / np.abs(nll_o)
        assert rel.max() <= 1e-5, (p, rel.max())
