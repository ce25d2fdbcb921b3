"""e2e probe: the reference-facing ffca_fit on pinned host buffers for c1,
timed on the host for several FFCA_FIT_CHUNKS settings, plus the raw pinned
H2D/D2H bandwidth of the box."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    from paper_2101_08563_b200 import _lib, synth
    cfg = synth.CONFIGS["c1"]
    x = synth.mixture(cfg)
    W0, L0, H0 = synth.init_params(cfg)
    F, M, N, T, iters = cfg.F, cfg.M, cfg.N, cfg.T, cfg.iters
    xr = torch.from_numpy(np.ascontiguousarray(np.swapaxes(x, -1, -2)).astype(np.complex128)).pin_memory()
    Wr = torch.from_numpy(np.ascontiguousarray(np.swapaxes(W0, -1, -2))).pin_memory()
    Lr = torch.from_numpy(np.ascontiguousarray(np.swapaxes(L0, -1, -2))).pin_memory()
    Hr0 = torch.from_numpy(np.ascontiguousarray(np.swapaxes(H0, -1, -2)))
    Hr = Hr0.clone().pin_memory()
    Wp, Lp = Wr.clone().pin_memory(), Lr.clone().pin_memory()
    nll = torch.zeros(iters + 1, dtype=torch.float64).pin_memory()
    d = _lib.Dims(1, F, M, N, T)
    opts = _lib.FitOpts(_lib.FLAVOR_EM, iters, 1, 0, 1, 0, _lib.PREC_FP32)
    ctx = _lib.Context(0)
    L_ = _lib.lib()
    for k in (1, 4):
        os.environ["FFCA_FIT_CHUNKS"] = str(k)
        ts = []
        for i in range(8):
            Hr.copy_(Hr0); Wp.copy_(Wr); Lp.copy_(Lr)
            t0 = time.perf_counter()
            _lib.check(L_.ffca_fit(ctx.handle, d, opts, _lib.ptr(xr), None, _lib.ptr(Wp), _lib.ptr(Lp),
                                   _lib.ptr(Hr), _lib.ptr(nll), None, None))
            ts.append(time.perf_counter() - t0)
        print(f"chunks {k}: e2e ms {['%.3f' % (1e3 * t) for t in ts[3:]]}")
    dev = torch.device("cuda", 0)
    big = torch.empty(xr.numel() * 2, dtype=torch.float64).pin_memory()
    g = torch.empty_like(big, device=dev)
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter(); g.copy_(big, non_blocking=True)
        torch.cuda.synchronize(); t1 = time.perf_counter(); big.copy_(g, non_blocking=True)
        torch.cuda.synchronize(); t2 = time.perf_counter()
    nb = big.numel() * 8
    print(f"pinned H2D {nb / (t1 - t0) / 1e9:.1f} GB/s, D2H {nb / (t2 - t1) / 1e9:.1f} GB/s ({nb / 1e6:.1f} MB)")


if __name__ == "__main__":
    main()
