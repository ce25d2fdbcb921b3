"""Profiling driver: one device-resident fastfca_fit of a BASELINE config
(optionally restricted to its first --bins bins / --iters iterations), timed
with CUDA events; --phases reads the per-phase cycle counters of the
diagnostics build (FFCA_LIB=.../libffca_timing.so, build.build_lib(variant=
"timing")).  Used under ncu for the captures in profiles/.

    python tools/prof_fit.py c3 --bins 296 --iters 3 --reps 3 [--phases]
"""
from __future__ import annotations

import argparse
import dataclasses
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

PHASES = ["A frames", "A reduce", "IP serial", "iter sync", "EM frames", "EM barrier",
          "EM update", "balance", "EM sum", "init"]
# fit_big.cuh (M = 8, N = 12 large-bin kernel) phase order
PHASES_BIG = ["U pass", "EM frames", "EM reduce", "balance", "A1", "A2 frames", "A2 reduce",
              "IP", "iter sync", "init"]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--bins", type=int, default=0)
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--fp64", action="store_true")
    ap.add_argument("--no-trace", action="store_true")
    ap.add_argument("--phases", action="store_true")
    ap.add_argument("--big", action="store_true", help="phase names of the large-bin kernel")
    a = ap.parse_args()
    import torch
    from paper_2101_08563_b200 import _lib, synth
    cfg = synth.CONFIGS[a.config]
    F = a.bins or cfg.F
    cfg = dataclasses.replace(cfg, iters=a.iters or cfg.iters)
    xs, Ws, Ls, Hs = [], [], [], []
    for b in range(cfg.batch):
        xs.append(synth.mixture(cfg, b, slice(0, F)) if F < cfg.F else synth.mixture(cfg, b))
        W, L, H = synth.init_params(cfg, b)
        Ws.append(W[:F]); Ls.append(L[:F]); Hs.append(H[:F])
    x, W0, L0, H0 = (np.concatenate(v) for v in (xs, Ws, Ls, Hs))
    P, M, N, T, iters = x.shape[0], cfg.M, cfg.N, cfg.T, cfg.iters
    dev = torch.device("cuda", 0)
    cdt, rdt = (torch.complex128, torch.float64) if a.fp64 else (torch.complex64, torch.float32)
    xd = torch.from_numpy(np.ascontiguousarray(np.swapaxes(x, -1, -2))).to(dev, cdt)
    Hi = torch.from_numpy(np.ascontiguousarray(np.swapaxes(H0, -1, -2))).to(dev, rdt)
    Wi = torch.from_numpy(np.ascontiguousarray(np.swapaxes(W0, -1, -2))).to(dev)
    Li = torch.from_numpy(np.ascontiguousarray(np.swapaxes(L0, -1, -2))).to(dev)
    Hd, Wd, Ld = Hi.clone(), Wi.clone(), Li.clone()
    power = torch.empty(P, dtype=torch.float64, device=dev)
    slots = torch.zeros((iters + 1, P), dtype=torch.float64, device=dev)
    status = torch.zeros(P, dtype=torch.int32, device=dev)
    ctx = _lib.Context(0)
    Lb = _lib.lib()
    prec = _lib.PREC_FP64 if a.fp64 else _lib.PREC_FP32
    # A dedicated stream: the library launches on the stream it is given (NULL
    # would mean the context's own stream, which torch's events do not see).
    ts = torch.cuda.Stream(dev)
    torch.cuda.set_stream(ts)
    stream = ts.cuda_stream
    _lib.check(Lb.ffca_power_scale_device(ctx.handle, P, M, T, prec, _lib.ptr(xd), _lib.ptr(power),
                                          stream))
    counters = None
    if a.phases:
        counters = torch.zeros((P, 16), dtype=torch.int64, device=dev)
        _lib.check(Lb.ffca_debug_set_timing(ctx.handle, _lib.ptr(counters)))
    o = _lib.FitOpts(_lib.FLAVOR_EM, iters, 0 if a.no_trace else 1, 0, 1, 0, prec)
    times = []
    for r in range(a.reps):
        Hd.copy_(Hi); Wd.copy_(Wi); Ld.copy_(Li)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ts)
        _lib.check(Lb.ffca_fit_device(ctx.handle, P, F, 0, M, N, T, o, _lib.ptr(xd),
                                      _lib.ptr(power), _lib.ptr(Wd), _lib.ptr(Ld), _lib.ptr(Hd),
                                      _lib.ptr(slots), _lib.ptr(status), stream))
        e1.record(ts)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    st = status.cpu().numpy()
    units = P * T * iters
    best = min(times)
    print(f"{a.config}: P={P} M={M} N={N} T={T} iters={iters}  ms={['%.3f' % t for t in times]}"
          f"  best {best:.3f} ms  {units / best * 1e3:.3e} TF-bin-updates/s  bad={int((st >= 2).sum())}")
    if counters is not None:
        c = counters.cpu().numpy()[:, :10].astype(np.float64)
        tot = c.sum(axis=1)
        print("phase cycles per bin (mean over bins, per iteration):")
        for k in range(10):
            print(f"  {(PHASES_BIG if a.big else PHASES)[k]:<11} {c[:, k].mean() / iters:10.0f}  ({100 * c[:, k].sum() / tot.sum():5.1f} %)")


if __name__ == "__main__":
    main()
