"""FastFCA IP+EM fit throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
                    [--impl ours|reference] [--no-cpu-baseline] [--scaling strong|weak]

A step is one full fastfca_fit (all `iters` IP+EM iterations) over the
workload's synthetic mixtures -- SURVEY §8(d): the work unit is one TF-bin EM
update, throughput = B*F*T*iters / t.

Workload: BASELINE.json configs[3] ("c3": M=8, N=12, F=2049, T=8000, 30 EM
iterations, one mixture) -- the configuration the metric ("... 1/2/4/8 B200")
is quoted on; it fits one GPU (x 1.05 GB + H 0.79 GB).  Under torchrun
(N > 1) the ONE mixture's 2049 bins (for c4: the 256 x 513 flattened
(mixture, bin) problems) are split into contiguous balanced ranges, one per
rank -- the reference's parallel_for over bins (parallel.cpp:16-45) moved
onto GPUs: no exchange during the fit, total work fixed as N grows (scaling
"strong").  The per-bin NLL slots are all-gathered over NCCL after the timed
region and each mixture's trace is summed in bin order, so the trace is
bit-identical for any N.  --scaling weak gives every rank its own mixture
instead.  Other configs (--config c0|c1|c2|c4) are parity cases / secondary
lines.

value : device-resident inputs (x, H, W, L already in HBM), one fit kernel per
        step timed with CUDA events on the launching stream, L2 flushed
        between steps (a 256 MiB write), max over ranks.
e2e   : the reference-facing C-ABI call ffca_fit with pinned HOST buffers in
        the reference's Eigen layout (complex<double> x, double W/L/H): H2D,
        boundary conversion, fit, unpack, D2H -- host clock around the
        synchronous call, max over ranks.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "TF-bin EM updates/sec (F*T*iters/s) and % of HBM roofline, 1/2/4/8 B200"
UNIT = "TF-bin-updates/s"


def peaks() -> dict:
    """HBM peak: the driver-written MEASURED_PEAKS.json, else the profiling
    recipe's fallback.  FP32 (CUDA-core FFMA) peak: the FFMA loop of
    tools/fp32_peak.cu measured on this pool's B200s (profiles/r2_fp32_peak.json,
    committed), else SURVEY 8(d)'s nominal 75 TFLOP/s."""
    out = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)",
           "fp32_tflops": 75.0, "fp32_source": "fallback (SURVEY 8(d) nominal)"}
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        out.update(hbm_gbs=d["hbm_gbs"], source="measured (MEASURED_PEAKS.json)")
    q = ROOT / "profiles" / "r2_fp32_peak.json"
    if q.exists():
        out.update(fp32_tflops=json.loads(q.read_text())["ffma_tflops"],
                   fp32_source="measured FFMA loop (tools/fp32_peak.cu, profiles/r2_fp32_peak.json)")
    return out


def alg_bytes(M: int, N: int) -> int:
    """Algorithmic bytes per TF-bin-iteration: x read once
    (complex64), v read and written once (fp32)."""
    return 8 * M + 8 * N


def alg_flops(M: int, N: int) -> int:
    """Algorithmic flops per TF-bin-iteration: Q 2M^3+5M^2+3M,
    U 8M^2+3M, sigma^2 2MN, EM 11MN, NLL 3M."""
    return 2 * M ** 3 + 13 * M ** 2 + 9 * M + 13 * M * N


def config_dict(cfg, batch: int, world: int, scaling: str) -> dict:
    """The line's `config` -- identical for the GPU arm and the reference arm."""
    return {"workload": cfg.name, "M": cfg.M, "N": cfg.N, "F": cfg.F, "T": cfg.T,
            "iters": cfg.iters, "batch": batch, "flavor": "em", "record_trace": True,
            "parallelism": f"freq-shard x{world} ({scaling})",
            "l2": "flushed between steps (256 MiB write)"}


from paper_2101_08563_b200.shard import bin_order_trace, gather_slots, shard  # noqa: E402


def workload(cfg, world: int, scaling: str = "strong"):
    """The benchmarked batch.  strong (default): the config as BASELINE.json
    states it, its (mixture, bin) problems split over the ranks.  weak: one
    copy of the config's batch per rank."""
    if scaling == "weak" and world > 1:
        return dataclasses.replace(cfg, batch=cfg.batch * world), "weak"
    return cfg, "strong"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples: list[list[str]] = []
        self._stop = threading.Event()
        self._t = None

    def _sample(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                  f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                 capture_output=True, text=True, timeout=5).stdout.strip()
            if out:
                self.samples.append([s.strip() for s in out.split(",")])
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def build_inputs(cfg, lo: int, hi: int):
    """Host inputs for problems [lo, hi) of the flattened (mixture, bin) index."""
    from paper_2101_08563_b200 import synth
    xs, Ws, Ls, Hs = [], [], [], []
    F = cfg.F
    for b in range(lo // F, (hi - 1) // F + 1):
        f0 = max(lo - b * F, 0)
        f1 = min(hi - b * F, F)
        x = synth.mixture(cfg, b, slice(f0, f1))
        W, L, H = synth.init_params(cfg, b)
        xs.append(x); Ws.append(W[f0:f1]); Ls.append(L[f0:f1]); Hs.append(H[f0:f1])
    return (np.concatenate(xs), np.concatenate(Ws), np.concatenate(Ls), np.concatenate(Hs))


def oracle_sample(cfg, args, budget_s: float = 10.0):
    """The bounded CPU sample: the first S bins of mixture 0, all frames and
    iterations.  S = all F bins when that fits ~budget_s of fastfca_fit on all
    host threads (calibrated on one bin), else the largest S that does."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle  # test infrastructure: the CPU baseline leg only
    from paper_2101_08563_b200 import synth
    cores = oracle.default_workers()
    if args.cpu_bins:
        S = min(cfg.F, args.cpu_bins)
    else:
        cal_it = min(cfg.iters, 3)
        x1 = synth.mixture(cfg, 0, slice(0, 1)).astype(np.complex128)
        W, L, H = synth.init_params(cfg, 0, nbins=1)
        _, _, _, _, _, s1 = oracle.fit(x1, W, L, H, cal_it, workers=1)
        per_bin = max(s1, 1e-6) * cfg.iters / cal_it
        S = int(min(cfg.F, max(cores, budget_s * cores / per_bin)))
    x = synth.mixture(cfg, 0, slice(0, S)).astype(np.complex128)
    W, L, H = synth.init_params(cfg, 0, nbins=S)
    sample = (f"{cfg.name}: first {S} of {cfg.F} bins of mixture 0, T={cfg.T}, {cfg.iters} "
              f"iters, fastfca_fit only, fp64 oracle port of the reference (the reference "
              f"itself needs Eigen3, absent)")
    return oracle, cores, S, (x, W[:S], L[:S], H[:S]), sample


def cpu_baseline(cfg, args, budget_s: float = 10.0) -> dict:
    """The oracle port on all host threads over the bounded sample, repeated
    until about budget_s of CPU time has been measured (the whole c1 fit is
    well under a second on the box's cores)."""
    oracle, cores, S, (x, W, L, H), sample = oracle_sample(cfg, args, budget_s=budget_s)
    total, reps = 0.0, 0
    while reps == 0 or total < budget_s:
        _, _, _, _, _, secs = oracle.fit(x, W, L, H, cfg.iters, record_trace=True, workers=cores)
        total += secs
        reps += 1
    return {"value": reps * S * cfg.T * cfg.iters / total, "unit": UNIT, "cores": cores,
            "kind": "port", "sample": sample + f" x {reps} repetitions ({total:.1f} s)"}


def run_reference(cfg, args, rank: int, world: int) -> None:
    if rank != 0:
        return
    # Each step is a bounded sample sized so the whole --steps/--warmup run
    # stays within about two minutes.
    budget = min(10.0, 120.0 / (args.steps + args.warmup))
    oracle, cores, S, (x, W, L, H), sample = oracle_sample(cfg, args, budget_s=budget)
    times = []
    for i in range(args.warmup + args.steps):
        _, _, _, _, _, secs = oracle.fit(x, W, L, H, cfg.iters, record_trace=True, workers=cores)
        if i >= args.warmup:
            times.append(secs)
    tot = sum(times)
    v = S * cfg.T * cfg.iters * len(times) / tot
    wl, scaling = workload(cfg, world, args.scaling)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json config shapes; paper data unavailable)",
        "config": config_dict(cfg, wl.batch, world, scaling),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample, "sample_bins": S},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("FFCA_BENCH_CONFIG", "c3"))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-separate", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: harness test on fewer GPUs than ranks (ranks share devices; the "
                         "slot all-gather runs on host tensors)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-bins", type=int, default=0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_2101_08563_b200 import synth
    cfg0 = synth.CONFIGS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(cfg0, args, rank, world)
        return

    import torch
    if args.dist_backend == "gloo":
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    from paper_2101_08563_b200 import _lib

    cfg, scaling = workload(cfg0, world, args.scaling)
    P = cfg.batch * cfg.F
    lo, hi = shard(P, world, rank)
    Pl = hi - lo
    M, N, T, iters = cfg.M, cfg.N, cfg.T, cfg.iters
    x, W0, L0, H0 = build_inputs(cfg, lo, hi)
    dev = torch.device("cuda", local)
    cdev = dev if args.dist_backend == "nccl" else torch.device("cpu")  # collectives' tensors
    fp64 = args.precision == "fp64"
    cdt = torch.complex128 if fp64 else torch.complex64
    rdt = torch.float64 if fp64 else torch.float32
    # Device layouts are the reference's per-bin order: x [P, T, M], H [P, T, N].
    x_d = torch.from_numpy(np.ascontiguousarray(np.swapaxes(x, -1, -2))).to(dev, cdt).contiguous()
    H_init = torch.from_numpy(np.ascontiguousarray(np.swapaxes(H0, -1, -2))).to(dev, rdt).contiguous()
    W_init = torch.from_numpy(np.ascontiguousarray(np.swapaxes(W0, -1, -2))).to(dev)  # col-major
    L_init = torch.from_numpy(np.ascontiguousarray(np.swapaxes(L0, -1, -2))).to(dev)
    H_d, W_d, L_d = H_init.clone(), W_init.clone(), L_init.clone()
    power = torch.empty(Pl, dtype=torch.float64, device=dev)
    slots = torch.zeros((iters + 1, Pl), dtype=torch.float64, device=dev)
    status = torch.zeros(Pl, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ctx = _lib.Context(local)
    L_ = _lib.lib()
    # A dedicated stream: every copy, flush, event and kernel is ordered on it
    # (the library launches on the stream it is given).
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    prec = _lib.PREC_FP64 if fp64 else _lib.PREC_FP32
    _lib.check(L_.ffca_power_scale_device(ctx.handle, Pl, M, T, prec, _lib.ptr(x_d),
                                          _lib.ptr(power), sp))
    opts = _lib.FitOpts(_lib.FLAVOR_EM, iters, 1, 0, 1, 0, prec)

    def reset():
        H_d.copy_(H_init); W_d.copy_(W_init); L_d.copy_(L_init)

    def fit_once():
        _lib.check(L_.ffca_fit_device(ctx.handle, Pl, cfg.F, lo, M, N, T, opts, _lib.ptr(x_d),
                                      _lib.ptr(power), _lib.ptr(W_d), _lib.ptr(L_d),
                                      _lib.ptr(H_d), _lib.ptr(slots), _lib.ptr(status), sp))
        return ctx.launches()

    for _ in range(args.warmup):
        reset(); fit_once()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches = 0
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            reset()
            flush.fill_(s & 0xff)  # evict L2 (126 MB) between timed steps
            ev[s][0].record(stream)
            launches += fit_once()
            ev[s][1].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = sum(step_ms)
    if dist:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    units = P * T * iters * args.steps
    value = units / (tot_ms / 1e3)

    # Trace assembly: all-gather the per-bin slots (NCCL), bin-order sums.
    st = status.cpu().numpy()
    bad = int((st >= 2).sum())
    all_slots = gather_slots(slots.to(cdev), P, world, rank, dist)
    if dist:
        badt = torch.tensor([bad], device=cdev)
        dist.all_reduce(badt)
        bad = int(badt.item())
    trace = bin_order_trace(all_slots, cfg.batch, cfg.F)  # [iters+1, batch]
    monotone = bool((trace[1:] <= trace[:-1] + 1e-5 * np.abs(trace[:-1])).all())

    # The same fit with record_trace off (timed with the trace
    # on -- the headline, as the parity runs -- and off).
    opts_nt = _lib.FitOpts(_lib.FLAVOR_EM, iters, 0, 0, 1, 0, prec)
    nt_ms = []
    for i in range(3 + 10):
        reset()
        flush.fill_(i & 0xff)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _lib.check(L_.ffca_fit_device(ctx.handle, Pl, cfg.F, lo, M, N, T, opts_nt, _lib.ptr(x_d),
                                      _lib.ptr(power), _lib.ptr(W_d), _lib.ptr(L_d),
                                      _lib.ptr(H_d), None, _lib.ptr(status), sp))
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            nt_ms.append(e0.elapsed_time(e1))
    trace_off = {"ms_per_step": statistics.median(nt_ms),
                 "value": P * T * iters / (statistics.median(nt_ms) / 1e3),
                 "note": "record_trace=false (no per-iteration NLL), median of 10, this rank"}

    # Separation (fastfca_separate) of the fitted parameters, device path.
    separate = None
    if not args.no_separate:
        img = torch.empty((N, Pl, T, M), dtype=cdt, device=dev)
        sep_ms = []
        for i in range(3 + 5):
            flush.fill_(i & 0xff)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _lib.check(L_.ffca_separate_device(ctx.handle, Pl, M, N, T, prec, _lib.ptr(x_d),
                                               _lib.ptr(W_d), _lib.ptr(L_d), _lib.ptr(H_d),
                                               _lib.ptr(img), sp))
            e1.record(stream)
            torch.cuda.synchronize()
            if i >= 3:
                sep_ms.append(e0.elapsed_time(e1))
        sep_s = statistics.median(sep_ms) / 1e3
        esz = 16 if fp64 else 8
        sep_bytes = Pl * T * (esz * M + (esz // 2) * N + esz * N * M)
        separate = {"ms": sep_s * 1e3, "bytes": int(sep_bytes), "GB_per_s": sep_bytes / sep_s / 1e9,
                    "frac_hbm": sep_bytes / sep_s / 1e9 / peaks()["hbm_gbs"],
                    "bytes_per_frame": "x read + H read + N images written"}
        del img

    # e2e through the reference-facing C-ABI with pinned host buffers.
    e2e = None
    if not args.no_e2e:
        xr = torch.from_numpy(np.ascontiguousarray(np.swapaxes(x, -1, -2)).astype(np.complex128)).pin_memory()
        Wr = torch.from_numpy(np.ascontiguousarray(np.swapaxes(W0, -1, -2))).pin_memory()
        Lr = torch.from_numpy(np.ascontiguousarray(np.swapaxes(L0, -1, -2))).pin_memory()
        Hr0 = np.ascontiguousarray(np.swapaxes(H0, -1, -2))
        Hr = torch.from_numpy(Hr0.copy()).pin_memory()
        Wpin, Lpin = Wr.clone().pin_memory(), Lr.clone().pin_memory()
        nll_h = torch.zeros(iters + 1, dtype=torch.float64).pin_memory()
        d = _lib.Dims(1, Pl, M, N, T)
        ectx = _lib.Context(local)
        times = []
        for i in range(args.warmup + args.steps):
            Hr.copy_(torch.from_numpy(Hr0)); Wpin.copy_(Wr); Lpin.copy_(Lr)
            flush.fill_(i & 0xff)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _lib.check(L_.ffca_fit(ectx.handle, d, opts, _lib.ptr(xr), None, _lib.ptr(Wpin),
                                   _lib.ptr(Lpin), _lib.ptr(Hr), _lib.ptr(nll_h), None, None))
            t1 = time.perf_counter()
            if i >= args.warmup:
                times.append(t1 - t0)
        et = sum(times)
        if dist:
            t = torch.tensor([et], dtype=torch.float64, device=cdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            et = float(t.item())
        # whole-job bytes per step (all ranks' shards)
        h2d = P * (T * M * 16 + T * N * 8 + M * M * 16 + M * N * 8)
        d2h = P * (T * N * 8 + M * M * 16 + M * N * 8) + world * (iters + 1) * 8
        e2e = {"value": P * T * iters * len(times) / et, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": 1e3 * et / len(times), "launches_per_step": ectx.launches(),
               "timing": "host clock around the synchronous C-ABI call, max over ranks"}

    # e2e through the reference's C++ API (include/fastfca, csrc/shim.cpp):
    # fastfca::fastfca_fit on host containers -- container -> pinned staging
    # copies on host threads, the same pipelined C-ABI call, copies back into
    # the result containers.  tools/cpp_e2e.cpp, rank 0 / single GPU only.
    e2e_cpp = None
    if not args.no_e2e and world == 1 and (ROOT / "tools" / "cpp_e2e.so").exists():
        import ctypes as C
        cpp = C.CDLL(str(ROOT / "tools" / "cpp_e2e.so"))
        nst = min(args.steps, 5)
        ms = np.zeros(nst)
        nll_last = C.c_double(0.0)
        err = C.create_string_buffer(512)
        xh = np.ascontiguousarray(np.swapaxes(x, -1, -2)).astype(np.complex128)
        Wh = np.ascontiguousarray(np.swapaxes(W0, -1, -2))
        Lh = np.ascontiguousarray(np.swapaxes(L0, -1, -2))
        Hh = np.ascontiguousarray(np.swapaxes(H0, -1, -2))
        cpp.ffca_cpp_e2e.argtypes = [C.c_int] * 7 + [C.c_void_p] * 5 + [C.POINTER(C.c_double),
                                                                      C.c_char_p, C.c_int]
        rc = cpp.ffca_cpp_e2e(Pl, M, N, T, iters, 2, nst, xh.ctypes.data, Wh.ctypes.data,
                              Lh.ctypes.data, Hh.ctypes.data, ms.ctypes.data, C.byref(nll_last),
                              err, 512)
        if rc == 0:
            med = float(np.median(ms))
            e2e_cpp = {"value": P * T * iters / (med / 1e3), "unit": UNIT, "ms_per_step": med,
                       "nll_last": nll_last.value,
                       "timing": "host clock around fastfca::fastfca_fit (SampleCovSet/FastFcaParams "
                                 f"in, FastFcaFitResult out), median of {nst} after 2 warm-ups"}
        else:
            e2e_cpp = {"error": err.value.decode(errors="replace")}
        del xh, Hh

    if rank == 0:
        pk = peaks()
        b_alg, f_alg = alg_bytes(M, N), alg_flops(M, N)
        kern_s = (tot_ms / 1e3) / args.steps
        units_launch = Pl * T * iters  # per GPU (rank 0's shard), one launch per step
        achieved = units_launch * b_alg / kern_s / 1e9
        fl_achieved = units_launch * f_alg / kern_s / 1e12
        frac_hbm, frac_fp32 = achieved / pk["hbm_gbs"], fl_achieved / pk["fp32_tflops"]
        traffic = None
        tp = ROOT / "profiles" / "ncu_traffic.json"
        if tp.exists():
            tj = json.loads(tp.read_text()).get(cfg0.name)
            if tj and world == 1:
                traffic = tj
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(cfg0, args)
        clocks = clk.summary()
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32" if not fp64 else "f64",
            "data": "synthetic (seeded, BASELINE.json config shapes; paper data unavailable)",
            "config": config_dict(cfg0, cfg.batch, world, scaling),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": frac_hbm, "traffic": traffic,
                         "peak_source": pk["source"],
                         "algorithmic_bytes_per_unit": b_alg,
                         "units_per_launch": units_launch,
                         "kernel": "the one fit kernel launched per step (big_fit_kernel for c3, "
                                   "fit_kernel otherwise) = 100 % of the timed region",
                         "fp32": {"bound": "fp32 CUDA cores", "achieved": fl_achieved,
                                  "peak": pk["fp32_tflops"], "unit": "TFLOP/s", "frac": frac_fp32,
                                  "algorithmic_flops_per_unit": f_alg,
                                  "peak_source": pk["fp32_source"]},
                         "min_bound": {"bound": "fp32" if frac_fp32 > frac_hbm else "hbm",
                                       "frac": max(frac_fp32, frac_hbm),
                                       "note": "fraction of min(HBM peak / B_alg, FP32 peak / F_alg)"
                                               " units/s -- the binding roofline of this config"},
                         "note": "algorithmic bytes (8M+8N per TF-bin-iteration, SURVEY 8(d)) x"
                                 " units per launch / kernel time; per-frame state stays on chip"
                                 " (shared / tensor memory) for the whole fit, so DRAM traffic"
                                 " (traffic) differs from the algorithmic bytes"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_cpp_api": e2e_cpp,
            "gpu_launches": launches,
            "trace_off": trace_off,
            "separate": separate,
            "clocks": clocks,
            "trace": {"nll_first": float(trace[0].sum()), "nll_last": float(trace[-1].sum()),
                      "monotone": monotone, "failed_bins": bad},
            "step_ms": step_ms,
        }
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
