"""Regenerate the committed golden fixtures in tests/golden/*.npz.

TEST INFRASTRUCTURE.  The reference itself cannot be built here (Eigen3 and
doctest are absent), so the expected outputs come from
the fp64 oracle restatement (oracle/oracle.cpp), which is pinned first by the
reference's own known-answer tests ported in oracle/kat_tests.cpp
(`make -C oracle kat_tests && oracle/kat_tests` must report 0 failures
before these files are trusted; tests/test_oracle_kat.py runs it).  Freezing the
oracle's outputs here does two things:
  * the CPU suite (tests/test_golden.py) catches any drift of the oracle from
    the pinned state, and
  * the GPU suite checks the CUDA path against stored vectors, without
    running the oracle on the GPU box.

Every fixture stores its inputs in full (x rounded to complex64 values,
initial W, L, H), so the files do not depend on synth.py staying unchanged.

Usage:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import oracle  # noqa: E402
import stft_oracle  # noqa: E402
from paper_2101_08563_b200 import synth  # noqa: E402

# name: (M, N, F, T, iters, flavor 0=em/1=mm, kind, seed, extra)
FIT_CASES = {
    "fit_m2n3_em": (2, 3, 4, 313, 25, 0, "jd", 11, {}),
    "fit_m2n2_em": (2, 2, 4, 400, 40, 0, "jd", 12, {}),
    "fit_m2n2_mm": (2, 2, 4, 400, 20, 1, "jd", 13, {}),
    "fit_m3n4_em": (3, 4, 3, 313, 20, 0, "jd", 14, {}),
    "fit_m1n2_em": (1, 2, 3, 200, 10, 0, "jd", 15, {}),
    "fit_m4n6_em_silent": (4, 6, 2, 500, 8, 0, "fullrank", 16, {}),
    "fit_m2n3_em_noscale": (2, 3, 3, 300, 10, 0, "jd", 17, {"normalize_scales": False}),
    "fit_m3n4_mm_fixL": (3, 4, 2, 300, 10, 1, "jd", 18, {"fix_loadings": True}),
}
ICA_CASE = ("ica_m2", 2, 3, 300, 15, 19)
# block-stationary input (sample_covs(spec, B), sigmodel.cpp:17-48):
# name: (M, N, F, T, B, iters, flavor, seed); T % B != 0 leaves a ragged tail block
BLOCK_CASES = {
    "block_m2n2_b10_em": (2, 2, 4, 505, 10, 20, 0, 21),
    "block_m3n4_b4_mm": (3, 4, 3, 313, 4, 10, 1, 22),
}


# STFT front end / iSTFT back end (stft.cpp:33-128): name: (channels, length,
# frame_len, shift, padding 0=centered/1=full_frames, seed)
STFT_CASES = {
    "stft_c2_n5000_f256_centered": (2, 5000, 256, 128, 0, 23),
    "stft_c3_n3001_f512_full": (3, 3001, 512, 256, 1, 24),
}


# batch of independent mixtures (config 4's shape family, fastfca_fit_batch):
# (batch, M, N, F, T, iters, seed)
BATCH_CASE = ("batch3_m3n4_em", 3, 3, 4, 3, 313, 12, 25)


def inputs(M, N, F, T, kind, seed):
    cfg = synth.small(M, N, F, T, seed=seed, kind=kind)
    x = synth.mixture(cfg).astype(np.complex64).astype(np.complex128)
    W, L, H = synth.init_params(cfg)
    return x, np.asarray(W, np.complex128), np.asarray(L, np.float64), np.asarray(H, np.float64)


def main() -> None:
    for name, (M, N, F, T, iters, flavor, kind, seed, extra) in FIT_CASES.items():
        x, W, L, H = inputs(M, N, F, T, kind, seed)
        Wo, Lo, Ho, nll, _, _ = oracle.fit(x, W, L, H, iters, flavor=flavor, **extra)
        out = dict(x=x.astype(np.complex64), W0=W, L0=L, H0=H, iters=iters, flavor=flavor,
                   normalize_scales=int(extra.get("normalize_scales", True)),
                   fix_loadings=int(extra.get("fix_loadings", False)),
                   W=Wo, L=Lo, H=Ho, nll=nll)
        if name == "fit_m2n3_em":
            out["images"] = oracle.separate(x, Wo, Lo, Ho).astype(np.complex128)
        np.savez_compressed(HERE / f"{name}.npz", **out)
        print(name, "nll", nll[0], "->", nll[-1])
    for name, (M, N, F, T, B, iters, flavor, seed) in BLOCK_CASES.items():
        x, W, L, _ = inputs(M, N, F, T, "jd", seed)
        J = -(-T // B)
        H = np.random.default_rng(seed + 1).lognormal(0.0, 1.0, (F, N, J))
        mats, power = oracle.block_covs(x, B)
        Wo, Lo, Ho, nll, _ = oracle.fit_covs(mats, W, L, H, iters, flavor=flavor, power=power)
        np.savez_compressed(HERE / f"{name}.npz", x=x.astype(np.complex64), block_size=B,
                            W0=W, L0=L, H0=H, iters=iters, flavor=flavor, mats=mats,
                            power=power, W=Wo, L=Lo, H=Ho, nll=nll)
        print(name, "nll", nll[0], "->", nll[-1])
    for name, (C, n, fl, sh, pad, seed) in STFT_CASES.items():
        wave = np.random.default_rng(seed).standard_normal((C, n))
        spec = stft_oracle.stft(wave, fl, sh, pad)
        back = stft_oracle.istft(spec, fl, sh, n, pad)
        np.savez_compressed(HERE / f"{name}.npz", wave=wave, frame_len=fl, shift=sh, pad=pad,
                            spec=spec, back=back)
        print(name, "spec", spec.shape, "round trip", float(np.abs(back - wave).max()))
    name, Bn, M, N, F, T, iters, seed = BATCH_CASE
    cases = [inputs(M, N, F, T, "jd", seed + b) for b in range(Bn)]
    x, W, L, H = (np.stack([c[k] for c in cases]) for k in range(4))
    Wo, Lo, Ho, nll, _, _ = oracle.fit(x, W, L, H, iters)  # batched: the loop of fastfca_fit
    np.savez_compressed(HERE / f"{name}.npz", x=x.astype(np.complex64), W0=W, L0=L, H0=H,
                        iters=iters, W=Wo, L=Lo, H=Ho, nll=nll)
    print(name, "nll", nll[:, 0], "->", nll[:, -1])
    name, M, F, T, iters, seed = ICA_CASE
    x, W, _, _ = inputs(M, M, F, T, "jd", seed)
    Wo, Lo, Ho, nll = oracle.ica_fit(x, W, iters)
    np.savez_compressed(HERE / f"{name}.npz", x=x.astype(np.complex64), W0=W, iters=iters,
                        W=Wo, L=Lo, H=Ho, nll=nll)
    print(name, "nll", nll[0], "->", nll[-1])


if __name__ == "__main__":
    main()
