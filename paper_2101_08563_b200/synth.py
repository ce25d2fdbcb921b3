"""Seeded synthetic mixtures for BASELINE.json configs 0-4.

The paper's evaluation data (real-room impulse responses, speech) is not in
this container, so these seeded generators stand in for it with the shapes
and value distributions BASELINE.json names.  numpy's PCG64 streams are
platform-independent for a fixed numpy version, so every host (this
container, the GPU box) draws identical inputs.  x is rounded to complex64,
and the oracle consumes exactly those complex64 values promoted to double.

Generative model (c0/c1/c3/c4, jointly diagonalizable):
  A_f ~ iid CN(0,1) (M x M);  d_nf ~ lognormal(0, 1) (M);
  v_nft ~ lognormal(0, sigma_v);  s_nft = sqrt(v) A_f diag(sqrt(d_nf)) z, z ~ CN(0, I)
  x_ft = sum_n s_nft + e_ft,  e ~ CN(0, 1e-3 I)
c2 (full-rank, not JD): R_nf = B B^H + 1e-2 I, s = sqrt(v) chol(R_nf) z,
  v ~ Gamma(0.5, 1) * a_n(floor(t/50)), a ~ Bernoulli(0.5); no noise.
Init (all): W_f = I, L = 1, H ~ lognormal(0, 1) from a separate init stream.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    M: int
    N: int
    F: int
    T: int
    iters: int
    batch: int = 1
    kind: str = "jd"       # "jd" or "fullrank"
    sigma_v: float = 1.5
    seed: int = 20210120


CONFIGS = {
    "c0": Config("c0", 2, 3, 513, 626, 50, sigma_v=1.5),
    "c1": Config("c1", 2, 2, 513, 1250, 100, sigma_v=1.5),
    "c2": Config("c2", 4, 6, 1025, 2000, 50, kind="fullrank"),
    "c3": Config("c3", 8, 12, 2049, 8000, 30, sigma_v=2.0),
    "c4": Config("c4", 3, 4, 513, 626, 50, batch=256, sigma_v=1.5),
}


def crandn(rng: np.random.Generator, shape) -> np.ndarray:
    """Circular complex Gaussian with E|z|^2 = 1."""
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2.0)


def _mixture_chunk(cfg: Config, rng: np.random.Generator, nb: int) -> np.ndarray:
    """nb bins of x, complex64 [nb, M, T], drawn from rng."""
    M, N, T = cfg.M, cfg.N, cfg.T
    if cfg.kind == "jd":
        A = crandn(rng, (nb, M, M))
        d = np.exp(rng.standard_normal((nb, N, M)))
        v = np.exp(cfg.sigma_v * rng.standard_normal((nb, N, T)))
        z = crandn(rng, (nb, N, M, T))
        # s_n = sqrt(v_n) * A diag(sqrt(d_n)) z_n
        y = z * np.sqrt(d)[..., None] * np.sqrt(v)[:, :, None, :]
        s = np.einsum("fab,fnbt->fat", A, y)
        s += np.sqrt(1e-3) * crandn(rng, (nb, M, T))
    else:
        B = crandn(rng, (nb, N, M, M))
        R = B @ np.conj(np.swapaxes(B, -1, -2)) + 1e-2 * np.eye(M)
        C = np.linalg.cholesky(R)
        act = rng.random((nb, N, (T + 49) // 50)) < 0.5
        a = np.repeat(act, 50, axis=-1)[..., :T]
        v = rng.gamma(0.5, 1.0, (nb, N, T)) * a
        z = crandn(rng, (nb, N, M, T))
        s = np.einsum("fnab,fnbt->fat", C, z * np.sqrt(v)[:, :, None, :])
    return s.astype(np.complex64)


# Configs above this many source-image samples (c3: 1.6e9) draw every chunk of
# bins from its own child stream, so chunks generate in parallel threads and a
# frequency shard generates only its own bins.
PARALLEL_STREAMS_ABOVE = 1 << 29


def mixture(cfg: Config, b: int = 0, bins: slice | None = None) -> np.ndarray:
    """x for mixture b: complex64 [F, M, T] (natural layout; the device SoA).
    `bins` (a contiguous slice) restricts the result to those bins."""
    M, N, F, T = cfg.M, cfg.N, cfg.F, cfg.T
    chunk = max(1, (1 << 22) // (N * M * T))
    lo, hi, step = (0, F, 1) if bins is None else bins.indices(F)
    assert step == 1
    if F * N * M * T <= PARALLEL_STREAMS_ABOVE:
        rng = np.random.Generator(np.random.PCG64([cfg.seed, 1, b]))
        x = np.empty((F, M, T), np.complex64)
        for f0 in range(0, F, chunk):
            f1 = min(F, f0 + chunk)
            x[f0:f1] = _mixture_chunk(cfg, rng, f1 - f0)
        return x if bins is None else x[bins]
    import concurrent.futures as cf
    import os
    x = np.empty((max(hi - lo, 0), M, T), np.complex64)

    def work(k: int) -> None:
        f0, f1 = k * chunk, min(F, (k + 1) * chunk)
        part = _mixture_chunk(cfg, np.random.Generator(np.random.PCG64([cfg.seed, 1, b, k])),
                              f1 - f0)
        a, e = max(f0, lo), min(f1, hi)
        x[a - lo:e - lo] = part[a - f0:e - f0]

    ks = range(lo // chunk, (max(hi, lo + 1) - 1) // chunk + 1) if hi > lo else range(0)
    with cf.ThreadPoolExecutor(min(32, os.cpu_count() or 4)) as ex:
        list(ex.map(work, ks))
    return x


def init_params(cfg: Config, b: int = 0, nbins: int | None = None):
    """(W, L, H) natural layout: W [F,M,M] complex128, L [F,M,N], H [F,N,T].
    nbins: only the first nbins bins (the same values: H is drawn bin by bin
    from one stream)."""
    M, N, F, T = cfg.M, cfg.N, cfg.F, cfg.T
    F = F if nbins is None else min(F, nbins)
    rng = np.random.Generator(np.random.PCG64([cfg.seed, 2, b]))
    W = np.broadcast_to(np.eye(M, dtype=np.complex128), (F, M, M)).copy()
    L = np.ones((F, M, N))
    H = np.exp(rng.standard_normal((F, N, T)))
    return W, L, H


def small(M: int, N: int, F: int, T: int, seed: int = 0, kind: str = "jd",
          sigma_v: float = 1.5, iters: int = 10) -> Config:
    """A reduced config with the same generative model (for parity tests)."""
    return Config(f"small{M}{N}{F}{T}", M, N, F, T, iters, kind=kind, sigma_v=sigma_v,
                  seed=seed)
