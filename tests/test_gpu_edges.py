"""Edge cases of the GPU fit against the oracle (through the C-ABI).

* empty spectrogram -> invalid argument (sigmodel.cpp:17-48 rejects it; the
  oracle raises the same);
* a rank-deficient bin (T = 1 < M): every Q_m is rank one, the IP's LU solve
  fails its residual check and the fit raises NumericalError
  (fastfca.cpp:53-65) -- the oracle raises too;
* ragged frame counts (T not a multiple of the CTA width, T < warp size,
  T = 2) and a single source (N = 1): trace parity at north_star tolerances;
* the degenerate single bin / channel / source case (M = N = F = 1).
"""
import numpy as np
import pytest

import oracle
from paper_2101_08563_b200 import api, synth
from paper_2101_08563_b200._lib import InvalidArgument, NumericalError

pytestmark = pytest.mark.gpu

NLL_TOL = {"fp32": 1e-5, "fp64": 1e-10}


def make(M, N, F, T, seed=3):
    cfg = synth.small(M, N, F, T, seed=seed)
    x = synth.mixture(cfg).astype(np.complex64).astype(np.complex128)
    W, L, H = synth.init_params(cfg)
    return x, W, L, H


def fit(x, W, L, H, iters, precision):
    covs = api.sample_covs(api.Spectrogram(x))
    return api.fastfca_fit(covs, api.FastFcaParams(W, L, H), 0, iters, precision=precision)


def test_empty_spectrogram_is_invalid(gpu):
    x = np.zeros((0, 2, 100), np.complex128)
    with pytest.raises(InvalidArgument):
        api.sample_covs(api.Spectrogram(x))
    with pytest.raises(oracle.OracleError):
        oracle.fit(x, np.zeros((0, 2, 2), complex), np.zeros((0, 2, 2)), np.zeros((0, 2, 100)), 3)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_rank_deficient_bin_raises_numerical_error(gpu, precision):
    x, W, L, H = make(2, 2, 3, 1)
    with pytest.raises(oracle.OracleError):
        oracle.fit(x, W, L, H, 5)
    with pytest.raises(NumericalError):
        fit(x, W, L, H, 5, precision)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("M,N,F,T", [(2, 3, 3, 33), (3, 1, 2, 129), (2, 2, 2, 2),
                                     (2, 2, 5, 1257), (4, 2, 2, 31), (1, 1, 1, 7)])
def test_ragged_shapes_match_oracle(gpu, precision, M, N, F, T):
    x, W, L, H = make(M, N, F, T)
    iters = 6
    nll_o = oracle.fit(x, W, L, H, iters)[3]
    r = fit(x, W, L, H, iters, precision)
    nll_g = np.asarray(r.nll)
    assert nll_g.shape == nll_o.shape
    rel = np.abs(nll_g - nll_o) / np.abs(nll_o)
    assert rel.max() <= NLL_TOL[precision], (rel.max(), int(rel.argmax()))
    assert (r.bin_status == 0).all()
