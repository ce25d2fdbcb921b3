"""B200-native FastFCA (arxiv 2101.08563) IP+EM hot path.

C++/CUDA library libffca.so (sm_100a) behind the reference's API; this
package is the Python mirror of that API plus build and data helpers.
"""
from .api import (FastFcaFitResult, FastFcaOptions, FastFcaParams, FitOptions,  # noqa: F401
                  LhFlavor, SampleCovSet, Spectrogram, fastfca_fit, fastfca_nll,
                  fastfca_nll_bins, fastfca_separate, sample_covs)
from ._lib import CudaError, FfcaError, InvalidArgument, NumericalError  # noqa: F401
