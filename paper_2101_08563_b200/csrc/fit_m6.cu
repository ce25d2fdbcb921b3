// fit_m6.cu -- fit kernel instantiations for dim = 6.
#include "fit_launch.cuh"
FFCA_DEFINE_FIT_LAUNCHER(6)
