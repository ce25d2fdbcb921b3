// fit_m8.cu -- fit kernel instantiations for dim = 8.
#include "fit_launch.cuh"
FFCA_DEFINE_FIT_LAUNCHER(8)
