// fit_m1.cu -- fit kernel instantiations for dim = 1.
#include "fit_launch.cuh"
FFCA_DEFINE_FIT_LAUNCHER(1)
