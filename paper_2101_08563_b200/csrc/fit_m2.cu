// fit_m2.cu -- fit kernel instantiations for dim = 2.
#include "fit_launch.cuh"
FFCA_DEFINE_FIT_LAUNCHER(2)
