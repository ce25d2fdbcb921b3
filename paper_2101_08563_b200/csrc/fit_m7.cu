// fit_m7.cu -- fit kernel instantiations for dim = 7.
#include "fit_launch.cuh"
FFCA_DEFINE_FIT_LAUNCHER(7)
