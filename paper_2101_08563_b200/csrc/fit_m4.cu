// fit_m4.cu -- fit kernel instantiations for dim = 4.
#include "fit_launch.cuh"
FFCA_DEFINE_FIT_LAUNCHER(4)
