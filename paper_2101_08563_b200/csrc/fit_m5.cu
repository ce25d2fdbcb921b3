// fit_m5.cu -- fit kernel instantiations for dim = 5.
#include "fit_launch.cuh"
FFCA_DEFINE_FIT_LAUNCHER(5)
