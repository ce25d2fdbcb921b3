// fit_m3.cu -- fit kernel instantiations for dim = 3.
#include "fit_launch.cuh"
FFCA_DEFINE_FIT_LAUNCHER(3)
