#include "hd_kernels.cuh"
HD_DEFINE_SLICE(lookup_f64_256, double, 256)
