#include "hd_kernels.cuh"
HD_DEFINE_SLICE(lookup_f64_576, double, 576)
