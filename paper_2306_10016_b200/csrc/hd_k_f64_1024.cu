#include "hd_kernels.cuh"
HD_DEFINE_SLICE(lookup_f64_1024, double, 1024)
