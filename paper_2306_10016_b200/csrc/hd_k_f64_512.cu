#include "hd_kernels.cuh"
HD_DEFINE_SLICE(lookup_f64_512, double, 512)
