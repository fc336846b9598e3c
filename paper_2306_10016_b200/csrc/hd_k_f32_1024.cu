#include "hd_kernels.cuh"
HD_DEFINE_SLICE(lookup_f32_1024, float, 1024)
