#include "hd_kernels.cuh"
HD_DEFINE_SLICE(lookup_f32_256, float, 256)
