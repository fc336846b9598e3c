#include "hd_kernels.cuh"
HD_DEFINE_SLICE(lookup_f32_512, float, 512)
