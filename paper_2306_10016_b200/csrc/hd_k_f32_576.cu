#include "hd_kernels.cuh"
HD_DEFINE_SLICE(lookup_f32_576, float, 576)
