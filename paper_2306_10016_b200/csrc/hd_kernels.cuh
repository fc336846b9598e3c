// hd_kernels.cuh -- launcher templates; each hd_k_<dtype>_<threads>.cu instantiates
// one (precision, threads-per-CTA) slice so the slices compile in parallel.
#pragma once
#include "hd_device.cuh"
#include "hd_internal.h"

namespace hd {

template <typename T, int M, int NT, int MODE>
static cudaError_t launch_pass_impl(const PassArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
  auto kern = pass_kernel<T, M, NT, MODE>;
  static size_t configured = 0;  // largest dynamic smem size already allowed
  if (smem > 48 * 1024 && smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  kern<<<grid, NT, smem, st>>>(a);
  return cudaGetLastError();
}

template <typename T, int NT, int MODE>
static LaunchFn pick_m(int m) {
  switch (m) {
    case 2: return launch_pass_impl<T, 2, NT, MODE>;
    case 4: return launch_pass_impl<T, 4, NT, MODE>;
    case 8: return launch_pass_impl<T, 8, NT, MODE>;
    case 16: return launch_pass_impl<T, 16, NT, MODE>;
    case 32: return launch_pass_impl<T, 32, NT, MODE>;
    case 64: return launch_pass_impl<T, 64, NT, MODE>;
    case 128: return launch_pass_impl<T, 128, NT, MODE>;
    case 256: return launch_pass_impl<T, 256, NT, MODE>;
    case 512: return launch_pass_impl<T, 512, NT, MODE>;
    case 1024: return launch_pass_impl<T, 1024, NT, MODE>;
    case 2048: return launch_pass_impl<T, 2048, NT, MODE>;
    case 4096: return launch_pass_impl<T, 4096, NT, MODE>;
    default: return nullptr;
  }
}

template <typename T, int NT>
static LaunchFn pick_mode(int m, int mode) {
  switch (mode) {
    case MODE_FWD: return pick_m<T, NT, MODE_FWD>(m);
    case MODE_INV: return pick_m<T, NT, MODE_INV>(m);
    case MODE_CONV: return pick_m<T, NT, MODE_CONV>(m);
    default: return nullptr;
  }
}

}  // namespace hd

#define HD_DEFINE_SLICE(NAME, T, NT) \
  namespace hd { LaunchFn NAME(int m, int mode) { return pick_mode<T, NT>(m, mode); } }
