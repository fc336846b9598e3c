// hd_kernels.cu -- instantiations of the pass kernels for every supported FFT size
// m = 2..4096 (powers of two), both precisions, and the three pass modes.
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

LaunchFn lookup_launcher(bool is_double, int m, int mode, int threads) {
  if (threads != 256) return nullptr;
  return is_double ? pick_mode<double, 256>(m, mode) : pick_mode<float, 256>(m, mode);
}

template <typename V>
static cudaError_t launch_pad_impl(const void* src, void* dst, const int64_t L[3], const int64_t P[3],
                                   int64_t nb, cudaStream_t st) {
  const int64_t total = nb * P[0] * P[1] * P[2];
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  pad_copy_kernel<V><<<(unsigned)blocks, 256, 0, st>>>((const V*)src, (V*)dst, L[0], L[1], L[2],
                                                       P[0], P[1], P[2], nb);
  return cudaGetLastError();
}
template <typename V>
static cudaError_t launch_crop_impl(const void* src, void* dst, const int64_t O[3], const int64_t P[3],
                                    int64_t nb, cudaStream_t st) {
  const int64_t total = nb * O[0] * O[1] * O[2];
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  crop_copy_kernel<V><<<(unsigned)blocks, 256, 0, st>>>((const V*)src, (V*)dst, O[0], O[1], O[2],
                                                        P[0], P[1], P[2], nb);
  return cudaGetLastError();
}

cudaError_t launch_pad(bool is_double, const void* src, void* dst, const int64_t L[3],
                       const int64_t P[3], int64_t nb, cudaStream_t st) {
  return is_double ? launch_pad_impl<double2>(src, dst, L, P, nb, st)
                   : launch_pad_impl<float2>(src, dst, L, P, nb, st);
}
cudaError_t launch_crop(bool is_double, const void* src, void* dst, const int64_t O[3],
                        const int64_t P[3], int64_t nb, cudaStream_t st) {
  return is_double ? launch_crop_impl<double2>(src, dst, O, P, nb, st)
                   : launch_crop_impl<float2>(src, dst, O, P, nb, st);
}

}  // namespace hd
