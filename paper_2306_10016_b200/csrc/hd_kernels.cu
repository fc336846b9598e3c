// hd_kernels.cu -- launcher lookup over the instantiated slices (hd_k_*.cu: every
// FFT size m = 2..4096, both precisions, 256 or 512 threads, three pass modes)
// and the explicit-padding copy kernels.
#include "hd_device.cuh"
#include "hd_internal.h"

namespace hd {

LaunchFn lookup_f64_256(int m, int mode);
LaunchFn lookup_f64_576(int m, int mode);
LaunchFn lookup_f64_1024(int m, int mode);
LaunchFn lookup_f32_256(int m, int mode);
LaunchFn lookup_f32_576(int m, int mode);
LaunchFn lookup_f32_1024(int m, int mode);

// the slice with the smallest register bound that admits `threads`
LaunchFn lookup_launcher(bool is_double, int m, int mode, int threads) {
  if (threads <= 256) return is_double ? lookup_f64_256(m, mode) : lookup_f32_256(m, mode);
  if (threads <= 576) return is_double ? lookup_f64_576(m, mode) : lookup_f32_576(m, mode);
  if (threads <= 1024) return is_double ? lookup_f64_1024(m, mode) : lookup_f32_1024(m, mode);
  return nullptr;
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
