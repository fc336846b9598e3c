// hd_kernels.cu -- launcher lookup over the instantiated slices (hd_k_*.cu: every
// FFT size m = 2..4096, both precisions, 256 or 512 threads, three pass modes)
// and the explicit-padding copy kernels.
#include <map>
#include <mutex>
#include <utility>

#include "hd_device.cuh"
#include "hd_internal.h"

namespace hd {

cudaError_t allow_dynamic_smem(const void* fn, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> allowed;  // (kernel, device) -> bytes
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = allowed[{fn, dev}];
  if (smem <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) cur = smem;
  return e;
}

int device_sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 1;
  static std::mutex mu;
  static std::map<int, int> sms;
  std::lock_guard<std::mutex> lk(mu);
  int& n = sms[dev];
  if (!n && cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n = 0;
  return n > 0 ? n : 1;
}

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

// ---------------------------------------------------------------------------
// Real-input path (hd_conv_real): pack the two halves of a real f along axis 0 as
// the real and imaginary parts of one complex array, and unpack the complex result
//   z[b][y][r] = f[b][y][r] + i f[b][y + A][r]            (y < A, 0 beyond Lf0)
//   h[b][y][r] = Re w[b][y][r] + Im w[b][y - A][r]         (each term where defined)
// R rows of `rest` elements each; memory-bound grid-stride loops.
// one CTA per (b, y) row at a time, threads along the contiguous rest: no per-element
// division, coalesced rows
template <typename R>
__global__ void real_pack_kernel(const R* __restrict__ f, typename cplx_of<R>::type* __restrict__ z,
                                 int64_t Lf0, int64_t A, int64_t rest, int64_t nb) {
  using V = typename cplx_of<R>::type;
  for (int64_t row = blockIdx.x; row < nb * A; row += gridDim.x) {
    const int64_t b = row / A, y = row - b * A;
    const R* fa = f + (b * Lf0 + y) * rest;
    const R* fb = (y + A < Lf0) ? fa + A * rest : nullptr;
    V* zr = z + row * rest;
    for (int64_t r = threadIdx.x; r < rest; r += blockDim.x) {
      V v;
      v.x = fa[r];
      v.y = fb ? fb[r] : (R)0;
      zr[r] = v;
    }
  }
}
template <typename R>
__global__ void real_to_complex_kernel(const R* __restrict__ g, typename cplx_of<R>::type* __restrict__ gc,
                                       int64_t n) {
  using V = typename cplx_of<R>::type;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    V v; v.x = g[i]; v.y = (R)0;
    gc[i] = v;
  }
}
template <typename R>
__global__ void real_unpack_kernel(const typename cplx_of<R>::type* __restrict__ w, R* __restrict__ h,
                                   int64_t Lout0, int64_t Ow0, int64_t A, int64_t rest, int64_t nb) {
  using V = typename cplx_of<R>::type;
  for (int64_t row = blockIdx.x; row < nb * Lout0; row += gridDim.x) {
    const int64_t b = row / Lout0, y = row - b * Lout0;
    const V* wa = (y < Ow0) ? w + (b * Ow0 + y) * rest : nullptr;
    const V* wb = (y >= A && y - A < Ow0) ? w + (b * Ow0 + y - A) * rest : nullptr;
    R* hr = h + row * rest;
    for (int64_t r = threadIdx.x; r < rest; r += blockDim.x) {
      R acc = wa ? wa[r].x : (R)0;
      if (wb) acc += wb[r].y;
      hr[r] = acc;
    }
  }
}

static unsigned grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (unsigned)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

cudaError_t launch_real_pack(bool is_double, const void* f, void* z, int64_t Lf0, int64_t A, int64_t rest,
                             int64_t nb, cudaStream_t st) {
  const unsigned g = grid_for(nb * A * 256);
  if (is_double) real_pack_kernel<double><<<g, 256, 0, st>>>((const double*)f, (double2*)z, Lf0, A, rest, nb);
  else real_pack_kernel<float><<<g, 256, 0, st>>>((const float*)f, (float2*)z, Lf0, A, rest, nb);
  return cudaGetLastError();
}
cudaError_t launch_real_to_complex(bool is_double, const void* g, void* gc, int64_t n, cudaStream_t st) {
  const unsigned gr = grid_for(n);
  if (is_double) real_to_complex_kernel<double><<<gr, 256, 0, st>>>((const double*)g, (double2*)gc, n);
  else real_to_complex_kernel<float><<<gr, 256, 0, st>>>((const float*)g, (float2*)gc, n);
  return cudaGetLastError();
}
cudaError_t launch_real_unpack(bool is_double, const void* w, void* h, int64_t Lout0, int64_t Ow0, int64_t A,
                               int64_t rest, int64_t nb, cudaStream_t st) {
  const unsigned g = grid_for(nb * Lout0 * 256);
  if (is_double)
    real_unpack_kernel<double><<<g, 256, 0, st>>>((const double2*)w, (double*)h, Lout0, Ow0, A, rest, nb);
  else real_unpack_kernel<float><<<g, 256, 0, st>>>((const float2*)w, (float*)h, Lout0, Ow0, A, rest, nb);
  return cudaGetLastError();
}

// fused real path (hd_conv_real): the Im parts of the w rows that overlap Re rows
__global__ void real_fixup_kernel(const double* __restrict__ side, double* h, int64_t rows, int64_t A,
                                  int64_t Lout0, int64_t rest) {
  const int64_t n = rows * rest;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = i / rest;
    if (y + A < Lout0) h[i + A * rest] += side[i];
  }
}
cudaError_t launch_real_fixup(const void* side, void* h, int64_t rows, int64_t A, int64_t Lout0, int64_t rest,
                              cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  real_fixup_kernel<<<grid_for(rows * rest), 256, 0, st>>>((const double*)side, (double*)h, rows, A, Lout0, rest);
  return cudaGetLastError();
}

// Row f1 matched product: H_{r_g}[l_g] = F_{q_g lambda + r_g}[l_f]
// G_{r_g}[l_g] * scale, l_f = l_g / Lambda, lambda = l_g mod Lambda; residue rows in
// the engine's spectral order (perm_g: position -> frequency of size Lambda m;
// iperm_f: frequency -> position of size m).  H overwrites G.
template <typename V>
__global__ void lambda_product_kernel(const V* __restrict__ Xf, V* Xg, const int32_t* __restrict__ perm_g,
                                      const int32_t* __restrict__ iperm_f, int64_t n, int m, int Lam, int qg,
                                      decltype(V::x) scale) {
  const int Lm = m * Lam;
  const int64_t M1 = (int64_t)qg * Lm;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = i / M1;
    const int64_t P = i - l * M1;
    const int rg = (int)(P / Lm), pos = (int)(P - (int64_t)rg * Lm);
    const int lg = __ldg(perm_g + pos);
    const int lam = lg % Lam, lf = lg / Lam;
    const int rf = qg * lam + rg;
    const V a = Xf[l * M1 + (int64_t)rf * m + __ldg(iperm_f + lf)];
    const V b = Xg[i];
    V c;
    c.x = (a.x * b.x - a.y * b.y) * scale;
    c.y = (a.x * b.y + a.y * b.x) * scale;
    Xg[i] = c;
  }
}

cudaError_t launch_lambda_product(bool is_double, const void* Xf, void* Xg, const int32_t* perm_g,
                                  const int32_t* iperm_f, int64_t nlines, int m, int Lam, int qg, double scale,
                                  cudaStream_t st) {
  const int64_t n = nlines * (int64_t)qg * m * Lam;
  const unsigned g = grid_for(n);
  if (is_double)
    lambda_product_kernel<double2><<<g, 256, 0, st>>>((const double2*)Xf, (double2*)Xg, perm_g, iperm_f, n, m,
                                                      Lam, qg, scale);
  else
    lambda_product_kernel<float2><<<g, 256, 0, st>>>((const float2*)Xf, (float2*)Xg, perm_g, iperm_f, n, m, Lam,
                                                     qg, (float)scale);
  return cudaGetLastError();
}

}  // namespace hd
