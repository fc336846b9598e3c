// hd_filter.cu -- the paper's image-filter pipeline around the convolution (SURVEY.md
// 8(f) row f3): a dictionary of eight small named kernels
// convolved with every channel of a real image, the real part of
// each channel's result kept (np.real(mainconvolve(v, data[:,:,i],
// ...))) and a window of it returned (the listing's crop; include/hdconv.h
// hd_conv_window for the mode formulas).  The convolutions are hd_conv_real calls (all
// channels as one batch); this file only holds the kernel table and two layout kernels
// (channel de-interleave, window crop + interleave).
#include "hdconv.h"
#include "hd_internal.h"

#include <cuda_runtime.h>

#include <cstring>
#include <string>

namespace {

thread_local std::string g_ferr;

hd_status_t ferr(hd_status_t st, const char* m) {
  g_ferr = m;
  return st;
}

struct FilterKernel {
  const char* name;
  int n;            // n x n
  double num, den;  // scale num / den
  int v[25];
};

// PAPER.md:1511-1518 (kernel .. kernel7), names of PAPER.md:1520 (kernels_dict)
const FilterKernel kKernels[HD_FILTER_COUNT] = {
    {"Identity", 3, 1, 1, {0, 0, 0, 0, 1, 0, 0, 0, 0}},
    {"Ridge_detection_1", 3, 1, 1, {-1, -1, -1, -1, 4, -1, -1, -1, -1}},
    {"Ridge_detection_2", 3, 1, 1, {-1, -1, -1, -1, 8, -1, -1, -1, -1}},
    {"Sharpen", 3, 1, 1, {0, -1, 0, -1, 5, -1, 0, -1, 0}},
    {"Box_blur", 3, 1, 9, {1, 1, 1, 1, 1, 1, 1, 1, 1}},
    {"Gaussian_blur", 3, 1, 16, {1, 2, 1, 2, 4, 2, 1, 2, 1}},
    {"Gaussian_blur_5", 5, 1, 256, {1, 4, 6, 4, 1, 4, 16, 24, 16, 4, 6, 24, 36, 24, 6, 4, 16, 24, 16, 4, 1, 4, 6, 4, 1}},
    {"Unsharpen_masking", 5, -1, 256,
     {1, 4, 6, 4, 1, 4, 16, 24, 16, 4, 6, 24, -476, 24, 6, 4, 16, 24, 16, 4, 1, 4, 6, 4, 1}},
};

struct KernelArg {
  double w[25];
};

// g[c][i][j] = kernel (replicated per channel: hd_conv_real takes one g per batch entry)
template <typename T>
__global__ void fill_kernel(T* g, KernelArg k, int nn, int C) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nn * C) g[i] = (T)k.w[i % nn];
}

// planes[c][y][x] = img[y][x][c]
template <typename T>
__global__ void deinterleave_kernel(const T* __restrict__ img, T* __restrict__ planes, int64_t HW, int C) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HW * C; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / HW, p = i % HW;
    planes[i] = img[p * C + c];
  }
}

// out = window [lo0, lo0 + n0) x [lo1, lo1 + n1) of full[c] (extent O0 x O1), laid out
// [n0][n1][C] (channel_last) or [C][n0][n1]
template <typename T>
__global__ void window_kernel(const T* __restrict__ full, T* __restrict__ out, int64_t O0, int64_t O1, int64_t lo0,
                              int64_t lo1, int64_t n0, int64_t n1, int C, int channel_last) {
  const int64_t total = n0 * n1 * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c, y, x;
    if (channel_last) { c = i % C; x = (i / C) % n1; y = i / (C * n1); }
    else { x = i % n1; y = (i / n1) % n0; c = i / (n0 * n1); }
    out[i] = full[(c * O0 + lo0 + y) * O1 + lo1 + x];
  }
}

unsigned blocks_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

template <typename T>
hd_status_t run(hd_ctx_t ctx, hd_dtype_t dtype, const void* img, int64_t H, int64_t W, int32_t C, int32_t channel_last,
                const FilterKernel& fk, const int64_t* lo, const int64_t* n, void* out, cudaStream_t st) {
  const int nn = fk.n * fk.n;
  const int64_t O0 = H + fk.n - 1, O1 = W + fk.n - 1;
  const size_t es = sizeof(T);
  const size_t bp = channel_last ? (size_t)C * H * W * es : 0;
  const size_t bg = ((size_t)C * nn * es + 255) & ~size_t(255);
  const size_t bf = (size_t)C * O0 * O1 * es;
  char* buf = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&buf), ((bp + 255) & ~size_t(255)) + bg + bf, st) != cudaSuccess)
    return ferr(HD_ERR_CUDA, "cudaMallocAsync(filter scratch)");
  T* planes = channel_last ? reinterpret_cast<T*>(buf) : const_cast<T*>(static_cast<const T*>(img));
  T* g = reinterpret_cast<T*>(buf + ((bp + 255) & ~size_t(255)));
  T* full = reinterpret_cast<T*>(reinterpret_cast<char*>(g) + bg);
  KernelArg k;
  for (int i = 0; i < nn; ++i) k.w[i] = fk.num * fk.v[i] / fk.den;
  fill_kernel<T><<<(unsigned)((nn * C + 63) / 64), 64, 0, st>>>(g, k, nn, C);
  if (channel_last) deinterleave_kernel<T><<<blocks_for(H * W * C), 256, 0, st>>>(static_cast<const T*>(img), planes, H * W, C);
  const int64_t Lf[2] = {H, W}, Lg[2] = {fk.n, fk.n};
  hd_status_t s = hd_conv_real(ctx, dtype, 2, C, planes, Lf, g, Lg, full, nullptr, st);
  if (s == HD_OK) {
    window_kernel<T><<<blocks_for(n[0] * n[1] * C), 256, 0, st>>>(full, static_cast<T*>(out), O0, O1, lo[0], lo[1],
                                                                  n[0], n[1], C, channel_last);
    if (cudaGetLastError() != cudaSuccess) s = ferr(HD_ERR_CUDA, "filter kernels");
  } else {
    g_ferr = hd_last_error(ctx);
  }
  cudaFreeAsync(buf, st);
  return s;
}

}  // namespace

extern "C" {

hd_status_t hd_filter_kernel(int32_t id, double* w, int32_t* n, const char** name) {
  if (id < 0 || id >= HD_FILTER_COUNT) return ferr(HD_ERR_INVALID, "filter id out of range");
  const FilterKernel& fk = kKernels[id];
  if (n) *n = fk.n;
  if (name) *name = fk.name;
  if (w)
    for (int i = 0; i < fk.n * fk.n; ++i) w[i] = fk.num * fk.v[i] / fk.den;
  return HD_OK;
}

const char* hd_filter_last_error(void) { return g_ferr.c_str(); }

hd_status_t hd_filter_image(hd_ctx_t ctx, hd_dtype_t dtype, const void* img, int64_t H, int64_t W, int32_t C,
                            int32_t channel_last, int32_t id, const int64_t* win_lo, const int64_t* win_n, void* out,
                            void* stream) {
  if (!ctx || !img || !out) return ferr(HD_ERR_INVALID, "null argument");
  if (dtype != HD_C64 && dtype != HD_C128) return ferr(HD_ERR_INVALID, "dtype must be HD_C64 (float) or HD_C128 (double)");
  if (H < 1 || W < 1 || C < 1 || C > 64) return ferr(HD_ERR_INVALID, "need H, W >= 1 and 1 <= C <= 64");
  if (id < 0 || id >= HD_FILTER_COUNT) return ferr(HD_ERR_INVALID, "filter id out of range");
  const FilterKernel& fk = kKernels[id];
  const int64_t O[2] = {H + fk.n - 1, W + fk.n - 1};
  int64_t lo[2] = {0, 0}, n[2] = {O[0], O[1]};
  if (win_lo && win_n) {
    for (int i = 0; i < 2; ++i) {
      if (win_lo[i] < 0 || win_n[i] < 1 || win_lo[i] + win_n[i] > O[i]) return ferr(HD_ERR_INVALID, "window outside the output");
      lo[i] = win_lo[i];
      n[i] = win_n[i];
    }
  }
  cudaStream_t st = (cudaStream_t)stream;
  return dtype == HD_C128 ? run<double>(ctx, dtype, img, H, W, C, channel_last, fk, lo, n, out, st)
                          : run<float>(ctx, dtype, img, H, W, C, channel_last, fk, lo, n, out, st);
}

}  // extern "C"
