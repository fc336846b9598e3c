// hd_internal.h -- declarations shared by the host driver (hd_api.cu) and the
// kernel instantiations (hd_kernels.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hd {
struct PassArgs;
using LaunchFn = cudaError_t (*)(const PassArgs&, dim3, int, size_t, cudaStream_t);
// nullptr if (m, mode) has no instantiation or threads exceeds every slice bound
LaunchFn lookup_launcher(bool is_double, int m, int mode, int threads);
// staged warp engine for m = 512 complex double (hd_s512.cuh); blockDim = 32 (q + 1) <= 384
LaunchFn lookup_s512(int mode, int q);
constexpr int kS512QMax = 11;
constexpr int kS512LeanQ = 5;  // q <= 5: two CTAs per SM (zeta_{M1}^s from global memory)
// 1-D convolution pass of long lines (hd_s512c.cuh): m = 512, a two-CTA cluster
// per line, 12 <= q <= 22
constexpr int kS512cQMin = 12, kS512cQMax = 22;
LaunchFn lookup_s512c();
// 1-D convolution pass of long lines at m = 2048, one CTA per line (hd_s2048r.cuh), q <= 8
LaunchFn lookup_s2048r();
int s2048r_threads();
int s2048r_qmax();
size_t s2048r_smem_bytes();
// 1-D convolution pass of long lines at m = 4096, one CTA per line (hd_s4096r.cuh), q <= 4, p <= 4
LaunchFn lookup_s4096r();
int s4096r_threads();
int s4096r_qmax();
int s4096r_pmax();
size_t s4096r_smem_bytes();
int s512c_threads(int q);
size_t s512c_smem_bytes();
size_t s512_smem_bytes(int q, int mode);
int s512_threads(int q, int mode);
// staged multi-pair convolution pass (MODE_MCONV): q <= s512_mconv_qmax()
LaunchFn lookup_s512_mconv(int q);
int s512_mconv_qmax();
// staged engine for m = 128 complex float, 4 lines per item (hd_s128.cuh);
// blockDim = 32 (q + 1), q <= kS128QMax
// in_kind / out_kind / out_slog: the launch's TMA descriptions (compile-time layouts)
LaunchFn lookup_s128(int mode, int q, int in_kind, int out_kind, int out_slog);
constexpr int kS128QMax = 8;
size_t s128_smem_bytes(int q, int mode, int64_t M1, int in_kind, int out_kind, int pg);
// its batch-grouped forward pass (4 batch entries x 4 lines per item), q = 5
LaunchFn lookup_s128_bg(int mode, int q);
int s128_bg_threads(int q);
size_t s128_bg_smem_bytes(int q, int64_t M1);
cudaError_t launch_pad(bool is_double, const void* src, void* dst, const int64_t L[3],
                       const int64_t P[3], int64_t nb, cudaStream_t st);
cudaError_t launch_crop(bool is_double, const void* src, void* dst, const int64_t O[3],
                        const int64_t P[3], int64_t nb, cudaStream_t st);
// real-input path (hd_conv_real): pack / promote / unpack kernels (hd_kernels.cu)
cudaError_t launch_real_pack(bool is_double, const void* f, void* z, int64_t Lf0, int64_t A, int64_t rest,
                             int64_t nb, cudaStream_t st);
cudaError_t launch_real_to_complex(bool is_double, const void* g, void* gc, int64_t n, cudaStream_t st);
cudaError_t launch_real_unpack(bool is_double, const void* w, void* h, int64_t Lout0, int64_t Ow0, int64_t A,
                               int64_t rest, int64_t nb, cudaStream_t st);
// fused real path: h[y + A] += side[y] for y < rows (rows of `rest` doubles, y + A < Lout0)
cudaError_t launch_real_fixup(const void* side, void* h, int64_t rows, int64_t A, int64_t Lout0, int64_t rest,
                              cudaStream_t st);
// row f1 (hd_conv1d_lambda): matched product of the Lambda > 1 residue construction
cudaError_t launch_lambda_product(bool is_double, const void* Xf, void* Xg, const int32_t* perm_g,
                                  const int32_t* iperm_f, int64_t nlines, int m, int Lam, int qg, double scale,
                                  cudaStream_t st);
constexpr size_t kMaxSmem = 227 * 1024;
// Launcher helpers (hd_kernels.cu), thread-safe and per device (the dynamic
// shared-memory opt-in is a per-device function attribute): allow `smem` bytes of
// dynamic shared memory for kernel `fn` on the current device (no-op at <= 48 KB
// or when already allowed), and the current device's SM count.
cudaError_t allow_dynamic_smem(const void* fn, size_t smem);
int device_sm_count();
// hd_dist.cu: release a context's communicator and exchange buffers (hd_destroy)
void dist_release(struct hd_ctx* ctx);
}  // namespace hd
