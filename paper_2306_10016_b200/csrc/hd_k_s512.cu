// hd_k_s512.cu -- launchers of the staged m = 512 warp engine (hd_s512.cuh):
// one persistent CTA per SM (two-stage cp.async ring, ~170 KB of shared memory),
// blockDim = 32 q.
#include <cstdlib>
#include "hd_internal.h"
#include "hd_s512.cuh"

namespace hd {

template <int MODE, int NTMAX, int QC, int LEAN = 0>
static cudaError_t launch_s512_impl(const PassArgs& a, dim3 grid, int nt, size_t smem, cudaStream_t st) {
  auto kern = s512::s512_kernel<MODE, NTMAX, QC, LEAN>;
  if (cudaError_t e = allow_dynamic_smem(reinterpret_cast<const void*>(kern), smem); e != cudaSuccess) return e;
  if (nt < 32 || nt > NTMAX || nt % 32) return cudaErrorInvalidConfiguration;
  // W8: setmaxnreg acts on whole warpgroups -- exactly three of them
  if (QC == 9 && NTMAX == 384 && nt != 384) return cudaErrorInvalidConfiguration;
  const int sms = device_sm_count();
  int occ = 1;
  if (LEAN) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
  }
  if ((int64_t)grid.x > (int64_t)sms * occ) grid.x = (unsigned)(sms * occ);
  kern<<<grid, nt, smem, st>>>(a);
  return cudaGetLastError();
}

// q = 9: eight compute warps at 232 registers (s512_kernel's W8 layout, blockDim 384),
// else nine at 168 (blockDim 320).  HD_S512_W8 (A/B switch) = bit mask: 1 the x passes
// (forward and inverse together: W8 stores residue 8's spectrum as two FFT-256 halves,
// an order both passes of an axis must share), 2 the convolution pass.
constexpr int kW8Default = 2;
static bool s512_w8(int mode) {
  static const int mask = [] {
    const char* e = getenv("HD_S512_W8");
    return e ? atoi(e) : kW8Default;
  }();
  return (mask >> (mode == MODE_CONV ? 1 : 0)) & 1;
}

// q = 9 (the BASELINE 2-D configs' axes) has a compile-time-q instantiation; other
// q get a runtime-q kernel.  blockDim = 32 (q + 1): q compute warps + the producer.
template <int MODE>
static LaunchFn pick_s512(int q) {
  if (q == 9) return s512_w8(MODE) ? launch_s512_impl<MODE, 384, 9> : launch_s512_impl<MODE, 320, 9>;
  if (q == 7) return launch_s512_impl<MODE, 256, 7>;  // BASELINE config 5's x axis
  if (q == 5) return launch_s512_impl<MODE, 192, 5, 1>;  // the real path's packed y axis (lean)
  if (q <= kS512LeanQ) return launch_s512_impl<MODE, 32 * (kS512LeanQ + 1), 0, 1>;
  return launch_s512_impl<MODE, 32 * (s512::kQMax + 1), 0>;
}
LaunchFn lookup_s512(int mode, int q) {
  switch (mode) {
    case MODE_FWD: return pick_s512<MODE_FWD>(q);
    case MODE_INV: return pick_s512<MODE_INV>(q);
    case MODE_CONV: return pick_s512<MODE_CONV>(q);
    default: return nullptr;
  }
}

template <int QC>
static cudaError_t launch_s512_mconv(const PassArgs& a, dim3 grid, int nt, size_t smem, cudaStream_t st) {
  constexpr int NT = 32 * (s512::kMconvQMax + 1);
  auto kern = s512::s512_mconv_kernel<NT, QC>;
  if (cudaError_t e = allow_dynamic_smem(reinterpret_cast<const void*>(kern), smem); e != cudaSuccess) return e;
  if (nt < 64 || nt > NT || nt % 32) return cudaErrorInvalidConfiguration;
  const int sms = device_sm_count();
  if ((int64_t)grid.x > sms) grid.x = (unsigned)sms;
  kern<<<grid, nt, smem, st>>>(a);
  return cudaGetLastError();
}

// q = 6 (BASELINE config 5's convolution axis) at compile time; other q at run time
LaunchFn lookup_s512_mconv(int q) { return q == 6 ? launch_s512_mconv<6> : launch_s512_mconv<0>; }
int s512_mconv_qmax() { return s512::kMconvQMax; }

// compute warps + the producer warp
int s512_threads(int q, int mode) {
  if (q == 9 && mode != MODE_MCONV && s512_w8(mode)) return 384;
  return 32 * (q + 1);
}

size_t s512_smem_bytes(int q, int mode) {
  if (mode == MODE_MCONV)
    return 128 + sizeof(double2) * (size_t)(kQF * kQF + w512::kTwRows * 32 + 512 + 2 * (2 * q * 512));
  const bool lean = q <= kS512LeanQ && q != 9;
  // W8: the FFT-256 twiddle columns; the convolution pass also G_8's halves (X)
  const bool w8 = q == 9 && s512_w8(mode);
  return 128 + sizeof(double2) * (size_t)(q * kQF + w512::kTwRows * 32 + (lean ? 0 : 512) +
                                          2 * (q * 512 + (mode == MODE_CONV ? 512 : 0)) +
                                          (w8 ? w256::kTwRows * 32 + (mode == MODE_CONV ? 512 : 0) : 0));
}

}  // namespace hd

// ---------------------------------------------------------------------------
// 1-D long lines: two-CTA clusters (hd_s512c.cuh), 12 <= q <= 22
// ---------------------------------------------------------------------------
#include "hd_s512c.cuh"
namespace hd {
static cudaError_t launch_s512c(const PassArgs& a, dim3 grid, int nt, size_t smem, cudaStream_t st) {
  constexpr int NT = 32 * s512c::kRMax;
  auto kern = s512c::s512c_kernel<NT>;
  if (cudaError_t e = allow_dynamic_smem(reinterpret_cast<const void*>(kern), smem); e != cudaSuccess) return e;
  if (nt < 32 || nt > NT || nt % 32) return cudaErrorInvalidConfiguration;
  const int sms = device_sm_count();
  // one cluster of two CTAs per line, persistent: at most one CTA per SM
  int64_t ncl = (int64_t)a.nlines;
  if (ncl > sms / 2) ncl = sms / 2;
  grid.x = (unsigned)(2 * ncl);
  grid.y = 1;
  grid.z = 1;
  kern<<<grid, nt, smem, st>>>(a);
  return cudaGetLastError();
}
LaunchFn lookup_s512c() { return launch_s512c; }
int s512c_threads(int q) {
  const int P = (q - 1) / 2, K0 = (q & 1) ? (P + 1) / 2 : P / 2;
  const int n0 = 1 + 2 * K0, n1 = 2 * (P - K0) + ((q & 1) ? 0 : 1);
  return 32 * (n0 > n1 ? n0 : n1);
}
size_t s512c_smem_bytes() { return s512c::smem_bytes(); }
}  // namespace hd

