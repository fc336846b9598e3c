// hd_k_s128.cu -- launchers of the staged m = 128 complex-float engine (hd_s128.cuh):
// persistent CTAs (as many per SM as shared memory allows), blockDim = 32 (q + 1).
#include <cstdlib>

#include "hd_internal.h"
#include "hd_s128.cuh"

namespace hd {

template <int MODE, int NT, int QC, int MINB = 2, int ILK = 0, int OUTK = 0>
static cudaError_t launch_s128_impl(const PassArgs& a, dim3 grid, int nt, size_t smem, cudaStream_t st) {
  auto kern = s128::s128_kernel<MODE, NT, QC, MINB, ILK, OUTK>;
  if (cudaError_t e = allow_dynamic_smem(reinterpret_cast<const void*>(kern), smem); e != cudaSuccess) return e;
  if (nt < 64 || nt > NT || nt % 32) return cudaErrorInvalidConfiguration;
  const int sms = device_sm_count();
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const int64_t cap = (int64_t)sms * occ;
  if ((int64_t)grid.x > cap) grid.x = (unsigned)cap;
  kern<<<grid, nt, smem, st>>>(a);
  return cudaGetLastError();
}

// q = 5 (BASELINE config 4: M1 = 640 on every axis) has a compile-time-q kernel;
// blockDim bound 192 (q <= 5: two CTAs per SM at <= 168 registers) or 288 (q <= 8)
// q = 5 with line-tiled input: the layouts of the 3-D pipeline's passes at compile
// time (conv_z in place; inv_y -> element tiles of 4; inv_x -> rows; fwd_y_g ->
// interleaved)
template <int MODE>
static LaunchFn pick_s128(int q, int in_kind, int out_kind, int out_slog) {
  const bool il = in_kind == TMA_LINE_TILED;
  if (q == 5 && il) {
    const bool ip = s128::inplace_of(MODE, in_kind, out_kind);
    if constexpr (MODE == MODE_CONV) {
      if (ip) return launch_s128_impl<MODE, 192, 5, 2, 1, 1>;
    } else if constexpr (MODE == MODE_INV) {
      if (out_kind == TMA_ELEM_TILED && out_slog == 2) return launch_s128_impl<MODE, 192, 5, 2, 1, 2>;
      if (out_kind == TMA_BULK) return launch_s128_impl<MODE, 192, 5, 2, 1, 3>;
    } else {
      if (out_kind == TMA_LINE_TILED) return launch_s128_impl<MODE, 192, 5, 2, 1, 4>;
    }
    return launch_s128_impl<MODE, 192, 5, 2, 1>;
  }
  if (q == 5) return launch_s128_impl<MODE, 192, 5, 2>;
  if (q < 5) return launch_s128_impl<MODE, 192, 0>;
  return launch_s128_impl<MODE, 32 * (s128::kQMax + 1), 0>;
}
LaunchFn lookup_s128(int mode, int q, int in_kind, int out_kind, int out_slog) {
  if (q < 1 || q > s128::kQMax) return nullptr;
  switch (mode) {
    case MODE_FWD: return pick_s128<MODE_FWD>(q, in_kind, out_kind, out_slog);
    case MODE_INV: return pick_s128<MODE_INV>(q, in_kind, out_kind, out_slog);
    case MODE_CONV: return pick_s128<MODE_CONV>(q, in_kind, out_kind, out_slog);
    default: return nullptr;
  }
}

static cudaError_t launch_s128_bg_fwd(const PassArgs& a, dim3 grid, int nt, size_t smem, cudaStream_t st) {
  constexpr int NT = 32 * (s128::kBG * 5 + 1);
  auto kern = s128::s128_bg_fwd_kernel<5>;
  if (cudaError_t e = allow_dynamic_smem(reinterpret_cast<const void*>(kern), smem); e != cudaSuccess) return e;
  if (nt != NT) return cudaErrorInvalidConfiguration;
  const int sms = device_sm_count();
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const int64_t cap = (int64_t)sms * occ;
  if ((int64_t)grid.x > cap) grid.x = (unsigned)cap;
  kern<<<grid, nt, smem, st>>>(a);
  return cudaGetLastError();
}

// batch-grouped forward pass (four batch entries x four lines per item): q = 5 only
LaunchFn lookup_s128_bg(int mode, int q) {
  return (mode == MODE_FWD && q == 5) ? launch_s128_bg_fwd : nullptr;
}
int s128_bg_threads(int q) { return 32 * (s128::kBG * q + 1); }
size_t s128_bg_smem_bytes(int q, int64_t M1) { return s128::bg_smem_bytes(q, (int)M1); }

size_t s128_smem_bytes(int q, int mode, int64_t M1, int in_kind, int out_kind, int pg) {
  return s128::smem_bytes(q, mode, (int)M1, s128::inplace_of(mode, in_kind, out_kind), pg);
}

}  // namespace hd
