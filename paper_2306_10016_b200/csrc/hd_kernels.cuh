// hd_kernels.cuh -- launcher templates; each hd_k_<dtype>_<NT>.cu instantiates one
// (precision, max threads-per-CTA) slice so the slices compile in parallel.  The
// template NT only bounds registers (__launch_bounds__); the block size is runtime.
#pragma once
#include "hd_device.cuh"
#include "hd_internal.h"

namespace hd {

template <typename T, int M, int NT, int MODE>
static cudaError_t launch_pass_impl(const PassArgs& a, dim3 grid, int nt, size_t smem, cudaStream_t st) {
  auto kern = pass_kernel<T, M, NT, MODE>;
  if (cudaError_t e = allow_dynamic_smem(reinterpret_cast<const void*>(kern), smem); e != cudaSuccess) return e;
  if (nt < 32 || nt > NT || nt % 32) return cudaErrorInvalidConfiguration;
  // persistent grid: every SM gets as many CTAs as fit; grid.x work items are
  // strided over them (grid.x on entry = total work items)
  const int sms = device_sm_count();
  thread_local int occ_nt = -1, occ_val = 1;  // per thread: no shared mutable state
  thread_local size_t occ_smem = 0;
  if (occ_nt != nt || occ_smem != smem) {
    int nb = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, nt, smem) != cudaSuccess || nb < 1) nb = 1;
    occ_nt = nt; occ_smem = smem; occ_val = nb;
  }
  const int64_t cap = (int64_t)sms * occ_val;
  if ((int64_t)grid.x > cap) grid.x = (unsigned)cap;
  kern<<<grid, nt, smem, st>>>(a);
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
