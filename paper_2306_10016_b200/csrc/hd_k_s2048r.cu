// hd_k_s2048r.cu -- launcher of the 1-D m = 2048 engine (hd_s2048r.cuh): one persistent
// CTA per SM (512 threads, two warp groups), one line per iteration.
#include "hd_internal.h"
#include "hd_s2048r.cuh"

namespace hd {

static cudaError_t launch_s2048r(const PassArgs& a, dim3 grid, int nt, size_t smem, cudaStream_t st) {
  auto kern = s2048r::s2048r_kernel;
  if (cudaError_t e = allow_dynamic_smem(reinterpret_cast<const void*>(kern), smem); e != cudaSuccess) return e;
  if (nt != s2048r::NT) return cudaErrorInvalidConfiguration;
  const int sms = device_sm_count();
  int64_t n = a.nlines < sms ? a.nlines : sms;
  grid.x = (unsigned)(n < 1 ? 1 : n);
  grid.y = 1;
  grid.z = 1;
  kern<<<grid, nt, smem, st>>>(a);
  return cudaGetLastError();
}

LaunchFn lookup_s2048r() { return launch_s2048r; }
int s2048r_threads() { return s2048r::NT; }
int s2048r_qmax() { return s2048r::kQMax; }
size_t s2048r_smem_bytes() {
  return sizeof(double2) * (size_t)(4 * 2048 + 7 * 256 + w256::kTwRows * 32 + s2048r::kQMax + 8 * s2048r::kQMax);
}

}  // namespace hd
