// hd_k_s4096r.cu -- launcher of the 1-D m = 4096 engine (hd_s4096r.cuh): one persistent
// CTA per SM (256 threads), one line per iteration.
#include "hd_internal.h"
#include "hd_s4096r.cuh"

namespace hd {

static cudaError_t launch_s4096r(const PassArgs& a, dim3 grid, int nt, size_t smem, cudaStream_t st) {
  auto kern = a.q <= 3 ? (a.out.j0 != 0 ? s4096r::s4096r_kernel<true, 3> : s4096r::s4096r_kernel<false, 3>)
                       : (a.out.j0 != 0 ? s4096r::s4096r_kernel<true, 4> : s4096r::s4096r_kernel<false, 4>);
  if (cudaError_t e = allow_dynamic_smem(reinterpret_cast<const void*>(kern), smem); e != cudaSuccess) return e;
  if (nt != s4096r::NT) return cudaErrorInvalidConfiguration;
  const int sms = device_sm_count();
  int64_t n = a.nlines < sms ? a.nlines : sms;
  grid.x = (unsigned)(n < 1 ? 1 : n);
  grid.y = 1;
  grid.z = 1;
  kern<<<grid, nt, smem, st>>>(a);
  return cudaGetLastError();
}

LaunchFn lookup_s4096r() { return launch_s4096r; }
int s4096r_threads() { return s4096r::NT; }
int s4096r_qmax() { return s4096r::kQMax; }
int s4096r_pmax() { return s4096r::kPMax; }
size_t s4096r_smem_bytes() {
  return sizeof(double2) * (size_t)(3 * 4096 + w512::kTwRows * 32 + 8 * s4096r::kQMax * s4096r::kPMax) + 16;
}

}  // namespace hd
