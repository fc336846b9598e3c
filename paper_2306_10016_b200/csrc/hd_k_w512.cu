// hd_k_w512.cu -- launchers of the warp-level m = 512 engine (hd_w512.cuh).
#include "hd_internal.h"
#include "hd_w512.cuh"

namespace hd {

template <int MODE>
static cudaError_t launch_w512_impl(const PassArgs& a, dim3 grid, int nt, size_t smem, cudaStream_t st) {
  auto kern = w512::w512_kernel<MODE>;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  if (nt < 32 || nt > 288 || nt % 32) return cudaErrorInvalidConfiguration;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  static int occ_nt = -1, occ_val = 1;
  static size_t occ_smem = 0;
  if (occ_nt != nt || occ_smem != smem) {
    int nb = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, nt, smem) != cudaSuccess || nb < 1) nb = 1;
    occ_nt = nt; occ_smem = smem; occ_val = nb;
  }
  // CONV parks F-hat in a scratch sized for <= 4 CTAs per SM (hd_api.cu)
  const int64_t cap = (int64_t)sms * (MODE == MODE_CONV ? (occ_val < 4 ? occ_val : 4) : occ_val);
  if ((int64_t)grid.x > cap) grid.x = (unsigned)cap;
  kern<<<grid, nt, smem, st>>>(a);
  return cudaGetLastError();
}

LaunchFn lookup_w512(int mode) {
  switch (mode) {
    case MODE_FWD: return launch_w512_impl<MODE_FWD>;
    case MODE_INV: return launch_w512_impl<MODE_INV>;
    case MODE_CONV: return launch_w512_impl<MODE_CONV>;
    default: return nullptr;
  }
}

}  // namespace hd
