// Microbenchmark: throughput of the warp-level FFT-512 (fwd + inv) with no global
// memory traffic, at several warps/CTA.  Build: nvcc -arch=sm_100a -O3 -I../../paper_2306_10016_b200/csrc
#include <cstdio>
#include "hd_w512.cuh"
using namespace hd;
using V = double2;

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) k_fft(double2* out, int iters) {
  extern __shared__ double2 E[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  V* tab = E + WARPS * 512;
  for (int i = threadIdx.x; i < w512::kTwRows * 32; i += blockDim.x) {
    const int row = i >> 5, u = i & 31;
    const int e = row < 15 ? (u * (row + 1)) % 512 : 16 * ((row - 15) + 8 * (u & 1));
    const double a = 2.0 * 3.14159265358979323846 * e / 512.0;
    tab[i] = make_double2(cos(a), sin(a));
  }
  __syncthreads();
  const V* tw = tab + lane;
  V* Fr = E + w * 512;
  V v[16];
  for (int i = 0; i < 16; ++i) v[i] = make_double2(lane * 0.001 + i, i * 0.5 - lane);
  for (int it = 0; it < iters; ++it) {
    w512::fft_fwd(v, Fr, lane, tw);
    for (int i = 0; i < 16; ++i) v[i] = cscale(v[i], 1.0 / 512.0);
    w512::fft_inv(v, Fr, lane, tw);
  }
  double2 s = v[0];
  for (int i = 1; i < 16; ++i) s = cadd(s, v[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int WARPS>
void run(int blocks_per_sm, int iters) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nb = sms * blocks_per_sm;
  double2* out; cudaMalloc(&out, (size_t)nb * WARPS * 32 * sizeof(double2));
  const size_t sm = (WARPS * 512 + w512::kTwRows * 32) * sizeof(double2);
  cudaFuncSetAttribute(k_fft<WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_fft<WARPS><<<nb, WARPS * 32, sm>>>(out, 2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_fft<WARPS><<<nb, WARPS * 32, sm>>>(out, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k_fft<WARPS>);
  const double ffts = (double)nb * WARPS * iters * 2;       // warp-FFT-512s (fwd + inv)
  const double pts = ffts * 512;
  printf("warps/CTA %2d CTAs/SM %d regs %d: %.3f ms, %.1f ns per warp-FFT per SM, %.2f Gpts/s/SM-pair\n",
         WARPS, blocks_per_sm, fa.numRegs, ms, ms * 1e6 / (ffts / sms), pts / (ms * 1e-3) / 1e9);
  cudaFree(out);
}

int main() {
  run<9>(1, 200); run<12>(1, 200); run<16>(1, 200); run<18>(1, 200);
  run<9>(2, 200); run<4>(4, 200); run<8>(2, 200); run<4>(3, 200); run<4>(2, 200); run<4>(1, 200);
  return 0;
}
