// Microbenchmark: warp FFT-512 throughput with two independent transforms interleaved
// stage by stage in one warp (the F and G transforms of a residue), vs one at a time,
// at 8 warps per SM (2 per sub-partition, up to 255 registers).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2306_10016_b200/csrc fft_dual.cu
#include <cstdio>
#include "hd_w512.cuh"
using namespace hd;
using namespace hd::w512;
using V = double2;

// two forward FFT-512s, interleaved stage by stage (same twiddle loads)
__device__ __forceinline__ void fft_fwd2(V* a, V* b, V* Ea, V* Eb, int lane, const V* tw) {
  dft16<+1>(a);
  dft16<+1>(b);
#pragma unroll
  for (int j = 1; j < 16; ++j) {
    const V w = tw[(j - 1) * 32];
    a[j] = cmul(a[j], w);
    b[j] = cmul(b[j], w);
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 16; ++j) { Ea[ex(j, lane)] = a[j]; Eb[ex(j, lane)] = b[j]; }
  __syncwarp();
  const int jj = lane >> 1, t2 = lane & 1;
#pragma unroll
  for (int i = 0; i < 16; ++i) { a[i] = Ea[ex(jj, t2 + 2 * i)]; b[i] = Eb[ex(jj, t2 + 2 * i)]; }
  dft16<+1>(a);
  dft16<+1>(b);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const V sa = t2 ? a[k] : a[k + 8], sb = t2 ? b[k] : b[k + 8];
    const V ra = shfl_x1(sa), rb = shfl_x1(sb);
    if (t2) { a[k] = ra; b[k] = rb; } else { a[k + 8] = ra; b[k + 8] = rb; }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const V w = tw[(15 + k) * 32];
    const V wa = cmul(a[k + 8], w), wb = cmul(b[k + 8], w);
    const V A = a[k], B = b[k];
    a[k] = cadd(A, wa); a[k + 8] = csub(A, wa);
    b[k] = cadd(B, wb); b[k + 8] = csub(B, wb);
  }
}

template <int WARPS, int DUAL>
__global__ void __launch_bounds__(WARPS * 32, 1) k_fft(double2* out, int iters) {
  extern __shared__ double2 E[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  V* tab = E + 2 * WARPS * 512;
  for (int i = threadIdx.x; i < kTwRows * 32; i += blockDim.x) {
    const int row = i >> 5, u = i & 31;
    const int e = row < 15 ? (u * (row + 1)) % 512 : 16 * ((row - 15) + 8 * (u & 1));
    const double ang = 2.0 * 3.14159265358979323846 * e / 512.0;
    tab[i] = make_double2(cos(ang), sin(ang));
  }
  __syncthreads();
  const V* tw = tab + lane;
  V* Ea = E + w * 1024;
  V* Eb = Ea + 512;
  V a[16], b[16];
  for (int i = 0; i < 16; ++i) { a[i] = make_double2(lane * 0.001 + i, i * 0.5 - lane); b[i] = make_double2(i - lane * 0.002, lane + 0.25 * i); }
  for (int it = 0; it < iters; ++it) {
    if (DUAL) {
      fft_fwd2(a, b, Ea, Eb, lane, tw);
    } else {
      fft_fwd(a, Ea, lane, tw);
      fft_fwd(b, Eb, lane, tw);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) { a[i] = cscale(a[i], 1.0 / 512.0); b[i] = cscale(b[i], 1.0 / 512.0); }
  }
  double2 s = a[0];
  for (int i = 1; i < 16; ++i) s = cadd(s, cadd(a[i], b[i]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int WARPS, int DUAL>
void run(int bps, int iters) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nb = sms * bps;
  double2* out; cudaMalloc(&out, (size_t)nb * WARPS * 32 * sizeof(double2));
  const size_t sm = (2 * WARPS * 512 + kTwRows * 32) * sizeof(double2);
  cudaFuncSetAttribute(k_fft<WARPS, DUAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_fft<WARPS, DUAL><<<nb, WARPS * 32, sm>>>(out, 2);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_fft<WARPS, DUAL><<<nb, WARPS * 32, sm>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k_fft<WARPS, DUAL>);
  const double ffts = (double)nb * WARPS * iters * 2;
  printf("warps/CTA %2d CTAs/SM %d dual %d regs %3d lmem %zu: %.1f ns per warp-FFT per SM %s\n", WARPS, bps, DUAL,
         fa.numRegs, fa.localSizeBytes, ms * 1e6 / (ffts / sms), err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(out);
}

int main() {
  run<8, 0>(1, 200); run<8, 1>(1, 200);
  run<9, 0>(1, 200); run<9, 1>(1, 200);
  run<10, 0>(1, 200); run<10, 1>(1, 200);
  run<12, 0>(1, 200); run<12, 1>(1, 200);
  run<16, 0>(1, 200); run<16, 1>(1, 200);
  run<4, 1>(2, 200); run<4, 1>(3, 200);
  return 0;
}
