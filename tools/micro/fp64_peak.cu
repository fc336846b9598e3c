// Microbenchmark: FP64 (and FP32) pipe throughput on this GPU, the ALU roof of the
// bench's roofline ("a measured FP64 peak").  Every thread runs 8
// independent dependency chains of DFMA (a = a * b + c) in registers, no memory
// traffic; grid = SMs x CTAs/SM, timed with CUDA events over several launches after
// warm-up.  Also DADD and DMUL chains (one flop per instruction) and FFMA for c64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
// Output: one JSON line with flop/s per instruction kind and the clock seen.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int KIND>  // 0: fma, 1: add, 2: mul
__global__ void __launch_bounds__(256) chains(T* out, int iters, T b, T c) {
  T a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = (T)(threadIdx.x + k) * (T)1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (KIND == 0) a[k] = fma(a[k], b, c);
        else if (KIND == 1) a[k] = a[k] + c;
        else a[k] = a[k] * b;
      }
  }
  T s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == (T)12345.678) out[threadIdx.x] = s;  // keeps the chains live
}

template <typename T, int KIND>
double run(int sms, int per_sm, int iters, float* ms_out) {
  T* out;
  cudaMalloc(&out, 1024 * sizeof(T));
  const int grid = sms * per_sm;
  const T b = (T)0.999999, c = (T)1e-7;
  for (int w = 0; w < 3; ++w) chains<T, KIND><<<grid, 256>>>(out, iters, b, c);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) chains<T, KIND><<<grid, 256>>>(out, iters, b, c);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  *ms_out = ms / reps;
  const double instr = (double)grid * 256 * iters * 16 * 8;  // per launch, thread-level
  const double flops_per = KIND == 0 ? 2.0 : 1.0;
  return instr * flops_per / (ms / reps * 1e-3);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int sms = p.multiProcessorCount;
  float ms;
  double best_fma = 0, best_add = 0, best_mul = 0, best_ffma = 0;
  int best_per_sm = 0;
  for (int per_sm : {2, 4, 8}) {
    const double v = run<double, 0>(sms, per_sm, 2000, &ms);
    if (v > best_fma) { best_fma = v; best_per_sm = per_sm; }
  }
  best_add = run<double, 1>(sms, best_per_sm, 2000, &ms);
  best_mul = run<double, 2>(sms, best_per_sm, 2000, &ms);
  for (int per_sm : {4, 8}) {
    const double v = run<float, 0>(sms, per_sm, 2000, &ms);
    if (v > best_ffma) best_ffma = v;
  }
  // the issue rate implied: DFMA thread-instructions per SM per clock at the rated clock
  const double lanes = best_fma / 2.0 / sms / (clk_khz * 1e3);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"rated_sm_mhz\": %.0f, \"ctas_per_sm\": %d, "
         "\"fp64_fma_tflops\": %.3f, \"fp64_add_tflops\": %.3f, \"fp64_mul_tflops\": %.3f, "
         "\"fp32_fma_tflops\": %.3f, \"dfma_lanes_per_sm_clk_at_rated\": %.2f}\n",
         p.name, sms, clk_khz / 1e3, best_per_sm, best_fma / 1e12, best_add / 1e12, best_mul / 1e12,
         best_ffma / 1e12, lanes);
  return 0;
}
