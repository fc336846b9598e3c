// Microbenchmark: HBM throughput of 32-byte pieces scattered with a large stride
// (the 3-D pipeline's y -> z transpose: item (z, kx-tile g) touches 640 rows
// ky of 32 B at stride 2.6 MB; consecutive items are consecutive z, i.e. adjacent
// 32-byte pieces).  Write vs read vs contiguous rows of the same bytes.
// Build: nvcc -arch=sm_100a -O3 scatter32.cu -o scatter32
#include <cstdio>
#include <cuda_runtime.h>

constexpr int KY = 640, NG = 160, NZ = 512;  // pieces: KY x NG x NZ of 32 B
__global__ void k_write(float4* buf) {  // buf[ky][g][z][2 x float4]
  const int items = NG * NZ;
  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    const int z = w % NZ, g = w / NZ;
    for (int ky = threadIdx.x; ky < KY; ky += blockDim.x) {
      float4* p = buf + (((size_t)ky * NG + g) * NZ + z) * 2;
      p[0] = make_float4(w, ky, 0, 0);
      p[1] = make_float4(0, 0, w, ky);
    }
  }
}
// pieces of 32 * W bytes: one item = W consecutive z (the same bytes in total)
template <int W>
__global__ void k_write_w(float4* buf) {
  const int items = NG * NZ / W;
  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    const int z0 = (w % (NZ / W)) * W, g = w / (NZ / W);
    for (int i = threadIdx.x; i < KY * 2 * W; i += blockDim.x) {
      const int ky = i / (2 * W), o = i % (2 * W);
      buf[(((size_t)ky * NG + g) * NZ + z0) * 2 + o] = make_float4(w, ky, o, 0);
    }
  }
}
__global__ void k_read(const float4* buf, float* out) {
  const int items = NG * NZ;
  float acc = 0;
  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    const int z = w % NZ, g = w / NZ;
    for (int ky = threadIdx.x; ky < KY; ky += blockDim.x) {
      const float4* p = buf + (((size_t)ky * NG + g) * NZ + z) * 2;
      const float4 a = __ldcs(p), b = __ldcs(p + 1);
      acc += a.x + a.y + b.z + b.w;
    }
  }
  if (acc == 123.f) out[0] = acc;
}
__global__ void k_contig(float4* buf) {  // same bytes, item writes one contiguous 20 KB row
  const int items = NG * NZ;
  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    float4* p = buf + (size_t)w * KY * 2;
    for (int i = threadIdx.x; i < KY * 2; i += blockDim.x) p[i] = make_float4(w, i, 0, 0);
  }
}

int main() {
  const size_t bytes = (size_t)KY * NG * NZ * 32;
  float4* buf;
  float* out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int bpsm : {2, 4, 8}) {
    const int grid = sms * bpsm;
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a); k_write<<<grid, 128>>>(buf); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("CTAs/SM %d scattered write: %.3f ms %.2f TB/s\n", bpsm, ms, bytes / ms / 1e9);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a); k_read<<<grid, 128>>>(buf, out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("CTAs/SM %d scattered read:  %.3f ms %.2f TB/s\n", bpsm, ms, bytes / ms / 1e9);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a); k_contig<<<grid, 128>>>(buf); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("CTAs/SM %d contiguous write: %.3f ms %.2f TB/s\n", bpsm, ms, bytes / ms / 1e9);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a); k_write_w<2><<<grid, 128>>>(buf); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("CTAs/SM %d 64-byte pieces write: %.3f ms %.2f TB/s\n", bpsm, ms, bytes / ms / 1e9);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a); k_write_w<4><<<grid, 128>>>(buf); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("CTAs/SM %d 128-byte pieces write: %.3f ms %.2f TB/s\n", bpsm, ms, bytes / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
