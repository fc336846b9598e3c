// Which hardware warp slot (%warpid; sub-partition = warpid % 4) does each warp of a
// 1-CTA-per-SM block land on?  (Used to check the sub-partition balance assumptions
// of the staged engine.)
#include <cstdio>
__global__ void k(int* out) {
  unsigned w;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(w));
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 32 + (threadIdx.x >> 5)] = (int)w;
}
int main() {
  int* d; cudaMalloc(&d, 148 * 32 * sizeof(int));
  for (int nt : {288, 320, 384}) {
    cudaMemset(d, 0xff, 148 * 32 * sizeof(int));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k<<<148, nt, 200 * 1024>>>(d);
    int h[148 * 32]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int b = 0; b < 3; ++b) {
      printf("nt=%d block %d:", nt, b);
      for (int i = 0; i < nt / 32; ++i) printf(" %d", h[b * 32 + i]);
      printf("\n");
    }
  }
  return 0;
}
