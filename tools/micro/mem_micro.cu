// Memory-pattern microbenchmark for the 2D pass layouts (complex double, 16 B):
//  copy      : contiguous read -> contiguous write (peak reference)
//  tile<S>   : read rows y (4096 x 4608 elements) -> write X[k/S][y][k%S]
//              (each warp writes 16 S-element tiles of consecutive rows; S=2 uses 256-bit stores)
//  coltile<S>: read X tiles back one column k at a time (what conv_y's fold does)
#include <cstdio>
#include <cstdint>
using V = double2;
constexpr int NY = 4096, NK = 4608;

__global__ void copy_k(const V* __restrict__ a, V* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}
template <int S, int C = 1>
__global__ void tile_k(const V* __restrict__ a, V* __restrict__ x) {
  // block handles C rows; threads sweep (row, k) with the row fastest so that the C
  // rows' S-segments of one tile (contiguous C*S elements) are written together
  const int y0 = blockIdx.x * C;
  for (int it = threadIdx.x; it < C * (NK / S); it += blockDim.x) {
    const int c = it % C, k0 = (it / C) * S, ky = y0 + c;
    V v[S];
    for (int s = 0; s < S; ++s) v[s] = a[(int64_t)ky * NK + k0 + s];
    V* d = x + ((int64_t)(k0 / S) * NY + ky) * S;
    for (int s = 0; s < S; ++s) d[s] = v[s];
  }
}
template <int S>
__global__ void coltile_k(const V* __restrict__ x, V* __restrict__ b) {
  // block handles column k; threads sweep y
  const int k = blockIdx.x;
  double sx = 0, sy = 0;
  for (int y = threadIdx.x; y < NY; y += blockDim.x) {
    V v = x[((int64_t)(k / S) * NY + y) * S + (k % S)];
    sx += v.x; sy += v.y;
  }
  if (threadIdx.x == 0) b[k] = make_double2(sx, sy);
}

// read C adjacent columns of a row-major [NY][NK] matrix per block (threads sweep y)
template <int C>
__global__ void colrm_k(const V* __restrict__ a, V* __restrict__ b) {
  const int k0 = blockIdx.x * C;
  double sx = 0, sy = 0;
  for (int it = threadIdx.x; it < NY * C; it += blockDim.x) {
    const int c = it % C, y = it / C;
    V v = a[(int64_t)y * NK + k0 + c];
    sx += v.x; sy += v.y;
  }
  if (threadIdx.x == 0) b[blockIdx.x] = make_double2(sx, sy);
}
// write C adjacent columns of a row-major [NY][NK] matrix per block
template <int C>
__global__ void colwrm_k(V* __restrict__ a) {
  const int k0 = blockIdx.x * C;
  for (int it = threadIdx.x; it < NY * C; it += blockDim.x) {
    const int c = it % C, y = it / C;
    a[(int64_t)y * NK + k0 + c] = make_double2(y, c);
  }
}

template <typename F> float timeit(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(e0); for (int i = 0; i < 10; ++i) f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / 10;
}

int main() {
  const int64_t n = (int64_t)NY * NK;
  V *a, *x, *b;
  cudaMalloc(&a, n * 16); cudaMalloc(&x, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  double gb = 2.0 * n * 16 / 1e9;
  float t = timeit([&] { copy_k<<<148 * 8, 256>>>(a, b, n); });
  printf("copy         %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { tile_k<1><<<NY, 256>>>(a, x); }); printf("tile S=1     %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { tile_k<2><<<NY, 256>>>(a, x); }); printf("tile S=2     %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { tile_k<4><<<NY, 256>>>(a, x); }); printf("tile S=4     %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { tile_k<8><<<NY, 256>>>(a, x); }); printf("tile S=8     %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { tile_k<16><<<NY, 256>>>(a, x); }); printf("tile S=16    %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { tile_k<2, 2><<<NY / 2, 256>>>(a, x); }); printf("tile S=2 C=2 %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { tile_k<2, 4><<<NY / 4, 256>>>(a, x); }); printf("tile S=2 C=4 %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { tile_k<4, 4><<<NY / 4, 256>>>(a, x); }); printf("tile S=4 C=4 %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { tile_k<1, 8><<<NY / 8, 256>>>(a, x); }); printf("tile S=1 C=8 %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  double gr = 1.0 * n * 16 / 1e9;
  t = timeit([&] { coltile_k<1><<<NK, 256>>>(x, b); }); printf("coltile S=1  %.3f ms  %.0f GB/s (read)\n", t, gr / t * 1e3);
  t = timeit([&] { coltile_k<2><<<NK, 256>>>(x, b); }); printf("coltile S=2  %.3f ms  %.0f GB/s (read)\n", t, gr / t * 1e3);
  t = timeit([&] { coltile_k<4><<<NK, 256>>>(x, b); }); printf("coltile S=4  %.3f ms  %.0f GB/s (read)\n", t, gr / t * 1e3);
  t = timeit([&] { coltile_k<16><<<NK, 256>>>(x, b); }); printf("coltile S=16 %.3f ms  %.0f GB/s (read)\n", t, gr / t * 1e3);
  t = timeit([&] { colrm_k<1><<<NK, 256>>>(a, b); }); printf("colrm C=1    %.3f ms  %.0f GB/s (read)\n", t, gr / t * 1e3);
  t = timeit([&] { colrm_k<2><<<NK / 2, 256>>>(a, b); }); printf("colrm C=2    %.3f ms  %.0f GB/s (read)\n", t, gr / t * 1e3);
  t = timeit([&] { colrm_k<4><<<NK / 4, 256>>>(a, b); }); printf("colrm C=4    %.3f ms  %.0f GB/s (read)\n", t, gr / t * 1e3);
  t = timeit([&] { colwrm_k<1><<<NK, 256>>>(x); }); printf("colwrm C=1   %.3f ms  %.0f GB/s (write)\n", t, gr / t * 1e3);
  t = timeit([&] { colwrm_k<2><<<NK / 2, 256>>>(x); }); printf("colwrm C=2   %.3f ms  %.0f GB/s (write)\n", t, gr / t * 1e3);
  t = timeit([&] { colwrm_k<4><<<NK / 4, 256>>>(x); }); printf("colwrm C=4   %.3f ms  %.0f GB/s (write)\n", t, gr / t * 1e3);
  return 0;
}
