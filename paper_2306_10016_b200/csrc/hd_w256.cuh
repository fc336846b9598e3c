// hd_w256.cuh -- register FFT of size 256 (complex double) for one warp, 8 values per
// lane: the sub-transforms of the 1-D engine's FFT-2048 (hd_s2048r.cuh).
//
// 256 = 8 x 32 with 32 = 8 x 4 ("W <- m F(W)", positive exponent):
//   L1  DFT-8 over x[u + 32 i] (lane u, register i), twiddle zeta_256^{u k1}
//   X1  warp-local transpose (256 slots, XOR swizzle: conflict-free both ways)
//   L2  lane v = (k1 = v >> 2, c = v & 3) holds Y1[k1][c + 4 j]: DFT-8 over j,
//       twiddle zeta_32^{c m}
//   X2  transpose: lane w = (k1, mm) gathers Z[k1][c][2 mm + b], c < 4, b < 2
//   L3  two DFT-4 over c:  register 4 b + k3 of lane w holds frequency
//       k1 + 8 (2 mm + b) + 64 k3           (k1 = w >> 2, mm = w & 3)
// 128-bit shared accesses are served per quarter warp (8 consecutive lanes): every
// exchange pattern below puts those 8 lanes on 8 distinct 16-byte bank groups.  The
// inverse is the exact adjoint (negative exponents).
#pragma once
#include "hd_device.cuh"

namespace hd {
namespace w256 {

using V = double2;
constexpr int kTwRows = 14;  // per-lane twiddle column: 7 rows zeta_256^{u k1}, 7 rows zeta_32^{(u&3) m}

// the twiddle column from a zeta_N^k table (N a multiple of 256)
__device__ __forceinline__ V tw_entry(const V* twN, int N, int row, int lane) {
  if (row < 7) return ldg(twN + ((N / 256) * lane * (row + 1)) % N);
  return ldg(twN + ((N / 32) * (lane & 3) * (row - 6)) % N);
}

// register index -> frequency after fft256_fwd
__device__ __forceinline__ int freq256(int lane, int reg) {
  return (lane >> 2) + 8 * (2 * (lane & 3) + (reg >> 2)) + 64 * (reg & 3);
}

// slot of Z[k1][c][m] in the second exchange: row (4 k1 + c), column m ^ ((k1 & 1) | 2c)
__device__ __forceinline__ int x2_slot(int k1, int c, int m) {
  return (4 * k1 + c) * 8 + (m ^ ((k1 & 1) | (c << 1)));
}

// Forward FFT-256.  In: a[i] = x[lane + 32 i].  Out: a[reg] = X[freq256(lane, reg)].
// E: this warp's 256 exchange slots; tw: this lane's twiddle column (tw[row * 32]).
__device__ __forceinline__ void fft256_fwd(V* a, V* E, int lane, const V* tw) {
  dft8<V, +1>(a);
#pragma unroll
  for (int k = 1; k < 8; ++k) a[k] = cmul(a[k], tw[(k - 1) * 32]);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) E[k * 32 + (lane ^ (4 * (k & 1)))] = a[k];
  __syncwarp();
  {
    const int k1 = lane >> 2, c = lane & 3;
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = E[k1 * 32 + ((c + 4 * j) ^ (4 * (k1 & 1)))];
  }
  dft8<V, +1>(a);
#pragma unroll
  for (int m = 1; m < 8; ++m) a[m] = cmul(a[m], tw[(6 + m) * 32]);
  __syncwarp();
  {
    const int sw = ((lane >> 2) & 1) | ((lane & 3) << 1);
#pragma unroll
    for (int m = 0; m < 8; ++m) E[lane * 8 + (m ^ sw)] = a[m];
  }
  __syncwarp();
  {
    const int k1 = lane >> 2, mm = lane & 3;
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) a[4 * b + c] = E[x2_slot(k1, c, 2 * mm + b)];
  }
  dft4<V, +1>(a);
  dft4<V, +1>(a + 4);
}

// Inverse FFT-256 (adjoint of fft256_fwd).  In: a[reg] = Y[freq256(lane, reg)].
// Out: a[i] = sum_f zeta_256^{-(lane + 32 i) f} Y[f].
__device__ __forceinline__ void fft256_inv(V* a, V* E, int lane, const V* tw) {
  dft4<V, -1>(a);
  dft4<V, -1>(a + 4);
  __syncwarp();
  {
    const int k1 = lane >> 2, mm = lane & 3;
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) E[x2_slot(k1, c, 2 * mm + b)] = a[4 * b + c];
  }
  __syncwarp();
  {
    const int sw = ((lane >> 2) & 1) | ((lane & 3) << 1);
#pragma unroll
    for (int m = 0; m < 8; ++m) a[m] = E[lane * 8 + (m ^ sw)];
  }
#pragma unroll
  for (int m = 1; m < 8; ++m) a[m] = cmulc(a[m], tw[(6 + m) * 32]);
  dft8<V, -1>(a);
  __syncwarp();
  {
    const int k1 = lane >> 2, c = lane & 3;
#pragma unroll
    for (int j = 0; j < 8; ++j) E[k1 * 32 + ((c + 4 * j) ^ (4 * (k1 & 1)))] = a[j];
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = E[k * 32 + (lane ^ (4 * (k & 1)))];
#pragma unroll
  for (int k = 1; k < 8; ++k) a[k] = cmulc(a[k], tw[(k - 1) * 32]);
  dft8<V, -1>(a);
}

}  // namespace w256
}  // namespace hd
