// hd_w512.cuh -- warp-level engine for FFT size m = 512 (complex double).
//
// One warp owns one residue r of one line: its size-512 FFT (PAPER.md:104,
// "W <- m F(W)") runs in registers as 512 = 16 x 16 x 2:
//   L1  radix-16 over x[lane + 32 i] (16 values per lane), twiddle zeta_512^{lane j}
//   --  warp-local transpose through shared memory (no CTA barrier)
//   L2  radix-16 over the stride-2 decimation of each 32-point sub-problem,
//       twiddle zeta_32^{(lane&1) k2}
//   L3  radix-2 between lane pairs (shuffle)
// Lane u then holds frequency f = (u>>1) + 16 k2 + 256 (u&1) in register k2.  The
// spectrum is stored in the SAME digit-reversed order as the generic radix-8 engine
// (position = base-8 digit reversal of f), so the internal spectral layout does not
// depend on which engine ran.  The inverse is the exact adjoint (negative exponent,
// PAPER.md:121).  The multi-pass structure (fold, product, unfold) is unchanged.
#pragma once
#include "hd_device.cuh"

namespace hd {
namespace w512 {

using V = double2;

// 16-point DFT in registers, y_k = sum_n v_n zeta_16^{S n k}, natural order out.
// 4 x 4 Cooley-Tukey: n = 4 n1 + n2, k = k1 + 4 k2.
template <int S> __device__ __forceinline__ void dft16(V* v) {
  const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
  const double h = 0.70710678118654752440;
  V A[4][4];
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    V t[4] = {v[n2], v[4 + n2], v[8 + n2], v[12 + n2]};
    dft4<V, S>(t);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) A[n2][k1] = t[k1];
  }
  // twiddles zeta_16^{S n2 k1}
  auto rot = [&](V a, double c, double s) {  // a * (c + i S s)
    return cmk<V>(fma(a.x, c, -S * a.y * s), fma(a.y, c, S * a.x * s));
  };
  A[1][1] = rot(A[1][1], c1, s1);                                   // 1
  A[1][2] = cmk<V>(h * (A[1][2].x - S * A[1][2].y), h * (A[1][2].y + S * A[1][2].x));  // 2
  A[1][3] = rot(A[1][3], s1, c1);                                   // 3
  A[2][1] = cmk<V>(h * (A[2][1].x - S * A[2][1].y), h * (A[2][1].y + S * A[2][1].x));  // 2
  A[2][2] = cmul_si<V, S>(A[2][2]);                                 // 4
  A[2][3] = cmk<V>(h * (-A[2][3].x - S * A[2][3].y), h * (-A[2][3].y + S * A[2][3].x));  // 6
  A[3][1] = rot(A[3][1], s1, c1);                                   // 3
  A[3][2] = cmk<V>(h * (-A[3][2].x - S * A[3][2].y), h * (-A[3][2].y + S * A[3][2].x));  // 6
  A[3][3] = rot(A[3][3], -c1, -s1);                                 // 9
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    V t[4] = {A[0][k1], A[1][k1], A[2][k1], A[3][k1]};
    dft4<V, S>(t);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = t[k2];
  }
}

// exchange slot of element (row j < 16, column t < 32) inside a 512-slot region
__device__ __forceinline__ int ex(int j, int t) { return j * 32 + (t ^ ((j & 3) << 1)); }

// zeta_32^k, k < 16 (constant bank operands, no load instructions)
__constant__ double2 c_w32[16] = {
    {1.0, 0.0},
    {0.98078528040323044913, 0.19509032201612826785},
    {0.92387953251128675613, 0.38268343236508977173},
    {0.83146961230254523708, 0.55557023301960222474},
    {0.70710678118654752440, 0.70710678118654752440},
    {0.55557023301960222474, 0.83146961230254523708},
    {0.38268343236508977173, 0.92387953251128675613},
    {0.19509032201612826785, 0.98078528040323044913},
    {0.0, 1.0},
    {-0.19509032201612826785, 0.98078528040323044913},
    {-0.38268343236508977173, 0.92387953251128675613},
    {-0.55557023301960222474, 0.83146961230254523708},
    {-0.70710678118654752440, 0.70710678118654752440},
    {-0.83146961230254523708, 0.55557023301960222474},
    {-0.92387953251128675613, 0.38268343236508977173},
    {-0.98078528040323044913, 0.19509032201612826785}};

// L1 twiddles w[j] = zeta_512^{lane j}, j = 1..15, from w1 = zeta_512^{lane} by a
// product tree of depth <= 4 (w[0] unused)
__device__ __forceinline__ void l1_twiddles(V w1, V* w) {
  w[1] = w1;
  w[2] = cmul(w1, w1);
  w[4] = cmul(w[2], w[2]);
  w[8] = cmul(w[4], w[4]);
  w[3] = cmul(w[2], w1);
  w[5] = cmul(w[4], w1);
  w[6] = cmul(w[4], w[2]);
  w[7] = cmul(w[4], w[3]);
#pragma unroll
  for (int j = 9; j < 16; ++j) w[j] = cmul(w[8], w[j - 8]);
}

__device__ __forceinline__ V shfl_x1(V a) {
  V r;
  r.x = __shfl_xor_sync(0xffffffffu, a.x, 1);
  r.y = __shfl_xor_sync(0xffffffffu, a.y, 1);
  return r;
}

// frequency held by (lane, k2) after the forward transform, and its position in the
// generic engine's digit-reversed order
__device__ __forceinline__ int freq_of(int lane, int k2) { return (lane >> 1) + 16 * k2 + 256 * (lane & 1); }
__device__ __forceinline__ int pos_of_freq(int f) { return ((f & 7) << 6) | (f & 56) | (f >> 6); }

// Forward FFT-512.  In: a[i] = x[lane + 32 i].  Out: a[k2] = X[freq_of(lane, k2)].
// E: this warp's 512-slot exchange region (E[ex(j,t)]); w1l = zeta_512^{lane}.
__device__ __forceinline__ void fft_fwd(V* a, V* E, int lane, V w1l) {
  dft16<+1>(a);
  {
    V w[16];
    l1_twiddles(w1l, w);
#pragma unroll
    for (int j = 1; j < 16; ++j) a[j] = cmul(a[j], w[j]);
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 16; ++j) E[ex(j, lane)] = a[j];
  __syncwarp();
  const int jj = lane >> 1, t2 = lane & 1;
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = E[ex(jj, t2 + 2 * i)];
  dft16<+1>(a);
#pragma unroll
  for (int k = 1; k < 16; ++k) {
    const V aw = cmul(a[k], c_w32[k]);
    a[k] = t2 ? aw : a[k];
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const V o = shfl_x1(a[k]);
    a[k] = t2 ? csub(o, a[k]) : cadd(a[k], o);
  }
}

// Inverse FFT-512 (adjoint of fft_fwd).  In: a[k2] = Y[freq_of(lane, k2)].
// Out: a[i] = sum_f zeta_512^{-(lane + 32 i) f} Y[f].
__device__ __forceinline__ void fft_inv(V* a, V* E, int lane, V w1l) {
  const int jj = lane >> 1, t2 = lane & 1;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const V o = shfl_x1(a[k]);
    a[k] = t2 ? csub(o, a[k]) : cadd(a[k], o);
  }
#pragma unroll
  for (int k = 1; k < 16; ++k) {
    const V aw = cmulc(a[k], c_w32[k]);
    a[k] = t2 ? aw : a[k];
  }
  dft16<-1>(a);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 16; ++i) E[ex(jj, t2 + 2 * i)] = a[i];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = E[ex(j, lane)];
  {
    V w[16];
    l1_twiddles(w1l, w);
#pragma unroll
    for (int j = 1; j < 16; ++j) a[j] = cmulc(a[j], w[j]);
  }
  dft16<-1>(a);
}

}  // namespace w512
}  // namespace hd
