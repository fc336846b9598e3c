// hd_w512.cuh -- register FFT of size m = 512 (complex double) for one warp.
//
// One warp owns one residue r of one line: its size-512 FFT (PAPER.md:104,
// "W <- m F(W)") runs in registers as 512 = 16 x 16 x 2:
//   L1  radix-16 over x[lane + 32 i] (16 values per lane), twiddle zeta_512^{lane j}
//   --  warp-local transpose through shared memory (no CTA barrier)
//   L2  radix-16 over the stride-2 decimation of each 32-point sub-problem
//   L3  radix-2 between lane pairs: each lane of a pair takes half of the 16
//       butterflies (one shuffle of 8 values each way), twiddle zeta_32^{k}
// Lane u then holds frequency freq_of(u, k) in register k.  The twiddles come from a
// per-lane shared-memory column (TwTab) filled once per CTA.  The inverse is the
// exact adjoint (negative exponent).
#pragma once
#include "hd_device.cuh"

namespace hd {
namespace w512 {

using V = double2;

// 16-point DFT in registers, y_k = sum_n v_n zeta_16^{S n k}, natural order out.
// 4 x 4 Cooley-Tukey: n = 4 n1 + n2, k = k1 + 4 k2.
// LOWHALF: the input's upper half v[8..15] is zero (a short input padded to 512,
// e.g. the kernel g with L_g <= 256); the first radix-4 layer then reduces to
// 2-point sums (32 fewer FP64 operations).
template <int S, bool LOWHALF = false, typename VT = V> __device__ __forceinline__ void dft16(VT* v) {
  using R = decltype(VT::x);
  using V = VT;  // complex double (FFT-512) or complex float (hd_s128.cuh)
  const R c1 = (R)0.92387953251128675613, s1 = (R)0.38268343236508977173;
  const R h = (R)0.70710678118654752440;
  V A[4][4];
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    if constexpr (LOWHALF) {
      const V x0 = v[n2], x1 = v[4 + n2];
      const V ix1 = cmul_si<V, S>(x1);
      A[n2][0] = cadd(x0, x1);
      A[n2][1] = cadd(x0, ix1);
      A[n2][2] = csub(x0, x1);
      A[n2][3] = csub(x0, ix1);
    } else {
      V t[4] = {v[n2], v[4 + n2], v[8 + n2], v[12 + n2]};
      dft4<V, S>(t);
#pragma unroll
      for (int k1 = 0; k1 < 4; ++k1) A[n2][k1] = t[k1];
    }
  }
  // twiddles zeta_16^{S n2 k1}
  auto rot = [&](V a, R c, R s) {  // a * (c + i S s)
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


// Per-lane twiddle column (shared memory, [kTwRows][32], read at tw[row * 32]):
//   rows 0..14:  zeta_512^{lane (j+1)}                (L1)
//   rows 15..22: zeta_32^{k + 8 (lane & 1)}, k < 8     (L3)
constexpr int kTwRows = 23;
__device__ __forceinline__ V tw_entry(const V* twm512, int row, int lane) {
  if (row < 15) return ldg(twm512 + (lane * (row + 1)) % 512);
  const int kk = (row - 15) + 8 * (lane & 1);
  return ldg(twm512 + 16 * kk);
}

// radix-2 butterfly with a twiddle, FMA-fused: (A + w B, A - w B) in 6 FP64 operations
// (A + w B by four chained FMAs, A - w B = 2A - (A + w B)) instead of 8
__device__ __forceinline__ void bfly_tw(V& A, V& B, V w) {
  V s;
  s.x = fma(B.x, w.x, A.x);
  s.x = fma(-B.y, w.y, s.x);
  s.y = fma(B.x, w.y, A.y);
  s.y = fma(B.y, w.x, s.y);
  B = cmk<V>(fma(2.0, A.x, -s.x), fma(2.0, A.y, -s.y));
  A = s;
}

__device__ __forceinline__ V shfl_x1(V a) {
  V r;
  r.x = __shfl_xor_sync(0xffffffffu, a.x, 1);
  r.y = __shfl_xor_sync(0xffffffffu, a.y, 1);
  return r;
}

// frequency held by register k of lane u after the forward transform
__device__ __forceinline__ int freq_of(int u, int k) {
  return (u >> 1) + 16 * ((k & 7) + 8 * (u & 1)) + 256 * (k >> 3);
}

// Forward FFT-512.  In: a[i] = x[lane + 32 i] (LOWHALF: a[8..15] = 0, not read).
// Out: a[k] = X[freq_of(lane, k)].
// E: this warp's 512-slot exchange region (E[ex(j,t)]); tw: this lane's twiddle column.
template <bool LOWHALF = false>
__device__ __forceinline__ void fft_fwd(V* a, V* E, int lane, const V* tw) {
  dft16<+1, LOWHALF>(a);
#pragma unroll
  for (int j = 1; j < 16; ++j) a[j] = cmul(a[j], tw[(j - 1) * 32]);
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 16; ++j) E[ex(j, lane)] = a[j];
  __syncwarp();
  const int jj = lane >> 1, t2 = lane & 1;
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = E[ex(jj, t2 + 2 * i)];
  dft16<+1>(a);
  // even lane holds A[k], odd lane B[k] (k < 16); after the exchange lane t2 holds
  // A[k + 8 t2] in a[k] and B[k + 8 t2] in a[k + 8], k < 8
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const V snd = t2 ? a[k] : a[k + 8];
    const V rcv = shfl_x1(snd);
    if (t2) a[k] = rcv; else a[k + 8] = rcv;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) bfly_tw(a[k], a[k + 8], tw[(15 + k) * 32]);  // zeta_32^{k + 8 t2} B
}

// Two forward FFT-512s interleaved stage by stage (independent data, so the radix-16
// stages of one overlap the other's shared-memory exchange); one 512-slot exchange
// area, used by a then b.  lowb: b's upper half is zero (fft_fwd<true>).
__device__ __forceinline__ void fft_fwd2(V* a, V* b, V* E, int lane, const V* tw, bool lowb) {
  dft16<+1>(a);
  if (lowb) dft16<+1, true>(b);
  else dft16<+1>(b);
#pragma unroll
  for (int j = 1; j < 16; ++j) {
    const V w = tw[(j - 1) * 32];
    a[j] = cmul(a[j], w);
    b[j] = cmul(b[j], w);
  }
  const int jj = lane >> 1, t2 = lane & 1;
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 16; ++j) E[ex(j, lane)] = a[j];
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = E[ex(jj, t2 + 2 * i)];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 16; ++j) E[ex(j, lane)] = b[j];
  dft16<+1>(a);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 16; ++i) b[i] = E[ex(jj, t2 + 2 * i)];
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
    bfly_tw(a[k], a[k + 8], w);
    bfly_tw(b[k], b[k + 8], w);
  }
}

// Inverse FFT-512 (adjoint of fft_fwd).  In: a[k] = Y[freq_of(lane, k)].
// Out: a[i] = sum_f zeta_512^{-(lane + 32 i) f} Y[f].
__device__ __forceinline__ void fft_inv(V* a, V* E, int lane, const V* tw) {
  const int jj = lane >> 1, t2 = lane & 1;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const V x0 = a[k], x1 = a[k + 8];
    a[k] = cadd(x0, x1);                                  // A'[k + 8 t2]
    a[k + 8] = cmulc(csub(x0, x1), tw[(15 + k) * 32]);    // B'[k + 8 t2]
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const V snd = t2 ? a[k] : a[k + 8];
    const V rcv = shfl_x1(snd);
    if (t2) a[k] = rcv; else a[k + 8] = rcv;
  }
  // even lane: a = A'[0..15]; odd lane: a = B'[0..15]
  dft16<-1>(a);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 16; ++i) E[ex(jj, t2 + 2 * i)] = a[i];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = E[ex(j, lane)];
#pragma unroll
  for (int j = 1; j < 16; ++j) a[j] = cmulc(a[j], tw[(j - 1) * 32]);
  dft16<-1>(a);
}

}  // namespace w512
}  // namespace hd
