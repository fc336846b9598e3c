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

// ---------------------------------------------------------------------------
// Pass kernel on the warp engine: one line per CTA, one warp per residue
// (blockDim = 32 q), D = q, fast fold/unfold (q <= 16, p <= 8).
// MODE_FWD / MODE_INV / MODE_CONV as in pass_kernel; CONV needs npairs == 1 and
// p_g == 1 (the short input's fold is done in registers, residue by residue).
// Shared memory: [zq: q][zt: 16x16][F: q*512] (each warp's F row doubles as its
// exchange area; in CONV the F-hat spectrum stays in registers while G is transformed)
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(288, 2) w512_kernel(const __grid_constant__ PassArgs a) {
  constexpr int M = 512;
  constexpr int EPR = 8;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V* smem = reinterpret_cast<V*>(smem_raw);
  const int q = a.q;
  const int k_arr = blockIdx.z;
  const int lane = threadIdx.x & 31;
  const int r = threadIdx.x >> 5;  // this warp's residue
  V* zq = smem;
  V* zt = zq + round_slots<EPR>(q);
  V* F = zt + round_slots<EPR>(kQF * kQF);
  // CONV: per-CTA global scratch (L2-resident) where each warp parks its F-hat
  V* Fh = MODE == MODE_CONV ? reinterpret_cast<V*>(a.scratch) + ((int64_t)blockIdx.x * q + (threadIdx.x >> 5)) * M
                            : nullptr;
  const V* twm = reinterpret_cast<const V*>(a.tw_m);
  const V* twM1 = reinterpret_cast<const V*>(a.tw_M1);
  const V w1l = ldg(twm + lane);  // zeta_512^{lane}: seeds this lane's L1 twiddles
  for (int i = threadIdx.x; i < q; i += (int)blockDim.x) zq[i] = ldg(twM1 + (int64_t)i * M);
  for (int i = threadIdx.x; i < kQF * kQF; i += (int)blockDim.x) {
    const int rr = i / kQF, t = i % kQF;
    zt[i] = ldg(twM1 + (int64_t)((rr * t) % q) * M);
  }
  __syncthreads();

  V* Fr = F + r * M;  // this warp's residue row (also its exchange region)
  const int64_t total = a.nbatch * a.ngroups;
  for (int64_t w = blockIdx.x; w < total; w += gridDim.x) {
    int64_t g, b;
    split_item(w, a.nbatch, a.ngroups, a.batch_fastest, b, g);
    if (threadIdx.x == 0 && w + gridDim.x < total) {
      int64_t gn, bn;
      split_item(w + gridDim.x, a.nbatch, a.ngroups, a.batch_fastest, bn, gn);
      prefetch_lines<V>(a.in_f, MODE == MODE_FWD ? k_arr : 0, bn, gn, 1, a.nlines);
      if (MODE == MODE_CONV) prefetch_lines<V>(a.in_g, 0, bn, gn, 1, a.nlines);
    }
    const bool live = g < a.nlines;
    if constexpr (MODE == MODE_FWD) {
      fold<V, M, 512>(F, a.in_f, k_arr, b, g, a.nlines, 1, 0, 0, q, q, zq, zt, twm, twM1);
      __syncthreads();
      V v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = Fr[swz<V>(r * M + lane + 32 * i) - r * M];
      fft_fwd(v, Fr, lane, w1l);
      if (live) {
        const LineOut& o = a.out;
        V* y = reinterpret_cast<V*>(o.ptr[k_arr]) + boff(b, o.nbi, o.s_bo, o.s_b) +
               line_off(o, g);
        const int sl = out_sl(o);
        const int64_t k0 = (int64_t)r * M;
        if (sl >= 1 && sl < 30 && o.s_js == 1) {
          // positions pos(f) and pos(f)+1 = pos(f+64): registers k2 and k2+4, k2 in {0..3, 8..11}
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int k2 = (kk & 3) + ((kk >> 2) << 3);
            const int p0 = pos_of_freq(freq_of(lane, k2));
            st256(y + jt_off(k0 + p0, sl, o.s_jt, o.s_js), v[k2], v[k2 + 4]);
          }
        } else {
#pragma unroll
          for (int k2 = 0; k2 < 16; ++k2)
            y[jt_off(k0 + pos_of_freq(freq_of(lane, k2)), sl, o.s_jt, o.s_js)] = v[k2];
        }
      }
      __syncthreads();
    } else if constexpr (MODE == MODE_INV) {
      {
        const LineIn& in = a.in_f;
        const V* x = reinterpret_cast<const V*>(in.ptr[0]) + boff(b, in.nbi, in.s_bo, in.s_b) +
                     line_off(in, g);
        V v[16];
        const int64_t k0 = (int64_t)r * M;
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2)
          v[k2] = live ? x[in_el(in, k0 + pos_of_freq(freq_of(lane, k2)))] : cmk<V>(0, 0);
        fft_inv(v, Fr, lane, w1l);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 16; ++i) Fr[swz<V>(r * M + lane + 32 * i) - r * M] = v[i];
      }
      __syncthreads();
      unfold<V, M, 512>(F, a.out, 0, b, g, a.nlines, 1, 0, 0, q, q, false, zq, zt, twm, twM1);
      __syncthreads();
    } else {
      fold<V, M, 512>(F, a.in_f, 0, b, g, a.nlines, 1, 0, 0, q, q, zq, zt, twm, twM1);
      __syncthreads();
      V v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = Fr[swz<V>(r * M + lane + 32 * i) - r * M];
      fft_fwd(v, Fr, lane, w1l);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 16; ++k) Fh[lane + 32 * k] = v[k];  // F-hat parked in L2 scratch
      // short input g: p_g == 1, fold in registers: w[s] = g[s] zeta_{M1}^{r s}, s = lane + 32 i
      {
        const LineIn& in = a.in_g;
        const V* x = reinterpret_cast<const V*>(in.ptr[0]) + boff(b, in.nbi, in.s_bo, in.s_b) + line_off(in, g);
        V wr = ldg(twM1 + (int64_t)r * lane);
        const V step = ldg(twM1 + (int64_t)r * 32);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int s = lane + 32 * i;
          const V u = (live && s < in.L) ? x[in_el(in, s)] : cmk<V>(0, 0);
          v[i] = cmul(u, wr);
          wr = cmul(wr, step);
        }
      }
      fft_fwd(v, Fr, lane, w1l);   // G's transform reuses this warp's SMEM row
      {
        const double sc = a.scale;
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = cscale(cmul(Fh[lane + 32 * k], v[k]), sc);  // (1/prod M1) F-hat G-hat
      }
      fft_inv(v, Fr, lane, w1l);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 16; ++i) Fr[swz<V>(r * M + lane + 32 * i) - r * M] = v[i];
      __syncthreads();
      unfold<V, M, 512>(F, a.out, 0, b, g, a.nlines, 1, 0, 0, q, q, false, zq, zt, twm, twM1);
      __syncthreads();
    }
  }
}

}  // namespace w512
}  // namespace hd
