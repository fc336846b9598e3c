// hd_s2048r.cuh -- 1-D convolution of long lines with m = 2048 (complex double), one
// CTA per line (persistent over lines): BASELINE config 2 (4096 pairs, L_f = 8192,
// L_g = 3000: q = 6 residues of M1 = 12288).
//
// A line's spectral state (M1 x 16 B = 192 KB) does not fit one SM next to its inputs,
// so the residues are processed in pairs: warp group A (warps 0-7) convolves residue
// r = 2 pr, group B (warps 8-15) residue 2 pr + 1, each with register FFT-2048s:
//   fold      y[s] = sum_{t<p} zeta_q^{r t} x[2048 t + s] straight from global
//             (L2), thread t of the group holding s = t + 256 i, i < 8 (Forward Eq.
//             PAPER.md:528 without its twiddle)
//   FFT-2048  (of x[s] = zeta_{M1}^{r s} y[s]) = DFT-8 over i of the
//             twisted y_i zeta_{8q}^{r i}, twiddle zeta_{M1}^{t (r + q k1)} (the residue
//             twiddle folded into the stage twiddle zeta_2048^{t k1}), a group-wide
//             transpose through shared memory, then warp w runs the FFT-256 of
//             sub-problem k1 = w in registers (hd_w256.cuh)
//   F parked in shared memory, G transformed the same way, product x 1/M1
//   (PAPER.md:190-192), inverse FFT-2048 (exact adjoint) ending with
//   zeta_{M1}^{-r s}: w_r[s] = zeta_{M1}^{-r s} V_r[s], stored to the CTA's residue
//   slots in global memory (PassArgs::scr; they stay in L2) for every pair but the
//   last, whose w_r go to the groups' shared rows
//   unfold    (all 512 threads, once per line) h[2048 t + s] = sum_{r<q} zeta_q^{-t r}
//             w_r[s] (Backward Eq. PAPER.md:531): h is written once
// The next line's f and g are prefetched into L2 (bulk prefetch) while this one runs.
// Shared memory: [E_A | E_B | P_A | P_B] (4 x 2048 slots) + stage twiddles zeta_2048^{t k1}
// (7 x 256) + FFT-256 twiddle columns (14 x 32) + zeta_q, zeta_{8q} (<= 72).
#pragma once
#include "hd_tma.cuh"
#include "hd_w256.cuh"

namespace hd {
namespace s2048r {

using V = double2;
constexpr int M = 2048;
constexpr int GT = 256;           // threads per warp group
constexpr int NT = 2 * GT;        // two groups
constexpr int kQMax = 8;

__device__ __forceinline__ void group_sync(int grp) {
  asm volatile("bar.sync %0, %1;" :: "r"(1 + grp), "r"(GT) : "memory");
}

// y_i (i < 8) for residue r: sum_{t<p} zeta_q^{r t} x[2048 t + s], s = tt + 256 i,
// twisted by zeta_{8q}^{r i}; x has L elements (zero beyond).  P: compile-time bound on
// p, blocks loaded two at a time (16 independent loads in flight per thread).
template <int P>
__device__ __forceinline__ void fold_r(V* y, const V* x, int L, int p, int r, int q, int tt, const V* zq,
                                      const V* z8q) {
#pragma unroll
  for (int i = 0; i < 8; ++i) y[i] = cmk<V>(0, 0);
#pragma unroll
  for (int t0 = 0; t0 < P; t0 += 2) {
    V v[2][8];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int t = t0 + u, idx = M * t + tt + GT * i;
        v[u][i] = (t < p && idx < L) ? ldg(x + idx) : cmk<V>(0, 0);
      }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const V c = zq[(r * (t0 + u)) % q];
#pragma unroll
      for (int i = 0; i < 8; ++i) y[i] = cfma(y[i], v[u][i], c);
    }
  }
#pragma unroll
  for (int i = 1; i < 8; ++i) y[i] = cmul(y[i], z8q[(r * i) % (8 * q)]);
}
__device__ __forceinline__ void fold_any(V* y, const V* x, int L, int p, int r, int q, int tt, const V* zq,
                                        const V* z8q) {
  if (p <= 2) fold_r<2>(y, x, L, p, r, q, tt, zq, z8q);
  else if (p <= 4) fold_r<4>(y, x, L, p, r, q, tt, zq, z8q);
  else fold_r<8>(y, x, L, p, r, q, tt, zq, z8q);
}

// forward FFT-2048 of the group's residue: in y (thread tt, s = tt + 256 i, already
// twisted), out the warp's sub-problem spectrum (8 values, w256 order).  The stage
// twiddle zeta_{M1}^{tt (r + q k1)} = zeta_{M1}^{r tt} zeta_2048^{tt k1} is applied as
// the thread's scalar c0 = zeta_{M1}^{r tt} on the DFT-8's inputs (it commutes with the
// DFT) and the table twiddle zeta_2048^{tt k1} (tw8) on its outputs.
__device__ __forceinline__ void fwd2048(V* y, V c0, const V* tw8, V* E, int grp, int tt, int wg, int lane,
                                       const V* tw) {
#pragma unroll
  for (int i = 0; i < 8; ++i) y[i] = cmul(y[i], c0);
  dft8<V, +1>(y);
#pragma unroll
  for (int k = 1; k < 8; ++k) y[k] = cmul(y[k], tw8[(k - 1) * GT + tt]);
  group_sync(grp);  // E free (the previous transform's warps are done with it)
#pragma unroll
  for (int k = 0; k < 8; ++k) E[k * GT + tt] = y[k];
  group_sync(grp);
  V* Ew = E + wg * GT;
#pragma unroll
  for (int j = 0; j < 8; ++j) y[j] = Ew[lane + 32 * j];
  __syncwarp();
  w256::fft256_fwd(y, Ew, lane, tw);
}

// inverse of fwd2048: in the warp's sub-problem spectrum, out w[i] = the group's
// inverse at s = tt + 256 i times conj(zeta_{M1}^{r s}) (conj twiddles, then the twist)
__device__ __forceinline__ void inv2048(V* v, V c0, const V* tw8, V* E, int grp, int tt, int wg, int lane,
                                       const V* tw, int r, int q, const V* z8q) {
  V* Ew = E + wg * GT;
  w256::fft256_inv(v, Ew, lane, tw);
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 8; ++j) Ew[lane + 32 * j] = v[j];
  group_sync(grp);
  v[0] = E[tt];
#pragma unroll
  for (int k = 1; k < 8; ++k) v[k] = cmulc(E[k * GT + tt], tw8[(k - 1) * GT + tt]);
  dft8<V, -1>(v);
  v[0] = cmulc(v[0], c0);
#pragma unroll
  for (int i = 1; i < 8; ++i) v[i] = cmulc(v[i], cmul(c0, z8q[(r * i) % (8 * q)]));
}

__global__ void __launch_bounds__(NT, 1) s2048r_kernel(const __grid_constant__ PassArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V* Ebase = reinterpret_cast<V*>(smem_raw);
  V* Pbase = Ebase + 2 * M;
  V* tw8 = Pbase + 2 * M;            // [k1 - 1][t] = zeta_2048^{t k1}
  V* tw256 = tw8 + 7 * GT;            // FFT-256 twiddle columns
  V* zq = tw256 + w256::kTwRows * 32; // zeta_q^e, e < q
  V* z8q = zq + kQMax;                // zeta_{8q}^e, e < 8q
  const int q = a.q;
  const int tid = threadIdx.x, grp = tid >> 8, tt = tid & (GT - 1);
  const int lane = tid & 31, wg = tt >> 5;
  const V* twm = reinterpret_cast<const V*>(a.tw_m);
  const V* twM1 = reinterpret_cast<const V*>(a.tw_M1);
  const int64_t M1 = a.M1;
  for (int i = tid; i < 7 * GT; i += NT) tw8[i] = ldg(twm + ((i & (GT - 1)) * ((i >> 8) + 1)) % M);
  for (int i = tid; i < w256::kTwRows * 32; i += NT) tw256[i] = w256::tw_entry(twm, M, i >> 5, i & 31);
  for (int i = tid; i < q; i += NT) zq[i] = ldg(twM1 + (int64_t)i * M);
  for (int i = tid; i < 8 * q; i += NT) z8q[i] = ldg(twM1 + (int64_t)i * (M / 8));
  __syncthreads();
  V* E = Ebase + grp * M;
  V* P = Pbase + grp * M;
  const V* tw = tw256 + lane;
  const LineIn& fi = a.in_f;
  const LineIn& gi = a.in_g;
  const LineOut& o = a.out;
  const int Lf = (int)fi.L, Lg = (int)gi.L, Lout = (int)o.L, T = o.T;
  const double scale = a.scale;
  const int npr = (q + 1) / 2;
  for (int64_t l = blockIdx.x; l < a.nlines; l += gridDim.x) {
    const V* f = reinterpret_cast<const V*>(fi.ptr[0]) + line_off(fi, l);
    const V* g = reinterpret_cast<const V*>(gi.ptr[0]) + line_off(gi, l);
    V* h = reinterpret_cast<V*>(o.ptr[0]) + line_off(o, l);
    if (tid == 0 && l + gridDim.x < a.nlines) {  // the next line's inputs into L2
      bulk_prefetch_l2(reinterpret_cast<const V*>(fi.ptr[0]) + line_off(fi, l + gridDim.x), (uint32_t)Lf * 16u);
      bulk_prefetch_l2(reinterpret_cast<const V*>(gi.ptr[0]) + line_off(gi, l + gridDim.x), (uint32_t)Lg * 16u);
    }
    V* slots = reinterpret_cast<V*>(a.scr) + (int64_t)blockIdx.x * (2 * (npr - 1)) * M;
    for (int pr = 0; pr < npr; ++pr) {
      const int r = 2 * pr + grp;
      const bool last = pr == npr - 1;
      if (r < q) {
        const V c0 = ldg(twM1 + ((int64_t)r * tt) % M1);  // zeta_{M1}^{r tt}
        V y[8];
        fold_any(y, f, Lf, fi.p, r, q, tt, zq, z8q);
        fwd2048(y, c0, tw8, E, grp, tt, wg, lane, tw);
        V* Pw = P + wg * GT;
#pragma unroll
        for (int k = 0; k < 8; ++k) Pw[k * 32 + lane] = y[k];  // F parked (own slice)
        fold_any(y, g, Lg, gi.p, r, q, tt, zq, z8q);
        fwd2048(y, c0, tw8, E, grp, tt, wg, lane, tw);
#pragma unroll
        for (int k = 0; k < 8; ++k) y[k] = cscale(cmul(Pw[k * 32 + lane], y[k]), scale);
        inv2048(y, c0, tw8, E, grp, tt, wg, lane, tw, r, q, z8q);
        V* w = last ? P : slots + (int64_t)r * M;  // w_r[s], s = tt + 256 i
#pragma unroll
        for (int i = 0; i < 8; ++i) w[tt + GT * i] = y[i];
      }
    }
    __syncthreads();
    // unfold of the line: h[2048 t + s] = sum_{r<q} zeta_q^{-t r} w_r[s]
    const int rl = 2 * (npr - 1);  // residues in shared memory: rl, rl + 1
#pragma unroll 1
    for (int c = 0; c < M / NT; ++c) {
      const int s = tid + NT * c;
      V w[kQMax];
#pragma unroll
      for (int r = 0; r < kQMax; ++r) {
        if (r >= q) w[r] = cmk<V>(0, 0);
        else if (r < rl) w[r] = __ldcs(slots + (int64_t)r * M + s);  // last use
        else w[r] = Pbase[(r - rl) * M + s];
      }
#pragma unroll
      for (int t = 0; t < kQMax; ++t) {
        if (t >= T || M * t + s >= Lout) break;
        V val = w[0];
#pragma unroll
        for (int r = 1; r < kQMax; ++r)
          if (r < q) val = cfmac(val, w[r], zq[(t * r) % q]);
        __stcs(h + M * t + s, val);  // streaming: keep L2 for the next lines' inputs and the slots
      }
    }
    __syncthreads();
  }
}

}  // namespace s2048r
}  // namespace hd
