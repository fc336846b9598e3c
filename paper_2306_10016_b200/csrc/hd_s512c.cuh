// hd_s512c.cuh -- 1-D convolution pass for long lines (m = 512, complex double,
// 12 <= q <= 22): a thread-block cluster of two CTAs per line.
//
// A line of M1 = q m outputs (BASELINE config 2: 3000 (*) 8192, M1 = 22 x 512)
// needs q residue rows of 8 KB: too many for one CTA's shared memory with the
// input staged beside them.  The two CTAs of a cluster split the residues (CTA 0:
// r = 0 and the pairs (k, q - k) for k <= K0; CTA 1: the other pairs and, for even
// q, r = q/2), so each CTA holds at most 11 rows, one compute warp per residue:
//
//   fold f   thread per column s, straight from global memory (p_f loads in
//            flight per thread): w_r[s] = zeta_{qm}^{rs} sum_t zeta_q^{rt} x[tm+s],
//            the q-point DFT in pairs (r, q - r) (Forward Eq. PAPER.md:528) -> row
//   FFT      warp per residue, FFT-512 in registers (hd_w512.cuh) -> F
//   fold g   the same for the short input -> rows;  warp: G = FFT(row)
//   product  (1/prod M1) F G, inverse FFT -> row
//   unfold   thread per column: partial h_t[s] = sum over THIS CTA's residues of
//            zeta_q^{-tr} zeta_{qm}^{-rs} V_r[s] for every output block t < T
//            (Backward Eq. PAPER.md:531, pairs (r, q - r) share their products);
//            the blocks the partner CTA owns are written into its shared memory
//            through the cluster's distributed shared memory (DSMEM), then each
//            CTA adds the two halves of its own blocks and stores them.
//
// Every input element is read twice (once per CTA, the second read mostly from
// L2) and every output written once.  The lane-major spectral order of the FFT
// never leaves registers.
#pragma once
#include <cooperative_groups.h>

#include "hd_internal.h"
#include "hd_tma.cuh"
#include "hd_w512.cuh"

namespace hd {
namespace s512c {

namespace cg = cooperative_groups;
using V = double2;
constexpr int M = 512;
constexpr int kQMin = 12, kQMax = 22;
constexpr int kRMax = 11;  // residues per CTA
constexpr int kPairs = kRMax / 2;  // pairs (k, q - k) per CTA
constexpr int kTMax = 32;          // blocks t of the fold (p) and of the unfold (T)

// residue groups of the two CTAs: P = floor((q-1)/2) pairs (k, q-k), k = 1..P;
// CTA 0: r = 0 and pairs 1..K0; CTA 1: pairs K0+1..P and r = q/2 (even q)
struct Split {
  int q, P, K0;
  __device__ __forceinline__ Split(int q_) : q(q_), P((q_ - 1) / 2), K0((q_ & 1) ? ((q_ - 1) / 2 + 1) / 2 : ((q_ - 1) / 2) / 2) {}
  __device__ __forceinline__ int nres(int c) const { return c == 0 ? 1 + 2 * K0 : 2 * (P - K0) + ((q & 1) ? 0 : 1); }
  __device__ __forceinline__ int npairs(int c) const { return c == 0 ? K0 : P - K0; }
  __device__ __forceinline__ int kfirst(int c) const { return c == 0 ? 1 : K0 + 1; }
  // row (= compute warp) of pair j's two members and of the singletons
  __device__ __forceinline__ int row_k(int c, int j) const { return c == 0 ? 1 + 2 * j : 2 * j; }
  __device__ __forceinline__ int row_qk(int c, int j) const { return row_k(c, j) + 1; }
  __device__ __forceinline__ int row_single(int c) const { return c == 0 ? 0 : 2 * (P - K0); }  // r = 0 / q/2
  __device__ __forceinline__ bool has_single(int c) const { return c == 0 || !(q & 1); }
  __device__ __forceinline__ int residue_of_row(int c, int w) const {
    if (c == 0) {
      if (w == 0) return 0;
      const int k = (w + 1) >> 1;
      return (w & 1) ? k : q - k;
    }
    if (w == 2 * (P - K0)) return q >> 1;
    const int k = K0 + 1 + (w >> 1);
    return (w & 1) ? q - k : k;
  }
};

// Fold of the CTA's residues for the columns of this thread, straight from global
// memory: x = the line, p blocks of M, length L; zkt[t * kPairs + j] = zeta_q^{k t}
// for the CTA's pair j (k = kfirst + j), t < kTMax (shared)
__device__ __forceinline__ void fold_line(V* rows, const V* x, int L, int p, const Split& sp, int c, const V* zkt,
                                          const V* twM1, int tid, int nth) {
  const int q = sp.q, np = sp.npairs(c), k0 = sp.kfirst(c);
  for (int s = tid; s < M; s += nth) {
    V acc0 = cmk<V>(0, 0);
    V pp[kRMax / 2 + 1], qq[kRMax / 2 + 1];
#pragma unroll
    for (int j = 0; j <= kRMax / 2; ++j) { pp[j] = cmk<V>(0, 0); qq[j] = cmk<V>(0, 0); }
    const int rem = L - s;
    // blocks in chunks of 8: the chunk's global loads are all in flight before use
    for (int t0 = 0; t0 < p; t0 += 8) {
      V uu[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        uu[i] = (t0 + i < p && (t0 + i) * M < rem) ? ldg(x + (t0 + i) * M + s) : cmk<V>(0, 0);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int t = t0 + i;
        const V u = uu[i];
        // singleton: r = 0 (sum) or r = q/2 (alternating sum)
        if (c == 0) acc0 = cadd(acc0, u);
        else if (!(q & 1)) acc0 = (t & 1) ? csub(acc0, u) : cadd(acc0, u);
        const V* zt = zkt + t * kPairs;
#pragma unroll
        for (int j = 0; j < kPairs; ++j) {
          if (j < np) {
            const V z = zt[j];
            pp[j].x = fma(z.x, u.x, pp[j].x); pp[j].y = fma(z.x, u.y, pp[j].y);
            qq[j].x = fma(z.y, u.x, qq[j].x); qq[j].y = fma(z.y, u.y, qq[j].y);
          }
        }
      }
    }
    if (sp.has_single(c)) {
      const int r = c == 0 ? 0 : q >> 1;
      rows[sp.row_single(c) * M + s] = cmul(acc0, ldg(twM1 + r * s));
    }
#pragma unroll
    for (int j = 0; j < kRMax / 2; ++j) {
      if (j < np) {
        const int k = k0 + j;
        // S_k = P + i Q, S_{q-k} = P - i Q (zeta_q^{(q-k) t} = conj zeta_q^{k t})
        rows[sp.row_k(c, j) * M + s] = cmul(cmk<V>(pp[j].x - qq[j].y, pp[j].y + qq[j].x), ldg(twM1 + k * s));
        rows[sp.row_qk(c, j) * M + s] = cmul(cmk<V>(pp[j].x + qq[j].y, pp[j].y - qq[j].x), ldg(twM1 + (q - k) * s));
      }
    }
  }
}

template <int NT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1) s512c_kernel(const __grid_constant__ PassArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V* twtab = reinterpret_cast<V*>(smem_raw);              // FFT-512 per-lane twiddle columns
  V* zkt = twtab + w512::kTwRows * 32;                     // zeta_q^{k t}: [t][pair]
  V* rows = zkt + kTMax * kPairs;                           // kRMax rows of M
  V* recv = rows + kRMax * M;                               // partner's partial sums, kRMax rows
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();                       // 0 or 1
  const int q = a.q;
  const Split sp(q);
  const int nres = sp.nres(c);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int nth = 32 * nres;
  const V* twm = reinterpret_cast<const V*>(a.tw_m);
  const V* twM1 = reinterpret_cast<const V*>(a.tw_M1);
  for (int i = tid; i < w512::kTwRows * 32; i += blockDim.x) twtab[i] = w512::tw_entry(twm, i >> 5, i & 31);
  for (int i = tid; i < kTMax * kPairs; i += blockDim.x) {
    const int t = i / kPairs, k = sp.kfirst(c) + i % kPairs;
    zkt[i] = ldg(twM1 + (int64_t)((k * t) % q) * M);
  }
  __syncthreads();
  V* partner_recv = cl.map_shared_rank(recv, c ^ 1);
  const int T = a.out.T;
  const int T0 = (T + 1) / 2;                               // CTA 0 owns blocks t < T0
  const int tlo = c == 0 ? 0 : T0, thi = c == 0 ? T0 : T;
  const V* tw = twtab + lane;
  const LineIn &fi = a.in_f, &gi = a.in_g;
  const LineOut& o = a.out;
  const int Lout = (int)(o.L + o.j0), j0 = (int)o.j0;
  const int64_t ncl = gridDim.x / 2;
  for (int64_t l = blockIdx.x / 2; l < a.nlines; l += ncl) {
    if (w < nres) {
      // 1. fold f into the rows, FFT of this warp's residue -> F (registers)
      const V* xf = reinterpret_cast<const V*>(fi.ptr[0]) + line_off(fi, l);
      fold_line(rows, xf, (int)fi.L, fi.p, sp, c, zkt, twM1, tid, nth);
      compute_sync(nth);
      V F[16];
      V* Er = rows + w * M;
#pragma unroll
      for (int i = 0; i < 16; ++i) F[i] = Er[lane + 32 * i];
      w512::fft_fwd(F, Er, lane, tw);
      compute_sync(nth);
      // 2. fold g, FFT -> G, product, inverse FFT -> V_r (natural order) in the row
      const V* xg = reinterpret_cast<const V*>(gi.ptr[0]) + line_off(gi, l);
      fold_line(rows, xg, (int)gi.L, gi.p, sp, c, zkt, twM1, tid, nth);
      compute_sync(nth);
      V G[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) G[i] = Er[lane + 32 * i];
      w512::fft_fwd(G, Er, lane, tw);
#pragma unroll
      for (int k = 0; k < 16; ++k) F[k] = cscale(cmul(F[k], G[k]), a.scale);
      w512::fft_inv(F, Er, lane, tw);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 16; ++i) Er[lane + 32 * i] = F[i];
      compute_sync(nth);
    }
    // 3. partial unfold over this CTA's residues for every block t < T
    cl.sync();  // the partner has consumed its receive buffer (previous line)
    if (w < nres) {
      const int np = sp.npairs(c), k0 = sp.kfirst(c);
      for (int s = tid; s < M; s += nth) {
        V v0 = cmk<V>(0, 0), A[kRMax / 2], B[kRMax / 2];
        if (sp.has_single(c)) {
          const int r = c == 0 ? 0 : q >> 1;
          v0 = cmulc(rows[sp.row_single(c) * M + s], ldg(twM1 + r * s));
        }
#pragma unroll
        for (int j = 0; j < kRMax / 2; ++j) {
          if (j < np) {
            const int k = k0 + j;
            const V vk = cmulc(rows[sp.row_k(c, j) * M + s], ldg(twM1 + k * s));
            const V vq = cmulc(rows[sp.row_qk(c, j) * M + s], ldg(twM1 + (q - k) * s));
            A[j] = cadd(vk, vq);
            B[j] = csub(vq, vk);
          }
        }
        for (int t = 0; t < T; ++t) {
          if (t * M + s >= Lout) break;
          // h_t = v0 (r = 0: 1; r = q/2: (-1)^t) + sum_k re_{tk} A_k + i im_{tk} B_k
          V h = (c == 0 || !(t & 1)) ? v0 : cmk<V>(-v0.x, -v0.y);
          const V* zt = zkt + t * kPairs;
#pragma unroll
          for (int j = 0; j < kPairs; ++j) {
            if (j < np) {
              const V z = zt[j];
              h.x = fma(z.x, A[j].x, h.x); h.x = fma(-z.y, B[j].y, h.x);
              h.y = fma(z.x, A[j].y, h.y); h.y = fma(z.y, B[j].x, h.y);
            }
          }
          if (t >= tlo && t < thi) rows[(t - tlo) * M + s] = h;              // own block (in place: column s)
          else partner_recv[(c == 0 ? t - T0 : t) * M + s] = h;              // the partner's block
        }
      }
    }
    cl.sync();  // partials exchanged
    if (w < nres) {
      V* y = reinterpret_cast<V*>(o.ptr[0]) + line_off(o, l);
      for (int i = tid; i < (thi - tlo) * M; i += nth) {
        const int t = tlo + i / M, s = i % M;
        const int j = t * M + s;
        if (j >= j0 && j < Lout) y[j - j0] = cadd(rows[i], recv[i]);
      }
    }
  }
}

// shared memory bytes of the kernel
inline size_t smem_bytes() {
  return sizeof(double2) * (size_t)(w512::kTwRows * 32 + kTMax * kPairs + 2 * kRMax * M);
}

}  // namespace s512c
}  // namespace hd
