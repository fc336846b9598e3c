// hd_s2048c.cuh -- 1-D convolution pass for long lines with FFT size m = 2048
// (complex double, 4 <= q <= 6): a two-CTA cluster per line, four warps per residue.
//
// BASELINE config 2 (3000 (*) 8192, L_out = 11191) is cheapest at m = 2048, q = 6:
// the q-point DFTs of the fold and unfold stay small (p_f = 4, p_g = 2, T = 6)
// while a residue row is 32 KB.  As in hd_s512c.cuh the two CTAs of a cluster
// split the residues by pairs (r, q - r) (at most 3 rows each), fold straight from
// global memory, and exchange the partial unfolds of the output blocks the partner
// owns through distributed shared memory.  The FFT-2048 of a residue runs on a
// group of 128 threads (4 warps, named barrier per group):
//
//   stage 1  thread t: radix-16 over x[t + 128 i] in registers, twiddle
//            zeta_2048^{t k1}, write row[k1 * 128 + t]           (group barrier)
//   stage 2  8-thread group (k1 = t / 8): FFT-128 of row segment k1 as in
//            hd_s128.cuh (radix-16, twiddle zeta_128^{u k}, swizzled 8-lane
//            transpose, two radix-8) -> frequencies k1 + 16 (2u + j + 16 k2)
//   inverse  the exact adjoint
//
// ("W <- m F(W)", 515-519: the size-m FFT of every residue.)
#pragma once
#include <cooperative_groups.h>

#include "hd_internal.h"
#include "hd_s512c.cuh"
#include "hd_tma.cuh"
#include "hd_w512.cuh"

namespace hd {
namespace s2048c {

namespace cg = cooperative_groups;
using V = double2;
using s512c::Split;
constexpr int M = 2048;
constexpr int kQMin = 4, kQMax = 6;
constexpr int kRMax = 3;          // residues per CTA
constexpr int kPairs = 1;         // pairs (k, q - k) per CTA
constexpr int kTMax = 32;         // blocks t of the fold (p) and of the unfold (T)
constexpr int kGT = 128;          // threads per residue group

__device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, %1;" :: "r"(2 + g), "r"(kGT) : "memory");
}

// 8-lane FFT-128 exchange slot of (k, v) within a 128-slot segment
__device__ __forceinline__ int ex128(int k, int v) { return (k << 3) + (v ^ (k >> 1)); }

// forward FFT-2048 of `row` (natural order in shared memory) -> a[8 j + k2]
// = X[k1 + 16 (2u + j + 16 k2)], k1 = t >> 3, u = t & 7
__device__ __forceinline__ void fft2048_fwd(V* a, V* row, int t, int g, const V* twm) {
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = row[t + kGT * i];
  w512::dft16<+1, false, V>(a);
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) a[k1] = cmul(a[k1], twm[t * k1]);
  group_sync(g);  // every thread has read the row
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) row[k1 * kGT + t] = a[k1];
  group_sync(g);
  const int k1 = t >> 3, u = t & 7;
  V* seg = row + k1 * kGT;
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = seg[u + 8 * i];
  w512::dft16<+1, false, V>(a);
#pragma unroll
  for (int k = 1; k < 16; ++k) a[k] = cmul(a[k], twm[16 * u * k]);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) seg[ex128(k, u)] = a[k];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int v = 0; v < 8; ++v) a[8 * j + v] = seg[ex128(2 * u + j, v)];
  dft8<V, +1>(a);
  dft8<V, +1>(a + 8);
}

// inverse (adjoint): a as produced by fft2048_fwd -> row (natural order, unnormalised)
__device__ __forceinline__ void fft2048_inv(V* a, V* row, int t, int g, const V* twm) {
  const int k1 = t >> 3, u = t & 7;
  V* seg = row + k1 * kGT;
  dft8<V, -1>(a);
  dft8<V, -1>(a + 8);
  group_sync(g);  // the row is free (previous readers done)
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int v = 0; v < 8; ++v) seg[ex128(2 * u + j, v)] = a[8 * j + v];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = seg[ex128(k, u)];
#pragma unroll
  for (int k = 1; k < 16; ++k) a[k] = cmulc(a[k], twm[16 * u * k]);
  w512::dft16<-1, false, V>(a);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 16; ++i) seg[u + 8 * i] = a[i];
  group_sync(g);
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) a[kk] = row[kk * kGT + t];
#pragma unroll
  for (int kk = 1; kk < 16; ++kk) a[kk] = cmulc(a[kk], twm[t * kk]);
  w512::dft16<-1, false, V>(a);
  group_sync(g);  // every thread has read the row
#pragma unroll
  for (int i = 0; i < 16; ++i) row[t + kGT * i] = a[i];
}

// fold of this CTA's residues (pair form) for the columns of this thread, straight
// from global memory; zkt[t] = zeta_q^{k t} of the CTA's pair (k = kfirst)
__device__ __forceinline__ void fold_line(V* rows, const V* x, int L, int p, const Split& sp, int c, const V* zkt,
                                          const V* twM1, int tid, int nth) {
  const int q = sp.q, np = sp.npairs(c), k0 = sp.kfirst(c);
  for (int s = tid; s < M; s += nth) {
    V acc0 = cmk<V>(0, 0), pp = cmk<V>(0, 0), qq = cmk<V>(0, 0);
    const int rem = L - s;
    for (int t0 = 0; t0 < p; t0 += 8) {
      V uu[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        uu[i] = (t0 + i < p && (t0 + i) * M < rem) ? ldg(x + (t0 + i) * M + s) : cmk<V>(0, 0);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int t = t0 + i;
        const V u = uu[i];
        if (c == 0) acc0 = cadd(acc0, u);
        else if (!(q & 1)) acc0 = (t & 1) ? csub(acc0, u) : cadd(acc0, u);
        if (np > 0) {
          const V z = zkt[t];
          pp.x = fma(z.x, u.x, pp.x); pp.y = fma(z.x, u.y, pp.y);
          qq.x = fma(z.y, u.x, qq.x); qq.y = fma(z.y, u.y, qq.y);
        }
      }
    }
    if (sp.has_single(c)) {
      const int r = c == 0 ? 0 : q >> 1;
      rows[sp.row_single(c) * M + s] = cmul(acc0, ldg(twM1 + r * s));
    }
    if (np > 0) {
      const int k = k0;
      rows[sp.row_k(c, 0) * M + s] = cmul(cmk<V>(pp.x - qq.y, pp.y + qq.x), ldg(twM1 + k * s));
      rows[sp.row_qk(c, 0) * M + s] = cmul(cmk<V>(pp.x + qq.y, pp.y - qq.x), ldg(twM1 + (q - k) * s));
    }
  }
}

template <int NT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1) s2048c_kernel(const __grid_constant__ PassArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V* zkt = reinterpret_cast<V*>(smem_raw);                 // zeta_q^{k t}, t < kTMax (the CTA's pair)
  V* tws = zkt + kTMax;                                     // zeta_2048^k, k < M (FFT twiddles)
  V* rows = tws + M;                                        // kRMax rows of M
  V* recv = rows + kRMax * M;                               // partner's partial sums
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  const int q = a.q;
  const Split sp(q);
  const int nres = sp.nres(c);
  const int tid = threadIdx.x;
  const int nth = kGT * nres;
  const int grp = tid / kGT, t = tid % kGT;                 // residue group (row), thread in group
  for (int i = tid; i < M; i += blockDim.x) tws[i] = ldg(reinterpret_cast<const V*>(a.tw_m) + i);
  const V* twm = tws;                                       // zeta_2048^k (shared)
  const V* twM1 = reinterpret_cast<const V*>(a.tw_M1);
  for (int i = tid; i < kTMax; i += blockDim.x) zkt[i] = ldg(twM1 + (int64_t)((sp.kfirst(c) * i) % q) * M);
  __syncthreads();
  V* partner_recv = cl.map_shared_rank(recv, c ^ 1);
  const int T = a.out.T;
  const int T0 = (T + 1) / 2;
  const int tlo = c == 0 ? 0 : T0, thi = c == 0 ? T0 : T;
  const LineIn &fi = a.in_f, &gi = a.in_g;
  const LineOut& o = a.out;
  const int Lout = (int)(o.L + o.j0), j0 = (int)o.j0;
  const int64_t ncl = gridDim.x / 2;
  for (int64_t l = blockIdx.x / 2; l < a.nlines; l += ncl) {
    if (tid == 0 && l + ncl < a.nlines) {  // the next line of f and g into L2
      prefetch_l2(reinterpret_cast<const V*>(fi.ptr[0]) + line_off(fi, l + ncl), fi.L * 16);
      prefetch_l2(reinterpret_cast<const V*>(gi.ptr[0]) + line_off(gi, l + ncl), gi.L * 16);
    }
    if (grp < nres) {
      V* row = rows + grp * M;
      const V* xf = reinterpret_cast<const V*>(fi.ptr[0]) + line_off(fi, l);
      s2048c::fold_line(rows, xf, (int)fi.L, fi.p, sp, c, zkt, twM1, tid, nth);
      compute_sync(nth);
      V F[16];
      fft2048_fwd(F, row, t, grp, twm);
      compute_sync(nth);  // every group is done with its row before the g fold
      const V* xg = reinterpret_cast<const V*>(gi.ptr[0]) + line_off(gi, l);
      s2048c::fold_line(rows, xg, (int)gi.L, gi.p, sp, c, zkt, twM1, tid, nth);
      compute_sync(nth);
      V G[16];
      fft2048_fwd(G, row, t, grp, twm);
#pragma unroll
      for (int k = 0; k < 16; ++k) F[k] = cscale(cmul(F[k], G[k]), a.scale);
      fft2048_inv(F, row, t, grp, twm);
      compute_sync(nth);
    }
    cl.sync();  // the partner has consumed its receive buffer (previous line)
    if (grp < nres) {
      const int np = sp.npairs(c), k0 = sp.kfirst(c);
      for (int s = tid; s < M; s += nth) {
        V v0 = cmk<V>(0, 0), A = cmk<V>(0, 0), B = cmk<V>(0, 0);
        if (sp.has_single(c)) {
          const int r = c == 0 ? 0 : q >> 1;
          v0 = cmulc(rows[sp.row_single(c) * M + s], ldg(twM1 + r * s));
        }
        if (np > 0) {
          const V vk = cmulc(rows[sp.row_k(c, 0) * M + s], ldg(twM1 + k0 * s));
          const V vq = cmulc(rows[sp.row_qk(c, 0) * M + s], ldg(twM1 + (q - k0) * s));
          A = cadd(vk, vq);
          B = csub(vq, vk);
        }
        for (int tb = 0; tb < T; ++tb) {
          if (tb * M + s >= Lout) break;
          V h = (c == 0 || !(tb & 1)) ? v0 : cmk<V>(-v0.x, -v0.y);
          if (np > 0) {
            const V z = zkt[tb];
            h.x = fma(z.x, A.x, h.x); h.x = fma(-z.y, B.y, h.x);
            h.y = fma(z.x, A.y, h.y); h.y = fma(z.y, B.x, h.y);
          }
          if (tb >= tlo && tb < thi) rows[(tb - tlo) * M + s] = h;
          else partner_recv[(c == 0 ? tb - T0 : tb) * M + s] = h;
        }
      }
    }
    cl.sync();
    if (grp < nres) {
      V* y = reinterpret_cast<V*>(o.ptr[0]) + line_off(o, l);
      for (int i = tid; i < (thi - tlo) * M; i += nth) {
        const int tb = tlo + i / M, s = i % M;
        const int j = tb * M + s;
        if (j >= j0 && j < Lout) y[j - j0] = cadd(rows[i], recv[i]);
      }
    }
  }
}

inline size_t smem_bytes() { return sizeof(double2) * (size_t)(kTMax + M + 2 * kRMax * M); }

}  // namespace s2048c
}  // namespace hd
