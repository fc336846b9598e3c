// hd_s4096r.cuh -- 1-D convolution of long lines with m = 4096 (complex double), one
// CTA per line (persistent over lines): BASELINE config 2 (4096 pairs, L_f = 8192,
// L_g = 3000, L_out = 11191: q = 3 residues of M1 = 12288, p_f = 2, p_g = 1).
//
// Eight compute warps (256 threads, one CTA per SM, up to 255 registers each: no
// spills).  Residues are processed one at a time, f and g side by side:
//   fold      y[n2] = sum_{t<p} zeta_{8q}^{r (8 t + n2)} x[n1 + 512 n2 + 4096 t]
//             = zeta_{8q}^{r n2} sum_t zeta_q^{r t} x[s + 4096 t], s = n1 + 512 n2
//             (Forward Eq. PAPER.md:528, the per-sample factor zeta_{M1}^{r s} split as
//             zeta_{M1}^{r n1} zeta_{8q}^{r n2}); thread tid holds n1 = tid, tid + 256
//   FFT-4096  (positive exponent, unnormalised) as 8 x 512:
//             DFT-8 over n2 in registers, twiddle zeta_{M1}^{n1 (r + q k2)} (the stage
//             twiddle zeta_4096^{n1 k2} times the residue's zeta_{M1}^{r n1}, which
//             commutes with the DFT-8), one CTA-wide exchange through shared memory,
//             then warp k2 runs the register FFT-512 over n1 (hd_w512.cuh) -- f and g
//             interleaved stage by stage (w512::fft_fwd2)
//   product   F G / M1 in registers
//   inverse   the exact adjoint: warp FFT-512^-1, exchange, conjugate
//             twiddles, DFT-8^-1 over k2 -> V''_r[n2] = zeta_{M1}^{-r n1} V_r[n1 + 512 n2]
//   unfold    h[4096 t + s] = sum_{r<q} zeta_{8q}^{-r (8 t + n2)} V''_r[n2]
//             (Backward Eq. PAPER.md:531: zeta_q^{-t r} zeta_{M1}^{-r s} folded into one
//             factor), once per line by the thread that owns s: every residue but the
//             last parks V''_r in per-CTA slots in global memory (PassArgs::scr, L2),
//             written and read back by the same thread (no synchronisation); h is
//             written once.
// The next line's f and g are prefetched into L2 (bulk prefetch) during the last residue.
// Shared memory: E_f | E_g (2 x 4096 slots: the stage exchange, then each warp's
// w512 exchange area inside its own slice), TW (4096: thread-private twiddles of the
// current residue), the FFT-512 twiddle columns, zeta_{8q}^e.
#pragma once
#include "hd_tma.cuh"
#include "hd_w512.cuh"

namespace hd {
namespace s4096r {

using V = double2;
constexpr int M = 4096;
constexpr int NT = 256;   // eight warps
constexpr int kQMax = 4;  // residues (slots: q - 1 per CTA)
constexpr int kPMax = 4;  // blocks per input

// residue slots stay in L2 (evict_last while parked, evict_first on the read back)
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_slot(V* dst, V v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" :: "l"(dst), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ V ld_slot(const V* src, uint64_t pol) {
  V v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(src), "l"(pol));
  return v;
}

__device__ __forceinline__ void cta_sync() { asm volatile("bar.sync 1, %0;" :: "r"(NT) : "memory"); }

// fold + DFT-8 of one input for the thread's two n1: u[c][k2] (the twiddle comes later)
// coef[t * 8 + n2] = zeta_{8q}^{r (8 t + n2)} of the residue
template <int P>
__device__ __forceinline__ void stage_fwd_p(V (*u)[8], const V* x, int L, int p, int tid, const V* coef) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int n1 = tid + 256 * c;
    V v[P][8];
#pragma unroll
    for (int t = 0; t < P; ++t)
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) {
        const int idx = n1 + 512 * n2 + M * t;
        v[t][n2] = (t < p && idx < L) ? ldg(x + idx) : cmk<V>(0, 0);
      }
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) {
      // sum_t zeta_q^{r t} x_t (coef[8 t] = zeta_q^{r t}), then the twist zeta_{8q}^{r n2}
      u[c][n2] = v[0][n2];
#pragma unroll
      for (int t = 1; t < P; ++t)
        if (t < p) u[c][n2] = cfma(u[c][n2], v[t][n2], coef[8 * t]);
      if (n2 > 0) u[c][n2] = cmul(u[c][n2], coef[n2]);
    }
    dft8<V, +1>(u[c]);
  }
}
__device__ __forceinline__ void stage_fwd(V (*u)[8], const V* x, int L, int p, int tid, const V* coef) {
  if (p <= 1) stage_fwd_p<1>(u, x, L, p, tid, coef);
  else if (p <= 2) stage_fwd_p<2>(u, x, L, p, tid, coef);
  else stage_fwd_p<kPMax>(u, x, L, p, tid, coef);
}

// the eight twiddles zeta_{M1}^{n1 (r + q k2)} = c om^{k2}, c = zeta_{M1}^{r n1},
// om = zeta_4096^{n1}, in registers (13 products)
__device__ __forceinline__ void tw_regs(V* t, V c_, V om) {
  const V w2 = cmul(om, om), w3 = cmul(w2, om), w4 = cmul(w2, w2);
  t[0] = c_;
  t[1] = cmul(c_, om); t[2] = cmul(c_, w2); t[3] = cmul(c_, w3); t[4] = cmul(c_, w4);
  t[5] = cmul(c_, cmul(w4, om)); t[6] = cmul(c_, cmul(w4, w2)); t[7] = cmul(c_, cmul(w4, w3));
}
// z^e for 0 <= e < QM
template <int QM>
__device__ __forceinline__ V zpow(V z, int e) {
  V p = cmk<V>(1, 0);
#pragma unroll
  for (int i = 0; i < QM - 1; ++i)
    if (i < e) p = cmul(p, z);
  return p;
}

// stage A of one item (fold, DFT-8, twiddles) for f into Ef and g into Eg, at the
// thread's own slots [k2 * 512 + n1]
template <int QM>
__device__ __forceinline__ void stage_item(V* Ef, V* Eg, const V* f, int Lf, int pf, const V* g, int Lg, int pg,
                                           int r, int tid, const V* cf, const V* z, const V* om) {
  V uf[2][8], ug[2][8];
  stage_fwd(uf, f, Lf, pf, tid, cf);
  stage_fwd(ug, g, Lg, pg, tid, cf);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    V t[8];
    tw_regs(t, zpow<QM>(z[c], r), om[c]);
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) {
      const int i = k2 * 512 + tid + 256 * c;
      Ef[i] = cmul(uf[c][k2], t[k2]);
      Eg[i] = cmul(ug[c][k2], t[k2]);
    }
  }
}

// Items (line l, residue r) in order.  Exchange areas: f alternates between EA and EC
// (the item's forward exchange, then each warp's w512 area and inverse output), g
// always EB.  Two CTA barriers per item: bar2 (stage A visible) and bar3 (inverse
// outputs visible); the next item's stage A runs before bar3 -- its f into the other
// f area (last read before this item's bar2), its g into EB once every warp has
// read its EB slice (an mbarrier with one arrival per warp, so the writers wait for
// the early reads, not for the other warps' transforms).
// WIN: an output window with a nonzero start (separate instantiation: the window-free
// kernel keeps its registers)
// QM: compile-time bound on q (3: config 2's lines; the smaller unfold measured 3.6 %
// faster than the general QM = 4)
template <bool WIN, int QM>
__global__ void __launch_bounds__(NT, 1) s4096r_kernel(const __grid_constant__ PassArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V* EA = reinterpret_cast<V*>(smem_raw);
  V* EC = EA + M;
  V* EB = EC + M;
  V* twt = EB + M;                      // FFT-512 twiddle columns
  V* coefs = twt + w512::kTwRows * 32;  // [r][t * 8 + n2] = zeta_{8q}^{r (8 t + n2)}
  uint64_t* bar_b = reinterpret_cast<uint64_t*>(coefs + kQMax * kPMax * 8);
  const int q = a.q;
  const int tid = threadIdx.x, wp = tid >> 5, lane = tid & 31;
  const V* twm = reinterpret_cast<const V*>(a.tw_m);     // zeta_4096^k
  const V* twM1 = reinterpret_cast<const V*>(a.tw_M1);   // zeta_{M1}^k
  // FFT-512 twiddle columns from the zeta_4096 table (zeta_512^j = zeta_4096^{8 j})
  for (int i = tid; i < w512::kTwRows * 32; i += NT) {
    const int row = i >> 5, ln = i & 31;
    const int e = row < 15 ? (ln * (row + 1)) % 512 : 16 * ((row - 15) + 8 * (ln & 1));
    twt[i] = ldg(twm + 8 * e);
  }
  for (int i = tid; i < kQMax * kPMax * 8; i += NT) {
    const int r = i / (kPMax * 8), tn = i % (kPMax * 8);
    coefs[i] = ldg(twM1 + (int64_t)((r * tn) % (8 * q)) * 512);  // zeta_{8q}^e = zeta_{M1}^{512 e}
  }
  if (tid == 0) mbar_init(bar_b, NT / 32);
  __syncthreads();
  const V* tw = twt + lane;
  const LineIn& fi = a.in_f;
  const LineIn& gi = a.in_g;
  const LineOut& o = a.out;
  // output window: positions [j0, j0 + Lout) of the full result,
  // element j at h[j - j0]; T = ceil((j0 + Lout) / 4096) blocks are unfolded
  const int Lf = (int)fi.L, Lg = (int)gi.L, T = o.T, j0 = WIN ? (int)o.j0 : 0, jend = j0 + (int)o.L;
  const double scale = a.scale;
  // per-CTA residue slots (absent for q = 1: never touched then)
  V* slots = a.scr ? reinterpret_cast<V*>(a.scr) + (int64_t)blockIdx.x * (kQMax - 1) * M : nullptr;
  const uint64_t pol = policy_evict_last(), pol_ef = policy_evict_first();
  const V* F0 = reinterpret_cast<const V*>(fi.ptr[0]);
  const V* G0 = reinterpret_cast<const V*>(gi.ptr[0]);
  const V z[2] = {ldg(twM1 + tid), ldg(twM1 + tid + 256)};  // zeta_{M1}^{n1}
  const V om[2] = {ldg(twm + tid), ldg(twm + tid + 256)};   // zeta_4096^{n1}
  int64_t l = blockIdx.x;
  if (l >= a.nlines) return;
  if (tid == 0 && l + gridDim.x < a.nlines) {
    bulk_prefetch_l2(F0 + line_off(fi, l + gridDim.x), (uint32_t)Lf * 16u);
    bulk_prefetch_l2(G0 + line_off(gi, l + gridDim.x), (uint32_t)Lg * 16u);
  }
  stage_item<QM>(EA, EB, F0 + line_off(fi, l), Lf, fi.p, G0 + line_off(gi, l), Lg, gi.p, 0, tid, coefs, z, om);
  int r = 0;
  uint32_t it = 0;
  bool cur_a = true;
#pragma unroll 1
  while (true) {
    V* Ecur = cur_a ? EA : EC;
    V* Enxt = cur_a ? EC : EA;
    V* Ew = Ecur + wp * 512;  // warp k2 = wp: its slice
    cta_sync();  // bar2: this item's stage A is visible
    {
      V a_[16], b_[16];
      const V* Bw = EB + wp * 512;
#pragma unroll
      for (int i = 0; i < 16; ++i) { a_[i] = Ew[lane + 32 * i]; b_[i] = Bw[lane + 32 * i]; }
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_b);  // this warp is done with its EB slice
      w512::fft_fwd2(a_, b_, Ew, lane, tw, false);
#pragma unroll
      for (int k = 0; k < 16; ++k) a_[k] = cscale(cmul(a_[k], b_[k]), scale);
      w512::fft_inv(a_, Ew, lane, tw);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 16; ++i) Ew[lane + 32 * i] = a_[i];
    }
    // the next item's stage A
    int64_t ln = l;
    int rn = r + 1;
    if (rn == q) { rn = 0; ln = l + gridDim.x; }
    const bool more = ln < a.nlines;
    if (more) {
      // the next line into L2 while this line's last residue runs (a whole line ahead
      // measured 0.1 ms slower on config 2: the early copies evict lines still in use)
      if (rn == q - 1 && tid == 0 && ln + gridDim.x < a.nlines) {
        bulk_prefetch_l2(F0 + line_off(fi, ln + gridDim.x), (uint32_t)Lf * 16u);
        bulk_prefetch_l2(G0 + line_off(gi, ln + gridDim.x), (uint32_t)Lg * 16u);
      }
      mbar_wait(bar_b, it & 1u);  // every warp has read its EB slice
      stage_item<QM>(Enxt, EB, F0 + line_off(fi, ln), Lf, fi.p, G0 + line_off(gi, ln), Lg, gi.p, rn, tid,
                 coefs + rn * (kPMax * 8), z, om);
    }
    cta_sync();  // bar3: this item's inverse outputs are visible
    // this item: conjugate twiddles and DFT-8^-1 over k2 for the thread's two n1
    V* hw = reinterpret_cast<V*>(o.ptr[0]) + line_off(o, l) - j0;  // element j at hw[j]
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      const int n1 = tid + 256 * c;
      V v[8];
      {
        V t[8];
        tw_regs(t, zpow<QM>(c ? z[1] : z[0], r), c ? om[1] : om[0]);
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) v[k2] = cmulc(Ecur[k2 * 512 + n1], t[k2]);
      }
      dft8<V, -1>(v);
      if (r < q - 1) {
#pragma unroll
        for (int n2 = 0; n2 < 8; ++n2) st_slot(slots + r * M + n1 + 512 * n2, v[n2], pol);
      } else {
        // unfold of the thread's positions s = n1 + 512 n2:
        // h[4096 t + s] = sum_rr conj(coef_rr[8 t + n2]) V''_rr[n2]
#pragma unroll
        for (int n2 = 0; n2 < 8; ++n2) {
          const int s = n1 + 512 * n2;
          V w[QM];
#pragma unroll
          for (int rr = 0; rr < QM; ++rr)
            w[rr] = rr == q - 1 ? v[n2] : (rr < q - 1 ? ld_slot(slots + rr * M + s, pol_ef) : cmk<V>(0, 0));
#pragma unroll
          for (int t = 0; t < QM; ++t) {
            const int j = M * t + s;
            if (t >= T || j >= jend) break;
            if (WIN && j < j0) continue;
            V val = w[0];
#pragma unroll
            for (int rr = 1; rr < QM; ++rr)
              if (rr < q) val = cfmac(val, w[rr], coefs[rr * (kPMax * 8) + 8 * t + n2]);
            __stcs(hw + j, val);
          }
        }
      }
    }
    if (!more) break;
    cur_a = !cur_a;
    l = ln;
    r = rn;
    ++it;
  }
}

}  // namespace s4096r
}  // namespace hd
