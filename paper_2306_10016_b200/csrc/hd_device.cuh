// hd_device.cuh -- device building blocks of the hybrid-dealiased convolution
// passes (sm_100a).  One CTA owns C lines of one axis (a "line group") and walks
// the q residues of that axis D at a time:
//
//   fold      w_r[s] = zeta_{qm}^{rs} * sum_{t<p} zeta_q^{rt} x[tm+s]
//             (Forward Eq. PAPER.md:528; Alg. Forward PAPER.md:90-102 incl. the
//             partial last block PAPER.md:100-101)               -> SMEM [c][d][s]
//   fft_fwd   size-m DIF FFT, positive exponent, unnormalised ("W <- m F(W)",
//             PAPER.md:104), radix-8/4/2 register butterflies, output left in
//             digit-reversed order (the internal spectral order)
//   product   H = (1/prod M1) * sum_k F_k G_k
//   fft_inv   size-m DIT FFT, negative exponent, digit-reversed in,
//             natural out -- the exact adjoint of fft_fwd
//   unfold    h[tm+s] += zeta_q^{-tr} zeta_{qm}^{-rs} V_r[s] for t < T
//             (Backward Eq. PAPER.md:531; Alg. Backward)
//
// Shared memory holds complex values in an XOR-swizzled layout so that both the
// unit-stride and the radix-strided butterfly accesses are bank-conflict free.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hd {

constexpr int kMaxPairs = 16;
constexpr int kFoldChunk = 8;  // residues held in registers by one fold/unfold sweep

template <typename T> struct cplx_of;
template <> struct cplx_of<double> { using type = double2; };
template <> struct cplx_of<float> { using type = float2; };

template <typename V> __device__ __forceinline__ V cmk(decltype(V::x) re, decltype(V::x) im) {
  V r; r.x = re; r.y = im; return r;
}
template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return cmk<V>(a.x + b.x, a.y + b.y); }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return cmk<V>(a.x - b.x, a.y - b.y); }
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
  return cmk<V>(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
template <typename V> __device__ __forceinline__ V cmulc(V a, V b) {
  return cmk<V>(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
// acc + a*b
template <typename V> __device__ __forceinline__ V cfma(V acc, V a, V b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
// acc + a*conj(b)
template <typename V> __device__ __forceinline__ V cfmac(V acc, V a, V b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.y, b.x, acc.y); acc.y = fma(-a.x, b.y, acc.y);
  return acc;
}
template <typename V> __device__ __forceinline__ V cscale(V a, decltype(V::x) s) { return cmk<V>(a.x * s, a.y * s); }
// multiply by (s * i), s = +-1
template <typename V, int S> __device__ __forceinline__ V cmul_si(V a) {
  return S > 0 ? cmk<V>(-a.y, a.x) : cmk<V>(a.y, -a.x);
}

// Read-only global load through the non-coherent path.
template <typename V> __device__ __forceinline__ V ldg(const V* p) { return __ldg(p); }

// XOR swizzle: permute the complex slots inside each 128-byte row by the row index.
template <typename V> __device__ __forceinline__ int swz(int i) {
  constexpr int EPR = 128 / (int)sizeof(V);  // 8 (double2) or 16 (float2)
  return i ^ ((i / EPR) & (EPR - 1));
}

// ---------------------------------------------------------------------------
// Radix schedule for m = 2^k: radix-8 stages, then one radix-4 or radix-2 stage.
// DIF stage s works on sub-transforms of size NK(s) with butterfly span NK/R.
// ---------------------------------------------------------------------------
template <int M> struct Sched {
  static constexpr int LOG = (M <= 1) ? 0 : 1 + Sched<M / 2>::LOG;
  static constexpr int N8 = LOG / 3;
  static constexpr int REM = LOG % 3;
  static constexpr int NST = N8 + (REM ? 1 : 0);
  __host__ __device__ static constexpr int radix(int s) { return s < N8 ? 8 : (REM == 1 ? 2 : 4); }
  __host__ __device__ static constexpr int nk(int s) {
    int n = M;
    for (int i = 0; i < s; ++i) n /= radix(i);
    return n;
  }
};
template <> struct Sched<1> { static constexpr int LOG = 0; };

// In-register DFT of size R with exponent sign S: y_j = sum_i v_i zeta_R^{S i j}.
template <typename V, int S> __device__ __forceinline__ void dft2(V& a, V& b) {
  V t = a; a = cadd(t, b); b = csub(t, b);
}
template <typename V, int S> __device__ __forceinline__ void dft4(V* v) {
  V a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
  V b0 = cadd(v[1], v[3]), b1 = cmul_si<V, S>(csub(v[1], v[3]));
  v[0] = cadd(a0, b0); v[2] = csub(a0, b0);
  v[1] = cadd(a1, b1); v[3] = csub(a1, b1);
}
template <typename V, int S> __device__ __forceinline__ void dft8(V* v) {
  using R = decltype(V::x);
  const R h = (R)0.70710678118654752440084436210484903928;
  // radix-2 DIF split: b_n = v_n + v_{n+4}, c_n = (v_n - v_{n+4}) zeta_8^{S n}
  V b[4], c[4];
#pragma unroll
  for (int n = 0; n < 4; ++n) { b[n] = cadd(v[n], v[n + 4]); c[n] = csub(v[n], v[n + 4]); }
  // zeta_8^{S} = h(1 + S i); zeta_8^{2S} = S i; zeta_8^{3S} = h(-1 + S i)
  c[1] = cmk<V>(h * (c[1].x - S * c[1].y), h * (c[1].y + S * c[1].x));
  c[2] = cmul_si<V, S>(c[2]);
  c[3] = cmk<V>(h * (-c[3].x - S * c[3].y), h * (-c[3].y + S * c[3].x));
  dft4<V, S>(b);
  dft4<V, S>(c);
#pragma unroll
  for (int k = 0; k < 4; ++k) { v[2 * k] = b[k]; v[2 * k + 1] = c[k]; }
}
template <typename V, int R, int S> __device__ __forceinline__ void dftR(V* v) {
  if constexpr (R == 2) dft2<V, S>(v[0], v[1]);
  else if constexpr (R == 4) dft4<V, S>(v);
  else dft8<V, S>(v);
}

// Twiddle powers w[j] = w1^j, j < R (w[0] unused), by repeated products of the
// one table entry w1 = zeta_NK^{o} (coalesced load; <= 3 products deep).
template <typename V, int R> __device__ __forceinline__ void tw_powers(V w1, V* w) {
  w[1] = w1;
  if constexpr (R >= 4) { w[2] = cmul(w1, w1); w[3] = cmul(w[2], w1); }
  if constexpr (R >= 8) {
    w[4] = cmul(w[2], w[2]); w[5] = cmul(w[4], w1); w[6] = cmul(w[4], w[2]); w[7] = cmul(w[4], w[3]);
  }
}

template <int M, int ST> struct StageC {
  static constexpr int R = Sched<M>::radix(ST);
  static constexpr int NK = Sched<M>::nk(ST);
  static constexpr int SPAN = NK / R;
  static constexpr int PER_ROW = M / R;
  static constexpr int TWSTEP = M / NK;
};

// Stage twiddle table (host-built per m, see hd_api.cu stage_table): for every
// stage with span > 1, a block [j-1][o] = zeta_NK^{o j}, j = 1..R-1, o < span,
// so that consecutive threads (consecutive o) load consecutive entries.
template <int M, int ST> struct StageOff {
  __host__ __device__ static constexpr int value() {
    int off = 0;
    for (int s = 0; s < ST; ++s) {
      const int R = Sched<M>::radix(s), NK = Sched<M>::nk(s), SP = NK / R;
      if (SP > 1) off += (R - 1) * SP;
    }
    return off;
  }
};

#ifndef HD_TW_LOADS
#define HD_TW_LOADS 1   // stage twiddles per butterfly loaded from the table (1: w1 only, 7: all)
#endif
// Stage twiddles w[j] = zeta_NK^{o j}, j = 1..R-1: HD_TW_LOADS == 1 loads w1 (coalesced
// across o) and forms the rest by <= 3-deep products; otherwise all R-1 are loaded.
template <typename V, int M, int ST>
__device__ __forceinline__ void stage_tw(int o, const V* __restrict__ twst, V* w) {
  using S = StageC<M, ST>;
  const V* tw = twst + StageOff<M, ST>::value() + o;
  if constexpr (HD_TW_LOADS == 1 && S::R > 2) {
    tw_powers<V, S::R>(ldg(tw), w);
  } else {
#pragma unroll
    for (int j = 1; j < S::R; ++j) w[j] = ldg(tw + (j - 1) * S::SPAN);
  }
}

// DIF butterfly of stage ST (forward, +exponent) on registers, offset o inside its block
template <typename V, int M, int ST>
__device__ __forceinline__ void dif_bfly(V* v, int o, const V* __restrict__ twst) {
  using S = StageC<M, ST>;
  dftR<V, S::R, +1>(v);
  if (S::SPAN > 1 && o > 0) {
    V w[S::R];
    stage_tw<V, M, ST>(o, twst, w);
#pragma unroll
    for (int j = 1; j < S::R; ++j) v[j] = cmul(v[j], w[j]);
  }
}
// DIT butterfly of stage ST (inverse, -exponent): adjoint of dif_bfly
template <typename V, int M, int ST>
__device__ __forceinline__ void dit_bfly(V* v, int o, const V* __restrict__ twst) {
  using S = StageC<M, ST>;
  if (S::SPAN > 1 && o > 0) {
    V w[S::R];
    stage_tw<V, M, ST>(o, twst, w);
#pragma unroll
    for (int j = 1; j < S::R; ++j) v[j] = cmulc(v[j], w[j]);
  }
  dftR<V, S::R, -1>(v);
}

// One DIF (forward) or DIT (inverse) stage over nrows rows of M in SMEM.
template <typename V, int M, int NT, int ST, bool INV>
__device__ __forceinline__ void fft_stage(V* buf, int nrows, const V* __restrict__ twm) {
  using S = StageC<M, ST>;
  const int items = nrows * S::PER_ROW;
  for (int it = threadIdx.x; it < items; it += (int)blockDim.x) {
    const int row = it / S::PER_ROW;
    const int w = it % S::PER_ROW;
    const int b = w / S::SPAN, o = w % S::SPAN;
    const int base = row * M + b * S::NK + o;
    V v[S::R];
#pragma unroll
    for (int i = 0; i < S::R; ++i) v[i] = buf[swz<V>(base + i * S::SPAN)];
    if constexpr (!INV) dif_bfly<V, M, ST>(v, o, twm);
    else dit_bfly<V, M, ST>(v, o, twm);
#pragma unroll
    for (int i = 0; i < S::R; ++i) buf[swz<V>(base + i * S::SPAN)] = v[i];
  }
}

// forward stages [ST, STOP) with a barrier after each
template <typename V, int M, int NT, int ST, int STOP>
__device__ __forceinline__ void fft_fwd_range(V* buf, int nrows, const V* twm) {
  if constexpr (ST < STOP) {
    fft_stage<V, M, NT, ST, false>(buf, nrows, twm);
    __syncthreads();
    fft_fwd_range<V, M, NT, ST + 1, STOP>(buf, nrows, twm);
  }
}
// inverse stages ST, ST-1, ..., 0 with a barrier after each
template <typename V, int M, int NT, int ST>
__device__ __forceinline__ void fft_inv_from(V* buf, int nrows, const V* twm) {
  if constexpr (ST >= 0) {
    fft_stage<V, M, NT, ST, true>(buf, nrows, twm);
    __syncthreads();
    fft_inv_from<V, M, NT, ST - 1>(buf, nrows, twm);
  }
}

// ---------------------------------------------------------------------------
// Pass arguments
// ---------------------------------------------------------------------------
struct LineIn {            // element j of line l = g*C + c, batch b, array k:
  const void* ptr[kMaxPairs];  //   ptr[k] + (b/nbi)*s_bo + (b%nbi)*s_b
  int64_t L;               //   + (l >> tl)*s_t + (l & (2^tl-1))*s_l + j*s_j
  int64_t nbi, s_bo;       // two-level batch index (nbi = nbatch: one level)
  int64_t s_b, s_t, s_l, s_j;
  int32_t p;               // ceil(L/m) blocks (fold)
  int32_t tl;              // log2 line-tile width of the layout (>= 30: untiled, l*s_l)
  int64_t jd, s_jt;        // element tiling: jd > 0: j -> (j / jd)*s_jt + (j % jd)*s_j
};
// offset of element j of an input line
__device__ __forceinline__ int64_t in_el(const LineIn& in, int64_t j) {
  if (in.jd <= 0) return j * in.s_j;
  const int64_t hi = j / in.jd;
  return hi * in.s_jt + (j - hi * in.jd) * in.s_j;
}
// two-level batch offset with 32-bit division (batch indices < 2^31)
__device__ __forceinline__ int64_t boff(int64_t b, int64_t nbi, int64_t s_bo, int64_t s_b) {
  const uint32_t ub = (uint32_t)b, un = (uint32_t)nbi;
  const uint32_t hi = ub / un;
  return (int64_t)hi * s_bo + (int64_t)(ub - hi * un) * s_b;
}
__device__ __forceinline__ int64_t line_off(const LineIn& in, int64_t l) {
  if (in.tl >= 30) return l * in.s_l;
  return (l >> in.tl) * in.s_t + (l & ((int64_t(1) << in.tl) - 1)) * in.s_l;
}
struct LineOut {           // element j of line l = g*C + c: ptr[k] + (b/nbi)*s_bo + (b%nbi)*s_b
  void* ptr[kMaxPairs];    //   + (l >> tl)*s_t + (l & (2^tl-1))*s_l + (j>>so_log2)*s_jt + (j&(2^so_log2-1))*s_js
  int64_t L;               // elements written per line
  int64_t nbi, s_bo;
  int64_t s_b, s_t, s_l, s_jt, s_js;
  int32_t so_log2;         // log2 tile width of the element axis (>= 30: plain, j*s_js)
  int32_t T;               // output blocks ceil(L/m) (unfold)
  int32_t tl;              // log2 line-tile width (>= 30: untiled)
  int32_t pad_;
  int64_t jd;              // > 0: element j -> (j / jd)*s_jt + (j % jd)*s_js (overrides so_log2)
  int64_t j0;              // output window: element j of the full line is written to
                           // position j - j0, kept when 0 <= j - j0 < L
};
// element-axis tile code for jt_off: log2 tile (0..29), plain (>= 30), or -width (general)
__device__ __forceinline__ int out_sl(const LineOut& o) { return o.jd > 0 ? -(int)o.jd : o.so_log2; }
__device__ __forceinline__ int64_t line_off(const LineOut& o, int64_t l) {
  if (o.tl >= 30) return l * o.s_l;
  return (l >> o.tl) * o.s_t + (l & ((int64_t(1) << o.tl) - 1)) * o.s_l;
}
// TMA description of a family of lines (hd_s512.cuh; host side: hd_api.cu tma_desc_*)
enum { TMA_NONE = 0, TMA_BULK = 1, TMA_LINE_TILED = 2, TMA_ELEM_TILED = 3, TMA_ELEM2 = 4 };
struct TmaLine {
  int32_t kind;            // TMA_NONE: per-thread copies; TMA_BULK: one 1-D bulk copy per line
  int32_t slog;            // log2 of the tile width S (LINE_TILED / ELEM2: lines, ELEM_TILED: elements)
  int32_t bcast;           // bit 0 / bit 1: batch dimension 3 / 4 has stride 0 (coordinate 0)
  int32_t box;             // ELEM2: elements per box (a divisor of jd, <= 256, multiple of 8)
  int64_t nbi;             // two-level batch split (coordinates b % nbi, b / nbi)
  int64_t jd;              // ELEM2 (input lines, element axis tiled by jd: the slab exchanges):
                           // dims {2S (line in tile), j % jd, j / jd, line tile, batch}
};
constexpr int kTmaArrays = 6;  // arrays (multiconv pairs) with their own tensor maps

struct PassArgs {
  LineIn in_f, in_g;
  LineOut out;
  TmaLine tm_in, tm_in_g, tm_out;
  CUtensorMap tm_in_map[kTmaArrays];
  CUtensorMap tm_in_g_map[kTmaArrays];
  CUtensorMap tm_out_map[kTmaArrays];
  unsigned long long* phase_prof;  // debug (HD_PHASE_PROF=1): per-phase SM cycles, else null
  const void* tw_m;        // zeta_m^k,  k < m
  const void* tw_M1;       // zeta_M1^k, k < M1
  const void* tw_st;       // stage twiddle table of m (see StageOff)
  int64_t nlines;          // lines per batch entry
  int64_t nbatch;
  int64_t ngroups;         // line groups per batch entry (work items = nbatch * ngroups)
  int64_t M1;
  double scale;            // 1 / prod M1 (CONV)
  int32_t q, D, C, c_log2; // residues, residues per group, lines per CTA (power of two)
  int32_t npairs;
  int32_t batch_fastest;
  // hd_conv_real fused into the staged m = 512 x passes (hd_s512.cuh, q = 9):
  // rp (forward): line y is two real rows, re = (double*)in_f.ptr[0] + y * in_f.s_l and
  //   im = re + rp_off (zero for y >= rp_rows): the packed z = f[y] + i f[y + A];
  // rs (inverse): output line y (of w) is split: Re -> (double*)out.ptr[0] + y * out.s_l,
  //   Im -> row y + rs_A of the same array when y >= rs_side_rows (rows >= rs_rows
  //   dropped), else row y of rs_side (added by a fix-up kernel afterwards).
  int32_t rp, rs;
  // fam2 (forward, q = 9): a second family of plain-row lines after the first (the
  // 2-D g rows in the same launch as the f rows): items >= nbatch * ngroups are lines
  // of in_g (nlines2 of them, one batch entry), stored through out2 / tm_out2 /
  // tm_out_map[1]; both families move by bulk loads and element-tiled TMA stores
  int32_t fam2, pad_f2;
  int64_t nlines2;
  LineOut out2;
  TmaLine tm_out2;
  int64_t rp_off, rp_rows;
  int64_t rs_A, rs_side_rows, rs_rows;
  void* rs_side;
  // residue range [r_lo, r_hi) of a generic-engine CONV pass (r_hi = 0: all q): the
  // output is the partial sum over those residues of the backward transform
  // (PAPER.md:531), e.g. one rank's share under residue sharding (hd_conv1d_dist)
  int32_t r_lo, r_hi;
  // the 1-D m = 2048 engine (hd_s2048r.cuh): per-CTA slots for the inverse-transformed
  // residues of all but the last pair of a line (gridDim.x x 2 (ceil(q/2) - 1) x 2048
  // elements), so that the line's unfold runs once over every residue
  void* scr;
  // debug (HD_DEBUG_SKIP, timing experiments only -- results are garbage): bit 0 the
  // staged engine's producer skips the stores, bit 1 the loads
  int32_t dbg;
};

enum { MODE_FWD = 0, MODE_INV = 1, MODE_CONV = 2, MODE_MCONV = 3 /* staged engine only */ };

constexpr int kQF = 16;    // fast q-point DFT paths: q <= 16
constexpr int kPF = 8;     // fast fold path: p <= 8

__device__ __forceinline__ int64_t jt_off(int64_t j, int sl, int64_t s_jt, int64_t s_js) {
  if (sl >= 30) return j * s_js;
  if (sl < 0) {  // general tile width -sl (division)
    const int64_t hi = j / (-sl);
    return hi * s_jt + (j + hi * sl) * s_js;
  }
  return (j >> sl) * s_jt + (j & ((int64_t(1) << sl) - 1)) * s_js;
}

// One (line, s) of the fast fold: P = compile-time bound on p (<= 8)
template <typename V, int M, int P>
__device__ __forceinline__ void fold_fast_one(V* buf, int cb, const V* xl, int64_t s_j, int64_t jd,
                                              int64_t s_jt, int64_t L,
                                              int s, bool live, int q, const V* zt,
                                              const V* __restrict__ twm, const V* __restrict__ twM1) {
  V u[P];
  const int64_t rem = live ? L - s : 0;   // block t is valid while t*M < rem
  if (jd <= 0) {
    const V* xs = xl + (int64_t)s * s_j;
    const int64_t step = (int64_t)M * s_j;
#pragma unroll
    for (int t = 0; t < P; ++t) u[t] = ((int64_t)t * M < rem) ? xs[t * step] : cmk<V>(0, 0);
  } else {
#pragma unroll
    for (int t = 0; t < P; ++t) {
      const int64_t j = (int64_t)t * M + s;
      const int64_t hi = j / jd;
      u[t] = ((int64_t)t * M < rem) ? xl[hi * s_jt + (j - hi * jd) * s_j] : cmk<V>(0, 0);
    }
  }
  V a0 = u[0];
#pragma unroll
  for (int t = 1; t < P; ++t) a0 = cadd(a0, u[t]);
  buf[swz<V>(cb + s)] = a0;
  const V w1 = ldg(twM1 + s);                 // zeta_{M1}^{s}
  const V wq = ldg(twm + s);                  // zeta_{M1}^{q s} = zeta_m^{s}
  V wr = w1;
#pragma unroll
  for (int r = 1; r <= kQF / 2; ++r) {
    if (2 * r > q) break;
    V A = u[0], B = cmk<V>(0, 0);             // t = 0 term: zeta^0 = 1
#pragma unroll
    for (int t = 1; t < P; ++t) {
      const V z = zt[r * kQF + t];            // zeta_q^{r t}
      A.x = fma(u[t].x, z.x, A.x); A.y = fma(u[t].y, z.x, A.y);
      B.x = fma(u[t].x, z.y, B.x); B.y = fma(u[t].y, z.y, B.y);
    }
    // a_r = A + iB, a_{q-r} = A - iB
    const V ar = cmk<V>(A.x - B.y, A.y + B.x);
    buf[swz<V>(cb + r * M + s)] = cmul(ar, wr);
    if (2 * r < q) {
      const V aq = cmk<V>(A.x + B.y, A.y - B.x);
      buf[swz<V>(cb + (q - r) * M + s)] = cmul(aq, cmulc(wq, wr));  // zeta^{(q-r)s} = zeta_m^s conj(zeta^{rs})
    }
    wr = cmul(wr, w1);
  }
}

// ---------------------------------------------------------------------------
// fold: w_r[s] = zeta_{M1}^{rs} sum_{t<p} zeta_q^{rt} x[tm+s] for r in [r0, r0+nd)
// Fast path (all residues, q <= 16, p <= 8): the q-point DFT over t is evaluated
// in symmetric pairs r, q-r (shared real products), the zeta_{M1}^{rs} twiddles
// by recurrence from one table entry.  Generic path: direct sums.
// ---------------------------------------------------------------------------
template <typename V, int M, int NT>
__device__ __forceinline__ void fold(V* buf, const LineIn& in, int k, int64_t b, int64_t g,
                                     int64_t nlines, int C, int clog, int r0, int nd, int q,
                                     const V* zq, const V* zt, const V* __restrict__ twm,
                                     const V* __restrict__ twM1, int tid = -1, int nth = 0) {
  if (tid < 0) { tid = threadIdx.x; nth = blockDim.x; }
  using R = decltype(V::x);
  const V* x = reinterpret_cast<const V*>(in.ptr[k]) + boff(b, in.nbi, in.s_bo, in.s_b);
  const int items = C * M;
  const bool cfast = (in.s_j != 1);
  const int p = in.p;
  const int64_t L = in.L;
  const bool fast = (nd == q) && (q <= kQF) && (p <= kPF);
  for (int it = tid; it < items; it += nth) {
    int c, s;
    if (cfast) { c = it & (C - 1); s = it >> clog; } else { s = it % M; c = it / M; }
    const bool live = (g * C + c) < nlines;
    const V* xl = x + line_off(in, g * C + c);
    const int cb = c * nd * M;  // swizzle indices are relative to buf
    if (fast) {
      if (p <= 1) fold_fast_one<V, M, 1>(buf, cb, xl, in.s_j, in.jd, in.s_jt, L, s, live, q, zt, twm, twM1);
      else if (p <= 2) fold_fast_one<V, M, 2>(buf, cb, xl, in.s_j, in.jd, in.s_jt, L, s, live, q, zt, twm, twM1);
      else if (p <= 4) fold_fast_one<V, M, 4>(buf, cb, xl, in.s_j, in.jd, in.s_jt, L, s, live, q, zt, twm, twM1);
      else fold_fast_one<V, M, kPF>(buf, cb, xl, in.s_j, in.jd, in.s_jt, L, s, live, q, zt, twm, twM1);
    } else {
      for (int d0 = 0; d0 < nd; d0 += kFoldChunk) {
        V acc[kFoldChunk];
        int e[kFoldChunk];  // (r * t) mod q, updated incrementally over t
#pragma unroll
        for (int d = 0; d < kFoldChunk; ++d) { acc[d] = cmk<V>(0, 0); e[d] = 0; }
        if (live) {
          for (int t = 0; t < p; ++t) {
            const int64_t j = (int64_t)t * M + s;
            if (j >= L) break;
            const V u = xl[in_el(in, j)];
#pragma unroll
            for (int d = 0; d < kFoldChunk; ++d) {
              if (d0 + d < nd) {
                acc[d] = cfma(acc[d], u, zq[e[d]]);
                e[d] += r0 + d0 + d;
                if (e[d] >= q) e[d] -= q;
              }
            }
          }
        }
#pragma unroll
        for (int d = 0; d < kFoldChunk; ++d) {
          if (d0 + d < nd) {
            const int r = r0 + d0 + d;
            buf[swz<V>(cb + (d0 + d) * M + s)] = cmul(acc[d], ldg(twM1 + (int64_t)r * s));
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// unfold: h[tm+s] (+)= sum_{r in group} zeta_q^{-tr} zeta_{M1}^{-rs} V_r[s], t < T
// Fast path (all residues, q <= 16): v_r in registers, output blocks in pairs t, q-t.
// ---------------------------------------------------------------------------
template <typename V, int M, int NT, int QM>
__device__ __forceinline__ void unfold_fast(const V* buf, V* y, const LineOut& out, int64_t g,
                                            int64_t nlines, int C, int clog, int q,
                                            const V* zt, const V* __restrict__ twm,
                                            const V* __restrict__ twM1, int tid, int nth) {
  const int items = C * M;
  const int sl = out_sl(out);
  const int so_l = (sl >= 0 && sl < 30) ? (sl < Sched<M>::LOG ? sl : Sched<M>::LOG) : Sched<M>::LOG;
  const int64_t L = out.L;
  const int T = out.T;
  for (int it = tid; it < items; it += nth) {
    const int s_lo = it & ((1 << so_l) - 1);
    const int rest = it >> so_l;
    const int c = rest & (C - 1);
    const int s = ((rest >> clog) << so_l) + s_lo;
    if ((g * C + c) >= nlines) continue;
    const int cb = c * q * M;
    V* yl = y + line_off(out, g * C + c);
    V v[QM];
    const V w1 = ldg(twM1 + s);
    V wr = cmk<V>(1, 0);
#pragma unroll
    for (int r = 0; r < QM; ++r) {
      v[r] = cmk<V>(0, 0);
      if (r < q) {
        v[r] = cmulc(buf[swz<V>(cb + r * M + s)], wr);
        wr = cmul(wr, w1);
      }
    }
    // t = 0
    {
      V h0 = v[0];
#pragma unroll
      for (int r = 1; r < QM; ++r) h0 = cadd(h0, v[r]);
      const int64_t p0 = s - out.j0;
      if (p0 >= 0 && p0 < L) yl[jt_off(p0, sl, out.s_jt, out.s_js)] = h0;
    }
#pragma unroll
    for (int t = 1; t <= QM / 2; ++t) {
      if (2 * t > q) break;
      V A = cmk<V>(0, 0), B = cmk<V>(0, 0);
#pragma unroll
      for (int r = 0; r < QM; ++r) {
        const V z = zt[t * kQF + r];              // zeta_q^{t r}
        A.x = fma(v[r].x, z.x, A.x); A.y = fma(v[r].y, z.x, A.y);
        B.x = fma(v[r].x, z.y, B.x); B.y = fma(v[r].y, z.y, B.y);
      }
      // h_t = sum v_r conj(z) = A - iB ; h_{q-t} = A + iB
      const int64_t p1 = (int64_t)t * M + s - out.j0;
      if (t < T && p1 >= 0 && p1 < L) yl[jt_off(p1, sl, out.s_jt, out.s_js)] = cmk<V>(A.x + B.y, A.y - B.x);
      if (2 * t < q) {
        const int64_t p2 = (int64_t)(q - t) * M + s - out.j0;
        if (q - t < T && p2 >= 0 && p2 < L) yl[jt_off(p2, sl, out.s_jt, out.s_js)] = cmk<V>(A.x - B.y, A.y + B.x);
      }
    }
  }
}

template <typename V, int M, int NT>
__device__ __forceinline__ void unfold(const V* buf, const LineOut& out, int k, int64_t b, int64_t g,
                                       int64_t nlines, int C, int clog, int r0, int nd, int q,
                                       bool accumulate, const V* zq, const V* zt,
                                       const V* __restrict__ twm, const V* __restrict__ twM1,
                                       int tid = -1, int nth = 0) {
  if (tid < 0) { tid = threadIdx.x; nth = blockDim.x; }
  V* y = reinterpret_cast<V*>(out.ptr[k]) + boff(b, out.nbi, out.s_bo, out.s_b);
  if (nd == q && !accumulate) {
    if (q <= 4) { unfold_fast<V, M, NT, 4>(buf, y, out, g, nlines, C, clog, q, zt, twm, twM1, tid, nth); return; }
    if (q <= 8) { unfold_fast<V, M, NT, 8>(buf, y, out, g, nlines, C, clog, q, zt, twm, twM1, tid, nth); return; }
    if (q <= 12) { unfold_fast<V, M, NT, 12>(buf, y, out, g, nlines, C, clog, q, zt, twm, twM1, tid, nth); return; }
    if (q <= kQF) { unfold_fast<V, M, NT, kQF>(buf, y, out, g, nlines, C, clog, q, zt, twm, twM1, tid, nth); return; }
  }
  const int items = C * M;
  const int sl = out_sl(out);
  const int so_l = (sl >= 0 && sl < 30) ? (sl < Sched<M>::LOG ? sl : Sched<M>::LOG) : Sched<M>::LOG;
  const int64_t L = out.L;
  const int T = out.T;
  for (int it = tid; it < items; it += nth) {
    const int s_lo = it & ((1 << so_l) - 1);
    const int rest = it >> so_l;
    const int c = rest & (C - 1);
    const int s = ((rest >> clog) << so_l) + s_lo;
    if ((g * C + c) >= nlines) continue;
    V* yl = y + line_off(out, g * C + c);
    const int cb = c * nd * M;
    for (int d0 = 0; d0 < nd; d0 += kFoldChunk) {
      V v[kFoldChunk];
#pragma unroll
      for (int d = 0; d < kFoldChunk; ++d) {
        v[d] = cmk<V>(0, 0);
        if (d0 + d < nd) {
          const int r = r0 + d0 + d;
          v[d] = cmulc(buf[swz<V>(cb + (d0 + d) * M + s)], ldg(twM1 + (int64_t)r * s));
        }
      }
      int e[kFoldChunk];
#pragma unroll
      for (int d = 0; d < kFoldChunk; ++d) e[d] = 0;
      const bool add = accumulate || d0 > 0;
      for (int t = 0; t < T; ++t) {
        const int64_t j = (int64_t)t * M + s - out.j0;  // position in the output window
        if (j >= L) break;
        V val = cmk<V>(0, 0);
#pragma unroll
        for (int d = 0; d < kFoldChunk; ++d) {
          if (d0 + d < nd) {
            val = cfmac(val, v[d], zq[e[d]]);
            e[d] += r0 + d0 + d;
            if (e[d] >= q) e[d] -= q;
          }
        }
        if (j < 0) continue;
        V* dst = yl + jt_off(j, sl, out.s_jt, out.s_js);
        if (add) { V o = *dst; val = cadd(o, val); }
        *dst = val;
      }
    }
  }
}

// 256-bit global store of two adjacent complex values (STG.E.ENL2.256 on sm_100a);
// p must be 32-byte aligned.  Falls back to two stores for float2.
template <typename V> __device__ __forceinline__ void st256(V* p, V a, V b) {
  if constexpr (sizeof(V) == 16) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" :: "l"(p), "d"((double)a.x), "d"((double)a.y),
                 "d"((double)b.x), "d"((double)b.y) : "memory");
  } else {
    p[0] = a; p[1] = b;
  }
}

// Last forward stage fused with the spectrum store: DIF stage NST-1 (span 1) on
// buf rows (c, d), results written straight to the output element
// kappa = (r0 + d) m + pos of line c.  Line index fastest across threads so
// that the C lines of one kappa land in one contiguous tile segment.
template <typename V, int M, int NT>
__device__ __forceinline__ void fwd_last_store(const V* buf, const LineOut& out, int k, int64_t b,
                                               int64_t g, int64_t nlines, int C, int clog, int r0,
                                               int nd, const V* __restrict__ twm) {
  constexpr int ST = Sched<M>::NST - 1;
  using S = StageC<M, ST>;
  static_assert(S::SPAN == 1, "last stage has unit span");
  V* y = reinterpret_cast<V*>(out.ptr[k]) + boff(b, out.nbi, out.s_bo, out.s_b);
  const int sl = out_sl(out);
  const int items = C * nd * S::PER_ROW;
  for (int it = threadIdx.x; it < items; it += (int)blockDim.x) {
    const int c = it & (C - 1);
    const int rest = it >> clog;
    const int w = rest % S::PER_ROW;
    const int d = rest / S::PER_ROW;
    const int base = (c * nd + d) * M + w * S::R;
    V v[S::R];
#pragma unroll
    for (int i = 0; i < S::R; ++i) v[i] = buf[swz<V>(base + i)];
    dif_bfly<V, M, ST>(v, 0, twm);
    if ((g * C + c) < nlines) {
      V* yl = y + line_off(out, g * C + c);
      const int64_t k0 = (int64_t)(r0 + d) * M + w * S::R;
      if (sizeof(V) == 16 && S::R >= 2 && sl >= 1 && out.s_js == 1) {
        // kappa pairs (even, odd) are adjacent: one 256-bit store per pair
#pragma unroll
        for (int i = 0; i < S::R; i += 2) st256(yl + jt_off(k0 + i, sl, out.s_jt, out.s_js), v[i], v[i + 1]);
      } else {
#pragma unroll
        for (int i = 0; i < S::R; ++i) yl[jt_off(k0 + i, sl, out.s_jt, out.s_js)] = v[i];
      }
    }
  }
}

// First inverse stage fused with the spectrum load: reads kappa = (r0+d) m + pos
// of line c from global, DIT stage NST-1 (span 1), writes buf rows (c, d).
template <typename V, int M, int NT>
__device__ __forceinline__ void inv_first_load(V* buf, const LineIn& in, int64_t b, int64_t g,
                                               int64_t nlines, int C, int clog, int r0, int nd,
                                               const V* __restrict__ twm) {
  constexpr int ST = Sched<M>::NST - 1;
  using S = StageC<M, ST>;
  const V* x = reinterpret_cast<const V*>(in.ptr[0]) + boff(b, in.nbi, in.s_bo, in.s_b);
  const int items = C * nd * S::PER_ROW;
  const bool cfast = (in.s_j != 1);
  for (int it = threadIdx.x; it < items; it += (int)blockDim.x) {
    int c, w, d;
    if (cfast) {
      c = it & (C - 1);
      const int rest = it >> clog;
      w = rest % S::PER_ROW;
      d = rest / S::PER_ROW;
    } else {
      w = it % S::PER_ROW;
      const int rest = it / S::PER_ROW;
      d = rest % nd;
      c = rest / nd;
    }
    V v[S::R];
    const int64_t k0 = (int64_t)(r0 + d) * M + w * S::R;
    const bool live = (g * C + c) < nlines;
    const V* xl = x + line_off(in, g * C + c);
#pragma unroll
    for (int i = 0; i < S::R; ++i) v[i] = live ? xl[in_el(in, k0 + i)] : cmk<V>(0, 0);
    dit_bfly<V, M, ST>(v, 0, twm);
    const int base = (c * nd + d) * M + w * S::R;
#pragma unroll
    for (int i = 0; i < S::R; ++i) buf[swz<V>(base + i)] = v[i];
  }
}

// The pointwise (multi-)product fused between the last forward stage and the
// first inverse stage: for every group of R positions,
// DIF_last(F) * DIF_last(G) is accumulated over the pairs k, scaled by 1/prod M1
// on the last pair and put through DIT_last, all in registers.
//   npairs == 1: result -> bufF;  else accumulator -> bufA
template <typename V, int M, int NT>
__device__ __forceinline__ void conv_mid(V* bufF, const V* bufG, V* bufA, int nrows, int kk,
                                         int npairs, decltype(V::x) scale, const V* __restrict__ twm) {
  constexpr int ST = Sched<M>::NST - 1;
  using S = StageC<M, ST>;
  const int items = nrows * S::PER_ROW;
  const bool last = (kk == npairs - 1);
  for (int it = threadIdx.x; it < items; it += (int)blockDim.x) {
    const int base = it * S::R;  // rows are contiguous: row*M + w*R == it*R
    V f[S::R], h[S::R];
#pragma unroll
    for (int i = 0; i < S::R; ++i) { f[i] = bufF[swz<V>(base + i)]; h[i] = bufG[swz<V>(base + i)]; }
    dif_bfly<V, M, ST>(f, 0, twm);
    dif_bfly<V, M, ST>(h, 0, twm);
#pragma unroll
    for (int i = 0; i < S::R; ++i) f[i] = cmul(f[i], h[i]);
    if (npairs > 1 && kk > 0) {
#pragma unroll
      for (int i = 0; i < S::R; ++i) f[i] = cadd(f[i], bufA[swz<V>(base + i)]);
    }
    V* dst = (npairs == 1) ? bufF : bufA;
    if (last) {
#pragma unroll
      for (int i = 0; i < S::R; ++i) f[i] = cscale(f[i], scale);
      dit_bfly<V, M, ST>(f, 0, twm);
    }
#pragma unroll
    for (int i = 0; i < S::R; ++i) dst[swz<V>(base + i)] = f[i];
  }
}

// work item w -> (batch b, line group g) with 32-bit division
__device__ __forceinline__ void split_item(int64_t w, int64_t nbatch, int64_t ngroups, int bf,
                                           int64_t& b, int64_t& g) {
  const uint32_t uw = (uint32_t)w;
  if (bf) { const uint32_t n = (uint32_t)nbatch; const uint32_t hi = uw / n; g = hi; b = uw - hi * n; }
  else { const uint32_t n = (uint32_t)ngroups; const uint32_t hi = uw / n; b = hi; g = uw - hi * n; }
}

// TMA bulk prefetch of [p, p + bytes) into L2 (UBLKPF); p 16-byte aligned.
__device__ __forceinline__ void prefetch_l2(const void* p, int64_t bytes) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  for (uintptr_t a = a0; a < a1; a += (uintptr_t(1) << 20)) {
    const uint32_t n = (uint32_t)((a1 - a) < (uintptr_t(1) << 20) ? (a1 - a) : (uintptr_t(1) << 20));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(a), "r"(n) : "memory");
  }
}

// Prefetch the input lines of work item (b, g) of array k into L2 (one thread).
template <typename V>
__device__ __forceinline__ void prefetch_lines(const LineIn& in, int k, int64_t b, int64_t g, int C,
                                               int64_t nlines) {
  const V* x = reinterpret_cast<const V*>(in.ptr[k]) + boff(b, in.nbi, in.s_bo, in.s_b);
  const int64_t l0 = g * C;
  const int64_t l1 = (l0 + C < nlines ? l0 + C : nlines) - 1;
  if (l1 < l0) return;
  if (in.tl >= 30) {
    for (int64_t l = l0; l <= l1; ++l)
      prefetch_l2(x + l * in.s_l, ((in.L - 1) * in.s_j + 1) * (int64_t)sizeof(V));
  } else {
    const int64_t S = int64_t(1) << in.tl;
    for (int64_t t = l0 >> in.tl; t <= (l1 >> in.tl); ++t)
      prefetch_l2(x + t * in.s_t, in.L * S * (int64_t)sizeof(V));
  }
}

template <int EPR> __host__ __device__ constexpr int64_t round_slots(int64_t n) {
  return (n + 8 * EPR - 1) / (8 * EPR) * (8 * EPR);
}

// ---------------------------------------------------------------------------
// The pass kernel.  MODE_FWD: fold+FFT -> spectrum; MODE_INV: spectrum ->
// IFFT+unfold; MODE_CONV: fold+FFT both inputs, sum of products, IFFT+unfold.
// Shared memory: [zq: q][zt: 16x16][bufF][bufG][bufA]
// ---------------------------------------------------------------------------
template <typename T, int M, int NT, int MODE>
__global__ void __launch_bounds__(NT) pass_kernel(const __grid_constant__ PassArgs a) {
  using V = typename cplx_of<T>::type;
  constexpr int EPR = 128 / (int)sizeof(V);
  constexpr int NST = Sched<M>::NST;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V* smem = reinterpret_cast<V*>(smem_raw);

  const int k_arr = blockIdx.z;
  const int C = a.C, clog = a.c_log2, D = a.D, q = a.q;
  const int64_t bufn = round_slots<EPR>((int64_t)C * D * M);

  V* zq = smem;                                  // zeta_q^k, k < q
  V* zt = zq + round_slots<EPR>(q);              // zeta_q^{(r t) mod q}, r, t < 16
  V* bufF = zt + round_slots<EPR>(kQF * kQF);
  V* bufG = bufF + bufn;
  V* bufA = bufG + bufn;
  const V* twm = reinterpret_cast<const V*>(a.tw_m);
  const V* twM1 = reinterpret_cast<const V*>(a.tw_M1);
  const V* twst = reinterpret_cast<const V*>(a.tw_st);
  for (int i = threadIdx.x; i < q; i += (int)blockDim.x) zq[i] = ldg(twM1 + (int64_t)i * M);
  for (int i = threadIdx.x; i < kQF * kQF; i += (int)blockDim.x) {
    const int r = i / kQF, t = i % kQF;
    zt[i] = ldg(twM1 + (int64_t)((r * t) % q) * M);
  }
  __syncthreads();

  // persistent loop over work items (batch entry b, line group g); the next item's
  // input is prefetched into L2 by a TMA bulk prefetch while this one computes
  const int64_t total = a.nbatch * a.ngroups;
  for (int64_t w = blockIdx.x; w < total; w += gridDim.x) {
  int64_t g, b;
  split_item(w, a.nbatch, a.ngroups, a.batch_fastest, b, g);
  if (threadIdx.x == 0 && w + gridDim.x < total) {
    int64_t gn, bn;
    split_item(w + gridDim.x, a.nbatch, a.ngroups, a.batch_fastest, bn, gn);
    if constexpr (MODE == MODE_CONV) {
      for (int kk = 0; kk < a.npairs; ++kk) {
        prefetch_lines<V>(a.in_f, kk, bn, gn, C, a.nlines);
        prefetch_lines<V>(a.in_g, kk, bn, gn, C, a.nlines);
      }
    } else {
      prefetch_lines<V>(a.in_f, MODE == MODE_FWD ? k_arr : 0, bn, gn, C, a.nlines);
    }
  }
  const int rlo = a.r_lo, rhi = a.r_hi > 0 ? a.r_hi : q;
  for (int r0 = rlo; r0 < rhi; r0 += D) {
    const int nd = (rhi - r0) < D ? (rhi - r0) : D;
    if constexpr (MODE == MODE_FWD) {
      fold<V, M, NT>(bufF, a.in_f, k_arr, b, g, a.nlines, C, clog, r0, nd, q, zq, zt, twm, twM1);
      __syncthreads();
      fft_fwd_range<V, M, NT, 0, NST - 1>(bufF, C * nd, twst);
      fwd_last_store<V, M, NT>(bufF, a.out, k_arr, b, g, a.nlines, C, clog, r0, nd, twst);
      __syncthreads();
    } else if constexpr (MODE == MODE_INV) {
      inv_first_load<V, M, NT>(bufF, a.in_f, b, g, a.nlines, C, clog, r0, nd, twst);
      __syncthreads();
      fft_inv_from<V, M, NT, NST - 2>(bufF, C * nd, twst);
      unfold<V, M, NT>(bufF, a.out, 0, b, g, a.nlines, C, clog, r0, nd, q, r0 > rlo, zq, zt, twm, twM1);
      __syncthreads();
    } else {
      const T scale = (T)a.scale;
      V* P = (a.npairs == 1) ? bufF : bufA;
      for (int kk = 0; kk < a.npairs; ++kk) {
        fold<V, M, NT>(bufF, a.in_f, kk, b, g, a.nlines, C, clog, r0, nd, q, zq, zt, twm, twM1);
        fold<V, M, NT>(bufG, a.in_g, kk, b, g, a.nlines, C, clog, r0, nd, q, zq, zt, twm, twM1);
        __syncthreads();
        // bufF and bufG are adjacent when the group is full: one sweep over both
        if (bufn == (int64_t)C * nd * M) {
          fft_fwd_range<V, M, NT, 0, NST - 1>(bufF, 2 * C * nd, twst);
        } else {
          fft_fwd_range<V, M, NT, 0, NST - 1>(bufF, C * nd, twst);
          fft_fwd_range<V, M, NT, 0, NST - 1>(bufG, C * nd, twst);
        }
        conv_mid<V, M, NT>(bufF, bufG, bufA, C * nd, kk, a.npairs, scale, twst);
        __syncthreads();
      }
      fft_inv_from<V, M, NT, NST - 2>(P, C * nd, twst);
      unfold<V, M, NT>(P, a.out, 0, b, g, a.nlines, C, clog, r0, nd, q, r0 > rlo, zq, zt, twm, twM1);
      __syncthreads();
    }
  }
  }  // work items
}

// Materialise explicit zero padding: dst[b][i0][i1][i2] = src[..] inside L, else 0.
template <typename V>
__global__ void pad_copy_kernel(const V* __restrict__ src, V* __restrict__ dst,
                                int64_t L0, int64_t L1, int64_t L2,
                                int64_t P0, int64_t P1, int64_t P2, int64_t nb) {
  const int64_t total = nb * P0 * P1 * P2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t i2 = i % P2, r = i / P2;
    int64_t i1 = r % P1; r /= P1;
    int64_t i0 = r % P0; int64_t bb = r / P0;
    V v = cmk<V>(0, 0);
    if (i0 < L0 && i1 < L1 && i2 < L2) v = src[((bb * L0 + i0) * L1 + i1) * L2 + i2];
    dst[i] = v;
  }
}

// Crop: dst[b][o0][o1][o2] = src[b][o0][o1][o2] with src extents P, dst extents O.
template <typename V>
__global__ void crop_copy_kernel(const V* __restrict__ src, V* __restrict__ dst,
                                 int64_t O0, int64_t O1, int64_t O2,
                                 int64_t P0, int64_t P1, int64_t P2, int64_t nb) {
  const int64_t total = nb * O0 * O1 * O2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t i2 = i % O2, r = i / O2;
    int64_t i1 = r % O1; r /= O1;
    int64_t i0 = r % O0; int64_t bb = r / O0;
    dst[i] = src[((bb * P0 + i0) * P1 + i1) * P2 + i2];
  }
}

}  // namespace hd
