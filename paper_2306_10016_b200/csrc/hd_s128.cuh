// hd_s128.cuh -- staged engine for FFT size m = 128, complex float (complex64).
//
// The m = 128 counterpart of hd_s512.cuh for the complex64 3-D configuration
// (BASELINE config 4: 512^3 (*) 129^3, M1 = 640 = 5 x 128 on every axis).  One
// persistent CTA runs q compute warps (warp r owns residue r) and one producer
// warp that issues every TMA copy; a work item is a group of C = 4 lines (the tile
// width S = 4 of the tiled intermediates), so one warp transforms residue r of four
// lines at once: lane (c, u) = (lane >> 3, lane & 7) holds 16 points of line c.
//
//   stage     rows j = t m + s of the 4 lines, in the layout of the input family:
//             interleaved [j][c] (lines tiled by 4: TMA tensor boxes of 128 x 4)
//             or line-major [c][j] (plain rows: one 1-D bulk copy per line)
//   fold      thread (c, s): w_r[s] = zeta_{qm}^{rs} sum_{t<p} zeta_q^{rt} x[tm+s]
//             (Forward Eq. PAPER.md:528; Alg. Forward) -> row r
//   FFT-128   warp r, line c: 128 = 16 x 8 -- radix-16 over x[u + 8i] in registers,
//             twiddle zeta_128^{u k1}, transpose within the 8-lane group through the
//             warp's own row (swizzled: conflict-free), two radix-8 DFTs per lane.
//             Lane u then holds frequency 2u + j + 16 k2 in register (j, k2)
//             (PAPER.md:104); the spectrum is stored at position 16 k2 + 8 j + u.
//   CONV      F(row r) G(row q + r) (1/prod M1) -> inverse FFT -> row r
//   INV       row r (spectrum, position order) -> inverse FFT -> row r
//   unfold    thread (c, s): h[tm+s] = sum_r zeta_q^{-tr} zeta_{qm}^{-rs} V_r[s], t < T
//             (Backward Eq. PAPER.md:531; Alg. Backward)
//
// Results are written in the layout of the output family: in place when it equals
// the input's, else into a separate output region (element-tiled outputs, or rows
// after tiled inputs), and leave by TMA (tensor boxes / bulk rows) or plain stores.
// The spectral position order is internal to the passes of one axis; hd_api.cu runs
// every pass of an axis on the same engine.
#pragma once
#include <cuda.h>

#include "hd_internal.h"
#include "hd_tma.cuh"
#include "hd_w512.cuh"
#include "hd_zq_table.h"

namespace hd {
namespace s128 {

using V = float2;
constexpr int M = 128;
constexpr int C = 4;       // lines per work item
constexpr int kQMax = 8;
constexpr int kPMax = 8;
constexpr int kBox = 128;  // elements per line per TMA tensor box
constexpr int kPad = 8;    // line-major stage: line stride rows * M + kPad (spreads banks)

// stage slot of element j of line c: c*sc + (j >> sl)*sjt + (j & (2^sl - 1))*sjs
struct Lay {
  int sc, sjt, sjs, sl;
  __device__ __forceinline__ int at(int c, int j) const {
    return c * sc + (j >> sl) * sjt + (j & ((1 << sl) - 1)) * sjs;
  }
};
__device__ __forceinline__ Lay lay_interleaved() { return Lay{1, 16, 4, 2}; }       // [j][c]
__device__ __forceinline__ Lay lay_rows(int rs) { return Lay{rs, 4, 1, 2}; }        // [c][j], stride rs
__device__ __forceinline__ Lay lay_elem(int slog) {                                 // [j >> S][c][j & (S-1)]
  return Lay{1 << slog, 4 << slog, 1, slog};
}

// ---------------------------------------------------------------------------
// loads of one work item (lines 4g .. 4g+3 of batch entry b)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t item_bytes(const TmaLine& t, const LineIn& in, int nlive) {
  const uint32_t L = (uint32_t)in.L;
  return t.kind == TMA_BULK ? (uint32_t)nlive * L * 8u : ((L + kBox - 1) / kBox) * kBox * C * 8u;
}

// one line family into the stage at row offset j_base (the f rows, or the g rows of CONV)
__device__ __forceinline__ void load_family(const TmaLine& t, const CUtensorMap* map, const LineIn& in, int kk,
                                            int64_t b, int64_t g, int nlive, V* buf, const Lay& ly, int j_base,
                                            uint64_t* bar) {
  const int L = (int)in.L;
  if (t.kind == TMA_BULK) {
    const V* x = reinterpret_cast<const V*>(in.ptr[kk]) + boff(b, in.nbi, in.s_bo, in.s_b);
    for (int c = 0; c < nlive; ++c)
      bulk_load(buf + ly.at(c, j_base), x + line_off(in, 4 * g + c), (uint32_t)L * 8u, bar);
  } else {
    int co[5];
    for (int j0 = 0; j0 < L; j0 += kBox) {
      tma_coords(t, b, 4 * g, j0, co);
      tma_load(buf + ly.at(0, j_base + j0), map, co, bar);
    }
  }
}

// per-thread fallback (layouts TMA cannot express): plain loads by the compute warps
__device__ __forceinline__ void load_family_st(const LineIn& in, int kk, int64_t b, int64_t g, int nlive, V* buf,
                                               const Lay& ly, int j_base, int tid, int nth) {
  const int L = (int)in.L;
  const V* x = reinterpret_cast<const V*>(in.ptr[kk]) + boff(b, in.nbi, in.s_bo, in.s_b);
  for (int i = tid; i < nlive * L; i += nth) {
    const int c = i / L, j = i - c * L;
    buf[ly.at(c, j_base + j)] = x[line_off(in, 4 * g + c) + in_el(in, j)];
  }
}

// ---------------------------------------------------------------------------
// stores of one work item: output slots j < out.L (+ out.j0, the window start)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void store_tma(const PassArgs& a, int kk, int64_t b, int64_t g, int nlive, const V* ob,
                                          const Lay& lo) {
  const LineOut& o = a.out;
  const int L = (int)o.L;
  if (a.tm_out.kind == TMA_BULK) {
    V* y = reinterpret_cast<V*>(o.ptr[kk]) + boff(b, o.nbi, o.s_bo, o.s_b);
    for (int c = 0; c < nlive; ++c) bulk_store(y + line_off(o, 4 * g + c), ob + lo.at(c, 0), (uint32_t)L * 8u);
  } else {
    int co[5];
    for (int j0 = 0; j0 < L; j0 += kBox) {
      tma_coords(a.tm_out, b, 4 * g, j0, co);
      tma_store(&a.tm_out_map[kk], co, ob + lo.at(0, j0));
    }
  }
}

__device__ __forceinline__ void store_st(const PassArgs& a, int kk, int64_t b, int64_t g, int nlive, const V* ob,
                                         const Lay& lo, int tid, int nth) {
  const LineOut& o = a.out;
  const int L = (int)o.L, j0 = (int)o.j0;
  V* y = reinterpret_cast<V*>(o.ptr[kk]) + boff(b, o.nbi, o.s_bo, o.s_b);
  const int sl = out_sl(o);
  if (o.tl < 30 && o.s_l == 1) {  // lines interleaved in memory: line index fastest (coalesced)
    for (int i = tid; i < C * L; i += nth) {
      const int c = i & 3, j = i >> 2;
      if (c < nlive) y[line_off(o, 4 * g + c) + jt_off(j, sl, o.s_jt, o.s_js)] = ob[lo.at(c, j + j0)];
    }
    return;
  }
  for (int i = tid; i < nlive * L; i += nth) {
    const int c = i / L, j = i - c * L;
    y[line_off(o, 4 * g + c) + jt_off(j, sl, o.s_jt, o.s_js)] = ob[lo.at(c, j + j0)];
  }
}

// ---------------------------------------------------------------------------
// fold / unfold of one column (line c, offset s) -- tables: tM1[k] = zeta_{M1}^k
// ---------------------------------------------------------------------------
// rows t < p of a family at row offset j_base -> rows r < q (in place)
__device__ __forceinline__ void fold_col(V* buf, const Lay& ly, int c, int s, int j_base, int L, int p, int q,
                                         int M1, const V* tM1) {
  V u[kPMax];
  const int base = ly.at(c, j_base + s);
  const int rstep = (M >> ly.sl) * ly.sjt;  // slot distance of one row (M is a multiple of the tile)
  const int rem = L - s;
#pragma unroll
  for (int t = 0; t < kPMax; ++t)
    u[t] = (t < p && t * M < rem) ? buf[base + t * rstep] : make_float2(0.f, 0.f);
  int krs = 0;  // r s mod M1
  for (int r = 0; r < q; ++r) {
    V acc = u[0];
    int k = r;  // r t mod q
#pragma unroll
    for (int t = 1; t < kPMax; ++t) {
      if (t < p) {
        acc = cfma(acc, u[t], tM1[k * M]);
        k += r; if (k >= q) k -= q;
      }
    }
    buf[base + r * rstep] = cmul(acc, tM1[krs]);
    krs += s; if (krs >= M1) krs -= M1;
  }
}

// rows r < q -> output slots t m + s < Lout, t < T (in place or into the output region)
__device__ __forceinline__ void unfold_col(const V* buf, const Lay& ly, V* ob, const Lay& lo, int c, int s, int q,
                                           int T, int Lout, int M1, const V* tM1) {
  V v[kQMax];
  const int base = ly.at(c, s);
  const int rstep = (M >> ly.sl) * ly.sjt;
  int krs = 0;
#pragma unroll
  for (int r = 0; r < kQMax; ++r) {
    if (r < q) {
      v[r] = cmulc(buf[base + r * rstep], tM1[krs]);
      krs += s; if (krs >= M1) krs -= M1;
    }
  }
  const int obase = lo.at(c, s);
  const int ostep = (M >> lo.sl) * lo.sjt;
  for (int t = 0; t < T; ++t) {
    if (t * M + s >= Lout) break;
    V acc = v[0];
    int k = t;  // t r mod q
#pragma unroll
    for (int r = 1; r < kQMax; ++r) {
      if (r < q) {
        acc = cfmac(acc, v[r], tM1[k * M]);
        k += t; if (k >= q) k -= q;
      }
    }
    ob[obase + t * ostep] = acc;
  }
}

// Compile-time q (QC) and block count P: the q-point DFT over the blocks in the
// pair form (rows r and q - r share the products with cos / sin of 2 pi r t / q,
// constant-bank operands from c_zqf), twiddles zeta_{M1}^{rs} = w1^r as products
// of w1 = zeta_{M1}^s.
template <int QC, int P>
__device__ __forceinline__ void fold_colq(V* buf, int base, int rstep, int rem, V w1) {
  V u[P];
#pragma unroll
  for (int t = 0; t < P; ++t) u[t] = (t * M < rem) ? buf[base + t * rstep] : make_float2(0.f, 0.f);
  V w[QC];
  w[0] = make_float2(1.f, 0.f);
#pragma unroll
  for (int r = 1; r < QC; ++r) w[r] = r == 1 ? w1 : cmul(w[r - 1], w1);
  V s0 = u[0];
#pragma unroll
  for (int t = 1; t < P; ++t) s0 = cadd(s0, u[t]);
  buf[base] = s0;
#pragma unroll
  for (int r = 1; 2 * r < QC; ++r) {
    V pp = u[0], qq = make_float2(0.f, 0.f);
#pragma unroll
    for (int t = 1; t < P; ++t) {
      const float2 z = c_zqf[QC][(r * t) % QC];
      pp.x = fmaf(z.x, u[t].x, pp.x); pp.y = fmaf(z.x, u[t].y, pp.y);
      qq.x = fmaf(z.y, u[t].x, qq.x); qq.y = fmaf(z.y, u[t].y, qq.y);
    }
    buf[base + r * rstep] = cmul(make_float2(pp.x - qq.y, pp.y + qq.x), w[r]);
    buf[base + (QC - r) * rstep] = cmul(make_float2(pp.x + qq.y, pp.y - qq.x), w[QC - r]);
  }
  if constexpr (QC % 2 == 0) {
    V a = u[0];
#pragma unroll
    for (int t = 1; t < P; ++t) a = (t & 1) ? csub(a, u[t]) : cadd(a, u[t]);
    buf[base + (QC / 2) * rstep] = cmul(a, w[QC / 2]);
  }
}

// h_t = sum_r zeta_q^{-tr} conj(w1^r) V_r, pair form over (r, q - r)
template <int QC>
__device__ __forceinline__ void unfold_colq(const V* buf, int base, int rstep, V* ob, int obase, int ostep, int T,
                                            int rem, V w1) {
  V v[QC];
  v[0] = buf[base];
  V w = w1;
#pragma unroll
  for (int r = 1; r < QC; ++r) {
    v[r] = cmulc(buf[base + r * rstep], w);
    if (r + 1 < QC) w = cmul(w, w1);
  }
  constexpr int NP = (QC - 1) / 2;
  V A[NP + 1], B[NP + 1];
#pragma unroll
  for (int r = 1; r <= NP; ++r) { A[r] = cadd(v[r], v[QC - r]); B[r] = csub(v[QC - r], v[r]); }
#pragma unroll
  for (int t = 0; t < QC; ++t) {
    if (t < T && t * M < rem) {
      V h = v[0];
#pragma unroll
      for (int r = 1; r <= NP; ++r) {
        const float2 z = c_zqf[QC][(t * r) % QC];
        h.x = fmaf(z.x, A[r].x, h.x); h.x = fmaf(-z.y, B[r].y, h.x);
        h.y = fmaf(z.x, A[r].y, h.y); h.y = fmaf(z.y, B[r].x, h.y);
      }
      if constexpr (QC % 2 == 0) h = (t & 1) ? csub(h, v[QC / 2]) : cadd(h, v[QC / 2]);
      ob[obase + t * ostep] = h;
    }
  }
}

// fold of one column with the block count dispatched to a compile-time P <= QC
template <int QC>
__device__ __forceinline__ void fold_dispatch(V* buf, int base, int rstep, int rem, int p, V w1) {
  switch (p) {
    case 1: fold_colq<QC, 1>(buf, base, rstep, rem, w1); break;
    case 2: if constexpr (QC >= 2) fold_colq<QC, 2>(buf, base, rstep, rem, w1); break;
    case 3: if constexpr (QC >= 3) fold_colq<QC, 3>(buf, base, rstep, rem, w1); break;
    case 4: if constexpr (QC >= 4) fold_colq<QC, 4>(buf, base, rstep, rem, w1); break;
    case 5: if constexpr (QC >= 5) fold_colq<QC, 5>(buf, base, rstep, rem, w1); break;
    case 6: if constexpr (QC >= 6) fold_colq<QC, 6>(buf, base, rstep, rem, w1); break;
    case 7: if constexpr (QC >= 7) fold_colq<QC, 7>(buf, base, rstep, rem, w1); break;
    default: if constexpr (QC >= 8) fold_colq<QC, 8>(buf, base, rstep, rem, w1); break;
  }
}

// ---------------------------------------------------------------------------
// FFT-128 of residue row R of line c (lane = 8 c + u), through the warp's own row
// ---------------------------------------------------------------------------
// exchange slot of (k1, u) of line c: eb + c*esc + ((k1 + c*erot) & 15)*8 + (u ^ (k1 >> 1))
struct Ex {
  int eb, esc, erot;
  __device__ __forceinline__ int at(int c, int k1, int u) const {
    return eb + c * esc + (((k1 + c * erot) & 15) << 3) + (u ^ (k1 >> 1));
  }
};
__device__ __forceinline__ Ex ex_of(const Lay& ly, bool il, int R) {
  return il ? Ex{R * M * C, M, 1} : Ex{R * M, ly.sc, 0};
}

// forward: a[i] = x[u + 8i] in, out: a[8 j + k2] = X[2u + j + 16 k2]
__device__ __forceinline__ void fft_fwd(V* a, V* buf, const Ex& e, int c, int u, const V* t128) {
  w512::dft16<+1, false, V>(a);
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) a[k1] = cmul(a[k1], t128[(u * k1) & (M - 1)]);
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) buf[e.at(c, k1, u)] = a[k1];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int v = 0; v < 8; ++v) a[8 * j + v] = buf[e.at(c, 2 * u + j, v)];
  dft8<V, +1>(a);
  dft8<V, +1>(a + 8);
}

// two forward FFT-128s (rows of their own: exchanges ea, eb) interleaved stage by stage
// -- independent chains for the convolution pass's F and G
__device__ __forceinline__ void fft_fwd2(V* a, V* b, V* buf, const Ex& ea, const Ex& eb, int c, int u,
                                         const V* t128) {
  w512::dft16<+1, false, V>(a);
  w512::dft16<+1, false, V>(b);
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) {
    const V w = t128[(u * k1) & (M - 1)];
    a[k1] = cmul(a[k1], w);
    b[k1] = cmul(b[k1], w);
  }
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) {
    buf[ea.at(c, k1, u)] = a[k1];
    buf[eb.at(c, k1, u)] = b[k1];
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      a[8 * j + v] = buf[ea.at(c, 2 * u + j, v)];
      b[8 * j + v] = buf[eb.at(c, 2 * u + j, v)];
    }
  dft8<V, +1>(a);
  dft8<V, +1>(a + 8);
  dft8<V, +1>(b);
  dft8<V, +1>(b + 8);
}

// inverse (adjoint): a[8 j + k2] = Y[2u + j + 16 k2] in; out: a[i] = sum_f zeta^{-(u + 8i) f} Y[f]
__device__ __forceinline__ void fft_inv(V* a, V* buf, const Ex& e, int c, int u, const V* t128) {
  dft8<V, -1>(a);
  dft8<V, -1>(a + 8);
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int v = 0; v < 8; ++v) buf[e.at(c, 2 * u + j, v)] = a[8 * j + v];
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) a[k1] = buf[e.at(c, k1, u)];
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) a[k1] = cmulc(a[k1], t128[(u * k1) & (M - 1)]);
  w512::dft16<-1, false, V>(a);
}

// time-order row R of line c: element R*M + u + 8i (a[i])
__device__ __forceinline__ void load_time(V* a, const V* buf, const Lay& ly, int c, int u, int R) {
  const int base = ly.at(c, R * M + u);  // stage layouts have tiles of <= 8 elements
  const int istep = (8 >> ly.sl) * ly.sjt;
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = buf[base + i * istep];
}
__device__ __forceinline__ void store_time(const V* a, V* buf, const Lay& ly, int c, int u, int R) {
  const int base = ly.at(c, R * M + u);
  const int istep = (8 >> ly.sl) * ly.sjt;
#pragma unroll
  for (int i = 0; i < 16; ++i) buf[base + i * istep] = a[i];
}
// spectrum row R of line c: position 16 k2 + 8 j + u holds a[8 j + k2]
__device__ __forceinline__ void store_spec(const V* a, V* buf, const Lay& ly, int c, int u, int R) {
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) buf[ly.at(c, R * M + 16 * k2 + 8 * j + u)] = a[8 * j + k2];
}
__device__ __forceinline__ void load_spec(V* a, const V* buf, const Lay& ly, int c, int u, int R) {
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) a[8 * j + k2] = buf[ly.at(c, R * M + 16 * k2 + 8 * j + u)];
}

// shared memory: barriers (128 B) | zeta_128 table | zeta_{M1} table | 2 stages
// stage = input rows (R_in = q, CONV: 2q) [+ output region of q rows unless in place]
// (measured: folding g on the fly per residue warp from its p_g raw rows saves
// shared memory but not time -- 2.30 vs 2.27 ms on config 4's conv_z, 2.58 ms
// when the saving is spent on a third CTA per SM at 96 registers)
__host__ __device__ inline int in_floats2(int q, int mode, int pg = 0) {
  (void)pg;
  return C * ((mode == MODE_CONV ? 2 * q : q) * M + kPad);
}
__host__ __device__ inline int out_floats2(int q) { return C * (q * M + kPad); }
__host__ __device__ inline int m1_slots(int M1) { return (M1 + 15) / 16 * 16; }
__host__ __device__ inline size_t smem_bytes(int q, int mode, int M1, bool inplace, int pg) {
  return 128 + sizeof(float2) * (size_t)(M + m1_slots(M1) +
                                         2 * (in_floats2(q, mode, pg) + (inplace ? 0 : out_floats2(q))));
}

// The convolution pass (2q input rows) works in place when the output family's stage
// layout equals the input's; the forward / inverse passes always use a separate
// output region, so the next item's loads need not wait for the stores to drain.
__host__ __device__ inline bool inplace_of(int mode, int in_kind, int out_kind) {
  if (mode != MODE_CONV) return false;
  const bool il_in = in_kind == TMA_LINE_TILED;
  if (out_kind == TMA_ELEM_TILED) return false;
  return il_in == (out_kind == TMA_LINE_TILED);
}

// ILK = 1: the input family is line-tiled (interleaved stage layout) at compile
// time, so every stage address is an immediate offset from a per-lane base.
// OUTK: the output stage layout at compile time (0: from the launch's TMA kinds;
// 1: in place; 2: element-tiled by 4, 3: plain rows, 4: interleaved -- separate region)
template <int MODE, int NT, int QC, int MINB = 2, int ILK = 0, int OUTK = 0>
__global__ void __launch_bounds__(NT, MINB) s128_kernel(const __grid_constant__ PassArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* done = full + 2;
  uint64_t* ofree = full + 4;
  V* t128 = reinterpret_cast<V*>(smem_raw + 128);
  V* tM1 = t128 + M;
  const int q = QC > 0 ? QC : a.q;
  const int M1 = (int)a.M1;
  V* stage0 = tM1 + m1_slots(M1);
  const int tid = threadIdx.x;
  const int nth = 32 * q;
  const int lane = tid & 31;
  const int r = tid >> 5;
  const int k_arr = blockIdx.z;
  const int kk_out = MODE == MODE_FWD ? k_arr : 0;
  const int kk_in = MODE == MODE_FWD ? k_arr : 0;
  const bool tma = a.tm_in.kind != TMA_NONE;
  const bool tma_st = tma && a.tm_out.kind != TMA_NONE;
  const bool il = ILK == 1 ? true : a.tm_in.kind == TMA_LINE_TILED;
  const bool inplace = OUTK == 1 ? true : OUTK > 1 ? false : inplace_of(MODE, a.tm_in.kind, a.tm_out.kind);
  const int IN = in_floats2(q, MODE, MODE == MODE_CONV ? a.in_g.p : 0);
  const int SB = IN + (inplace ? 0 : out_floats2(q));
  const Lay li = il ? lay_interleaved() : lay_rows(IN / C);
  const Lay lo = OUTK == 2 ? lay_elem(2) : OUTK == 3 ? lay_rows(q * M + kPad) : OUTK == 4 ? lay_interleaved()
                 : inplace ? li
                 : a.tm_out.kind == TMA_ELEM_TILED ? lay_elem(a.tm_out.slog)
                 : a.tm_out.kind == TMA_LINE_TILED ? lay_interleaved()
                                                   : lay_rows(q * M + kPad);
  const int Rg = q;  // first row of g in CONV
  {
    const V* twm = reinterpret_cast<const V*>(a.tw_m);
    const V* twM1 = reinterpret_cast<const V*>(a.tw_M1);
    for (int i = tid; i < M; i += blockDim.x) t128[i] = ldg(twm + i);
    for (int i = tid; i < M1; i += blockDim.x) tM1[i] = ldg(twM1 + i);
  }
  if (tid == 0) {
    mbar_init(&full[0], 1); mbar_init(&full[1], 1);
    mbar_init(&done[0], nth); mbar_init(&done[1], nth);
    mbar_init(&ofree[0], 1); mbar_init(&ofree[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t total = a.nbatch * a.ngroups;

  // ------------------------------------------------------------ producer warp
  if (tid >= nth) {
    if (!tma || tid != nth) return;
    auto load_item = [&](int64_t w, int s2) {
      int64_t g, b;
      split_item(w, a.nbatch, a.ngroups, a.batch_fastest, b, g);
      const int nlive = (int)(a.nlines - 4 * g < C ? a.nlines - 4 * g : C);
      V* buf = stage0 + s2 * SB;
      uint32_t bytes = item_bytes(a.tm_in, a.in_f, nlive);
      if (MODE == MODE_CONV) bytes += item_bytes(a.tm_in_g, a.in_g, nlive);
      mbar_expect_tx(&full[s2], bytes);
      load_family(a.tm_in, &a.tm_in_map[kk_in], a.in_f, kk_in, b, g, nlive, buf, li, 0, &full[s2]);
      if (MODE == MODE_CONV)
        load_family(a.tm_in_g, &a.tm_in_g_map[0], a.in_g, 0, b, g, nlive, buf, li, Rg * M, &full[s2]);
    };
    int64_t wl = blockIdx.x;
    for (int s2 = 0; s2 < 2 && wl < total; ++s2, wl += gridDim.x) load_item(wl, s2);
    int it = 0;
    for (int64_t w = blockIdx.x; w < total; w += gridDim.x, ++it) {
      const int st = it & 1;
      mbar_wait(&done[st], (uint32_t)(it >> 1) & 1u);
      if (tma_st) {
        int64_t g, b;
        split_item(w, a.nbatch, a.ngroups, a.batch_fastest, b, g);
        const int nlive = (int)(a.nlines - 4 * g < C ? a.nlines - 4 * g : C);
        V* ob = stage0 + st * SB + (inplace ? 0 : IN);
        store_tma(a, kk_out, b, g, nlive, ob, lo);
        bulk_commit();
        if (inplace) bulk_wait_read0();
      }
      if (wl < total) { load_item(wl, st); wl += gridDim.x; }
      if (tma_st && !inplace) { bulk_wait_read0(); mbar_arrive(&ofree[st]); }
    }
    if (tma_st) bulk_wait0();
    return;
  }

  // ------------------------------------------------------------ compute warps
  const int c = lane >> 3, u = lane & 7;
  int it = 0;
  for (int64_t w = blockIdx.x; w < total; w += gridDim.x, ++it) {
    const int st = it & 1;
    V* buf = stage0 + st * SB;
    V* ob = inplace ? buf : buf + IN;
    int64_t g, b;
    split_item(w, a.nbatch, a.ngroups, a.batch_fastest, b, g);
    const int nlive = (int)(a.nlines - 4 * g < C ? a.nlines - 4 * g : C);
    if (tma) {
      mbar_wait(&full[st], (uint32_t)(it >> 1) & 1u);
    } else {
      load_family_st(a.in_f, kk_in, b, g, nlive, buf, li, 0, tid, nth);
      if (MODE == MODE_CONV) load_family_st(a.in_g, 0, b, g, nlive, buf, li, Rg * M, tid, nth);
      compute_sync(nth);
    }
    // columns (c, s): c fastest for the interleaved layout (consecutive slots)
    if constexpr (MODE == MODE_INV) {
      V v[16];
      const Ex e = ex_of(li, il, r);
      load_spec(v, buf, li, c, u, r);
      fft_inv(v, buf, e, c, u, t128);
      __syncwarp();
      store_time(v, buf, li, c, u, r);
    } else {
      const int rstep = (M >> li.sl) * li.sjt;
      for (int i = tid; i < C * M; i += nth) {
        const int cc = il ? (i & 3) : (i >> 7), s = il ? (i >> 2) : (i & (M - 1));
        if constexpr (QC > 0) {
          const V w1 = tM1[s];
          fold_dispatch<QC>(buf, li.at(cc, s), rstep, (int)a.in_f.L - s, a.in_f.p, w1);
          if (MODE == MODE_CONV)
            fold_dispatch<QC>(buf, li.at(cc, Rg * M + s), rstep, (int)a.in_g.L - s, a.in_g.p, w1);
        } else {
          fold_col(buf, li, cc, s, 0, (int)a.in_f.L, a.in_f.p, q, M1, tM1);
          if (MODE == MODE_CONV) fold_col(buf, li, cc, s, Rg * M, (int)a.in_g.L, a.in_g.p, q, M1, tM1);
        }
      }
    }
    compute_sync(nth);
    const bool wait_out = tma_st && !inplace && it >= 2;
    if constexpr (MODE == MODE_FWD) {
      V v[16];
      load_time(v, buf, li, c, u, r);
      fft_fwd(v, buf, ex_of(li, il, r), c, u, t128);
      __syncwarp();
      if (wait_out) mbar_wait(&ofree[st], (uint32_t)((it >> 1) + 1) & 1u);
      store_spec(v, ob, lo, c, u, r);
    } else if constexpr (MODE == MODE_CONV) {
      V F[16], G[16];
      load_time(F, buf, li, c, u, r);
      load_time(G, buf, li, c, u, Rg + r);
      fft_fwd2(F, G, buf, ex_of(li, il, r), ex_of(li, il, Rg + r), c, u, t128);
      const float sc = (float)a.scale;
#pragma unroll
      for (int k = 0; k < 16; ++k) F[k] = cscale(cmul(F[k], G[k]), sc);
      fft_inv(F, buf, ex_of(li, il, r), c, u, t128);
      __syncwarp();
      store_time(F, buf, li, c, u, r);
    }
    if constexpr (MODE != MODE_FWD) {
      compute_sync(nth);
      if (wait_out) mbar_wait(&ofree[st], (uint32_t)((it >> 1) + 1) & 1u);
      const int T = a.out.T, Lout = (int)(a.out.L + a.out.j0);
      const int rstep = (M >> li.sl) * li.sjt, ostep = (M >> lo.sl) * lo.sjt;
      for (int i = tid; i < C * M; i += nth) {
        const int cc = il ? (i & 3) : (i >> 7), s = il ? (i >> 2) : (i & (M - 1));
        if constexpr (QC > 0)
          unfold_colq<QC>(buf, li.at(cc, s), rstep, ob, lo.at(cc, s), ostep, T, Lout - s, tM1[s]);
        else
          unfold_col(buf, li, ob, lo, cc, s, q, T, Lout, M1, tM1);
      }
    }
    if (tma_st) {
      fence_async_smem();
      mbar_arrive(&done[st]);
    } else {
      compute_sync(nth);
      store_st(a, kk_out, b, g, nlive, ob, lo, tid, nth);
      if (tma) { fence_async_smem(); mbar_arrive(&done[st]); }
      else compute_sync(nth);
    }
  }
}

// ---------------------------------------------------------------------------
// Batch-grouped forward pass (BG = 4): one work item = four consecutive batch
// entries b = 4 b4 + k of one group of four tiled lines, i.e. 16 lines, for the
// y -> z transpose of the 3-D pipeline (fwd_y: batch = z with stride 4 elements =
// the line tile), where four batch entries x four lines of one output element are
// 128 contiguous bytes.  Loads: TMA tensor boxes per sub-item (as s128_kernel);
// transform in place per sub-item (warp (k, r): residue r of sub-item k); stores:
// plain 16-byte stores from every thread, eight threads per 128-byte piece
// (tools/micro/scatter32.cu: 128-byte pieces at 5.0 TB/s vs 1.1 TB/s for the 32-byte
// pieces of one 4-line item).  Host conditions: hd_api.cu use_s128_bg.
// ---------------------------------------------------------------------------
constexpr int kBG = 4;
__host__ __device__ inline size_t bg_smem_bytes(int q, int M1) {
  return 128 + sizeof(float2) * (size_t)(M + m1_slots(M1) + 2 * kBG * in_floats2(q, MODE_FWD));
}

template <int QC>
__global__ void __launch_bounds__(32 * (kBG * QC + 1), 1) s128_bg_fwd_kernel(const __grid_constant__ PassArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* done = full + 2;
  V* t128 = reinterpret_cast<V*>(smem_raw + 128);
  V* tM1 = t128 + M;
  constexpr int q = QC;
  const int M1 = (int)a.M1;
  V* stage0 = tM1 + m1_slots(M1);
  const int tid = threadIdx.x;
  constexpr int nth1 = 32 * q, nth = kBG * nth1;
  const int lane = tid & 31;
  const int wi = tid >> 5;
  const int k = wi / q, r = wi - k * q;  // sub-item, residue (compute warps)
  const int k_arr = blockIdx.z;
  const int IN = in_floats2(q, MODE_FWD);
  const int SB = kBG * IN;
  const Lay li = lay_interleaved();
  for (int i = tid; i < M; i += blockDim.x) t128[i] = ldg(reinterpret_cast<const V*>(a.tw_m) + i);
  for (int i = tid; i < M1; i += blockDim.x) tM1[i] = ldg(reinterpret_cast<const V*>(a.tw_M1) + i);
  if (tid == 0) {
    mbar_init(&full[0], 1); mbar_init(&full[1], 1);
    mbar_init(&done[0], nth); mbar_init(&done[1], nth);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nb4 = a.nbatch / kBG;
  const int64_t total = nb4 * a.ngroups;

  if (tid >= nth) {  // producer
    if (tid != nth) return;
    auto load_item = [&](int64_t w, int s2) {
      int64_t g, b4;
      split_item(w, nb4, a.ngroups, 1, b4, g);
      const int nlive = (int)(a.nlines - 4 * g < C ? a.nlines - 4 * g : C);
      V* buf = stage0 + s2 * SB;
      mbar_expect_tx(&full[s2], kBG * item_bytes(a.tm_in, a.in_f, nlive));
      for (int kk = 0; kk < kBG; ++kk)
        load_family(a.tm_in, &a.tm_in_map[k_arr], a.in_f, k_arr, 4 * b4 + kk, g, nlive, buf + kk * IN, li, 0,
                    &full[s2]);
    };
    int64_t wl = blockIdx.x;
    for (int s2 = 0; s2 < 2 && wl < total; ++s2, wl += gridDim.x) load_item(wl, s2);
    int it = 0;
    for (int64_t w = blockIdx.x; w < total; w += gridDim.x, ++it) {
      const int st = it & 1;
      mbar_wait(&done[st], (uint32_t)(it >> 1) & 1u);
      if (wl < total) { load_item(wl, st); wl += gridDim.x; }
    }
    return;
  }

  const int c = lane >> 3, u = lane & 7;
  const int tl = tid - k * nth1;
  const LineOut& o = a.out;
  const int Lout = (int)o.L;
  int it = 0;
  for (int64_t w = blockIdx.x; w < total; w += gridDim.x, ++it) {
    const int st = it & 1;
    V* buf = stage0 + st * SB;
    V* bk = buf + k * IN;
    int64_t g, b4;
    split_item(w, nb4, a.ngroups, 1, b4, g);
    const int nlive = (int)(a.nlines - 4 * g < C ? a.nlines - 4 * g : C);
    mbar_wait(&full[st], (uint32_t)(it >> 1) & 1u);
    {
      const int rstep = (M >> li.sl) * li.sjt;
      for (int i = tl; i < C * M; i += nth1) {
        const int cc = i & 3, s = i >> 2;
        fold_dispatch<QC>(bk, li.at(cc, s), rstep, (int)a.in_f.L - s, a.in_f.p, tM1[s]);
      }
    }
    compute_sync(nth);
    {
      V v[16];
      load_time(v, bk, li, c, u, r);
      fft_fwd(v, bk, ex_of(li, true, r), c, u, t128);
      __syncwarp();
      store_spec(v, bk, li, c, u, r);
    }
    compute_sync(nth);
    // 16-byte stores: thread i -> element j = i >> 3, sub-item (i >> 1) & 3, line pair i & 1
    V* y = reinterpret_cast<V*>(o.ptr[k_arr]);
    const int64_t l0 = 4 * g;
    for (int i = tid; i < Lout * 8; i += nth) {
      const int j = i >> 3, kk = (i >> 1) & 3, cp = i & 1;
      const V* src = buf + kk * IN + li.at(2 * cp, j);
      V* dst = y + boff(4 * b4 + kk, o.nbi, o.s_bo, o.s_b) + line_off(o, l0 + 2 * cp) + (int64_t)j * o.s_js;
      if (2 * cp + 1 < nlive) {
        *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(src);
      } else if (2 * cp < nlive) {
        *dst = *src;
      }
    }
    fence_async_smem();
    mbar_arrive(&done[st]);
  }
}

}  // namespace s128
}  // namespace hd
