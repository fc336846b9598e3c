// hd_s512.cuh -- staged warp engine for FFT size m = 512 (complex double).
//
// One persistent CTA per SM, one line per work item, q compute warps (warp r owns
// residue r) plus one producer warp that issues every TMA copy and bulk wait, so
// compute warps never stall on copy issue (blockDim = 32 (q + 1), q <= 11).  Lines move between HBM and a two-stage shared
// memory ring by TMA: strided / tiled lines as 5-D tensor boxes of 256 elements
// (cp.async.bulk.tensor, zero fill past the line end), plain rows as one 1-D bulk
// copy; loads complete on an mbarrier, stores are bulk-async groups.  The next
// item's loads are issued once the current item's first step is done, so they
// overlap its FFTs and unfold.  Every step works in place on the stage:
//
//   stage [t][s] = x[t m + s]        (TMA load, rows t < p; the rest unread)
//   fold     thread s:  w_r[s] = zeta_{qm}^{rs} sum_{t<p} zeta_q^{rt} x[tm+s]
//            (Forward Eq. PAPER.md:528; Alg. Forward)   -> row r
//   FFT      warp r: size-512 FFT of row r in registers (hd_w512.cuh)
//   FWD      spectrum -> row r in lane-major order (position k2*32 + lane holds
//            frequency freq_of(lane, k2)) -> TMA store of the line
//   CONV     G's transform (short input, p_g = 1), product (1/prod M1) F G
//            (PAPER.md:190-192), inverse FFT in registers -> row r
//   INV      row r (lane-major spectrum) -> inverse FFT -> row r
//   unfold   thread s: h[tm+s] = sum_r zeta_q^{-tr} zeta_{qm}^{-rs} V_r[s], t < T
//            (Backward Eq. PAPER.md:531; Alg. Backward) -> stage
//            [t][s] in place -> TMA store of the output line
//
// The lane-major spectral order is internal to the x (and 3-D y) passes of one
// axis; hd_api.cu runs every pass of an axis on the same engine.
#pragma once
#include <cuda.h>

#include "hd_internal.h"
#include "hd_tma.cuh"
#include "hd_w512.cuh"
#include "hd_w256.cuh"
#include "hd_zq_table.h"

namespace hd {
namespace s512 {

using V = double2;
constexpr int M = 512;
constexpr int kQMax = kS512QMax;  // q + 1 warps at <= 3 per SM sub-partition (168 registers)
constexpr int kBox = 256;         // elements per TMA box

// per-thread fallback for layouts TMA cannot express (general element tiling)
__device__ __forceinline__ void cp16(V* dst, const V* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Debug phase timing (library built with NVCC_APPEND_FLAGS=-DHD_PHASE_PROF_BUILD and
// run with HD_PHASE_PROF=1): lane 0 of every warp accumulates SM clock cycles per
// phase and adds them to a.phase_prof at exit.  Compiled out otherwise (the
// disabled probes cost ~2 % of the convolution pass's instructions).
constexpr int kPhases = 8;
#ifdef HD_PHASE_PROF_BUILD
constexpr bool kPhaseProf = true;
#else
constexpr bool kPhaseProf = false;
#endif
struct PhaseClock {
  unsigned long long acc[kPhases];
  long long t0;
  bool on;
  __device__ __forceinline__ void start(bool enable) {
    on = kPhaseProf && enable;
#pragma unroll
    for (int i = 0; i < kPhases; ++i) acc[i] = 0;
    if (on) t0 = clock64();
  }
  __device__ __forceinline__ void mark(int ph) {
    if (on) { const long long t = clock64(); acc[ph] += (unsigned long long)(t - t0); t0 = t; }
  }
  __device__ __forceinline__ void flush(unsigned long long* out) {
    if (on && (threadIdx.x & 31) == 0) {
#pragma unroll
      for (int i = 0; i < kPhases; ++i) atomicAdd(out + i, acc[i]);
      // per warp: every phase
#pragma unroll
      for (int i = 0; i < kPhases; ++i) atomicAdd(out + kPhases * (1 + (threadIdx.x >> 5)) + i, acc[i]);
    }
  }
};

// ---------------------------------------------------------------------------
// Loads of one work item: in_f line (+ in_g line in CONV) -> stage slot j = element j
// ---------------------------------------------------------------------------
// Loads of one work item in the slot range [j0, j1) of the in_f line (the whole
// short line g in CONV goes with the first range: it lands beyond the output slots).
// issue_loads_arm sets the mbarrier's byte count for the whole item first.
// real-pair input (a.rp): the re row at the stage start, the im row from double rp_im_slot
__device__ __forceinline__ int rp_im_slot(const PassArgs& a) { return (int)((a.in_f.L + 1) / 2 * 2); }

template <int MODE>
__device__ __forceinline__ void issue_loads_arm(const PassArgs& a, int64_t g, uint64_t* bar) {
  uint32_t bytes = 0;
  if (MODE == MODE_FWD && a.rp) {
    if (g < a.nlines) bytes = (uint32_t)a.in_f.L * 8u * (g < a.rp_rows ? 2u : 1u);
    mbar_expect_tx(bar, bytes);
    return;
  }
  if (g < a.nlines) {
    const int L = (int)a.in_f.L;
    bytes += a.tm_in.kind == TMA_BULK    ? (uint32_t)L * 16u
             : a.tm_in.kind == TMA_ELEM2 ? (uint32_t)L * 16u  // boxes tile [0, L) exactly
                                         : (uint32_t)((L + kBox - 1) / kBox) * kBox * 16u;
    if (MODE == MODE_CONV)
      bytes += a.tm_in_g.kind == TMA_BULK ? (uint32_t)a.in_g.L * 16u
                                           : (uint32_t)((a.in_g.L + kBox - 1) / kBox) * kBox * 16u;
  }
  mbar_expect_tx(bar, bytes);
}

template <int MODE>
__device__ __forceinline__ void issue_loads_range(const PassArgs& a, int k_arr, int64_t b, int64_t g, V* buf,
                                                  uint64_t* bar, int j0, int j1) {
  if (g >= a.nlines) return;
  const LineIn& in = a.in_f;
  const int L = (int)in.L;
  if (MODE == MODE_FWD && a.rp) {  // both real rows with the first range
    if (j0 != 0) return;
    const double* re = reinterpret_cast<const double*>(in.ptr[0]) + line_off(in, g);
    double* sb = reinterpret_cast<double*>(buf);
    bulk_load(sb, re, (uint32_t)L * 8u, bar);
    if (g < a.rp_rows) bulk_load(sb + rp_im_slot(a), re + a.rp_off, (uint32_t)L * 8u, bar);
    return;
  }
  j1 = j1 < L ? j1 : L;
  const int kk = MODE == MODE_FWD ? k_arr : 0;
  if (j0 < j1) {
    if (a.tm_in.kind == TMA_BULK) {
      const V* x = reinterpret_cast<const V*>(in.ptr[kk]) + boff(b, in.nbi, in.s_bo, in.s_b) + line_off(in, g);
      bulk_load(buf + j0, x + j0, (uint32_t)(j1 - j0) * 16u, bar);
    } else {
      const CUtensorMap* map = &a.tm_in_map[kk];
      const int step = a.tm_in.kind == TMA_ELEM2 ? a.tm_in.box : kBox;  // ELEM2: one range only
      int c[5];
      for (int jb = j0; jb < j1; jb += step) {
        tma_coords(a.tm_in, b, g, jb, c);
        tma_load(buf + jb, map, c, bar);
      }
    }
  }
  if (MODE == MODE_CONV && j0 == 0) {
    const LineIn& ig = a.in_g;
    if (a.tm_in_g.kind == TMA_BULK) {
      const V* xg = reinterpret_cast<const V*>(ig.ptr[0]) + boff(b, ig.nbi, ig.s_bo, ig.s_b) + line_off(ig, g);
      bulk_load(buf + a.q * M, xg, (uint32_t)ig.L * 16u, bar);
    } else {
      int c[5];
      for (int jb = 0; jb < (int)ig.L; jb += kBox) {
        tma_coords(a.tm_in_g, b, g, jb, c);
        tma_load(buf + a.q * M + jb, &a.tm_in_g_map[0], c, bar);
      }
    }
  }
}

template <int MODE>
__device__ __forceinline__ void issue_loads_tma(const PassArgs& a, int k_arr, int64_t b, int64_t g, V* buf,
                                                uint64_t* bar) {
  issue_loads_arm<MODE>(a, g, bar);
  issue_loads_range<MODE>(a, k_arr, b, g, buf, bar, 0, 1 << 30);
}

// L2 prefetch of a contiguous input line one item further ahead than the loads
// (tensor-map lines are not prefetched: the strided prefetch competes with the
// loads for the TMA unit and measured slower)
template <int MODE>
__device__ __forceinline__ void issue_prefetch(const PassArgs& a, int k_arr, int64_t b, int64_t g) {
  if (g >= a.nlines || a.tm_in.kind != TMA_BULK || (MODE == MODE_FWD && a.rp)) return;
  const LineIn& in = a.in_f;
  const int kk = MODE == MODE_FWD ? k_arr : 0;
  bulk_prefetch_l2(reinterpret_cast<const V*>(in.ptr[kk]) + boff(b, in.nbi, in.s_bo, in.s_b) + line_off(in, g),
                   (uint32_t)in.L * 16u);
}

template <int MODE>
__device__ __forceinline__ void issue_loads_cp(const PassArgs& a, int k_arr, int64_t b, int64_t g, V* buf,
                                               int tid, int nth) {
  if (g < a.nlines) {
    const LineIn& in = a.in_f;
    const V* x = reinterpret_cast<const V*>(in.ptr[MODE == MODE_FWD ? k_arr : 0]) +
                 boff(b, in.nbi, in.s_bo, in.s_b) + line_off(in, g);
    for (int j = tid; j < (int)in.L; j += nth) cp16(buf + j, x + in_el(in, j));
    if constexpr (MODE == MODE_CONV) {
      const LineIn& ig = a.in_g;
      const V* xg = reinterpret_cast<const V*>(ig.ptr[0]) + boff(b, ig.nbi, ig.s_bo, ig.s_b) + line_off(ig, g);
      for (int j = tid; j < (int)ig.L; j += nth) cp16(buf + a.q * M + j, xg + in_el(ig, j));
    }
  }
  cp_commit();
}

// ---------------------------------------------------------------------------
// Stores of one work item: stage slots j < out.L -> output line
// ---------------------------------------------------------------------------
// Stores of the output positions [p0, p1) (stage slots p + out.j0: the output
// window) as one bulk-async group.  Tensor boxes start at 8-aligned slots (128-byte
// shared-memory alignment); positions before the window are clipped by TMA.
__device__ __forceinline__ void issue_stores_range_o(const LineOut& o, const TmaLine& tmo, const CUtensorMap* map,
                                                     int kk, int64_t b, int64_t g, const V* buf, int p0, int p1) {
  const int L = (int)o.L;
  const int j0 = (int)o.j0;
  p1 = p1 < L ? p1 : L;
  if (p0 < p1) {
    if (tmo.kind == TMA_BULK) {
      V* y = reinterpret_cast<V*>(o.ptr[kk]) + boff(b, o.nbi, o.s_bo, o.s_b) + line_off(o, g);
      bulk_store(y + p0, buf + j0 + p0, (uint32_t)(p1 - p0) * 16u);
    } else {
      // boxes start at 8-aligned slots: positions p0 - sh + 256 k (the first group's
      // head before the first aligned slot goes by plain stores; later groups rewrite
      // sh positions of the group before with the same values).  Element-tiled lines with a window
      // go through per-thread stores instead (hd_api.cu prepare_tma).
      const int sh = j0 & 7;
      int pb = p0 - sh;
      if (pb < 0) {  // positions before the first 8-aligned slot: plain stores
        V* yl = reinterpret_cast<V*>(o.ptr[kk]) + boff(b, o.nbi, o.s_bo, o.s_b) + line_off(o, g);
        const int hp = (8 - sh) < p1 ? (8 - sh) : p1;
        for (int p = 0; p < hp; ++p) yl[jt_off(p, out_sl(o), o.s_jt, o.s_js)] = buf[j0 + p];
        pb += 8;
      }
      int c[5];
      for (; pb < p1; pb += kBox) {
        tma_coords(tmo, b, g, pb, c);
        tma_store(map, c, buf + j0 + pb);
      }
    }
  }
  bulk_commit();
}
__device__ __forceinline__ void issue_stores_range(const PassArgs& a, int kk, int64_t b, int64_t g, const V* buf,
                                                   int p0, int p1) {
  issue_stores_range_o(a.out, a.tm_out, &a.tm_out_map[kk], kk, b, g, buf, p0, p1);
}

__device__ __forceinline__ void issue_stores_tma(const PassArgs& a, int kk, int64_t b, int64_t g, const V* buf) {
  issue_stores_range(a, kk, b, g, buf, 0, 1 << 30);
}

template <int N> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_read_n(int n) {
  if (n >= 3) bulk_wait_read<3>();
  else if (n == 2) bulk_wait_read<2>();
  else if (n == 1) bulk_wait_read<1>();
  else bulk_wait_read<0>();
}

// The producer's hand-over of one stage: the stores of the finished item go out in
// kGroups slot ranges (bulk groups, in order), and the next item's loads into the
// same stage follow range by range, each waiting only until the store groups that
// overlap its slots have been read out of shared memory.
constexpr int kGroups = 4;
constexpr int T9SLOTS = 9 * M;  // real split: the Im array starts at double 9 m of the stage
// second-family (a.fam2) item: the stores of line gs of out2, the bulk load of line
// gl of in_g (whole, after every store group has been read)
__device__ __forceinline__ void handover_fam2(const PassArgs& a, bool store, int st_fam, int64_t gs, bool load,
                                              int ld_fam, int64_t gl, V* buf, uint64_t* bar) {
  store = store && !(a.dbg & 1);
  if (load && (a.dbg & 2)) { mbar_expect_tx(bar, 0); load = false; }
  if (store) {
    if (st_fam == 2) issue_stores_range_o(a.out2, a.tm_out2, &a.tm_out_map[1], 1, 0, gs, buf, 0, 1 << 30);
    else issue_stores_range(a, 0, 0, gs, buf, 0, 1 << 30);
  }
  if (!load) return;
  if (ld_fam == 1) {  // the first family as in any forward pass (plain rows or real pairs)
    issue_loads_arm<MODE_FWD>(a, gl, bar);
    if (store) bulk_wait_read_n(0);
    issue_loads_range<MODE_FWD>(a, 0, 0, gl, buf, bar, 0, 1 << 30);
    return;
  }
  const LineIn& in = a.in_g;
  mbar_expect_tx(bar, (uint32_t)in.L * 16u);
  if (store) bulk_wait_read_n(0);
  bulk_load(buf, reinterpret_cast<const V*>(in.ptr[0]) + line_off(in, gl), (uint32_t)in.L * 16u, bar);
}

template <int MODE>
__device__ __forceinline__ void handover(const PassArgs& a, int k_arr, int kk_out, bool store, int64_t bs,
                                         int64_t gs, bool load, int64_t bl, int64_t gl, V* buf, uint64_t* bar) {
  store = store && !(a.dbg & 1);
  if (load && (a.dbg & 2)) gl = a.nlines;  // an empty item: the barrier completes at once
  if ((MODE == MODE_INV && a.rs) || (MODE == MODE_FWD && a.rp)) {
    if (store) {
      if (MODE == MODE_INV && a.rs) {  // Re row and Im row of the output line (real split)
        const LineOut& o = a.out;
        const uint32_t nb = (uint32_t)o.L * 8u;
        const double* sb = reinterpret_cast<const double*>(buf);
        double* h = reinterpret_cast<double*>(o.ptr[0]);
        bulk_store(h + gs * o.s_l, sb, nb);
        const int64_t yi = gs + a.rs_A;
        if (gs < a.rs_side_rows) bulk_store(reinterpret_cast<double*>(a.rs_side) + gs * o.s_l, sb + T9SLOTS, nb);
        else if (yi < a.rs_rows) bulk_store(h + yi * o.s_l, sb + T9SLOTS, nb);
        bulk_commit();
      } else {
        issue_stores_range(a, kk_out, bs, gs, buf, 0, 1 << 30);
      }
    }
    if (!load) return;
    issue_loads_arm<MODE>(a, gl, bar);
    if (store) bulk_wait_read_n(0);
    issue_loads_range<MODE>(a, k_arr, bl, gl, buf, bar, 0, 1 << 30);
    return;
  }
  if (a.tm_in.kind == TMA_ELEM2) {  // boxes of jd-tiled lines: every store read out, then one load range
    if (store) issue_stores_range(a, kk_out, bs, gs, buf, 0, 1 << 30);
    if (!load) return;
    issue_loads_arm<MODE>(a, gl, bar);
    if (store) bulk_wait_read_n(0);
    issue_loads_range<MODE>(a, k_arr, bl, gl, buf, bar, 0, 1 << 30);
    return;
  }
  const int Ls = store ? (int)a.out.L : 0;
  const int Ll = load ? (int)a.in_f.L : 0;
  const int Lmax = Ls > Ll ? Ls : Ll;
  const int chunk = ((Lmax + kGroups - 1) / kGroups + kBox - 1) / kBox * kBox;
  if (store)
    for (int k = 0; k < kGroups; ++k) issue_stores_range(a, kk_out, bs, gs, buf, k * chunk, (k + 1) * chunk);
  if (!load) return;
  issue_loads_arm<MODE>(a, gl, bar);
  for (int k = 0; k < kGroups; ++k) {
    if (store) bulk_wait_read_n(kGroups - 1 - k);
    issue_loads_range<MODE>(a, k_arr, bl, gl, buf, bar, k * chunk, k == kGroups - 1 ? (1 << 30) : (k + 1) * chunk);
  }
}

__device__ __forceinline__ void stores_st(const PassArgs& a, int kk, int64_t b, int64_t g, const V* buf,
                                          int tid, int nth) {
  const LineOut& o = a.out;
  V* y = reinterpret_cast<V*>(o.ptr[kk]) + boff(b, o.nbi, o.s_bo, o.s_b) + line_off(o, g);
  const int sl = out_sl(o);
  for (int j = tid; j < (int)o.L; j += nth) y[jt_off(j, sl, o.s_jt, o.s_js)] = buf[j + o.j0];
}

// ---------------------------------------------------------------------------
// zeta_q^{rt}: compile-time q (QC > 0) from the constant table (constant-bank
// operands), else the SMEM table zt[r*16 + t] = zeta_q^{(r t) mod q}
// ---------------------------------------------------------------------------
template <int QC>
__device__ __forceinline__ V zq_rt(const V* zt, int r, int t) {
  if constexpr (QC > 0) return c_zq[QC][(r * t) % QC];
  else return zt[r * kQF + t];
}

// q = 9 codelets: the 9-point DFT y_r = sum_t zeta_9^{S r t} x_t as 3 x 3
// (t = 3 t1 + t2, r = r1 + 3 r2: radix-3 over t1, twiddle zeta_9^{S r1 t2},
// radix-3 over t2), 88 FP64 operations instead of the pair form's ~150.
template <int S> __device__ __forceinline__ void dft3(V& x0, V& x1, V& x2) {
  constexpr double h = 0.86602540378443864676;  // sin(2 pi / 3)
  const V sm = cadd(x1, x2), df = csub(x1, x2);
  const V mid = cmk<V>(fma(-0.5, sm.x, x0.x), fma(-0.5, sm.y, x0.y));
  x0 = cadd(x0, sm);
  // x1 = mid + S i h df, x2 = mid - S i h df
  x1 = cmk<V>(fma(-S * h, df.y, mid.x), fma(S * h, df.x, mid.y));
  x2 = cmk<V>(fma(S * h, df.y, mid.x), fma(-S * h, df.x, mid.y));
}
template <int S> __device__ __forceinline__ void dft9(V* x) {
  dft3<S>(x[0], x[3], x[6]);
  dft3<S>(x[1], x[4], x[7]);
  dft3<S>(x[2], x[5], x[8]);
  // twiddles zeta_9^{S r1 t2}: (r1, t2) = (1,1): 1, (2,1): 2, (1,2): 2, (2,2): 4
  const V z1 = c_zq[9][1], z2 = c_zq[9][2], z4 = c_zq[9][4];
  x[4] = S > 0 ? cmul(x[4], z1) : cmulc(x[4], z1);
  x[7] = S > 0 ? cmul(x[7], z2) : cmulc(x[7], z2);
  x[5] = S > 0 ? cmul(x[5], z2) : cmulc(x[5], z2);
  x[8] = S > 0 ? cmul(x[8], z4) : cmulc(x[8], z4);
  // radix-3 over t2 for each r1: inputs (x[3 r1'...]) -- element (r1, t2) sits at 3 t2' ...
  dft3<S>(x[0], x[1], x[2]);  // r1 = 0 -> y_0, y_3, y_6
  dft3<S>(x[3], x[4], x[5]);  // r1 = 1 -> y_1, y_4, y_7
  dft3<S>(x[6], x[7], x[8]);  // r1 = 2 -> y_2, y_5, y_8
}
// After dft9, x[3 r1 + r2] holds y_{r1 + 3 r2}.
__device__ __forceinline__ int dft9_slot(int r) { return 3 * (r % 3) + r / 3; }

// NC columns per call (NC = 2: two independent columns interleaved for ILP)
template <int P, int NC>
__device__ __forceinline__ void fold_col9(V* buf, const int* s, const int* rem, const V* w1) {
  V x[NC][9];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int t = 0; t < 9; ++t) x[c][t] = (t < P && t * M < rem[c]) ? buf[t * M + s[c]] : cmk<V>(0, 0);
#pragma unroll
  for (int c = 0; c < NC; ++c) dft9<+1>(x[c]);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    buf[s[c]] = x[c][0];
    // twiddles zeta_{M1}^{r s}: two interleaved recurrences (odd / even r)
    const V w2 = cmul(w1[c], w1[c]);
    V wo = w1[c], we = w2;
#pragma unroll
    for (int r = 1; r < 9; ++r) {
      const V y = x[c][dft9_slot(r)];
      if (r & 1) { buf[r * M + s[c]] = cmul(y, wo); wo = cmul(wo, w2); }
      else { buf[r * M + s[c]] = cmul(y, we); we = cmul(we, w2); }
    }
  }
}

// fold_col9 for the real-pair input (a.rp): x[t m + s] = (re[t m + s], im[t m + s]) from
// the two real rows at the stage start; every compute thread joins the barrier that
// separates the loads (columns of other threads) from the in-place residue stores.
template <int P>
__device__ __forceinline__ void fold9_rp(V* buf, int L, bool live, bool im_ok, int im_slot, const V* twcol,
                                         int tid, int nth) {
  constexpr int NC = 2;
  const bool act = tid < M / 2;
  const int s[NC] = {tid, tid + M / 2};
  V x[NC][9];
  const double* re = reinterpret_cast<const double*>(buf);
  const double* im = re + im_slot;
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      const bool ok = act && live && t < P && t * M + s[c] < L;
      x[c][t] = cmk<V>(ok ? re[t * M + s[c]] : 0.0, (ok && im_ok) ? im[t * M + s[c]] : 0.0);
    }
  compute_sync(nth);
  if (!act) return;
#pragma unroll
  for (int c = 0; c < NC; ++c) dft9<+1>(x[c]);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const V w1 = twcol[s[c]];
    buf[s[c]] = x[c][0];
    const V w2 = cmul(w1, w1);
    V wo = w1, we = w2;
#pragma unroll
    for (int r = 1; r < 9; ++r) {
      const V y = x[c][dft9_slot(r)];
      if (r & 1) { buf[r * M + s[c]] = cmul(y, wo); wo = cmul(wo, w2); }
      else { buf[r * M + s[c]] = cmul(y, we); we = cmul(we, w2); }
    }
  }
}

// unfold_col9 with the real-split output (a.rs): Re of h[t m + s] -> double t m + s of
// the stage, Im -> double T9SLOTS + t m + s, after a barrier (the doubles overlap
// other columns' residues)
template <bool SPLIT8 = false>  // row 8 as two halves (see unfold_col9)
__device__ __forceinline__ void unfold9_rs(V* buf, int T, const V* twcol, int tid, int nth) {
  constexpr int NC = 2;
  const bool act = tid < M / 2;
  const int s[NC] = {tid, tid + M / 2};
  V x[NC][9];
  if (act) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const V w1 = twcol[s[c]];
      x[c][0] = buf[s[c]];
      const V w2 = cmul(w1, w1);
      V wo = w1, we = w2;
#pragma unroll
      for (int r = 1; r < 9; ++r) {
        V y = buf[r * M + s[c]];
        if (SPLIT8 && r == 8) {
          const V lo = buf[8 * M + tid], hi = buf[8 * M + 256 + tid];
          y = c == 0 ? cadd(lo, hi) : csub(lo, hi);
        }
        if (r & 1) { x[c][r] = cmulc(y, wo); wo = cmul(wo, w2); }
        else { x[c][r] = cmulc(y, we); we = cmul(we, w2); }
      }
    }
  }
  compute_sync(nth);
  if (!act) return;
  double* dre = reinterpret_cast<double*>(buf);
  double* dim = dre + T9SLOTS;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    dft9<-1>(x[c]);
#pragma unroll
    for (int t = 0; t < 9; ++t)
      if (t < T) {
        const V v = x[c][dft9_slot(t)];
        dre[t * M + s[c]] = v.x;
        dim[t * M + s[c]] = v.y;
      }
  }
}

// SPLIT8: row 8 holds residue 8's inverse as two halves a (slots [0, 256)) and
// zeta_512^{-n} b (slots [256, 512)) of the last radix-2 step; V_8[n] = a +- zeta^{-n} b
// is formed here (columns s and s + 256 of one thread: NC = 2, s = {t, t + 256}).
template <int NC, bool SPLIT8 = false>
__device__ __forceinline__ void unfold_col9(V* buf, const int* s, int T, const V* w1) {
  V x[NC][9];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    x[c][0] = buf[s[c]];
    const V w2 = cmul(w1[c], w1[c]);
    V wo = w1[c], we = w2;
#pragma unroll
    for (int r = 1; r < 9; ++r) {
      V y = buf[r * M + s[c]];
      if (SPLIT8 && r == 8) {
        const V lo = buf[8 * M + (s[c] & 255)], hi = buf[8 * M + 256 + (s[c] & 255)];
        y = s[c] < 256 ? cadd(lo, hi) : csub(lo, hi);
      }
      if (r & 1) { x[c][r] = cmulc(y, wo); wo = cmul(wo, w2); }
      else { x[c][r] = cmulc(y, we); we = cmul(we, w2); }
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) dft9<-1>(x[c]);
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int t = 0; t < 9; ++t)
      if (t < T) buf[t * M + s[c]] = x[c][dft9_slot(t)];
}

// In-place fold of column s: rows t < p hold x[t m + s] (beyond the line: zero
// by predicate), rows r < q receive w_r[s].  The q-point DFT over t is evaluated
// in symmetric pairs (a_r, a_{q-r} share all real products).
template <int QC, int P>
__device__ __forceinline__ void fold_col(V* buf, int s, int rem, int qrt, const V* zt, V w1, V wq) {
  const int q = QC > 0 ? QC : qrt;
  V u[P];
#pragma unroll
  for (int t = 0; t < P; ++t) u[t] = (t * M < rem) ? buf[t * M + s] : cmk<V>(0, 0);
  V a0 = u[0];
#pragma unroll
  for (int t = 1; t < P; ++t) a0 = cadd(a0, u[t]);
  buf[s] = a0;
  V wr = w1;
#pragma unroll
  for (int r = 1; r <= kQMax / 2; ++r) {
    if (2 * r > q) break;
    V A = u[0], B = cmk<V>(0, 0);
#pragma unroll
    for (int t = 1; t < P; ++t) {
      const V z = zq_rt<QC>(zt, r, t);  // zeta_q^{r t}
      A.x = fma(u[t].x, z.x, A.x); A.y = fma(u[t].y, z.x, A.y);
      B.x = fma(u[t].x, z.y, B.x); B.y = fma(u[t].y, z.y, B.y);
    }
    buf[r * M + s] = cmul(cmk<V>(A.x - B.y, A.y + B.x), wr);  // a_r zeta^{rs}
    if (2 * r < q) buf[(q - r) * M + s] = cmul(cmk<V>(A.x + B.y, A.y - B.x), cmulc(wq, wr));
    wr = cmul(wr, w1);
  }
}

template <int QC>
__device__ __forceinline__ void fold_all(V* buf, int p, int L, bool live, int q, const V* zt, const V* twm,
                                         const V* twcol, int tid, int nth) {
  if constexpr (QC == 9) {
    // threads < 256 take columns s and s + 256 together (nth >= 256)
    if (tid < M / 2) {
      const int sc[2] = {tid, tid + M / 2};
      const int rm[2] = {live ? L - sc[0] : 0, live ? L - sc[1] : 0};
      const V w1[2] = {twcol[sc[0]], twcol[sc[1]]};
      if (p <= 4) fold_col9<4, 2>(buf, sc, rm, w1);
      else fold_col9<8, 2>(buf, sc, rm, w1);
    }
  } else {
    for (int s = tid; s < M; s += nth) {
      const int rem = live ? L - s : 0;
      const V w1 = twcol[s], wq = ldg(twm + s);
      if (p <= 1) fold_col<QC, 1>(buf, s, rem, q, zt, w1, wq);
      else if (p <= 2) fold_col<QC, 2>(buf, s, rem, q, zt, w1, wq);
      else if (p <= 4) fold_col<QC, 4>(buf, s, rem, q, zt, w1, wq);
      else fold_col<QC, 8>(buf, s, rem, q, zt, w1, wq);
    }
  }
}

// q = 9 fold of one item by the 6 warps that do not share the SM sub-partition of
// warps 0, 4, 8 (warp w runs on sub-partition (w + c) mod 4, so warps 0, 4, 8 always
// share one and carry 3 of the 9 residues there): light thread lt < 192 folds the
// columns lt, lt + 192 and (lt < 128) lt + 384.
__device__ __forceinline__ void fold9_light(V* buf, int p, int L, bool live, const V* twcol, int lt) {
  if (lt < 128) {
    const int sc[3] = {lt, lt + 192, lt + 384};
    const int rm[3] = {live ? L - sc[0] : 0, live ? L - sc[1] : 0, live ? L - sc[2] : 0};
    const V w1[3] = {twcol[sc[0]], twcol[sc[1]], twcol[sc[2]]};
    if (p <= 4) fold_col9<4, 3>(buf, sc, rm, w1);
    else fold_col9<8, 3>(buf, sc, rm, w1);
  } else {
    const int sc[2] = {lt, lt + 192};
    const int rm[2] = {live ? L - sc[0] : 0, live ? L - sc[1] : 0};
    const V w1[2] = {twcol[sc[0]], twcol[sc[1]]};
    if (p <= 4) fold_col9<4, 2>(buf, sc, rm, w1);
    else fold_col9<8, 2>(buf, sc, rm, w1);
  }
}

// In-place unfold of column s: rows r < q hold V_r[s]; rows t < T receive
// h[tm+s] = sum_r zeta_q^{-tr} conj(zeta_{M1}^{rs}) V_r[s], in pairs (t, q-t).
template <int QC, int QM>
__device__ __forceinline__ void unfold_col(V* buf, int s, int qrt, int T, const V* zt, V w1) {
  const int q = QC > 0 ? QC : qrt;
  V v[QM];
  v[0] = buf[s];
  {
    // conj twiddles zeta_{M1}^{-rs}: odd and even r by two interleaved recurrences
    const V w2 = cmul(w1, w1);
    V we = w2, wo = w1;
#pragma unroll
    for (int r = 1; r < QM; ++r) {
      v[r] = cmk<V>(0, 0);
      if (r < q) {
        if (r & 1) { v[r] = cmulc(buf[r * M + s], wo); wo = cmul(wo, w2); }
        else { v[r] = cmulc(buf[r * M + s], we); we = cmul(we, w2); }
      }
    }
  }
  V h0 = v[0];
#pragma unroll
  for (int r = 1; r < QM; ++r) h0 = cadd(h0, v[r]);
  buf[s] = h0;
#pragma unroll
  for (int t = 1; t <= QM / 2; ++t) {
    if (2 * t > q) break;
    V A = cmk<V>(0, 0), B = cmk<V>(0, 0);
#pragma unroll
    for (int r = 0; r < QM; ++r) {
      if (r < q) {
        const V z = zq_rt<QC>(zt, t, r);  // zeta_q^{t r}
        A.x = fma(v[r].x, z.x, A.x); A.y = fma(v[r].y, z.x, A.y);
        B.x = fma(v[r].x, z.y, B.x); B.y = fma(v[r].y, z.y, B.y);
      }
    }
    if (t < T) buf[t * M + s] = cmk<V>(A.x + B.y, A.y - B.x);
    if (2 * t < q && q - t < T) buf[(q - t) * M + s] = cmk<V>(A.x - B.y, A.y + B.x);
  }
}

template <int QC, bool SPLIT8 = false>
__device__ __forceinline__ void unfold_all(V* buf, int q, int T, const V* zt, const V* twcol, int tid, int nth) {
  if constexpr (QC == 9) {
    if (tid < M / 2) {
      const int sc[2] = {tid, tid + M / 2};
      const V w1[2] = {twcol[sc[0]], twcol[sc[1]]};
      unfold_col9<2, SPLIT8>(buf, sc, T, w1);
    }
  } else {
    for (int s = tid; s < M; s += nth) {
      const V w1 = twcol[s];
      if constexpr (QC > 0) unfold_col<QC, QC>(buf, s, q, T, zt, w1);
      else if (q <= 4) unfold_col<0, 4>(buf, s, q, T, zt, w1);
      else if (q <= 8) unfold_col<0, 8>(buf, s, q, T, zt, w1);
      else unfold_col<0, kQMax>(buf, s, q, T, zt, w1);
    }
  }
}

// ---------------------------------------------------------------------------
// The kernel.  MODE_FWD: fold + FFT -> spectrum line (array blockIdx.z);
// MODE_INV: spectrum line -> IFFT + unfold; MODE_CONV: fold + FFT of f, twiddle +
// FFT of the short g (p_g = 1), product, IFFT, unfold (npairs == 1).
// QC: compile-time q (0: runtime q, twiddles from the SMEM table).
//
// Roles (TMA mode): warp q is the producer.  It keeps two items in flight: loads
// of item i land on full[i&1]; the compute warps (named barrier 1 among
// themselves) process item i and arrive on done[i&1]; the producer then stores
// item i from that stage, waits until the store has read the stage, and loads
// item i + 2 into it.  Fallback mode (a layout TMA cannot express): the compute
// warps copy with cp.async / plain stores and the producer warp idles.
// Shared memory: [full x2, done x2 | pad][zt q x 16][tw 23x32][col 512 (not LEAN)]
//                [stage 0][stage 1], stage = q*512 (+512 CONV).
// ---------------------------------------------------------------------------
// The short input's transform for residue r (p_g = 1): w[s] = (1/prod M1)
// zeta_{M1}^{r s} g[s], s = lane + 32 i, then the size-512 FFT (E: exchange area).
// LOWHALF (L_g <= 256): the upper half of w is zero.  Twiddles by four
// interleaved recurrences of step zeta_{M1}^{128 r}.
// g_transform's input step alone (all 16 values; zero beyond L_g)
__device__ __forceinline__ void g_twist(V* v, const V* gbuf, int Lg, int r, int lane, const V* twM1, double scale) {
  const V st1 = ldg(twM1 + r * 32);
  const V st4 = ldg(twM1 + r * 128);
  V wc[4];
  wc[0] = cscale(ldg(twM1 + r * lane), scale);
  wc[1] = cmul(wc[0], st1);
  wc[2] = cmul(wc[1], st1);
  wc[3] = cmul(wc[2], st1);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int s = lane + 32 * i;
    v[i] = (s < Lg) ? cmul(gbuf[s], wc[i & 3]) : cmk<V>(0, 0);
    if ((i & 3) == 3) {
#pragma unroll
      for (int k = 0; k < 4; ++k) wc[k] = cmul(wc[k], st4);
    }
  }
}

template <bool LOWHALF>
__device__ __forceinline__ void g_transform(V* v, const V* gbuf, int Lg, int r, int lane, const V* twM1,
                                            double scale, V* E, const V* tw) {
  const V st1 = ldg(twM1 + r * 32);
  const V st4 = ldg(twM1 + r * 128);
  V wc[4];
  wc[0] = cscale(ldg(twM1 + r * lane), scale);
  wc[1] = cmul(wc[0], st1);
  wc[2] = cmul(wc[1], st1);
  wc[3] = cmul(wc[2], st1);
#pragma unroll
  for (int i = 0; i < (LOWHALF ? 8 : 16); ++i) {
    const int s = lane + 32 * i;
    v[i] = (s < Lg) ? cmul(gbuf[s], wc[i & 3]) : cmk<V>(0, 0);
    if ((i & 3) == 3) {
#pragma unroll
      for (int k = 0; k < 4; ++k) wc[k] = cmul(wc[k], st4);
    }
  }
  __syncwarp();
  w512::fft_fwd<LOWHALF>(v, E, lane, tw);
}


// LEAN (q <= 5): zeta_{M1}^s is read from global memory instead of a shared-memory
// column, so that two CTAs fit one SM (q + 1 <= 6 warps each at <= 168 registers):
// the small-q passes (the real-input path's packed convolution axis, q = 5) then
// run 12 warps per SM instead of 6.
//
// W8 (q = 9, blockDim 384 = three warpgroups): eight compute warps (warpgroups 0, 1)
// grown to 232 registers with setmaxnreg, the producer in warpgroup 2 shrunk to 40
// (its other three warps exit).  Two compute warps per SM sub-partition and no
// register spills; residue 8 runs as FFT-256 halves (hd_w256.cuh, one radix-2 step
// of the FFT-512): CONV: warps 4, 5 transform F_8's halves, warps 6, 7 G_8's (into
// the area X after the stages), warps 0, 1 multiply and inverse-transform half 0 / 1
// after their own residue (named barriers 5, 3, 4), the unfold combines the halves;
// FWD / INV (HD_S512_W8 bit 1): warps 2, 3 take the halves.  Every sub-partition then
// carries 6.5-7 of the 27 transforms of a column instead of 6-9.
template <int MODE, int NTMAX, int QC, int LEAN = 0>
__global__ void __launch_bounds__(NTMAX, LEAN ? 2 : 1) s512_kernel(const __grid_constant__ PassArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* done = full + 2;
  constexpr bool kW8 = QC == 9 && NTMAX == 384;
  const int q = QC > 0 ? QC : a.q;
  V* zt = reinterpret_cast<V*>(smem_raw + 128);  // zt[r * kQF + t], r < q
  V* twtab = zt + q * kQF;
  V* twcol = twtab + w512::kTwRows * 32;   // zeta_{M1}^s, s < 512 (not LEAN)
  constexpr bool kHalf8 = kW8;  // residue 8 as FFT-256 halves
  V* tw256 = LEAN ? twcol : twcol + M;     // FFT-256 twiddle columns (kHalf8)
  V* stage0 = tw256 + (kHalf8 ? w256::kTwRows * 32 : 0);
  const int tid = threadIdx.x;
  const int nth = kW8 ? 256 : 32 * q;      // compute threads; the next warp is the producer
  const int lane = tid & 31;
  const int r = tid >> 5;                  // this warp's residue (compute warps)
  const int k_arr = blockIdx.z;
  const int SB = q * M + (MODE == MODE_CONV ? M : 0);
  // loads by the producer's TMA (tma) or by every compute thread (cp.async);
  // stores by the producer's TMA (tma_st) or by every compute thread (plain
  // stores: lines TMA could only write in 16-byte pieces, see hd_api.cu)
  const bool tma = a.tm_in.kind != TMA_NONE;
  const bool tma_st = tma && a.tm_out.kind != TMA_NONE;
  // (measured for W8 too -- light warps 0, 4-7 folding during the others' fourth
  // transform: conv_y 308 -> 323 us -- so W8 folds every item up front)
  constexpr bool kPipeFold = (MODE == MODE_CONV && QC == 9 && !kW8);
  const V* twm = reinterpret_cast<const V*>(a.tw_m);
  const V* twM1 = reinterpret_cast<const V*>(a.tw_M1);
  if (QC == 0) {
    for (int i = tid; i < q * kQF; i += blockDim.x) {
      const int rr = i / kQF, t = i % kQF;
      zt[i] = ldg(twM1 + (int64_t)((rr * t) % q) * M);
    }
  }
  for (int i = tid; i < w512::kTwRows * 32; i += blockDim.x) twtab[i] = w512::tw_entry(twm, i >> 5, i & 31);
  if (!LEAN)
    for (int i = tid; i < M; i += blockDim.x) twcol[i] = ldg(twM1 + i);
  if (kHalf8)
    for (int i = tid; i < w256::kTwRows * 32; i += blockDim.x) tw256[i] = w256::tw_entry(twm, M, i >> 5, i & 31);
  const V* twc = LEAN ? twM1 : twcol;
  if (tid == nth) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&done[0], nth);
    mbar_init(&done[1], nth);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t total1 = a.nbatch * a.ngroups;
  const bool fam2 = QC == 9 && MODE == MODE_FWD && a.fam2;
  const int64_t total = total1 + (fam2 ? a.nlines2 : 0);
  const int kk_out = MODE == MODE_FWD ? k_arr : 0;
  if constexpr (kW8) {  // every warp of a warpgroup executes its group's setmaxnreg
    if (tid >= nth) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;" ::: "memory");
    else asm volatile("setmaxnreg.inc.sync.aligned.u32 232;" ::: "memory");
  }

  // ------------------------------------------------------------ producer warp
  if (tid >= nth) {
    if (!tma || tid != nth) return;
    if (fam2) {  // two line families, plain rows (one batch entry each)
      int64_t wl = blockIdx.x;
      for (int s2 = 0; s2 < 2 && wl < total; ++s2, wl += gridDim.x)
        handover_fam2(a, false, 1, 0, true, wl < total1 ? 1 : 2, wl < total1 ? wl : wl - total1,
                      stage0 + s2 * SB, &full[s2]);
      int it = 0;
      for (int64_t w = blockIdx.x; w < total; w += gridDim.x, ++it) {
        const int st = it & 1;
        mbar_wait(&done[st], (uint32_t)(it >> 1) & 1u);
        const bool load = wl < total;
        handover_fam2(a, true, w < total1 ? 1 : 2, w < total1 ? w : w - total1, load, wl < total1 ? 1 : 2,
                      wl < total1 ? wl : wl - total1, stage0 + st * SB, &full[st]);
        if (load) wl += gridDim.x;
      }
      bulk_wait0();
      return;
    }
    int64_t wl = blockIdx.x;  // next item to load
    for (int s2 = 0; s2 < 2 && wl < total; ++s2, wl += gridDim.x) {
      int64_t g, b;
      split_item(wl, a.nbatch, a.ngroups, a.batch_fastest, b, g);
      issue_loads_tma<MODE>(a, k_arr, b, g, stage0 + s2 * SB, &full[s2]);
    }
    if (wl < total) {
      int64_t g, b;
      split_item(wl, a.nbatch, a.ngroups, a.batch_fastest, b, g);
      issue_prefetch<MODE>(a, k_arr, b, g);
    }
    int it = 0;
    for (int64_t w = blockIdx.x; w < total; w += gridDim.x, ++it) {
      const int st = it & 1;
      V* buf = stage0 + st * SB;
      mbar_wait(&done[st], (uint32_t)(it >> 1) & 1u);
      int64_t gs, bs, gl = 0, bl = 0;
      split_item(w, a.nbatch, a.ngroups, a.batch_fastest, bs, gs);
      const bool load = wl < total;
      if (load) split_item(wl, a.nbatch, a.ngroups, a.batch_fastest, bl, gl);
      handover<MODE>(a, k_arr, kk_out, tma_st && gs < a.nlines, bs, gs, load, bl, gl, buf, &full[st]);
      if (load) {
        wl += gridDim.x;
        if (wl < total) {  // and the item after it into L2
          int64_t g, b;
          split_item(wl, a.nbatch, a.ngroups, a.batch_fastest, b, g);
          issue_prefetch<MODE>(a, k_arr, b, g);
        }
      }
    }
    if (tma_st) bulk_wait0();
    return;
  }

  // ------------------------------------------------------------ compute warps
  const V* tw = twtab + lane;  // this lane's FFT twiddle column
  PhaseClock pc;
  pc.start(a.phase_prof != nullptr);
  if (!tma && blockIdx.x < total) {
    int64_t g0, b0;
    split_item(blockIdx.x, a.nbatch, a.ngroups, a.batch_fastest, b0, g0);
    issue_loads_cp<MODE>(a, k_arr, b0, g0, stage0, tid, nth);
  }
  int it = 0;
  for (int64_t w = blockIdx.x; w < total; w += gridDim.x, ++it) {
    const int st = it & 1;
    V* buf = stage0 + st * SB;
    V* gbuf = buf + q * M;
    int64_t g, b;
    const bool in2 = fam2 && w >= total1;  // an item of the second family
    if (fam2) { b = 0; g = in2 ? w - total1 : w; }
    else split_item(w, a.nbatch, a.ngroups, a.batch_fastest, b, g);
    const bool live = g < (in2 ? a.nlines2 : a.nlines);
    V* Fr = buf + r * M;  // this warp's residue row (also its FFT exchange area)
    pc.mark(7);
    // CONV, q = 9, TMA: the fold of item it + 1 is done by the light warps during
    // item it's transforms (kPipeFold); only the first item is folded up front.
    const bool pipe_fold = kPipeFold && tma;
    const bool folded = pipe_fold && it > 0;
    if (!folded) {
      if (tma) mbar_wait(&full[st], (uint32_t)(it >> 1) & 1u);
      else { cp_wait0(); compute_sync(nth); }
    }
    pc.mark(0);

    // step 1: fold (FWD, CONV) or the inverse FFT of the spectrum (INV)
    if (folded) {
      // done during the previous item
    } else if constexpr (MODE == MODE_INV) {
      {
        V v[16];
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) v[k2] = Fr[k2 * 32 + lane];
        w512::fft_inv(v, Fr, lane, tw);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 16; ++i) Fr[lane + 32 * i] = v[i];
      }
      if (kW8 && (r == 2 || r == 3)) {  // residue 8's inverse halves (combined in the unfold)
        const int h = r - 2;
        V* E = buf + 8 * M + 256 * h;
        V a8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) a8[k] = E[k * 32 + lane];
        __syncwarp();
        w256::fft256_inv(a8, E, lane, tw256 + lane);
        if (h) {
#pragma unroll
          for (int i = 0; i < 8; ++i) a8[i] = cmulc(a8[i], ldg(twm + lane + 32 * i));
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) E[lane + 32 * i] = a8[i];
      }
    } else {
      if (QC == 9 && MODE == MODE_FWD && a.rp && !in2) {
        if (a.in_f.p <= 4) fold9_rp<4>(buf, (int)a.in_f.L, live, g < a.rp_rows, rp_im_slot(a), twc, tid, nth);
        else fold9_rp<8>(buf, (int)a.in_f.L, live, g < a.rp_rows, rp_im_slot(a), twc, tid, nth);
      } else {
        const LineIn& fin = in2 ? a.in_g : a.in_f;
        fold_all<QC>(buf, fin.p, (int)fin.L, live, q, zt, twm, twc, tid, nth);
      }
    }
    pc.mark(1);
    compute_sync(nth);
    pc.mark(2);
    if (!tma) {  // fallback: the compute warps copy the next item into the other stage
      const int64_t wn = w + gridDim.x;
      if (wn < total) {
        int64_t gn, bn;
        split_item(wn, a.nbatch, a.ngroups, a.batch_fastest, bn, gn);
        V* nb = stage0 + (st ^ 1) * SB;
        issue_loads_cp<MODE>(a, k_arr, bn, gn, nb, tid, nth);
      }
    }
    pc.mark(3);
    if constexpr (MODE == MODE_FWD) {
      if (kW8 && (r == 2 || r == 3)) {  // residue 8's forward halves: X[2k] / X[2k+1]
        const int h = r - 2;
        V* R8 = buf + 8 * M;
        V* E = R8 + 256 * h;
        V a8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const V x0 = R8[lane + 32 * i], x1 = R8[lane + 32 * i + 256];
          a8[i] = h ? cmul(csub(x0, x1), ldg(twm + lane + 32 * i)) : cadd(x0, x1);
        }
        asm volatile("bar.sync 5, 64;" ::: "memory");  // both halves read row 8
        w256::fft256_fwd(a8, E, lane, tw256 + lane);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) E[k * 32 + lane] = a8[k];
      }
      V v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = Fr[lane + 32 * i];
      w512::fft_fwd(v, Fr, lane, tw);
      __syncwarp();
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) Fr[k2 * 32 + lane] = v[k2];  // lane-major spectrum
    } else if constexpr (MODE == MODE_CONV && kW8) {
      // Residue 8 runs as six FFT-256 half jobs (one radix-2 step of the size-512
      // transform): forward X[2k] = FFT256(w[n] + w[n+256]), X[2k+1] =
      // FFT256((w[n] - w[n+256]) zeta_512^n); inverse halves a = IFFT256(Y[2k]),
      // b = IFFT256(Y[2k+1]) zeta_512^{-n}, combined y = a +- b in the unfold.
      //   warps 4, 5: F_8 halves 0, 1 (row 8 -> row 8, slots [256 h, 256 h + 256))
      //   warps 6, 7: G_8 halves 0, 1 (twisted g -> X)
      //   warps 0, 1: product and inverse of half 0, 1 (row 8), after their own residue
      // so every warp carries three transforms and at most one half (sub-partitions
      // (w + c) mod 4: 7, 7, 6.5, 6.5 transforms).  Named barriers: 5 (warps 4, 5: both
      // halves read row 8 before either overwrites it), 3 / 4 (half 0 / 1 ready:
      // arrive by the F and G warps, sync by warp 0 / 1).
      V* R8 = buf + 8 * M;
      V* X = stage0 + 2 * SB;
      const int Lg = live ? (int)a.in_g.L : 0;
      const V* tq = tw256 + lane;
      V F[16], v[16];
      if (r >= 4) {
        const int h = r & 1;
        const bool isF = r < 6;
        V* E = (isF ? R8 : X) + 256 * h;
        V a8[8];
        if (isF) {
#pragma unroll
          for (int i = 0; i < 8; ++i) { v[i] = R8[lane + 32 * i]; v[i + 8] = R8[lane + 32 * i + 256]; }
        } else {
          g_twist(v, gbuf, Lg, 8, lane, twM1, a.scale);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
          a8[i] = h ? cmul(csub(v[i], v[i + 8]), ldg(twm + lane + 32 * i)) : cadd(v[i], v[i + 8]);
        if (isF) asm volatile("bar.sync 5, 64;" ::: "memory");
        __syncwarp();
        w256::fft256_fwd(a8, E, lane, tq);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) E[k * 32 + lane] = a8[k];
        if (h) asm volatile("bar.arrive 4, 96;" ::: "memory");
        else asm volatile("bar.arrive 3, 96;" ::: "memory");
      }
      // F_r and G_r together (one exchange area: row r), product
#pragma unroll
      for (int i = 0; i < 16; ++i) F[i] = Fr[lane + 32 * i];
      g_twist(v, gbuf, Lg, r, lane, twM1, a.scale);
      w512::fft_fwd2(F, v, Fr, lane, tw, Lg <= M / 2);
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = cmul(F[k], v[k]);
      __syncwarp();
      w512::fft_inv(v, Fr, lane, tw);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 16; ++i) Fr[lane + 32 * i] = v[i];
      if (r < 2) {  // half r of residue 8: product, inverse FFT-256
        const int h = r;
        if (h) asm volatile("bar.sync 4, 96;" ::: "memory");
        else asm volatile("bar.sync 3, 96;" ::: "memory");
        V* E = R8 + 256 * h;
        const V* Xh = X + 256 * h;
        V a8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) a8[k] = cmul(E[k * 32 + lane], Xh[k * 32 + lane]);
        __syncwarp();
        w256::fft256_inv(a8, E, lane, tq);
        if (h) {
#pragma unroll
          for (int i = 0; i < 8; ++i) a8[i] = cmulc(a8[i], ldg(twm + lane + 32 * i));
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) E[lane + 32 * i] = a8[i];
      }
    } else if constexpr (MODE == MODE_CONV) {
      V F[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) F[i] = Fr[lane + 32 * i];
      w512::fft_fwd(F, Fr, lane, tw);
      V v[16];
      {
        const int Lg = live ? (int)a.in_g.L : 0;
        __syncwarp();
        if (Lg <= M / 2) g_transform<true>(v, gbuf, Lg, r, lane, twM1, a.scale, Fr, tw);
        else g_transform<false>(v, gbuf, Lg, r, lane, twM1, a.scale, Fr, tw);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = cmul(F[k], v[k]);
      w512::fft_inv(v, Fr, lane, tw);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 16; ++i) Fr[lane + 32 * i] = v[i];
    }
    if (pipe_fold && (r & 3) != 0) {  // light warps: fold the next item now
      const int64_t wn = w + gridDim.x;
      if (wn < total) {
        int64_t gn, bn;
        split_item(wn, a.nbatch, a.ngroups, a.batch_fastest, bn, gn);
        mbar_wait(&full[st ^ 1], (uint32_t)((it + 1) >> 1) & 1u);
        const int lt = (r - 1 - (r > 4 ? 1 : 0)) * 32 + lane;
        fold9_light(stage0 + (st ^ 1) * SB, a.in_f.p, (int)a.in_f.L, gn < a.nlines, twc, lt);
      }
    }
    pc.mark(4);
    if constexpr (MODE != MODE_FWD) {
      compute_sync(nth);
      pc.mark(5);
      if (QC == 9 && MODE == MODE_INV && a.rs) unfold9_rs<kHalf8>(buf, a.out.T, twc, tid, nth);
      else unfold_all<QC, kHalf8>(buf, q, a.out.T, zt, twc, tid, nth);
    }
    pc.mark(6);
    // results are in stage slots j < out.L
    if (tma_st) {
      fence_async_smem();
      mbar_arrive(&done[st]);  // the producer stores them
    } else if (tma) {
      compute_sync(nth);
      if (live) stores_st(a, kk_out, b, g, buf, tid, nth);
      mbar_arrive(&done[st]);  // stage free once every thread's stores have read it
    } else {
      compute_sync(nth);
      if (live) stores_st(a, kk_out, b, g, buf, tid, nth);
      compute_sync(nth);
    }
  }
  pc.flush(a.phase_prof);
}

// ---------------------------------------------------------------------------
// MODE_MCONV: the convolution pass for N pairs (multi-convolution, PAPER.md:19;
// h = sum_k f_k * g_k, BASELINE config 5) and short inputs of several blocks
// (p_g <= 8).  One work item = one line; the producer streams its N pairs through
// the two-stage ring (stage = 2q rows: f_k folded into rows 0..q-1, g_k into rows
// q..2q-1).  Warp r keeps the running sum of F_k G_k of residue r in registers:
//   fold f_k, g_k (thread per column) -> F-FFT and G-FFT of rows r and q + r
//   interleaved in registers (w512::fft_fwd2) -> acc += F G;  after the last pair:
//   inverse FFT of (1/prod M1) acc -> row r -> unfold -> the producer stores.
// q <= 6 (two stages of 2q rows), blockDim = 32 (q + 1): at most two warps per
// SM sub-partition, so acc and a transform fit in registers.
// ---------------------------------------------------------------------------
constexpr int kMconvQMax = 6;

__device__ __forceinline__ void issue_loads_pair(const PassArgs& a, int64_t b, int64_t g, int k, V* buf,
                                                 uint64_t* bar) {
  const bool live = g < a.nlines;
  const int Lf = (int)a.in_f.L, Lg = (int)a.in_g.L;
  mbar_expect_tx(bar, live ? (uint32_t)(((Lf + kBox - 1) / kBox + (Lg + kBox - 1) / kBox) * kBox * 16) : 0u);
  if (!live) return;
  int c[5];
  for (int j0 = 0; j0 < Lf; j0 += kBox) {
    tma_coords(a.tm_in, b, g, j0, c);
    tma_load(buf + j0, &a.tm_in_map[k], c, bar);
  }
  V* gb = buf + a.q * M;
  for (int j0 = 0; j0 < Lg; j0 += kBox) {
    tma_coords(a.tm_in_g, b, g, j0, c);
    tma_load(gb + j0, &a.tm_in_g_map[k], c, bar);
  }
}

template <int NTMAX, int QC = 0>
__global__ void __launch_bounds__(NTMAX, 1) s512_mconv_kernel(const __grid_constant__ PassArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* done = full + 2;
  V* zt = reinterpret_cast<V*>(smem_raw + 128);
  V* twtab = zt + kQF * kQF;
  V* twcol = twtab + w512::kTwRows * 32;
  V* stage0 = twcol + M;
  const int q = QC > 0 ? QC : a.q, N = a.npairs;
  const int tid = threadIdx.x, lane = tid & 31, r = tid >> 5;
  const int nth = 32 * q;
  const int SB = 2 * q * M;
  const V* twm = reinterpret_cast<const V*>(a.tw_m);
  const V* twM1 = reinterpret_cast<const V*>(a.tw_M1);
  for (int i = tid; i < kQF * kQF; i += blockDim.x) {
    const int rr = i / kQF, t = i % kQF;
    zt[i] = ldg(twM1 + (int64_t)((rr * t) % q) * M);
  }
  for (int i = tid; i < w512::kTwRows * 32; i += blockDim.x) twtab[i] = w512::tw_entry(twm, i >> 5, i & 31);
  for (int i = tid; i < M; i += blockDim.x) twcol[i] = ldg(twM1 + i);
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&done[0], nth);
    mbar_init(&done[1], nth);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t total = a.nbatch * a.ngroups;
  const int64_t nit = total > blockIdx.x ? (total - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nsteps = nit * N;  // (line, pair) steps of this CTA

  if (tid >= nth) {  // producer warp (lane 0)
    if (tid != nth) return;
    auto step_item = [&](int64_t sg, int64_t& b, int64_t& g, int& k) {
      const int64_t it = sg / N;
      k = (int)(sg - it * N);
      split_item(blockIdx.x + it * gridDim.x, a.nbatch, a.ngroups, a.batch_fastest, b, g);
    };
    int64_t sl = 0;
    for (; sl < 2 && sl < nsteps; ++sl) {
      int64_t b, g; int k;
      step_item(sl, b, g, k);
      issue_loads_pair(a, b, g, k, stage0 + (sl & 1) * SB, &full[sl & 1]);
    }
    for (int64_t sg = 0; sg < nsteps; ++sg) {
      const int st = (int)(sg & 1);
      V* buf = stage0 + st * SB;
      mbar_wait(&done[st], (uint32_t)(sg >> 1) & 1u);
      int64_t b, g; int k;
      step_item(sg, b, g, k);
      if (k == N - 1 && g < a.nlines) issue_stores_tma(a, 0, b, g, buf);
      if (sl < nsteps) {
        bulk_wait_read0();
        step_item(sl, b, g, k);
        issue_loads_pair(a, b, g, k, buf, &full[st]);
        ++sl;
      }
    }
    bulk_wait0();
    return;
  }

  const V* tw = twtab + lane;
  const double scale = a.scale;
  int64_t sg = 0;
  for (int64_t it = 0; it < nit; ++it) {
    int64_t g, b;
    split_item(blockIdx.x + it * gridDim.x, a.nbatch, a.ngroups, a.batch_fastest, b, g);
    const bool live = g < a.nlines;
    V acc[16];
    for (int k = 0; k < N; ++k, ++sg) {
      const int st = (int)(sg & 1);
      V* buf = stage0 + st * SB;
      V* Fr = buf + r * M;
      V* Gr = buf + (q + r) * M;
      mbar_wait(&full[st], (uint32_t)(sg >> 1) & 1u);
      fold_all<QC>(buf, a.in_f.p, (int)a.in_f.L, live, q, zt, twm, twcol, tid, nth);
      fold_all<QC>(buf + q * M, a.in_g.p, (int)a.in_g.L, live, q, zt, twm, twcol, tid, nth);
      compute_sync(nth);
      // F_k and G_k of residue r transformed together, stage by stage (w512::fft_fwd2:
      // independent chains; the single transforms back to back left the warp latency-bound)
      V v[16], u[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) { v[i] = Fr[lane + 32 * i]; u[i] = Gr[lane + 32 * i]; }
      __syncwarp();
      w512::fft_fwd2(v, u, Fr, lane, tw, false);
      if (k == 0) {
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) acc[k2] = cmul(v[k2], u[k2]);
      } else {
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) acc[k2] = cfma(acc[k2], v[k2], u[k2]);
      }
      if (k < N - 1) {
        mbar_arrive(&done[st]);  // stage free for the producer
        continue;
      }
      // last pair: inverse transform of the scaled sum, unfold, store
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) acc[k2] = cscale(acc[k2], scale);
      __syncwarp();
      w512::fft_inv(acc, Fr, lane, tw);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 16; ++i) Fr[lane + 32 * i] = acc[i];
      compute_sync(nth);
      unfold_all<QC>(buf, q, a.out.T, zt, twcol, tid, nth);
      fence_async_smem();
      mbar_arrive(&done[st]);
    }
  }
}

}  // namespace s512
}  // namespace hd
