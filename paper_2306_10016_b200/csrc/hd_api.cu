// hd_api.cu -- host side of libhdconv.so: plans,
// twiddle tables, the multi-pass drivers for 1D/2D/3D/multiconv
// (PAPER.md:716-739, 1438-1489), the explicit baseline, the
// on-device tuning sweep and the C ABI (include/hdconv.h).
#include "hdconv.h"
#include "hd_device.cuh"
#include "hd_internal.h"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <string>
#include <vector>

using hd::LineIn;
using hd::LineOut;
using hd::PassArgs;

namespace {
thread_local std::string g_tls_error;
}  // namespace

struct hd_ctx {
  int device = 0;
  std::string err;
  std::recursive_mutex mu;            // held for a whole entry point (entries nest: real -> run_entry)
  std::map<int64_t, void*> tw64, tw32;  // N -> device zeta_N^k tables
  std::map<int64_t, void*> st64, st32;  // m -> device stage twiddle tables
  std::map<int64_t, int32_t*> perm;     // 2n (+1: inverse) -> device spectral permutation
  void* ws = nullptr;
  size_t ws_size = 0;
  void* io = nullptr;                   // device buffers for hd_conv_host
  size_t io_size = 0;
  void* rio = nullptr;                  // hd_conv_real: packed input, complex g, complex result
  size_t rio_size = 0;
  struct HostSlot {                     // hd_conv_host_async: triple-buffered host I/O
    void* io = nullptr;
    size_t size = 0;
    cudaStream_t st = nullptr;
  };
  static constexpr int kHostSlots = 3;  // copy-in k+2 | compute k+1 | copy-out k
  HostSlot hslot[kHostSlots];
  int hnext = 0;
  // Context scratch (ws, io, rio, host slots) is shared by every call that passes
  // no workspace, whatever stream it is on: each such call waits for the previous
  // one's last scratch use (scratch_done) and records its own.
  cudaEvent_t scratch_done = nullptr;
  bool scratch_pending = false;
  std::map<std::string, hd_plan_t> plan_cache;
  std::vector<std::pair<hd_plan_t, double>> tune_log;
  // profiling
  bool profiling = false;
  struct ProfEntry {
    std::string name;
    double ms = 0;
    int64_t launches = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
  };
  std::vector<ProfEntry> prof;
  int64_t launches = 0;
  int64_t engine_launches[7] = {0, 0, 0, 0, 0, 0, 0};  // pass launches per engine (HD_ENGINE_*)
  // HD_FLAG_GRAPH: captured pass sequences keyed by their full argument list
  std::map<std::string, cudaGraphExec_t> graphs;
  cudaStream_t capture_stream = nullptr;
  bool capturing = false;
  int64_t graph_replays = 0;
};

namespace {

hd_status_t fail(hd_ctx* ctx, hd_status_t st, const std::string& msg) {
  if (ctx) ctx->err = msg; else g_tls_error = msg;
  g_tls_error = msg;
  return st;
}
hd_status_t cuda_fail(hd_ctx* ctx, cudaError_t e, const char* what) {
  return fail(ctx, HD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
int ilog2(int64_t v) { int r = 0; while ((int64_t(1) << r) < v) ++r; return r; }
size_t elem_bytes(hd_dtype_t dt) { return dt == HD_C128 ? 16 : 8; }

// Order a call that uses context scratch after the previous such call (any stream).
// Not during graph capture: a captured launch sequence is ordered by its replay.
hd_status_t scratch_acquire(hd_ctx* ctx, cudaStream_t st) {
  if (ctx->capturing) return HD_OK;
  if (!ctx->scratch_done) {
    cudaError_t e = cudaEventCreateWithFlags(&ctx->scratch_done, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaEventCreate(scratch)");
  }
  if (ctx->scratch_pending) {
    cudaError_t e = cudaStreamWaitEvent(st, ctx->scratch_done, 0);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamWaitEvent(scratch)");
  }
  return HD_OK;
}
hd_status_t scratch_release(hd_ctx* ctx, cudaStream_t st) {
  if (ctx->capturing || !ctx->scratch_done) return HD_OK;
  cudaError_t e = cudaEventRecord(ctx->scratch_done, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaEventRecord(scratch)");
  ctx->scratch_pending = true;
  return HD_OK;
}
// Grow one context scratch buffer.  Captured graphs may address any scratch buffer,
// so they are dropped first; cudaFree waits for in-flight work on the device.
hd_status_t grow_scratch(hd_ctx* ctx, void** buf, size_t* size, size_t need, const char* what) {
  if (*size >= need) return HD_OK;
  for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
  ctx->graphs.clear();
  if (*buf) cudaFree(*buf);
  *buf = nullptr; *size = 0;
  cudaError_t e = cudaMalloc(buf, need);
  if (e != cudaSuccess) return cuda_fail(ctx, e, what);
  *size = need;
  return HD_OK;
}

// ---------------------------------------------------------------------------
// twiddle tables zeta_N^k = exp(2 pi i k / N), k < N, computed in long double
// with the integer k reduced to the first octant's symmetric argument.
// ---------------------------------------------------------------------------
void host_twiddles(int64_t N, std::vector<double>& out) {
  out.resize(2 * N);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int64_t k = 0; k < N; ++k) {
    // reduce: angle = 2 pi k / N; use k' = min(k, N-k) for accuracy of sin/cos
    long double ang = two_pi * (long double)k / (long double)N;
    long double c = cosl(ang), s = sinl(ang);
    if (4 * k == N) { c = 0; s = 1; }
    if (2 * k == N) { c = -1; s = 0; }
    if (4 * k == 3 * N) { c = 0; s = -1; }
    out[2 * k] = (double)c;
    out[2 * k + 1] = (double)s;
  }
}

hd_status_t get_table(hd_ctx* ctx, int64_t N, bool dbl, const void** out) {
  auto& cache = dbl ? ctx->tw64 : ctx->tw32;
  auto it = cache.find(N);
  if (it != cache.end()) { *out = it->second; return HD_OK; }
  std::vector<double> h;
  host_twiddles(N, h);
  void* d = nullptr;
  size_t bytes = dbl ? 16 * (size_t)N : 8 * (size_t)N;
  cudaError_t e = cudaMalloc(&d, bytes);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(twiddles)");
  if (dbl) {
    e = cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice);
  } else {
    std::vector<float> hf(2 * N);
    for (int64_t i = 0; i < 2 * N; ++i) hf[i] = (float)h[i];
    e = cudaMemcpy(d, hf.data(), bytes, cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) { cudaFree(d); return cuda_fail(ctx, e, "cudaMemcpy(twiddles)"); }
  cache[N] = d;
  *out = d;
  return HD_OK;
}

// Stage twiddle table of the size-m FFT (layout of hd_device.cuh StageOff): for
// every DIF stage s with span SP > 1 (radix-8 stages, then one radix-4/2), the
// entries [j-1][o] = zeta_NK^{o j}, j = 1..R-1, o < SP, NK = m / prod(radix < s).
hd_status_t get_stage_table(hd_ctx* ctx, int m, bool dbl, const void** out) {
  auto& cache = dbl ? ctx->st64 : ctx->st32;
  auto it = cache.find(m);
  if (it != cache.end()) { *out = it->second; return HD_OK; }
  const int lg = ilog2(m);
  std::vector<int> rad;
  for (int i = 0; i < lg / 3; ++i) rad.push_back(8);
  if (lg % 3 == 1) rad.push_back(2);
  if (lg % 3 == 2) rad.push_back(4);
  std::vector<double> full;
  host_twiddles(m, full);  // zeta_m^k
  std::vector<double> tab;
  int NK = m;
  for (size_t st = 0; st < rad.size(); ++st) {
    const int R = rad[st], SP = NK / R;
    if (SP > 1)
      for (int j = 1; j < R; ++j)
        for (int o = 0; o < SP; ++o) {
          const int64_t e = (int64_t)o * j * (m / NK);  // zeta_NK^{o j} = zeta_m^{o j m/NK}
          tab.push_back(full[2 * e]);
          tab.push_back(full[2 * e + 1]);
        }
    NK = SP;
  }
  if (tab.empty()) { tab.push_back(1.0); tab.push_back(0.0); }
  const size_t n = tab.size() / 2;
  void* d = nullptr;
  cudaError_t e = cudaMalloc(&d, dbl ? 16 * n : 8 * n);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(stage twiddles)");
  if (dbl) e = cudaMemcpy(d, tab.data(), 16 * n, cudaMemcpyHostToDevice);
  else {
    std::vector<float> f(tab.begin(), tab.end());
    e = cudaMemcpy(d, f.data(), 8 * n, cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) { cudaFree(d); return cuda_fail(ctx, e, "cudaMemcpy(stage twiddles)"); }
  cache[m] = d;
  *out = d;
  return HD_OK;
}

// ---------------------------------------------------------------------------
// plans
// ---------------------------------------------------------------------------
struct AxisInfo {
  int64_t Lf, Lg, Lout, M, M1, O;  // O: output extent (Lout, or M1 if aliased; the window size)
  int64_t o0;                      // output window start (0: from the first output)
  int m, q, pf, pg, T, C, S, D, lines, threads;
  bool auto_engine;                // plan threads == 0: warp engine where it applies
};

// lines per CTA used by passes along axis i (the paper's C, "copies of the FFT
// computed simultaneously"); S is the tile width of the transposed
// intermediate those passes read (strided-pass staging width)
int lines_for(const hd_axis_plan_t& a, int i, int ndim) { (void)i; (void)ndim; return a.C; }

int64_t round_slots(int64_t n, size_t eb) {
  const int64_t epr = 128 / (int64_t)eb;
  return (n + 8 * epr - 1) / (8 * epr) * (8 * epr);
}
size_t pass_smem(size_t eb, int q, int lines, int D, int m, int nbuf) {
  return eb * (size_t)(round_slots(q, eb) + round_slots(hd::kQF * hd::kQF, eb) +
                       nbuf * round_slots((int64_t)lines * D * m, eb));
}
int conv_nbuf(int npairs) { return npairs == 1 ? 2 : 3; }

bool valid_lines(int v) { return v == 1 || v == 2 || v == 4 || v == 8 || v == 16; }
// Block size matched to the FFT butterfly sweep (lines * D * m / R items): the
// multiple of 32 in [128, 576] that wastes the fewest thread slots, largest first.
int default_threads(int lines, int D, int m) {
  const int R = m >= 8 ? 8 : m;
  const int64_t items = (int64_t)lines * D * (m / R);
  int best = 576;
  double best_eff = 0;
  for (int nt = 576; nt >= 128; nt -= 32) {
    const double eff = (double)items / (double)(cdiv(items, nt) * nt);
    if (eff > best_eff + 0.01) { best_eff = eff; best = nt; }
  }
  return best;
}
bool valid_threads(int t) { return t >= 32 && t <= 1024 && t % 32 == 0; }
// automatic CTA size: passes whose shared memory leaves room for one CTA per SM
// get 1024 threads (latency hiding by width; config 2: 3.0 -> 2.5 ms at m = 1024)
int auto_threads(int lines, int D, int m, size_t smem) {
  if (smem > hd::kMaxSmem / 2 && (int64_t)lines * D * (m / 8) >= 512) return 1024;
  return default_threads(lines, D, m);
}

hd_status_t complete_plan(hd_ctx* ctx, hd_dtype_t dt, int ndim, int npairs, const int64_t* Lf,
                          const int64_t* Lg, const int64_t* M, hd_plan_t* plan, AxisInfo* ax) {
  if (dt != HD_C64 && dt != HD_C128) return fail(ctx, HD_ERR_INVALID, "dtype must be HD_C64 or HD_C128");
  if (ndim < 1 || ndim > HD_MAX_DIM) return fail(ctx, HD_ERR_INVALID, "ndim must be 1, 2 or 3");
  if (npairs < 1 || npairs > HD_MAX_PAIRS) return fail(ctx, HD_ERR_INVALID, "N must be in [1, 16]");
  if (plan->ndim != ndim) return fail(ctx, HD_ERR_INVALID, "plan.ndim does not match ndim");
  const size_t eb = elem_bytes(dt);
  for (int i = 0; i < ndim; ++i) {
    hd_axis_plan_t& a = plan->axis[i];
    AxisInfo& x = ax[i];
    if (Lf[i] < 1 || Lg[i] < 1) return fail(ctx, HD_ERR_INVALID, "extents must be >= 1");
    x.Lf = Lf[i]; x.Lg = Lg[i];
    x.Lout = Lf[i] + Lg[i] - 1;
    x.M = (M && M[i] > 0) ? M[i] : x.Lout;
    if (!is_pow2(a.m) || a.m < 2 || a.m > 4096)
      return fail(ctx, HD_ERR_INVALID, "axis " + std::to_string(i) + ": m must be a power of two in [2, 4096]");
    x.m = a.m;
    x.q = (int)cdiv(x.M, a.m);
    x.M1 = (int64_t)x.q * a.m;
    if (x.M1 < x.Lout && !(plan->flags & HD_FLAG_ALLOW_ALIAS))
      return fail(ctx, HD_ERR_INVALID, "axis " + std::to_string(i) + ": M < L_f + L_g - 1 would alias (PAPER.md:592)");
    x.O = std::min(x.Lout, x.M1);
    x.o0 = 0;
    x.pf = (int)cdiv(x.Lf, a.m);
    x.pg = (int)cdiv(x.Lg, a.m);
    x.T = (int)cdiv(x.O, a.m);
    if (a.C == 0) a.C = 1;
    if (a.S == 0) a.S = 1;
    if (!valid_lines(a.C) || !valid_lines(a.S)) return fail(ctx, HD_ERR_INVALID, "C and S must be 1, 2, 4, 8 or 16");
    x.C = a.C; x.S = a.S;
    if (a.D == 0) a.D = x.q;
    if (a.D < 1 || a.D > x.q) return fail(ctx, HD_ERR_INVALID, "D must be in [1, q]");
    x.D = a.D;
    if (a.D == 0) a.D = x.q;
    x.auto_engine = (a.threads == 0);
    x.threads = a.threads ? a.threads
                          : auto_threads(lines_for(a, i, ndim), a.D, a.m,
                                         pass_smem(eb, x.q, lines_for(a, i, ndim), a.D, a.m,
                                                   (i == 0) ? conv_nbuf(npairs) : 1));
    if (!valid_threads(x.threads))
      return fail(ctx, HD_ERR_INVALID, "threads must be 0 or a multiple of 32 in [32, 1024]");
    x.lines = lines_for(a, i, ndim);
    const int nbuf = (i == 0) ? conv_nbuf(npairs) : 1;
    // the 1-D two-CTA cluster pass (hd_s512c.cuh) holds at most 11 residue rows per CTA;
    // the 1-D m = 2048 engine (hd_s2048r.cuh) keeps two residues in shared memory at a time
    const bool cluster_q = (x.m == 512 && x.q >= hd::kS512cQMin && x.q <= hd::kS512cQMax) ||
                           (x.m == 2048 && x.q <= hd::s2048r_qmax() && x.pf <= 8 && x.pg <= 8) ||
                           (x.m == 4096 && x.q <= hd::s4096r_qmax() && x.pf <= hd::s4096r_pmax() &&
                            x.pg <= hd::s4096r_pmax());
    const bool cluster_1d = dt == HD_C128 && ndim == 1 && npairs == 1 && cluster_q && x.D == x.q &&
                            x.lines == 1 && x.auto_engine && !(plan->flags & HD_FLAG_GENERIC_FFT);
    if (!cluster_1d && pass_smem(eb, x.q, x.lines, x.D, x.m, nbuf) > hd::kMaxSmem)
      return fail(ctx, HD_ERR_INVALID, "axis " + std::to_string(i) + ": lines*D*m too large for shared memory");
    a.p_f = x.pf; a.p_g = x.pg; a.q = x.q; a.M1 = x.M1;
  }
  return HD_OK;
}

// Output window: keep outputs
// [lo[i], lo[i] + n[i]) of each axis; the last pass of every axis writes only those.
hd_status_t apply_window(hd_ctx* ctx, int ndim, const int64_t* lo, const int64_t* n, AxisInfo* ax) {
  if (!lo || !n) return HD_OK;
  for (int i = 0; i < ndim; ++i) {
    AxisInfo& x = ax[i];
    if (lo[i] < 0 || n[i] < 1 || lo[i] + n[i] > x.O)
      return fail(ctx, HD_ERR_INVALID, "axis " + std::to_string(i) + ": window outside the output");
    x.o0 = lo[i];
    x.O = n[i];
    x.T = (int)cdiv(x.o0 + x.O, x.m);
  }
  return HD_OK;
}

// static cost model for the default plan (per line of the axis)
double axis_cost(int64_t Lf, int64_t Lg, int64_t Lout, int64_t M, int m, bool conv) {
  const int64_t q = cdiv(M, m), M1 = q * m;
  const int64_t pf = cdiv(Lf, m), pg = cdiv(Lg, m), T = cdiv(Lout, m);
  double fold = (double)M1 * (double)(pf + pg);
  double fft = (double)M1 * 3.0 * 1.25 * ilog2(m);
  double unfold = (double)T * m * (double)q;
  double bytes = conv ? 0.0 : 10.0 * (double)M1;
  return fold + fft + unfold + bytes;
}

hd_status_t default_plan(hd_ctx* ctx, hd_dtype_t dt, int ndim, int npairs, const int64_t* Lf,
                         const int64_t* Lg, const int64_t* M, hd_plan_t* out) {
  if (ndim < 1 || ndim > HD_MAX_DIM) return fail(ctx, HD_ERR_INVALID, "ndim must be 1, 2 or 3");
  const size_t eb = elem_bytes(dt);
  hd_plan_t p;
  std::memset(&p, 0, sizeof(p));
  p.ndim = ndim;
  for (int i = 0; i < ndim; ++i) {
    if (Lf[i] < 1 || Lg[i] < 1) return fail(ctx, HD_ERR_INVALID, "extents must be >= 1");
    const int64_t Lout = Lf[i] + Lg[i] - 1;
    const int64_t Mi = (M && M[i] > 0) ? M[i] : Lout;
    const bool conv = (i == 0);
    const int nbuf = conv ? conv_nbuf(npairs) : 1;
    double best = 1e300;
    int bm = 2, bD = 1, bl = 1;
    for (int lines : {2, 1}) {
      if (ndim == 1 && lines > 1) continue;
      for (int m = 2; m <= 4096; m *= 2) {
        const int q = (int)cdiv(Mi, m);
        int D = q;
        while (D > 1 && pass_smem(eb, q, lines, D, m, nbuf) > hd::kMaxSmem) --D;
        if (pass_smem(eb, q, lines, D, m, nbuf) > hd::kMaxSmem) continue;
        double c = axis_cost(Lf[i], Lg[i], Lout, Mi, m, conv);
        const int groups = (int)cdiv(q, D);
        if (groups > 1) c += (double)(groups - 1) * (double)(Lf[i] + Lg[i] + 2 * Lout) * 16.0;
        if (c < best * 0.999) { best = c; bm = m; bD = D; bl = lines; }
      }
    }
    // multi-D complex double: prefer m = 512 where the staged engine runs every pass
    // of the axis (q <= 11, p <= 8; the convolution axis with several pairs: the
    // multi-pair pass, q <= 6) -- measured faster than the cost model's pick (config
    // 5's y axis: 0.92 ms staged vs 1.98 ms at m = 1024 generic)
    if (dt == HD_C128 && ndim > 1 && bm != 512) {
      const int64_t q5 = cdiv(Mi, 512);
      const bool p_ok = cdiv(Lf[i], 512) <= 8 && cdiv(Lg[i], 512) <= 8;
      const bool q_ok = (conv && npairs > 1) ? q5 <= 6 : q5 <= hd::kS512QMax;
      if (p_ok && q_ok) { bm = 512; bD = (int)q5; }
    }
    // 1-D complex double, long lines: m = 4096 where the one-CTA-per-line engine
    // hd_s4096r.cuh runs (2 <= q <= 4, p <= 4; config 2: 1.43 ms at m = 2048 -> see DESIGN)
    if (dt == HD_C128 && ndim == 1 && npairs == 1 && bm >= 1024 && !getenv("HD_NO_S4096R")) {
      const int64_t q4 = cdiv(Mi, 4096);
      if (q4 >= 2 && q4 <= hd::s4096r_qmax() && cdiv(Lf[i], 4096) <= hd::s4096r_pmax() &&
          cdiv(Lg[i], 4096) <= hd::s4096r_pmax()) { bm = 4096; bD = (int)q4; }
    }
    // 1-D complex double at m = 2048: every residue in one pass (the one-CTA-per-line
    // engine, hd_s2048r.cuh, q <= 8, p <= 8)
    if (dt == HD_C128 && ndim == 1 && bm == 2048) {
      const int64_t q2 = cdiv(Mi, 2048);
      if (q2 <= hd::s2048r_qmax() && cdiv(Lf[i], 2048) <= 8 && cdiv(Lg[i], 2048) <= 8) bD = (int)q2;
    }
    // one line per CTA where the staged m = 512 engine applies (hd_s512.cuh); four
    // lines per item and tiles of four for the staged complex-float m = 128 engine
    // (hd_s128.cuh) in 2-D / 3-D
    const int qb = (int)cdiv(Mi, bm);
    const bool s128 = dt == HD_C64 && ndim > 1 && bm == 128 && bD == qb && qb <= hd::kS128QMax &&
                      cdiv(Lf[i], bm) <= 8 && cdiv(Lg[i], bm) <= 8;
    const int lines = (dt == HD_C128 && bm == 512 && bD == qb && bD <= hd::kS512QMax) ? 1 : s128 ? 4 : bl;
    p.axis[i].m = bm;
    p.axis[i].D = bD;
    p.axis[i].C = lines;
    p.axis[i].S = (ndim == 1) ? 1 : s128 ? 4 : 2;
    p.axis[i].threads = 0;  // automatic engine choice
  }
  *out = p;
  return HD_OK;
}

// ---------------------------------------------------------------------------
// launching
// ---------------------------------------------------------------------------
struct Launch {
  uint32_t flags;
  bool auto_engine;
  bool s512_axis;   // the staged engine may run this pass (same engine for every pass of the axis)
  bool s128_axis;   // likewise for the m = 128 complex-float staged engine
  bool s512c_axis;  // the 1-D two-CTA cluster pass may run (automatic engine on a 1-D problem)
  int mode;
  const char* name;
  PassArgs a;
  int m, lines, nbuf, threads;
  int64_t ngroups, nbatch, narrays;
};

void init_in(LineIn& in) { std::memset(&in, 0, sizeof(in)); in.nbi = 1; }
void init_out(LineOut& o) { std::memset(&o, 0, sizeof(o)); o.nbi = 1; o.so_log2 = 0; }

// ---------------------------------------------------------------------------
// TMA descriptions of line families for the staged engine (hd_s512.cuh).
// A line family is described by LineIn / LineOut; the kernel moves whole lines
// in boxes of 256 elements (tensor maps) or one bulk copy (plain rows).
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;  // contexts on several threads may ask first
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// dims (innermost first, complex values as 2 scalars): {d0 scalars, d1, d2, nbi, nbo};
// strides in complex elements (16 B, or 8 B when f32) for dims 1..4 (0 = broadcast
// dimension of size 1)
bool encode_lines(CUtensorMap* map, const void* base, const uint64_t dims[5], const int64_t strides[4],
                  const uint32_t box[5], bool f32 = false) {
  const cuuint64_t eb = f32 ? 8 : 16;
  auto enc = tensor_map_encoder();
  if (!enc || !base || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
  cuuint64_t gd[5];
  cuuint64_t gs[4];
  cuuint32_t bx[5], es[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 5; ++i) { gd[i] = dims[i] ? dims[i] : 1; bx[i] = box[i]; }
  for (int i = 0; i < 4; ++i) {
    if (strides[i] < 0) return false;
    gs[i] = strides[i] > 0 ? (cuuint64_t)strides[i] * eb : 16;
    if (gs[i] % 16) return false;
    if (strides[i] == 0) gd[i + 1] = 1;
    if (gs[i] >= (cuuint64_t(1) << 40)) return false;
  }
  for (int i = 0; i < 5; ++i) if (gd[i] > 0xffffffffull) return false;
  return enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<void*>(base), gd, gs, bx, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// 1-D bulk copies of complex-float rows need 16-byte aligned starts and lengths
bool bulk_ok_f32(const void* const* ptr, int narr, std::initializer_list<int64_t> v) {
  for (int k = 0; k < narr; ++k)
    if (reinterpret_cast<uintptr_t>(ptr[k]) & 15) return false;
  for (int64_t x : v) if (x & 1) return false;
  return true;
}

// input lines -> TMA_BULK (plain rows) or TMA_LINE_TILED (lines tiled by S, element stride s_j);
// with elem2 (the staged m = 512 engine), lines whose element axis is tiled by jd < L
// (the slab exchanges' pieces) -> TMA_ELEM2 when jd divides L and has a divisor
// <= 256 that is a multiple of 8 (the box).
// c64 (the m = 128 engine, 4 lines per item): boxes of 128 elements x 4 lines (S >= 4).
bool tma_desc_in(const LineIn& in, int64_t nlines, int64_t nbatch, int narr, hd::TmaLine& t,
                 CUtensorMap* maps, bool c64 = false, bool elem2 = false) {
  t.kind = hd::TMA_NONE; t.slog = 0; t.nbi = in.nbi > 0 ? in.nbi : 1;
  t.bcast = (in.s_b == 0 ? 1 : 0) | (in.s_bo == 0 ? 2 : 0);
  t.box = 0; t.jd = 0;
  if (narr > hd::kTmaArrays) return false;
  if (in.jd > 0 && in.jd < in.L) {
    if (!elem2 || c64 || in.L % in.jd != 0 || t.nbi != nbatch) return false;
    if (in.tl < 30 && in.s_l != 1) return false;
    int box = 0;
    for (int d = 256; d >= 8; d -= 8)
      if (in.jd % d == 0) { box = d; break; }
    if (!box) return false;
    const int64_t S = in.tl < 30 ? (int64_t(1) << in.tl) : 1;
    const int64_t nlt = in.tl < 30 ? ceil_div64(nlines, S) : nlines;
    const uint64_t dims[5] = {(uint64_t)(2 * S), (uint64_t)in.jd, (uint64_t)(in.L / in.jd), (uint64_t)nlt,
                              (uint64_t)nbatch};
    const int64_t str[4] = {in.s_j, in.s_jt, in.tl < 30 ? in.s_t : in.s_l, in.s_b};
    const uint32_t box5[5] = {2u, (uint32_t)box, 1, 1, 1};
    for (int k = 0; k < narr; ++k)
      if (!encode_lines(&maps[k], in.ptr[k], dims, str, box5)) return false;
    t.kind = hd::TMA_ELEM2; t.slog = in.tl < 30 ? in.tl : 0; t.box = box; t.jd = in.jd;
    return true;
  }
  if (in.tl >= 30) {
    if (in.s_j != 1) return false;
    if (c64 && !bulk_ok_f32(in.ptr, narr, {in.L, in.s_l, in.s_b, in.s_bo})) return false;
    t.kind = hd::TMA_BULK;
    return true;
  }
  if (in.s_l != 1 || (c64 && in.tl < 2)) return false;
  const int64_t S = int64_t(1) << in.tl;
  const uint64_t dims[5] = {(uint64_t)(2 * S), (uint64_t)in.L, (uint64_t)ceil_div64(nlines, S), (uint64_t)t.nbi,
                            (uint64_t)ceil_div64(nbatch, t.nbi)};
  const int64_t str[4] = {in.s_j, in.s_t, in.s_b, in.s_bo};
  const uint32_t box[5] = {c64 ? 8u : 2u, c64 ? 128u : 256u, 1, 1, 1};
  for (int k = 0; k < narr; ++k)
    if (!encode_lines(&maps[k], in.ptr[k], dims, str, box, c64)) return false;
  t.kind = hd::TMA_LINE_TILED; t.slog = in.tl;
  return true;
}

// output lines -> TMA_BULK (plain rows), TMA_ELEM_TILED (element axis tiled by S <= 16)
// or TMA_LINE_TILED (lines tiled by S, element stride s_js)
bool tma_desc_out(const LineOut& o, int64_t nlines, int64_t nbatch, int narr, hd::TmaLine& t,
                  CUtensorMap* maps, bool c64 = false) {
  t.kind = hd::TMA_NONE; t.slog = 0; t.nbi = o.nbi > 0 ? o.nbi : 1;
  t.bcast = (o.s_b == 0 ? 1 : 0) | (o.s_bo == 0 ? 2 : 0);
  if ((o.jd > 0 && o.jd < o.L + o.j0) || narr > hd::kTmaArrays) return false;
  const int64_t nbo = ceil_div64(nbatch, t.nbi);
  if (o.tl >= 30 && o.so_log2 >= 30) {
    if (o.s_js != 1) return false;
    if (c64 && !bulk_ok_f32(const_cast<const void* const*>(o.ptr), narr, {o.L, o.s_l, o.s_b, o.s_bo}))
      return false;
    t.kind = hd::TMA_BULK;
    return true;
  }
  if (o.tl >= 30) {
    if (o.s_js != 1 || o.so_log2 > 4) return false;
    const int64_t S = int64_t(1) << o.so_log2;
    const uint64_t dims[5] = {(uint64_t)(2 * S), (uint64_t)nlines, (uint64_t)ceil_div64(o.L, S), (uint64_t)t.nbi,
                              (uint64_t)nbo};
    const int64_t str[4] = {o.s_l, o.s_jt, o.s_b, o.s_bo};
    const uint32_t box[5] = {(uint32_t)(2 * S), c64 ? 4u : 1u, (uint32_t)((c64 ? 128 : 256) / S), 1, 1};
    for (int k = 0; k < narr; ++k)
      if (!encode_lines(&maps[k], o.ptr[k], dims, str, box, c64)) return false;
    t.kind = hd::TMA_ELEM_TILED; t.slog = o.so_log2;
    return true;
  }
  if (o.so_log2 < 30 || o.s_l != 1 || (c64 && o.tl < 2)) return false;
  const int64_t S = int64_t(1) << o.tl;
  const uint64_t dims[5] = {(uint64_t)(2 * S), (uint64_t)o.L, (uint64_t)ceil_div64(nlines, S), (uint64_t)t.nbi,
                            (uint64_t)nbo};
  const int64_t str[4] = {o.s_js, o.s_t, o.s_b, o.s_bo};
  const uint32_t box[5] = {c64 ? 8u : 2u, c64 ? 128u : 256u, 1, 1, 1};
  for (int k = 0; k < narr; ++k)
    if (!encode_lines(&maps[k], o.ptr[k], dims, str, box, c64)) return false;
  t.kind = hd::TMA_LINE_TILED; t.slog = o.tl;
  return true;
}

// Fill the staged engine's TMA descriptions of a launch (falls back to per-thread
// copies for anything a tensor map cannot express).
void prepare_tma(Launch& L, bool c64 = false, bool elem2 = false) {
  PassArgs& a = L.a;
  const int narr_in = L.mode == hd::MODE_FWD ? (int)L.narrays : (L.mode == hd::MODE_CONV ? a.npairs : 1);
  const int narr_out = L.mode == hd::MODE_FWD ? (int)L.narrays : 1;
  if (!tma_desc_in(a.in_f, a.nlines, a.nbatch, narr_in, a.tm_in, a.tm_in_map, c64, elem2 && !a.rp))
    a.tm_in.kind = hd::TMA_NONE;
  if (L.mode == hd::MODE_CONV) {
    // both inputs of the convolution pass move by TMA or both by per-thread copies
    if (!tma_desc_in(a.in_g, a.nlines, a.nbatch, a.npairs, a.tm_in_g, a.tm_in_g_map, c64) ||
        a.tm_in.kind == hd::TMA_NONE) {
      a.tm_in.kind = hd::TMA_NONE; a.tm_in_g.kind = hd::TMA_NONE;
    }
  }
  if (!tma_desc_out(a.out, a.nlines, a.nbatch, narr_out, a.tm_out, a.tm_out_map, c64)) a.tm_out.kind = hd::TMA_NONE;
  if (a.fam2) {  // the second line family of a merged forward launch (see PassArgs fam2)
    if (!tma_desc_in(a.in_g, a.nlines2, 1, 1, a.tm_in_g, a.tm_in_g_map)) a.tm_in_g.kind = hd::TMA_NONE;
    if (!tma_desc_out(a.out2, a.nlines2, 1, 1, a.tm_out2, &a.tm_out_map[1])) a.tm_out2.kind = hd::TMA_NONE;
  }
  // a window start that is not tile-aligned cannot be expressed by element-tiled boxes
  // (the m = 128 engine stores every window by plain stores)
  if (a.out.j0 != 0 && (c64 || a.tm_out.kind == hd::TMA_ELEM_TILED)) a.tm_out.kind = hd::TMA_NONE;
  // loads by TMA need the producer warp; without them the stores go per thread too
  if (a.tm_in.kind == hd::TMA_NONE) { a.tm_in_g.kind = hd::TMA_NONE; a.tm_out.kind = hd::TMA_NONE; }
}

// The staged warp engine (m = 512, hd_s512.cuh) applies to one line per CTA, all
// residues at once (D = q <= 12), the fast fold (p <= 8) and, for the convolution
// pass, one pair with a short input of a single block (p_g = 1).
bool use_s512(hd_dtype_t dt, const Launch& L) {
  if (dt != HD_C128 || L.m != 512 || L.lines != 1 || (L.flags & HD_FLAG_GENERIC_FFT)) return false;
  if (!L.auto_engine || !L.s512_axis) return false;
  if (L.a.D != L.a.q || L.a.q > hd::kS512QMax) return false;
  if (L.mode == hd::MODE_FWD) return L.a.in_f.p <= 8;
  if (L.mode == hd::MODE_CONV) return L.a.npairs == 1 && L.a.in_f.p <= 8 && L.a.in_g.p == 1;
  return true;
}

// The staged multi-pair convolution pass (MODE_MCONV): N <= 6 pairs or p_g > 1,
// q <= 6, both inputs by TMA.
bool use_s512_mconv(hd_dtype_t dt, const Launch& L) {
  if (dt != HD_C128 || L.m != 512 || L.lines != 1 || (L.flags & HD_FLAG_GENERIC_FFT)) return false;
  if (!L.auto_engine || !L.s512_axis || L.mode != hd::MODE_CONV) return false;
  if (L.a.D != L.a.q || L.a.q > hd::s512_mconv_qmax()) return false;
  return L.a.npairs <= hd::kTmaArrays && L.a.in_f.p <= 8 && L.a.in_g.p <= 8;
}

// The staged m = 128 complex-float engine (hd_s128.cuh): four lines per CTA item
// (C = 4), all residues at once (D = q <= 8), p <= 8, one pair in the convolution pass.
bool use_s128(hd_dtype_t dt, const Launch& L) {
  if (dt != HD_C64 || L.m != 128 || L.lines != 4 || (L.flags & HD_FLAG_GENERIC_FFT)) return false;
  if (!L.auto_engine || !L.s128_axis) return false;
  if (L.a.D != L.a.q || L.a.q > hd::kS128QMax || L.a.in_f.p > 8) return false;
  if (L.mode == hd::MODE_CONV) return L.a.npairs == 1 && L.a.in_g.p <= 8;
  return true;
}

// The batch-grouped forward pass of the m = 128 engine (hd_s128.cuh
// s128_bg_fwd_kernel): four consecutive batch entries x four lines per item, where
// the output keeps the line tile (4) innermost and the batch entries adjacent
// (stride 4 elements), so each output element of an item is 128 contiguous bytes
// (the 3-D fwd_y pass).  Needs tensor-box input loads (prepare_tma first).
bool use_s128_bg(const Launch& L) {
  const PassArgs& a = L.a;
  const LineOut& o = a.out;
  if (L.mode != hd::MODE_FWD || a.q != 5 || a.tm_in.kind != hd::TMA_LINE_TILED) return false;
  if (o.tl != 2 || o.s_l != 1 || o.so_log2 < 30 || o.jd > 0 || o.j0 != 0 || o.s_b != 4) return false;
  if (o.nbi % 4 || a.nbatch % 4 || !a.batch_fastest || L.narrays > hd::kTmaArrays) return false;
  if ((o.s_t | o.s_bo | o.s_js) & 1) return false;
  for (int k = 0; k < (int)L.narrays; ++k)
    if (reinterpret_cast<uintptr_t>(o.ptr[k]) & 15) return false;
  return true;
}

// The 1-D convolution pass of long lines on two-CTA clusters (hd_s512c.cuh): m = 512,
// complex double, all residues (D = q), 12 <= q <= 22, one pair, plain rows.
bool use_s512c(hd_dtype_t dt, const Launch& L) {
  if (dt != HD_C128 || L.m != 512 || L.lines != 1 || L.mode != hd::MODE_CONV || (L.flags & HD_FLAG_GENERIC_FFT))
    return false;
  if (!L.auto_engine || !L.s512c_axis || L.a.D != L.a.q) return false;
  if (L.a.q < hd::kS512cQMin || L.a.q > hd::kS512cQMax) return false;
  const PassArgs& a = L.a;
  return a.npairs == 1 && a.nbatch == 1 && a.in_f.p <= 32 && a.in_g.p <= 32 && a.out.T <= 32 && a.in_f.tl >= 30 && a.in_f.s_j == 1 && a.in_g.tl >= 30 &&
         a.in_g.s_j == 1 && a.out.tl >= 30 && a.out.so_log2 >= 30 && a.out.s_js == 1 && a.in_f.jd <= 0 &&
         a.in_g.jd <= 0 && a.out.jd <= 0;
}

// The 1-D m = 2048 engine (hd_s2048r.cuh): one pair of plain rows per line, every
// residue (D = q <= 8), p <= 8, no output window offset.  HD_NO_S2048R=1: A/B switch.
bool use_s2048r(hd_dtype_t dt, const Launch& L) {
  static const bool off = getenv("HD_NO_S2048R") != nullptr;
  if (off || dt != HD_C128 || L.m != 2048 || L.mode != hd::MODE_CONV || (L.flags & HD_FLAG_GENERIC_FFT)) return false;
  if (!L.auto_engine || !L.s512c_axis || L.a.D != L.a.q || L.a.q > hd::s2048r_qmax()) return false;
  const PassArgs& a = L.a;
  const LineIn &f = a.in_f, &g = a.in_g;
  const LineOut& o = a.out;
  if (a.q > 2 && a.scr == nullptr) return false;  // no residue slots (ws_regions)
  return a.npairs == 1 && a.nbatch == 1 && f.p <= 8 && g.p <= 8 && f.tl >= 30 && f.s_j == 1 && f.jd <= 0 &&
         g.tl >= 30 && g.s_j == 1 && g.jd <= 0 && o.tl >= 30 && o.so_log2 >= 30 && o.s_js == 1 && o.jd <= 0 &&
         o.j0 == 0 && o.L <= (int64_t)o.T * 2048 && f.L < (1 << 30) && g.L < (1 << 30);
}

// The 1-D m = 4096 engine (hd_s4096r.cuh): one pair of plain rows per line, every
// residue (D = q <= 4), p <= 4, output windows.  HD_NO_S4096R=1: A/B switch.
bool use_s4096r(hd_dtype_t dt, const Launch& L) {
  static const bool off = getenv("HD_NO_S4096R") != nullptr;
  if (off || dt != HD_C128 || L.m != 4096 || L.mode != hd::MODE_CONV || (L.flags & HD_FLAG_GENERIC_FFT)) return false;
  if (!L.auto_engine || !L.s512c_axis || L.a.D != L.a.q || L.a.q > hd::s4096r_qmax()) return false;
  const PassArgs& a = L.a;
  const LineIn &f = a.in_f, &g = a.in_g;
  const LineOut& o = a.out;
  if (a.q > 1 && a.scr == nullptr) return false;  // no residue slots (ws_regions)
  return a.npairs == 1 && a.nbatch == 1 && f.p <= hd::s4096r_pmax() && g.p <= hd::s4096r_pmax() && f.tl >= 30 &&
         f.s_j == 1 && f.jd <= 0 && g.tl >= 30 && g.s_j == 1 && g.jd <= 0 && o.tl >= 30 && o.so_log2 >= 30 &&
         o.s_js == 1 && o.jd <= 0 && o.j0 + o.L <= (int64_t)o.T * 4096 && f.L < (1 << 30) && g.L < (1 << 30);
}

hd_status_t launch(hd_ctx* ctx, hd_dtype_t dt, Launch& L, cudaStream_t st) {
  const bool dbl = dt == HD_C128;
  hd::LaunchFn fn = nullptr;
  size_t smem = 0;
  int threads = L.threads;
  const bool s4096r = use_s4096r(dt, L);
  const bool s2048r = !s4096r && use_s2048r(dt, L);
  bool staged = !s2048r && !s4096r && use_s512(dt, L);
  bool mconv = false;
  const bool s128 = use_s128(dt, L);
  const bool s512c = !staged && !s2048r && !s4096r && use_s512c(dt, L);
  if (L.a.fam2 && (!staged || s128 || s512c)) return HD_ERR_UNSUPPORTED;
  if (s4096r) {
    fn = hd::lookup_s4096r();
    threads = hd::s4096r_threads();
    smem = hd::s4096r_smem_bytes();
  } else if (s2048r) {
    fn = hd::lookup_s2048r();
    threads = hd::s2048r_threads();
    smem = hd::s2048r_smem_bytes();
  } else if (s512c) {
    fn = hd::lookup_s512c();
    threads = hd::s512c_threads(L.a.q);
    smem = hd::s512c_smem_bytes();
  } else if (s128) {
    prepare_tma(L, true);
    if (use_s128_bg(L)) {
      fn = hd::lookup_s128_bg(L.mode, L.a.q);
      threads = hd::s128_bg_threads(L.a.q);
      smem = hd::s128_bg_smem_bytes(L.a.q, L.a.M1);
    } else {
      fn = hd::lookup_s128(L.mode, L.a.q, L.a.tm_in.kind, L.a.tm_out.kind, L.a.tm_out.slog);
      threads = 32 * (L.a.q + 1);
      smem = hd::s128_smem_bytes(L.a.q, L.mode, L.a.M1, L.a.tm_in.kind, L.a.tm_out.kind, L.a.in_g.p);
    }
  } else if (!staged && use_s512_mconv(dt, L)) {
    prepare_tma(L);
    mconv = L.a.tm_in.kind == hd::TMA_LINE_TILED || L.a.tm_in.kind == hd::TMA_BULK;
  }
  if (s128 || s512c || s2048r || s4096r) {
    // set above
  } else if (mconv) {
    fn = hd::lookup_s512_mconv(L.a.q);
    threads = 32 * (L.a.q + 1);
    smem = hd::s512_smem_bytes(L.a.q, hd::MODE_MCONV);
  } else if (staged) {
    fn = hd::lookup_s512(L.mode, L.a.q);
    threads = hd::s512_threads(L.a.q, L.mode);
    smem = hd::s512_smem_bytes(L.a.q, L.mode);
    prepare_tma(L, false, true);
    static const int dbg_skip = getenv("HD_DEBUG_SKIP") ? atoi(getenv("HD_DEBUG_SKIP")) : 0;
    L.a.dbg = dbg_skip;
    if (L.a.fam2 && !(L.mode == hd::MODE_FWD && L.a.q == 9 && L.narrays == 1 && L.a.nbatch == 1 &&
                      L.a.tm_in.kind == hd::TMA_BULK && L.a.tm_in_g.kind == hd::TMA_BULK &&
                      L.a.tm_out.kind != hd::TMA_NONE && L.a.tm_out2.kind != hd::TMA_NONE && L.a.out.j0 == 0 &&
                      L.a.out2.j0 == 0))
      return HD_ERR_UNSUPPORTED;  // silently: the caller falls back to one launch per family
  } else {
    if (L.a.fam2) return HD_ERR_UNSUPPORTED;
    fn = hd::lookup_launcher(dbl, L.m, L.mode, L.threads);
    // a 1-D plan validated for a one-CTA-per-line engine (D = q, hd_s2048r / hd_s4096r)
    // that falls back here (e.g. an output window on s2048r) walks its residues in
    // groups that fit (the results do not depend on D)
    while (L.a.D > 1 && pass_smem(elem_bytes(dt), L.a.q, L.lines, L.a.D, L.m, L.nbuf) > hd::kMaxSmem) --L.a.D;
    smem = pass_smem(elem_bytes(dt), L.a.q, L.lines, L.a.D, L.m, L.nbuf);
  }
  if (!fn) return fail(ctx, HD_ERR_UNSUPPORTED, "no kernel instantiation for this m/threads");
  if (smem > hd::kMaxSmem) return fail(ctx, HD_ERR_INVALID, "pass shared memory exceeds 227 KB");
  dim3 grid;
  const int64_t total = L.ngroups * L.nbatch;
  if (L.ngroups < 1 || L.nbatch < 1 || L.narrays > 65535 || total > 0x7fffffffLL)
    return fail(ctx, HD_ERR_UNSUPPORTED, "grid too large for one launch");
  L.a.ngroups = L.ngroups;
  grid.x = (unsigned)total;  // capped to the persistent CTA count by the launcher
  grid.y = 1;
  grid.z = (unsigned)L.narrays;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ctx->profiling) {
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
  }
  // debug: HD_PHASE_PROF=1 prints the staged engine's cycles per warp and work item
  // for the phases 0 wait-load, 1 fold/step 1, 2 barrier, 3 issue next loads,
  // 4 FFTs, 5 barrier, 6 unfold, 7 store + loop
  static const bool phase_prof = getenv("HD_PHASE_PROF") != nullptr;
  static unsigned long long* d_phase = nullptr;
  L.a.phase_prof = nullptr;
  if (phase_prof && use_s512(dt, L)) {
    if (!d_phase) cudaMalloc(&d_phase, 8 * 17 * sizeof(unsigned long long));
    cudaMemsetAsync(d_phase, 0, 8 * 17 * sizeof(unsigned long long), st);
    L.a.phase_prof = d_phase;
  }
  // debug: HD_DEBUG_LAUNCH=1 prints each pass's engine, TMA kinds and shape
  static const bool dbg_launch = getenv("HD_DEBUG_LAUNCH") != nullptr;
  if (dbg_launch)
    fprintf(stderr, "[launch] %-8s engine=%s m=%d C=%d q=%d D=%d items=%lld threads=%d smem=%zu tma in=%d g=%d out=%d\n",
            L.name, s4096r ? "s4096r" : s2048r ? "s2048r" : s512c ? "s512c" : s128 ? "s128" : mconv ? "s512_mconv" : staged ? "s512" : "generic", L.m,
            L.lines, L.a.q, L.a.D,
            (long long)total, threads, smem, L.a.tm_in.kind, L.a.tm_in_g.kind, L.a.tm_out.kind);
  cudaError_t e = fn(L.a, grid, threads, smem, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, L.name);
  if (L.a.phase_prof) {
    unsigned long long h[8 * 17];
    cudaMemcpyAsync(h, d_phase, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const int cw = threads == 384 ? 8 : threads / 32 - 1;  // compute warps (hd_s512.cuh: W8 or q + producer)
    const double n = (double)total * cw;
    fprintf(stderr, "[phase] %-8s", L.name);
    for (int i = 0; i < 8; ++i) fprintf(stderr, " %7.0f", h[i] / n);
    fprintf(stderr, "\n");
    for (int w = 0; w < 16 && w < cw; ++w) {
      fprintf(stderr, "[phase] %-8s warp %2d", L.name, w);
      for (int i = 0; i < 8; ++i) fprintf(stderr, " %7.0f", h[8 * (1 + w) + i] / (double)total);
      fprintf(stderr, "\n");
    }
  }
  if (!ctx->capturing) ctx->launches += 1;
  if (!ctx->capturing) ctx->engine_launches[s4096r ? HD_ENGINE_S4096R : s2048r ? HD_ENGINE_S2048R : s512c ? HD_ENGINE_S512C : s128 ? HD_ENGINE_S128
                       : mconv ? HD_ENGINE_S512_MCONV : staged ? HD_ENGINE_S512 : HD_ENGINE_GENERIC] += 1;
  if (ctx->profiling) {
    cudaEventRecord(e1, st);
    hd_ctx::ProfEntry* pe = nullptr;
    for (auto& p : ctx->prof) if (p.name == L.name) pe = &p;
    if (!pe) { ctx->prof.push_back({}); pe = &ctx->prof.back(); pe->name = L.name; }
    pe->pending.push_back({e0, e1});
    pe->launches += 1;
  }
  return HD_OK;
}
}  // namespace

namespace {

struct Problem {
  hd_dtype_t dt = HD_C128;
  int ndim = 1, N = 1;
  int64_t batch = 1;
  bool shared_g = false;
  const void* f[HD_MAX_PAIRS] = {};
  const void* g[HD_MAX_PAIRS] = {};
  void* h = nullptr;
  AxisInfo ax[HD_MAX_DIM] = {};
  bool s512[HD_MAX_DIM] = {};  // every pass along axis i may run on the staged m = 512 engine
  bool s128[HD_MAX_DIM] = {};  // ... on the staged m = 128 complex-float engine
  hd_plan_t plan{};
  // hd_conv_real fused into the 2-D x passes (fwd_x_f reads the real row pairs, inv_x
  // writes the real split; see PassArgs rp / rs): f real [Lf0][Lf1], h real
  // [Lout0][Lout1], side buffer of Lg0 - 1 rows
  struct RealFuse {
    bool on = false;
    const void* f = nullptr;
    void* h = nullptr;
    void* side = nullptr;
    int64_t Lf0 = 0, A = 0, Lg0 = 0, Lout0 = 0;
  } rf;
};

// One engine per axis: the staged engine's spectral order (lane-major) differs from
// the generic engine's, so the forward and inverse passes of an axis must agree.
// The convolution axis (0) has a single pass, so only that pass's conditions matter.
void choose_engines(Problem& P) {
  for (int i = 0; i < P.ndim; ++i) {
    const AxisInfo& x = P.ax[i];
    bool ok = P.dt == HD_C128 && x.m == 512 && x.lines == 1 && x.auto_engine && x.D == x.q &&
              x.q <= hd::kS512QMax && !(P.plan.flags & HD_FLAG_GENERIC_FFT);
    if (i > 0) ok = ok && x.pf <= 8 && x.pg <= 8;
    P.s512[i] = ok;
    bool ok128 = P.dt == HD_C64 && x.m == 128 && x.lines == 4 && x.auto_engine && x.D == x.q &&
                 x.q <= hd::kS128QMax && x.pf <= 8 && !(P.plan.flags & HD_FLAG_GENERIC_FFT);
    if (i > 0) ok128 = ok128 && x.pg <= 8;
    P.s128[i] = ok128;
  }
}

size_t align256(size_t v) { return (v + 255) / 256 * 256; }

// Workspace regions (elements) of the multi-pass pipeline; returns total bytes.
// Spectral extents tiled by a tile width <= 16 are padded to a multiple of 16.
int64_t pad16(int64_t v) { return cdiv(v, 16) * 16; }
size_t ws_regions(const Problem& P, std::vector<int64_t>& elems) {
  elems.clear();
  const int64_t B = P.batch, Bg = P.shared_g ? 1 : P.batch;
  const AxisInfo* a = P.ax;
  if (P.ndim == 1) {
    // residue slots of the 1-D m = 2048 engine (PassArgs::scr): one CTA per SM or line
    const AxisInfo& x = a[0];
    if (P.dt == HD_C128 && x.m == 2048 && x.q > 2 && x.q <= hd::s2048r_qmax() && P.N == 1) {
      const int64_t ctas = std::min<int64_t>(B, hd::device_sm_count());
      elems.push_back(ctas * 2 * (cdiv(x.q, 2) - 1) * 2048);
    }
    // residue slots of the 1-D m = 4096 engine: q - 1 per CTA (hd_s4096r.cuh)
    if (P.dt == HD_C128 && x.m == 4096 && x.q > 1 && x.q <= hd::s4096r_qmax() && P.N == 1) {
      const int64_t ctas = std::min<int64_t>(B, hd::device_sm_count());
      elems.push_back(ctas * (hd::s4096r_qmax() - 1) * 4096);
    }
  } else if (P.ndim == 2) {
    const int64_t Kxp = pad16(a[1].M1), Sx = a[1].S;
    const int64_t Oyp = cdiv(a[0].O, Sx) * Sx;
    for (int k = 0; k < P.N; ++k) elems.push_back(B * Kxp * a[0].Lf);
    for (int k = 0; k < P.N; ++k) elems.push_back(Bg * Kxp * a[0].Lg);
    elems.push_back(B * Oyp * Kxp);
  } else if (P.ndim == 3) {
    const int64_t Kxp = pad16(a[2].M1), Ky = a[1].M1, Sx = a[2].S;
    const int64_t Oyp = cdiv(a[1].O, Sx) * Sx;
    for (int k = 0; k < P.N; ++k) elems.push_back(B * a[0].Lf * Kxp * a[1].Lf);
    for (int k = 0; k < P.N; ++k) elems.push_back(Bg * a[0].Lg * Kxp * a[1].Lg);
    for (int k = 0; k < P.N; ++k) elems.push_back(B * Ky * Kxp * a[0].Lf);
    for (int k = 0; k < P.N; ++k) elems.push_back(Bg * Ky * Kxp * a[0].Lg);
    elems.push_back(B * a[0].O * Kxp * Ky);
    elems.push_back(B * a[0].O * Oyp * Kxp);
  }
  size_t total = 0;
  for (int64_t e : elems) total += align256((size_t)e * elem_bytes(P.dt));
  return total;
}

// layout helpers (strides in elements)
void in_rows(LineIn& in, int64_t row) { in.tl = 40; in.s_l = row; in.s_j = 1; }
void in_tiled(LineIn& in, int64_t S, int64_t tile) { in.tl = ilog2(S); in.s_t = tile; in.s_l = 1; in.s_j = S; }
void out_rows(LineOut& o, int64_t row) { o.tl = 40; o.s_l = row; o.so_log2 = 40; o.s_jt = 0; o.s_js = 1; }
// lines linear (stride line), element axis tiled by S with tile stride `tile`
void out_elem_tiled(LineOut& o, int64_t line, int64_t S, int64_t tile) {
  o.tl = 40; o.s_l = line; o.so_log2 = ilog2(S); o.s_jt = tile; o.s_js = 1;
}
// lines tiled by S (tile stride `tile`, lane stride 1), element axis plain (stride `elem`)
void out_line_tiled(LineOut& o, int64_t S, int64_t tile, int64_t elem) {
  o.tl = ilog2(S); o.s_t = tile; o.s_l = 1; o.so_log2 = 40; o.s_jt = 0; o.s_js = elem;
}

Launch make_launch(hd_ctx* ctx, const Problem& P, int mode, const char* name, int axis,
                   const void* twm, const void* twM1, const void* twst) {
  const AxisInfo& x = P.ax[axis];
  Launch L;
  std::memset(&L, 0, sizeof(L));
  L.mode = mode;
  L.name = name;
  L.m = x.m;
  L.lines = x.lines;
  L.threads = x.threads;
  L.auto_engine = x.auto_engine;
  L.s512_axis = P.s512[axis];
  L.s128_axis = P.s128[axis];
  L.s512c_axis = P.ndim == 1;
  L.nbuf = (mode == hd::MODE_CONV) ? conv_nbuf(P.N) : 1;
  init_in(L.a.in_f);
  init_in(L.a.in_g);
  init_out(L.a.out);
  L.a.tw_m = twm;
  L.a.tw_M1 = twM1;
  L.a.tw_st = twst;
  L.a.q = x.q;
  L.a.D = x.D;
  L.a.C = x.lines;
  L.a.c_log2 = ilog2(x.lines);
  L.a.M1 = x.M1;
  L.a.npairs = (mode == hd::MODE_CONV) ? P.N : 1;
  L.a.scale = 1.0;
  L.narrays = 1;
  L.flags = P.plan.flags;
  (void)ctx;
  return L;
}

hd_status_t run_pipeline(hd_ctx* ctx, Problem& P, void* ws, size_t ws_bytes, cudaStream_t st) {
  const bool dbl = P.dt == HD_C128;
  const size_t eb = elem_bytes(P.dt);
  const void* twm[HD_MAX_DIM] = {};
  const void* twM1[HD_MAX_DIM] = {};
  const void* twst[HD_MAX_DIM] = {};
  for (int i = 0; i < P.ndim; ++i) {
    hd_status_t s = get_table(ctx, P.ax[i].m, dbl, &twm[i]);
    if (s != HD_OK) return s;
    s = get_stage_table(ctx, P.ax[i].m, dbl, &twst[i]);
    if (s != HD_OK) return s;
    s = get_table(ctx, P.ax[i].M1, dbl, &twM1[i]);
    if (s != HD_OK) return s;
  }
  double scale = 1.0;
  for (int i = 0; i < P.ndim; ++i) scale /= (double)P.ax[i].M1;

  std::vector<int64_t> el;
  const size_t need = ws_regions(P, el);
  if (need > 0) {
    if (!ws) {
      hd_status_t sg = grow_scratch(ctx, &ctx->ws, &ctx->ws_size, need, "cudaMalloc(workspace)");
      if (sg != HD_OK) return sg;
      ws = ctx->ws;
    } else if (ws_bytes < need) {
      return fail(ctx, HD_ERR_WORKSPACE, "workspace too small");
    }
  }
  std::vector<char*> reg;
  {
    char* base = (char*)ws;
    for (int64_t e : el) { reg.push_back(base); base += align256((size_t)e * eb); }
  }
  const int64_t B = P.batch, Bg = P.shared_g ? 1 : P.batch;
  const int N = P.N;
  const AxisInfo* a = P.ax;

  if (P.ndim == 1) {
    const AxisInfo& x = a[0];
    Launch L = make_launch(ctx, P, hd::MODE_CONV, "conv1d", 0, twm[0], twM1[0], twst[0]);
    for (int k = 0; k < N; ++k) { L.a.in_f.ptr[k] = P.f[k]; L.a.in_g.ptr[k] = P.g[k]; }
    L.a.in_f.L = x.Lf; L.a.in_f.p = x.pf; in_rows(L.a.in_f, x.Lf);
    L.a.in_g.L = x.Lg; L.a.in_g.p = x.pg; in_rows(L.a.in_g, P.shared_g ? 0 : x.Lg);
    L.a.out.ptr[0] = P.h; L.a.out.L = x.O; L.a.out.T = x.T; out_rows(L.a.out, x.O);
    L.a.out.j0 = x.o0;
    L.a.scale = scale;
    L.a.nlines = B; L.a.nbatch = 1;
    L.ngroups = cdiv(B, x.lines); L.nbatch = 1;
    if (!reg.empty()) L.a.scr = reg[0];
    return launch(ctx, P.dt, L, st);
  }

  if (P.ndim == 2) {
    const AxisInfo &y = a[0], &x = a[1];
    const int64_t Kx = x.M1, Kxp = pad16(Kx), Cx = x.lines, Cy = y.lines;
    const int64_t Sy = y.S, Sx = x.S;           // X tiles (read by conv_y), Y tiles (read by inv_x)
    const int64_t Oyp = cdiv(y.O, Sx) * Sx;
    char** Xf = &reg[0];
    char** Xg = &reg[N];
    char* Y = reg[2 * N];
    // pass A: forward along x for the rows of every f_k, then every g_k -> X[kx/Sy][y][kx%Sy]
    // (one pair, one batch entry, staged q = 9 x axis: both families in one launch,
    // so the g rows fill the f rows' last wave instead of a launch of their own)
    bool merged = false;
    if (P.s512[1] && x.q == 9 && x.lines == 1 && N == 1 && B == 1 && Bg == 1) {
      Launch L = make_launch(ctx, P, hd::MODE_FWD, "fwd_x", 1, twm[1], twM1[1], twst[1]);
      L.a.in_f.ptr[0] = P.f[0]; L.a.out.ptr[0] = Xf[0];
      L.a.in_f.L = x.Lf; L.a.in_f.p = x.pf; in_rows(L.a.in_f, x.Lf);
      L.a.out.s_b = Kxp * y.Lf; out_elem_tiled(L.a.out, Sy, Sy, y.Lf * Sy);
      L.a.out.L = Kx;
      L.a.nlines = y.Lf; L.a.nbatch = 1;
      L.ngroups = y.Lf; L.nbatch = 1; L.narrays = 1;
      L.a.fam2 = 1;
      L.a.in_g.ptr[0] = P.g[0]; L.a.in_g.L = x.Lg; L.a.in_g.p = x.pg; in_rows(L.a.in_g, x.Lg);
      init_out(L.a.out2);
      L.a.out2.ptr[0] = Xg[0]; L.a.out2.s_b = Kxp * y.Lg; out_elem_tiled(L.a.out2, Sy, Sy, y.Lg * Sy);
      L.a.out2.L = Kx;
      L.a.nlines2 = y.Lg;
      if (P.rf.on) {  // the f rows as real row pairs (hd_conv_real, fused pack)
        L.a.rp = 1;
        L.a.in_f.ptr[0] = P.rf.f;
        L.a.rp_off = P.rf.A * x.Lf;
        L.a.rp_rows = P.rf.Lf0 - P.rf.A;
      }
      hd_status_t s = launch(ctx, P.dt, L, st);
      if (s == HD_OK) merged = true;
      else if (s != HD_ERR_UNSUPPORTED) return s;
    }
    for (int which = 0; which < 2 && !merged; ++which) {
      const int64_t rows = which == 0 ? y.Lf : y.Lg;
      const int64_t len = which == 0 ? x.Lf : x.Lg;
      const int64_t nb = which == 0 ? B : Bg;
      Launch L = make_launch(ctx, P, hd::MODE_FWD, which == 0 ? "fwd_x_f" : "fwd_x_g", 1, twm[1], twM1[1], twst[1]);
      for (int k = 0; k < N; ++k) {
        L.a.in_f.ptr[k] = which == 0 ? P.f[k] : P.g[k];
        L.a.out.ptr[k] = which == 0 ? Xf[k] : Xg[k];
      }
      L.a.in_f.L = len; L.a.in_f.p = which == 0 ? x.pf : x.pg;
      L.a.in_f.nbi = nb; L.a.in_f.s_b = rows * len; in_rows(L.a.in_f, len);
      if (which == 0 && P.rf.on) {  // rows y and y + A of the real f (doubles)
        L.a.rp = 1;
        L.a.in_f.ptr[0] = P.rf.f;
        L.a.rp_off = P.rf.A * len;
        L.a.rp_rows = P.rf.Lf0 - P.rf.A;
      }
      L.a.out.nbi = nb; L.a.out.s_b = Kxp * rows; out_elem_tiled(L.a.out, Sy, Sy, rows * Sy);
      L.a.out.L = Kx;
      L.a.nlines = rows; L.a.nbatch = nb;
      L.ngroups = cdiv(rows, Cx); L.nbatch = nb; L.narrays = N;
      hd_status_t s = launch(ctx, P.dt, L, st);
      if (s != HD_OK) return s;
    }
    // Y: with the staged engine on x, plain rows Y[y][kx] (pass C loads each row with
    // one bulk copy; pass B, compute-bound, stores its columns in 16-byte TMA pieces
    // that L2 merges with the neighbouring columns'); otherwise Y[y/Sx][kx][y%Sx]
    const bool yrows = P.s512[1] && y.lines == 1;
    // pass B: convolution along y for every spectral column (sum over pairs) -> Y
    {
      Launch L = make_launch(ctx, P, hd::MODE_CONV, "conv_y", 0, twm[0], twM1[0], twst[0]);
      for (int k = 0; k < N; ++k) { L.a.in_f.ptr[k] = Xf[k]; L.a.in_g.ptr[k] = Xg[k]; }
      L.a.in_f.L = y.Lf; L.a.in_f.p = y.pf; L.a.in_f.nbi = B;
      L.a.in_f.s_b = Kxp * y.Lf; in_tiled(L.a.in_f, Sy, y.Lf * Sy);
      L.a.in_g.L = y.Lg; L.a.in_g.p = y.pg; L.a.in_g.nbi = B;
      L.a.in_g.s_b = P.shared_g ? 0 : Kxp * y.Lg; in_tiled(L.a.in_g, Sy, y.Lg * Sy);
      L.a.out.ptr[0] = Y; L.a.out.nbi = B; L.a.out.s_b = Oyp * Kxp;
      if (yrows) {  // lines kx (tile width 1), element y at stride Kxp
        L.a.out.tl = 0; L.a.out.s_t = 1; L.a.out.s_l = 1; L.a.out.so_log2 = 40; L.a.out.s_jt = 0;
        L.a.out.s_js = Kxp;
      } else {
        out_elem_tiled(L.a.out, Sx, Sx, Kxp * Sx);
      }
      L.a.out.L = y.O; L.a.out.T = y.T; L.a.out.j0 = y.o0;
      L.a.scale = scale;
      L.a.nlines = Kx; L.a.nbatch = B;
      L.ngroups = cdiv(Kx, Cy); L.nbatch = B;
      hd_status_t s = launch(ctx, P.dt, L, st);
      if (s != HD_OK) return s;
    }
    // pass C: inverse along x for every output row
    {
      Launch L = make_launch(ctx, P, hd::MODE_INV, "inv_x", 1, twm[1], twM1[1], twst[1]);
      L.a.in_f.ptr[0] = Y; L.a.in_f.nbi = B; L.a.in_f.s_b = Oyp * Kxp;
      if (yrows) in_rows(L.a.in_f, Kxp);
      else in_tiled(L.a.in_f, Sx, Kxp * Sx);
      L.a.in_f.L = Kx;
      L.a.out.ptr[0] = P.h; L.a.out.nbi = B; L.a.out.s_b = y.O * x.O; out_rows(L.a.out, x.O);
      L.a.out.L = x.O; L.a.out.T = x.T; L.a.out.j0 = x.o0;
      if (P.rf.on) {  // real split into h (doubles) and the side buffer
        L.a.rs = 1;
        L.a.out.ptr[0] = P.rf.h;
        L.a.rs_A = P.rf.A;
        L.a.rs_side_rows = P.rf.Lg0 - 1;
        L.a.rs_rows = P.rf.Lout0;
        L.a.rs_side = P.rf.side;
      }
      L.a.nlines = y.O; L.a.nbatch = B;
      L.ngroups = cdiv(y.O, Cx); L.nbatch = B;
      return launch(ctx, P.dt, L, st);
    }
  }

  // ndim == 3: axes z (0), y (1), x (2)
  const AxisInfo &z = a[0], &y = a[1], &x = a[2];
  const int64_t Kx = x.M1, Kxp = pad16(Kx), Ky = y.M1;
  const int64_t Cx = x.lines, Cy = y.lines, Cz = z.lines;
  const int64_t S1 = y.S, S0 = z.S, Sx = x.S;  // X1 / Zl kx-tiles, XY kx-tiles, W y-tiles
  const int64_t Oyp = cdiv(y.O, Sx) * Sx;
  char** X1f = &reg[0];
  char** X1g = &reg[N];
  char** XYf = &reg[2 * N];
  char** XYg = &reg[3 * N];
  char* Zl = reg[4 * N];
  char* W = reg[4 * N + 1];
  for (int which = 0; which < 2; ++which) {
    const int64_t Fz = which == 0 ? z.Lf : z.Lg, Fy = which == 0 ? y.Lf : y.Lg, Fx = which == 0 ? x.Lf : x.Lg;
    const int64_t nb = which == 0 ? B : Bg;
    // pass 1: forward along x; batch = (b, z) combined, lines = y -> X1[b][z][kx/S1][y][kx%S1]
    {
      Launch L = make_launch(ctx, P, hd::MODE_FWD, which == 0 ? "fwd_x_f" : "fwd_x_g", 2, twm[2], twM1[2], twst[2]);
      for (int k = 0; k < N; ++k) {
        L.a.in_f.ptr[k] = which == 0 ? P.f[k] : P.g[k];
        L.a.out.ptr[k] = which == 0 ? X1f[k] : X1g[k];
      }
      L.a.in_f.L = Fx; L.a.in_f.p = which == 0 ? x.pf : x.pg;
      L.a.in_f.nbi = nb * Fz; L.a.in_f.s_b = Fy * Fx; in_rows(L.a.in_f, Fx);
      L.a.out.nbi = nb * Fz; L.a.out.s_b = Kxp * Fy; out_elem_tiled(L.a.out, S1, S1, Fy * S1);
      L.a.out.L = Kx;
      L.a.nlines = Fy; L.a.nbatch = nb * Fz;
      L.ngroups = cdiv(Fy, Cx); L.nbatch = nb * Fz; L.narrays = N;
      hd_status_t s = launch(ctx, P.dt, L, st);
      if (s != HD_OK) return s;
    }
    // pass 2: forward along y; batch = (b, z), lines = kx -> XY[b][ky][kx/S0][z][kx%S0]
    {
      Launch L = make_launch(ctx, P, hd::MODE_FWD, which == 0 ? "fwd_y_f" : "fwd_y_g", 1, twm[1], twM1[1], twst[1]);
      for (int k = 0; k < N; ++k) {
        L.a.in_f.ptr[k] = which == 0 ? X1f[k] : X1g[k];
        L.a.out.ptr[k] = which == 0 ? XYf[k] : XYg[k];
      }
      L.a.in_f.L = Fy; L.a.in_f.p = which == 0 ? y.pf : y.pg;
      L.a.in_f.nbi = Fz; L.a.in_f.s_bo = Fz * Kxp * Fy; L.a.in_f.s_b = Kxp * Fy;
      in_tiled(L.a.in_f, S1, Fy * S1);
      L.a.out.nbi = Fz; L.a.out.s_bo = Ky * Kxp * Fz; L.a.out.s_b = S0;
      out_line_tiled(L.a.out, S0, Fz * S0, Kxp * Fz);
      L.a.out.L = Ky;
      L.a.batch_fastest = 1;
      L.a.nlines = Kx; L.a.nbatch = nb * Fz;
      L.ngroups = cdiv(Kx, Cy); L.nbatch = nb * Fz; L.narrays = N;
      hd_status_t s = launch(ctx, P.dt, L, st);
      if (s != HD_OK) return s;
    }
  }
  // pass 3: convolution along z; batch = (b, ky), lines = kx -> Zl[b][z][kx/S1][ky][kx%S1]
  {
    Launch L = make_launch(ctx, P, hd::MODE_CONV, "conv_z", 0, twm[0], twM1[0], twst[0]);
    for (int k = 0; k < N; ++k) { L.a.in_f.ptr[k] = XYf[k]; L.a.in_g.ptr[k] = XYg[k]; }
    L.a.in_f.L = z.Lf; L.a.in_f.p = z.pf; L.a.in_f.nbi = Ky; L.a.in_f.s_bo = Ky * Kxp * z.Lf;
    L.a.in_f.s_b = Kxp * z.Lf; in_tiled(L.a.in_f, S0, z.Lf * S0);
    L.a.in_g.L = z.Lg; L.a.in_g.p = z.pg; L.a.in_g.nbi = Ky; L.a.in_g.s_bo = P.shared_g ? 0 : Ky * Kxp * z.Lg;
    L.a.in_g.s_b = Kxp * z.Lg; in_tiled(L.a.in_g, S0, z.Lg * S0);
    L.a.out.ptr[0] = Zl; L.a.out.nbi = Ky; L.a.out.s_bo = z.O * Kxp * Ky; L.a.out.s_b = S1;
    out_line_tiled(L.a.out, S1, Ky * S1, Kxp * Ky);
    L.a.out.L = z.O; L.a.out.T = z.T; L.a.out.j0 = z.o0;
    L.a.scale = scale;
    L.a.batch_fastest = 1;
    L.a.nlines = Kx; L.a.nbatch = B * Ky;
    L.ngroups = cdiv(Kx, Cz); L.nbatch = B * Ky;
    hd_status_t s = launch(ctx, P.dt, L, st);
    if (s != HD_OK) return s;
  }
  // pass 4: inverse along y; batch = (b, z_out) combined, lines = kx -> W[b][z][y/Sx][kx][y%Sx]
  {
    Launch L = make_launch(ctx, P, hd::MODE_INV, "inv_y", 1, twm[1], twM1[1], twst[1]);
    L.a.in_f.ptr[0] = Zl; L.a.in_f.nbi = B * z.O; L.a.in_f.s_b = Kxp * Ky; in_tiled(L.a.in_f, S1, Ky * S1);
    L.a.in_f.L = Ky;
    L.a.out.ptr[0] = W; L.a.out.nbi = B * z.O; L.a.out.s_b = Oyp * Kxp; out_elem_tiled(L.a.out, Sx, Sx, Kxp * Sx);
    L.a.out.L = y.O; L.a.out.T = y.T; L.a.out.j0 = y.o0;
    L.a.nlines = Kx; L.a.nbatch = B * z.O;
    L.ngroups = cdiv(Kx, Cy); L.nbatch = B * z.O;
    hd_status_t s = launch(ctx, P.dt, L, st);
    if (s != HD_OK) return s;
  }
  // pass 5: inverse along x; batch = (b, z_out), lines = y_out
  {
    Launch L = make_launch(ctx, P, hd::MODE_INV, "inv_x", 2, twm[2], twM1[2], twst[2]);
    L.a.in_f.ptr[0] = W; L.a.in_f.nbi = B * z.O; L.a.in_f.s_b = Oyp * Kxp; in_tiled(L.a.in_f, Sx, Kxp * Sx);
    L.a.in_f.L = Kx;
    L.a.out.ptr[0] = P.h; L.a.out.nbi = B * z.O; L.a.out.s_b = y.O * x.O; out_rows(L.a.out, x.O);
    L.a.out.L = x.O; L.a.out.T = x.T; L.a.out.j0 = x.o0;
    L.a.nlines = y.O; L.a.nbatch = B * z.O;
    L.ngroups = cdiv(y.O, Cx); L.nbatch = B * z.O;
    return launch(ctx, P.dt, L, st);
  }
}

std::string problem_key(hd_dtype_t dt, int ndim, int N, int64_t batch, const int64_t* Lf,
                        const int64_t* Lg, const int64_t* M, uint32_t flags) {
  std::string k = std::to_string((int)dt) + "|" + std::to_string(ndim) + "|" + std::to_string(N) +
                  "|" + std::to_string(batch) + "|" + std::to_string(flags);
  for (int i = 0; i < ndim; ++i)
    k += "|" + std::to_string(Lf[i]) + "," + std::to_string(Lg[i]) + "," +
         std::to_string(M ? M[i] : 0);
  return k;
}

// Build a Problem from the public arguments (plan: explicit, cached or default).
hd_status_t setup(hd_ctx* ctx, Problem& P, hd_dtype_t dt, int ndim, int N, int64_t batch,
                  const void* const* f, const int64_t* Lf, const void* const* g, const int64_t* Lg,
                  void* h, const int64_t* M, const hd_plan_t* plan, bool need_ptrs = true,
                  const int64_t* win_lo = nullptr, const int64_t* win_n = nullptr) {
  if (!ctx) return fail(nullptr, HD_ERR_INVALID, "null context");
  if (dt != HD_C64 && dt != HD_C128) return fail(ctx, HD_ERR_INVALID, "dtype must be HD_C64 or HD_C128");
  if (ndim < 1 || ndim > HD_MAX_DIM) return fail(ctx, HD_ERR_INVALID, "ndim must be 1, 2 or 3");
  if (N < 1 || N > HD_MAX_PAIRS) return fail(ctx, HD_ERR_INVALID, "N must be in [1, 16]");
  if (batch < 1) return fail(ctx, HD_ERR_INVALID, "batch must be >= 1");
  if (!Lf || !Lg) return fail(ctx, HD_ERR_INVALID, "null extents");
  P.dt = dt; P.ndim = ndim; P.N = N; P.batch = batch;
  if (need_ptrs) {
    if (!f || !g || !h) return fail(ctx, HD_ERR_INVALID, "null data pointer");
    for (int k = 0; k < N; ++k) {
      if (!f[k] || !g[k]) return fail(ctx, HD_ERR_INVALID, "null input pointer");
      const uintptr_t al = elem_bytes(dt);
      if (((uintptr_t)f[k] % al) || ((uintptr_t)g[k] % al) || ((uintptr_t)h % al))
        return fail(ctx, HD_ERR_INVALID, "misaligned data pointer");
      if (f[k] == h || g[k] == h) return fail(ctx, HD_ERR_INVALID, "h must not alias f or g");
      P.f[k] = f[k]; P.g[k] = g[k];
    }
    P.h = h;
  }
  hd_plan_t pl;
  if (plan) {
    pl = *plan;
  } else {
    auto it = ctx->plan_cache.find(problem_key(dt, ndim, N, batch, Lf, Lg, M, 0));
    if (it != ctx->plan_cache.end()) pl = it->second;
    else {
      hd_status_t s = default_plan(ctx, dt, ndim, N, Lf, Lg, M, &pl);
      if (s != HD_OK) return s;
    }
  }
  P.shared_g = (pl.flags & HD_FLAG_SHARED_G) != 0;
  hd_status_t s = complete_plan(ctx, dt, ndim, N, Lf, Lg, M, &pl, P.ax);
  if (s != HD_OK) return s;
  s = apply_window(ctx, ndim, win_lo, win_n, P.ax);
  if (s != HD_OK) return s;
  P.plan = pl;
  choose_engines(P);
  return HD_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int hd_abi_version(void) { return HD_ABI_VERSION; }

hd_status_t hd_create(hd_ctx_t* out, int device) {
  if (!out) return fail(nullptr, HD_ERR_INVALID, "null ctx pointer");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return fail(nullptr, HD_ERR_CUDA, "no CUDA device available");
  if (device < 0 || device >= n) return fail(nullptr, HD_ERR_INVALID, "device ordinal out of range");
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaSetDevice");
  hd_ctx* c = new hd_ctx();
  c->device = device;
  *out = c;
  return HD_OK;
}

hd_status_t hd_destroy(hd_ctx_t ctx) {
  if (!ctx) return HD_OK;
  cudaSetDevice(ctx->device);
  hd::dist_release(ctx);
  for (auto& kv : ctx->tw64) cudaFree(kv.second);
  for (auto& kv : ctx->tw32) cudaFree(kv.second);
  for (auto& kv : ctx->st64) cudaFree(kv.second);
  for (auto& kv : ctx->perm) cudaFree(kv.second);
  for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
  if (ctx->capture_stream) cudaStreamDestroy(ctx->capture_stream);
  for (auto& kv : ctx->st32) cudaFree(kv.second);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->io) cudaFree(ctx->io);
  if (ctx->rio) cudaFree(ctx->rio);
  for (auto& sl : ctx->hslot) {
    if (sl.st) { cudaStreamSynchronize(sl.st); cudaStreamDestroy(sl.st); }
    if (sl.io) cudaFree(sl.io);
  }
  if (ctx->scratch_done) cudaEventDestroy(ctx->scratch_done);
  for (auto& p : ctx->prof)
    for (auto& ev : p.pending) { cudaEventDestroy(ev.first); cudaEventDestroy(ev.second); }
  delete ctx;
  return HD_OK;
}

const char* hd_last_error(hd_ctx_t ctx) {
  return ctx ? ctx->err.c_str() : g_tls_error.c_str();
}

hd_status_t hd_plan_default(hd_dtype_t dtype, int32_t ndim, int32_t npairs, const int64_t* Lf,
                            const int64_t* Lg, const int64_t* M, hd_plan_t* out) {
  if (!Lf || !Lg || !out) return fail(nullptr, HD_ERR_INVALID, "null argument");
  if (dtype != HD_C64 && dtype != HD_C128) return fail(nullptr, HD_ERR_INVALID, "bad dtype");
  if (npairs < 1 || npairs > HD_MAX_PAIRS) return fail(nullptr, HD_ERR_INVALID, "N must be in [1, 16]");
  return default_plan(nullptr, dtype, ndim, npairs, Lf, Lg, M, out);
}

hd_status_t hd_plan_complete(hd_dtype_t dtype, int32_t ndim, int32_t npairs, const int64_t* Lf,
                             const int64_t* Lg, const int64_t* M, hd_plan_t* plan) {
  if (!Lf || !Lg || !plan) return fail(nullptr, HD_ERR_INVALID, "null argument");
  AxisInfo ax[HD_MAX_DIM];
  return complete_plan(nullptr, dtype, ndim, npairs, Lf, Lg, M, plan, ax);
}

hd_status_t hd_spectral_permutation(int32_t m, int32_t* perm) {
  if (!perm || !is_pow2(m) || m < 2 || m > 4096)
    return fail(nullptr, HD_ERR_INVALID, "m must be a power of two in [2, 4096]");
  // radix schedule of hd_device.cuh Sched<m>: radix-8 stages then one radix-4/2
  const int lg = ilog2(m);
  std::vector<int> rad;
  for (int i = 0; i < lg / 3; ++i) rad.push_back(8);
  if (lg % 3 == 1) rad.push_back(2);
  if (lg % 3 == 2) rad.push_back(4);
  // DIF: position j*(n/R) + o' of a size-n block holds R*perm_{n/R}(o') + j
  for (int pos = 0; pos < m; ++pos) {
    int n = m, p = pos, mul = 1, freq = 0;
    for (size_t s = 0; s < rad.size(); ++s) {
      const int R = rad[s];
      const int sub = n / R;
      const int j = p / sub;
      freq += mul * j;
      mul *= R;
      p %= sub;
      n = sub;
    }
    perm[pos] = freq;
  }
  return HD_OK;
}

size_t hd_workspace_bytes(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t npairs, int64_t batch,
                          const int64_t* Lf, const int64_t* Lg, const int64_t* M,
                          const hd_plan_t* plan) {
  Problem P;
  if (setup(ctx, P, dtype, ndim, npairs, batch, nullptr, Lf, nullptr, Lg, nullptr, M, plan, false) != HD_OK)
    return 0;
  std::vector<int64_t> el;
  return ws_regions(P, el);
}

static hd_status_t run_graph_or_pipeline(hd_ctx_t ctx, Problem& P, hd_dtype_t dt, int ndim, int N, int64_t batch,
                                         const int64_t* Lf, const int64_t* Lg, void* h, const int64_t* M,
                                         const Problem::RealFuse* rf, void* ws, size_t ws_bytes, void* stream);

static hd_status_t run_entry(hd_ctx_t ctx, hd_dtype_t dt, int ndim, int N, int64_t batch,
                             const void* const* f, const int64_t* Lf, const void* const* g,
                             const int64_t* Lg, void* h, const int64_t* M, const hd_plan_t* plan,
                             void* ws, size_t ws_bytes, void* stream, const int64_t* win_lo = nullptr,
                             const int64_t* win_n = nullptr, const Problem::RealFuse* rf = nullptr) {
  Problem P;
  hd_status_t s = setup(ctx, P, dt, ndim, N, batch, f, Lf, g, Lg, h, M, plan, true, win_lo, win_n);
  if (s != HD_OK) return s;
  if (rf) P.rf = *rf;
  std::lock_guard<std::recursive_mutex> lk(ctx->mu);
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  if (ws) return run_graph_or_pipeline(ctx, P, dt, ndim, N, batch, Lf, Lg, h, M, rf, ws, ws_bytes, stream);
  s = scratch_acquire(ctx, st);
  if (s != HD_OK) return s;
  s = run_graph_or_pipeline(ctx, P, dt, ndim, N, batch, Lf, Lg, h, M, rf, ws, ws_bytes, stream);
  hd_status_t r = scratch_release(ctx, st);
  return s != HD_OK ? s : r;
}

static hd_status_t run_graph_or_pipeline(hd_ctx_t ctx, Problem& P, hd_dtype_t dt, int ndim, int N, int64_t batch,
                                         const int64_t* Lf, const int64_t* Lg, void* h, const int64_t* M,
                                         const Problem::RealFuse* rf, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  hd_status_t s;
  if (!(P.plan.flags & HD_FLAG_GRAPH) || rf || ctx->profiling) return run_pipeline(ctx, P, ws, ws_bytes, st);
  // HD_FLAG_GRAPH: replay the captured launches of an identical earlier call
  std::string key = problem_key(dt, ndim, N, batch, Lf, Lg, M, P.plan.flags);
  char buf[64];
  auto add = [&](const void* p) { snprintf(buf, sizeof(buf), "|%p", p); key += buf; };
  for (int k = 0; k < N; ++k) { add(P.f[k]); add(P.g[k]); }
  add(h); add(ws); add(stream);
  key += "|" + std::to_string(ws_bytes);
  for (int i = 0; i < ndim; ++i) {
    const AxisInfo& x = P.ax[i];
    key += "|" + std::to_string(x.m) + "," + std::to_string(x.lines) + "," + std::to_string(x.S) + "," +
           std::to_string(x.D) + "," + std::to_string(x.threads) + "," + std::to_string(x.auto_engine) + "," +
           std::to_string(x.o0) + "," + std::to_string(x.O);
  }
  auto it = ctx->graphs.find(key);
  if (it != ctx->graphs.end()) {
    cudaError_t e = cudaGraphLaunch(it->second, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaGraphLaunch");
    ctx->graph_replays += 1;
    return HD_OK;
  }
  s = run_pipeline(ctx, P, ws, ws_bytes, st);  // this call's result
  if (s != HD_OK) return s;
  if (!ctx->capture_stream) {
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->capture_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamCreate(capture)");
  }
  cudaError_t e = cudaStreamBeginCapture(ctx->capture_stream, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamBeginCapture");
  ctx->capturing = true;
  hd_status_t sc = run_pipeline(ctx, P, ws, ws_bytes, ctx->capture_stream);
  ctx->capturing = false;
  cudaGraph_t gr = nullptr;
  e = cudaStreamEndCapture(ctx->capture_stream, &gr);
  if (sc != HD_OK) { if (gr) cudaGraphDestroy(gr); return sc; }
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamEndCapture");
  cudaGraphExec_t ex = nullptr;
  e = cudaGraphInstantiate(&ex, gr, 0);
  cudaGraphDestroy(gr);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaGraphInstantiate");
  if (ctx->graphs.size() >= 64) {  // bounded cache: start over rather than grow without limit
    for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
    ctx->graphs.clear();
  }
  ctx->graphs[key] = ex;
  return HD_OK;
}

hd_status_t hd_conv_window(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N, int64_t batch,
                          const void* const* f, const int64_t* Lf, const void* const* g,
                          const int64_t* Lg, void* h, const int64_t* M, const int64_t* win_lo,
                          const int64_t* win_n, const hd_plan_t* plan, void* ws, size_t ws_bytes,
                          void* stream) {
  if (!win_lo || !win_n) return fail(ctx, HD_ERR_INVALID, "null window");
  return run_entry(ctx, dtype, ndim, N, batch, f, Lf, g, Lg, h, M, plan, ws, ws_bytes, stream, win_lo, win_n);
}

// The real path's pack / unpack fuse into the x passes when the packed 2-D problem
// runs its x axis on the staged engine with q = 9 (the compile-time-q kernel that
// has the real-pair / real-split modes) and every real row moves by 16-byte bulk copies.
static bool real_fusable(hd_ctx_t ctx, hd_dtype_t dtype, int ndim, int64_t batch, const void* f, const int64_t* Lz,
                         const int64_t* Lf, const int64_t* Lg, const void* h, const hd_plan_t* plan) {
  if (dtype != HD_C128 || ndim != 2 || batch != 1) return false;
  static const bool off = getenv("HD_NO_REAL_FUSE") != nullptr;  // A/B switch
  if (off) return false;
  const int64_t Lout1 = Lf[1] + Lg[1] - 1;
  if ((Lf[1] & 1) || (Lout1 & 1) || (reinterpret_cast<uintptr_t>(f) & 15) || (reinterpret_cast<uintptr_t>(h) & 15))
    return false;
  Problem P;
  const void* fa[1] = {f};
  const void* ga[1] = {f};
  if (setup(ctx, P, dtype, 2, 1, 1, fa, Lz, ga, Lg, nullptr, nullptr, plan, false) != HD_OK) return false;
  const AxisInfo& x = P.ax[1];
  return P.s512[1] && x.q == 9 && x.lines == 1 && x.D == 9 && x.pf <= 8 && x.o0 == 0 && x.O == Lout1;
}

static hd_status_t real_locked(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int64_t batch, const void* f,
                               const int64_t* Lf, const void* g, const int64_t* Lg, void* h, const hd_plan_t* plan,
                               void* stream, int64_t A, const int64_t* Lz, int64_t rest_f, int64_t rest_g,
                               int64_t rest_o, size_t bz, size_t bgc, int64_t Ow0, int64_t Lout0);

hd_status_t hd_conv_real(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int64_t batch, const void* f,
                         const int64_t* Lf, const void* g, const int64_t* Lg, void* h, const hd_plan_t* plan,
                         void* stream) {
  if (!ctx) return fail(nullptr, HD_ERR_INVALID, "null context");
  if (!f || !g || !h || !Lf || !Lg) return fail(ctx, HD_ERR_INVALID, "null argument");
  if (dtype != HD_C64 && dtype != HD_C128) return fail(ctx, HD_ERR_INVALID, "dtype must be HD_C64 or HD_C128");
  if (ndim < 1 || ndim > HD_MAX_DIM || batch < 1) return fail(ctx, HD_ERR_INVALID, "bad ndim or batch");
  for (int i = 0; i < ndim; ++i)
    if (Lf[i] < 1 || Lg[i] < 1) return fail(ctx, HD_ERR_INVALID, "extents must be >= 1");
  const bool dbl = dtype == HD_C128;
  const size_t rb = dbl ? 8 : 4, cb = 2 * rb;
  // z: the two halves of f along axis 0 (A = ceil(Lf0 / 2) rows each, zero-padded)
  const int64_t A = (Lf[0] + 1) / 2;
  int64_t Lz[HD_MAX_DIM];
  int64_t rest_f = 1, rest_g = 1, rest_o = 1;
  for (int i = 0; i < ndim; ++i) Lz[i] = Lf[i];
  Lz[0] = A;
  for (int i = 1; i < ndim; ++i) { rest_f *= Lf[i]; rest_g *= Lg[i]; rest_o *= Lf[i] + Lg[i] - 1; }
  const int64_t Ow0 = A + Lg[0] - 1, Lout0 = Lf[0] + Lg[0] - 1;
  const size_t bz = align256((size_t)(batch * A * rest_f) * cb);
  const size_t bgc = align256((size_t)(batch * Lg[0] * rest_g) * cb);
  const size_t bw = align256((size_t)(batch * Ow0 * rest_o) * cb);
  cudaStream_t st = (cudaStream_t)stream;
  std::lock_guard<std::recursive_mutex> lk(ctx->mu);  // held while rio is in use
  cudaSetDevice(ctx->device);
  hd_status_t sg = grow_scratch(ctx, &ctx->rio, &ctx->rio_size, bz + bgc + bw, "cudaMalloc(real path)");
  if (sg != HD_OK) return sg;
  sg = scratch_acquire(ctx, st);
  if (sg != HD_OK) return sg;
  hd_status_t sr = real_locked(ctx, dtype, ndim, batch, f, Lf, g, Lg, h, plan, stream, A, Lz, rest_f, rest_g, rest_o,
                               bz, bgc, Ow0, Lout0);
  sg = scratch_release(ctx, st);
  return sr != HD_OK ? sr : sg;
}

static hd_status_t real_locked(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int64_t batch, const void* f,
                               const int64_t* Lf, const void* g, const int64_t* Lg, void* h, const hd_plan_t* plan,
                               void* stream, int64_t A, const int64_t* Lz, int64_t rest_f, int64_t rest_g,
                               int64_t rest_o, size_t bz, size_t bgc, int64_t Ow0, int64_t Lout0) {
  const bool dbl = dtype == HD_C128;
  cudaStream_t st = (cudaStream_t)stream;
  char* z = (char*)ctx->rio;
  char* gc = z + bz;
  char* w = gc + bgc;
  if (real_fusable(ctx, dtype, ndim, batch, f, Lz, Lf, Lg, h, plan)) {
    // pack / unpack inside the x passes: only g is promoted; the Im rows of w that
    // overlap Re rows (Lg0 - 1 of them) go to a side buffer (w's space) and are added
    cudaError_t e = hd::launch_real_to_complex(dbl, g, gc, Lg[0] * rest_g, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "real to complex");
    Problem::RealFuse rf;
    rf.on = true; rf.f = f; rf.h = h; rf.side = w;
    rf.Lf0 = Lf[0]; rf.A = A; rf.Lg0 = Lg[0]; rf.Lout0 = Lout0;
    const void* fa[1] = {f};
    const void* ga[1] = {gc};
    hd_status_t s = run_entry(ctx, dtype, ndim, 1, 1, fa, Lz, ga, Lg, h, nullptr, plan, nullptr, 0, stream,
                              nullptr, nullptr, &rf);
    if (s != HD_OK) return s;
    e = hd::launch_real_fixup(w, h, Lg[0] - 1, A, Lout0, rest_o, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "real fix-up");
    return HD_OK;
  }
  cudaError_t e = hd::launch_real_pack(dbl, f, z, Lf[0], A, rest_f, batch, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "real pack");
  e = hd::launch_real_to_complex(dbl, g, gc, batch * Lg[0] * rest_g, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "real to complex");
  const void* fa[1] = {z};
  const void* ga[1] = {gc};
  hd_status_t s = run_entry(ctx, dtype, ndim, 1, batch, fa, Lz, ga, Lg, w, nullptr, plan, nullptr, 0, stream);
  if (s != HD_OK) return s;
  e = hd::launch_real_unpack(dbl, w, h, Lout0, Ow0, A, rest_o, batch, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "real unpack");
  return HD_OK;
}

hd_status_t hd_conv1d(hd_ctx_t ctx, hd_dtype_t dtype, int64_t batch, const void* f, int64_t Lf,
                      const void* g, int64_t Lg, void* h, int64_t M, const hd_plan_t* plan,
                      void* ws, size_t ws_bytes, void* stream) {
  const void* fa[1] = {f};
  const void* ga[1] = {g};
  int64_t Mv[1] = {M};
  return run_entry(ctx, dtype, 1, 1, batch, fa, &Lf, ga, &Lg, h, Mv, plan, ws, ws_bytes, stream);
}

hd_status_t hd_conv2d(hd_ctx_t ctx, hd_dtype_t dtype, int64_t batch, const void* f, const int64_t Lf[2],
                      const void* g, const int64_t Lg[2], void* h, const int64_t M[2],
                      const hd_plan_t* plan, void* ws, size_t ws_bytes, void* stream) {
  const void* fa[1] = {f};
  const void* ga[1] = {g};
  return run_entry(ctx, dtype, 2, 1, batch, fa, Lf, ga, Lg, h, M, plan, ws, ws_bytes, stream);
}

hd_status_t hd_conv3d(hd_ctx_t ctx, hd_dtype_t dtype, int64_t batch, const void* f, const int64_t Lf[3],
                      const void* g, const int64_t Lg[3], void* h, const int64_t M[3],
                      const hd_plan_t* plan, void* ws, size_t ws_bytes, void* stream) {
  const void* fa[1] = {f};
  const void* ga[1] = {g};
  return run_entry(ctx, dtype, 3, 1, batch, fa, Lf, ga, Lg, h, M, plan, ws, ws_bytes, stream);
}

hd_status_t hd_multiconv(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N,
                         const void* const* f, const int64_t* Lf, const void* const* g,
                         const int64_t* Lg, void* h, const int64_t* M, const hd_plan_t* plan,
                         void* ws, size_t ws_bytes, void* stream) {
  return run_entry(ctx, dtype, ndim, N, 1, f, Lf, g, Lg, h, M, plan, ws, ws_bytes, stream);
}

static hd_status_t explicit_locked(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N, const void* const* f,
                                   const int64_t* Lf, const void* const* g, const int64_t* Lg, void* h, Problem& E,
                                   const int64_t* Me, const int64_t* Lo, size_t inb, size_t wsb, cudaStream_t st);

hd_status_t hd_conv_explicit(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N,
                             const void* const* f, const int64_t* Lf, const void* const* g,
                             const int64_t* Lg, void* h, const hd_plan_t* plan, void* stream) {
  // Validate against the hybrid problem first (also gives the user's m, C, S).  A plan
  // flagged HD_FLAG_EXPLICIT_PLAN is the padded problem's own (hd_tune_explicit).
  const bool own = plan && (plan->flags & HD_FLAG_EXPLICIT_PLAN);
  Problem H;
  hd_status_t s = setup(ctx, H, dtype, ndim, N, 1, f, Lf, g, Lg, h, nullptr, own ? nullptr : plan);
  if (s != HD_OK) return s;
  std::lock_guard<std::recursive_mutex> lk(ctx->mu);
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t eb = elem_bytes(dtype);
  int64_t Me[HD_MAX_DIM], Lo[HD_MAX_DIM];
  int64_t nin = 1;
  for (int i = 0; i < ndim; ++i) {
    Lo[i] = Lf[i] + Lg[i] - 1;
    Me[i] = 1;
    while (Me[i] < Lo[i]) Me[i] *= 2;
    nin *= Me[i];
  }
  // explicit plan: the caller's own (HD_FLAG_EXPLICIT_PLAN), else the tuned one cached
  // by hd_tune_explicit, else the hybrid plan's m (capped by M_exp), C, S; D reduced
  // until the pass fits shared memory
  hd_plan_t pe = H.plan;
  if (own) {
    pe = *plan;
  } else if (!plan) {
    auto it = ctx->plan_cache.find(problem_key(dtype, ndim, N, 1, Lf, Lg, nullptr, HD_FLAG_EXPLICIT_PLAN));
    if (it != ctx->plan_cache.end()) pe = it->second;
  }
  pe.flags = HD_FLAG_ALLOW_ALIAS;
  for (int i = 0; i < ndim; ++i) {
    hd_axis_plan_t& a = pe.axis[i];
    a.m = (int)std::min<int64_t>(a.m, Me[i]);
    const int q = (int)(Me[i] / a.m);
    const int lines = lines_for(a, i, ndim);
    const int nbuf = (i == 0) ? conv_nbuf(N) : 1;
    if (!own || a.D <= 0 || a.D > q) a.D = q;
    while (a.D > 1 && pass_smem(eb, q, lines, a.D, a.m, nbuf) > hd::kMaxSmem) --a.D;
  }
  // scratch: N padded f, N padded g, padded output, pipeline workspace
  Problem E;
  E.dt = dtype; E.ndim = ndim; E.N = N; E.batch = 1;
  s = complete_plan(ctx, dtype, ndim, N, Me, Me, Me, &pe, E.ax);
  if (s != HD_OK) return s;
  E.plan = pe;
  std::vector<int64_t> el;
  const size_t wsb = ws_regions(E, el);
  const size_t inb = align256((size_t)nin * eb);
  const size_t need = (2 * N + 1) * inb + wsb;
  s = grow_scratch(ctx, &ctx->io, &ctx->io_size, need, "cudaMalloc(explicit scratch)");
  if (s != HD_OK) return s;
  s = scratch_acquire(ctx, st);
  if (s != HD_OK) return s;
  s = explicit_locked(ctx, dtype, ndim, N, f, Lf, g, Lg, h, E, Me, Lo, inb, wsb, st);
  hd_status_t r = scratch_release(ctx, st);
  return s != HD_OK ? s : r;
}

static hd_status_t explicit_locked(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N, const void* const* f,
                                   const int64_t* Lf, const void* const* g, const int64_t* Lg, void* h, Problem& E,
                                   const int64_t* Me, const int64_t* Lo, size_t inb, size_t wsb, cudaStream_t st) {
  hd_status_t s;
  char* base = (char*)ctx->io;
  int64_t L3[3], P3[3];
  auto to3 = [&](const int64_t* v, int64_t* o) {
    for (int i = 0; i < 3; ++i) o[i] = 1;
    for (int i = 0; i < ndim; ++i) o[3 - ndim + i] = v[i];
  };
  to3(Me, P3);
  for (int k = 0; k < N; ++k) {
    to3(Lf, L3);
    cudaError_t e = hd::launch_pad(dtype == HD_C128, f[k], base + k * inb, L3, P3, 1, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "pad_copy");
    to3(Lg, L3);
    e = hd::launch_pad(dtype == HD_C128, g[k], base + (N + k) * inb, L3, P3, 1, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "pad_copy");
    ctx->launches += 2;
    E.f[k] = base + k * inb;
    E.g[k] = base + (N + k) * inb;
  }
  E.h = base + 2 * N * inb;
  s = run_pipeline(ctx, E, base + (2 * N + 1) * inb, wsb, st);
  if (s != HD_OK) return s;
  to3(Lo, L3);
  cudaError_t e = hd::launch_crop(dtype == HD_C128, E.h, h, L3, P3, 1, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "crop_copy");
  ctx->launches += 1;
  return HD_OK;
}

hd_status_t hd_conv_host(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N, int64_t batch,
                         const void* const* f, const int64_t* Lf, const void* const* g,
                         const int64_t* Lg, void* h, const int64_t* M, const hd_plan_t* plan,
                         void* stream) {
  Problem P;
  hd_status_t s = setup(ctx, P, dtype, ndim, N, batch, f, Lf, g, Lg, h, M, plan);
  if (s != HD_OK) return s;
  std::lock_guard<std::recursive_mutex> lk(ctx->mu);
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t eb = elem_bytes(dtype);
  int64_t nf = batch, ng = P.shared_g ? 1 : batch, nh = batch;
  for (int i = 0; i < ndim; ++i) { nf *= Lf[i]; ng *= Lg[i]; nh *= P.ax[i].O; }
  const size_t bf = align256((size_t)nf * eb), bg = align256((size_t)ng * eb), bh = align256((size_t)nh * eb);
  const size_t need = N * (bf + bg) + bh;
  s = grow_scratch(ctx, &ctx->io, &ctx->io_size, need, "cudaMalloc(host io)");
  if (s != HD_OK) return s;
  s = scratch_acquire(ctx, st);
  if (s != HD_OK) return s;
  char* base = (char*)ctx->io;
  for (int k = 0; k < N; ++k) {
    char* df = base + k * bf;
    char* dg = base + N * bf + k * bg;
    cudaError_t e = cudaMemcpyAsync(df, f[k], (size_t)nf * eb, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemcpyAsync(f)");
    e = cudaMemcpyAsync(dg, g[k], (size_t)ng * eb, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemcpyAsync(g)");
    P.f[k] = df;
    P.g[k] = dg;
  }
  void* hh = h;
  P.h = base + N * (bf + bg);
  s = run_pipeline(ctx, P, nullptr, 0, st);
  if (s != HD_OK) return s;
  cudaError_t e = cudaMemcpyAsync(hh, P.h, (size_t)nh * eb, cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemcpyAsync(h)");
  s = scratch_release(ctx, st);
  if (s != HD_OK) return s;
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamSynchronize");
  return HD_OK;
}

hd_status_t hd_conv_host_async(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N, int64_t batch,
                               const void* const* f, const int64_t* Lf, const void* const* g,
                               const int64_t* Lg, void* h, const int64_t* M, const hd_plan_t* plan) {
  Problem P;
  hd_status_t s = setup(ctx, P, dtype, ndim, N, batch, f, Lf, g, Lg, h, M, plan);
  if (s != HD_OK) return s;
  std::lock_guard<std::recursive_mutex> lk(ctx->mu);
  cudaSetDevice(ctx->device);
  hd_ctx::HostSlot& sl = ctx->hslot[ctx->hnext];
  ctx->hnext = (ctx->hnext + 1) % hd_ctx::kHostSlots;
  cudaError_t e;
  if (!sl.st) {
    e = cudaStreamCreateWithFlags(&sl.st, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamCreate");
  }
  const size_t eb = elem_bytes(dtype);
  int64_t nf = batch, ng = P.shared_g ? 1 : batch, nh = batch;
  for (int i = 0; i < ndim; ++i) { nf *= Lf[i]; ng *= Lg[i]; nh *= P.ax[i].O; }
  const size_t bf = align256((size_t)nf * eb), bg = align256((size_t)ng * eb), bh = align256((size_t)nh * eb);
  const size_t need = N * (bf + bg) + bh;
  if (sl.size < need) {
    cudaStreamSynchronize(sl.st);
    if (sl.io) cudaFree(sl.io);
    sl.io = nullptr; sl.size = 0;
    e = cudaMalloc(&sl.io, need);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(host io slot)");
    sl.size = need;
  }
  // copy-in on this slot's stream (after the slot's previous copy-out: same stream)
  char* base = (char*)sl.io;
  for (int k = 0; k < N; ++k) {
    char* df = base + k * bf;
    char* dg = base + N * bf + k * bg;
    e = cudaMemcpyAsync(df, f[k], (size_t)nf * eb, cudaMemcpyHostToDevice, sl.st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemcpyAsync(f)");
    e = cudaMemcpyAsync(dg, g[k], (size_t)ng * eb, cudaMemcpyHostToDevice, sl.st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemcpyAsync(g)");
    P.f[k] = df;
    P.g[k] = dg;
  }
  P.h = base + N * (bf + bg);
  // the convolutions share the context workspace: run after the previous user of it
  s = scratch_acquire(ctx, sl.st);
  if (s != HD_OK) return s;
  s = run_pipeline(ctx, P, nullptr, 0, sl.st);
  if (s != HD_OK) return s;
  s = scratch_release(ctx, sl.st);
  if (s != HD_OK) return s;
  e = cudaMemcpyAsync(h, P.h, (size_t)nh * eb, cudaMemcpyDeviceToHost, sl.st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemcpyAsync(h)");
  return HD_OK;
}

hd_status_t hd_host_sync(hd_ctx_t ctx) {
  if (!ctx) return fail(nullptr, HD_ERR_INVALID, "null context");
  cudaSetDevice(ctx->device);
  for (auto& sl : ctx->hslot) {
    if (!sl.st) continue;
    cudaError_t e = cudaStreamSynchronize(sl.st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamSynchronize(host slot)");
  }
  return HD_OK;
}

}  // extern "C"

namespace {
// forward / backward residue passes of nlines plain rows (generic engine, spectral
// order of hd_spectral_permutation); the caller holds ctx->mu
hd_status_t forward_residues_locked(hd_ctx_t ctx, hd_dtype_t dtype, int64_t nlines, const void* x, int64_t L,
                                    int32_t m, int32_t q, void* X, cudaStream_t stream) {
  const bool dbl = dtype == HD_C128;
  const size_t eb = elem_bytes(dtype);
  Problem P;
  P.dt = dtype; P.N = 1;
  AxisInfo& a = P.ax[0];
  a.m = m; a.q = q; a.M1 = (int64_t)q * m; a.Lf = L; a.pf = (int)cdiv(L, m);
  a.lines = 1;
  a.D = q;
  while (a.D > 1 && pass_smem(eb, q, 1, a.D, m, 1) > hd::kMaxSmem) --a.D;
  a.threads = auto_threads(1, a.D, m, pass_smem(eb, q, 1, a.D, m, 1));
  a.auto_engine = true;
  const void *twm, *twM1;
  hd_status_t s = get_table(ctx, m, dbl, &twm);
  if (s != HD_OK) return s;
  s = get_table(ctx, a.M1, dbl, &twM1);
  if (s != HD_OK) return s;
  const void* twst;
  s = get_stage_table(ctx, m, dbl, &twst);
  if (s != HD_OK) return s;
  Launch Lh = make_launch(ctx, P, hd::MODE_FWD, "fwd_residues", 0, twm, twM1, twst);
  Lh.a.in_f.ptr[0] = x; Lh.a.in_f.L = L; Lh.a.in_f.p = a.pf; in_rows(Lh.a.in_f, L);
  Lh.a.out.ptr[0] = X; out_rows(Lh.a.out, a.M1); Lh.a.out.L = a.M1;
  Lh.a.nlines = nlines; Lh.a.nbatch = 1;
  Lh.ngroups = nlines; Lh.nbatch = 1;
  return launch(ctx, dtype, Lh, stream);
}

hd_status_t backward_residues_locked(hd_ctx_t ctx, hd_dtype_t dtype, int64_t nlines, const void* X, int32_t m,
                                     int32_t q, void* x, int64_t Lout, cudaStream_t stream) {
  const bool dbl = dtype == HD_C128;
  const size_t eb = elem_bytes(dtype);
  Problem P;
  P.dt = dtype; P.N = 1;
  AxisInfo& a = P.ax[0];
  a.m = m; a.q = q; a.M1 = (int64_t)q * m; a.O = Lout; a.T = (int)cdiv(Lout, m);
  a.lines = 1;
  a.D = q;
  while (a.D > 1 && pass_smem(eb, q, 1, a.D, m, 1) > hd::kMaxSmem) --a.D;
  a.threads = auto_threads(1, a.D, m, pass_smem(eb, q, 1, a.D, m, 1));
  a.auto_engine = true;
  const void *twm, *twM1;
  hd_status_t s = get_table(ctx, m, dbl, &twm);
  if (s != HD_OK) return s;
  s = get_table(ctx, a.M1, dbl, &twM1);
  if (s != HD_OK) return s;
  const void* twst;
  s = get_stage_table(ctx, m, dbl, &twst);
  if (s != HD_OK) return s;
  Launch Lh = make_launch(ctx, P, hd::MODE_INV, "bwd_residues", 0, twm, twM1, twst);
  Lh.a.in_f.ptr[0] = X; in_rows(Lh.a.in_f, a.M1); Lh.a.in_f.L = a.M1;
  Lh.a.out.ptr[0] = x; out_rows(Lh.a.out, Lout); Lh.a.out.L = Lout; Lh.a.out.T = a.T;
  Lh.a.nlines = nlines; Lh.a.nbatch = 1;
  Lh.ngroups = nlines; Lh.nbatch = 1;
  return launch(ctx, dtype, Lh, stream);
}

// device copy of the spectral permutation of size n (pos -> frequency) or its inverse
hd_status_t get_perm(hd_ctx* ctx, int32_t n, bool inverse, const int32_t** out) {
  const int64_t key = 2 * (int64_t)n + (inverse ? 1 : 0);
  auto it = ctx->perm.find(key);
  if (it != ctx->perm.end()) { *out = it->second; return HD_OK; }
  std::vector<int32_t> p(n), v(n);
  hd_status_t s = hd_spectral_permutation(n, p.data());
  if (s != HD_OK) return s;
  for (int32_t i = 0; i < n; ++i) v[inverse ? p[i] : i] = inverse ? i : p[i];
  int32_t* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(int32_t) * n);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(permutation)");
  e = cudaMemcpy(d, v.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { cudaFree(d); return cuda_fail(ctx, e, "cudaMemcpy(permutation)"); }
  ctx->perm[key] = d;
  *out = d;
  return HD_OK;
}
}  // namespace

extern "C" {

hd_status_t hd_forward_residues(hd_ctx_t ctx, hd_dtype_t dtype, int64_t nlines, const void* x,
                                int64_t L, int32_t m, int32_t q, void* X, void* stream) {
  if (!ctx) return fail(nullptr, HD_ERR_INVALID, "null context");
  if (!x || !X || nlines < 1 || L < 1) return fail(ctx, HD_ERR_INVALID, "bad arguments");
  if (!is_pow2(m) || m < 2 || m > 4096 || q < 1 || (int64_t)q * m < L)
    return fail(ctx, HD_ERR_INVALID, "need m a power of two in [2,4096] and q*m >= L");
  std::lock_guard<std::recursive_mutex> lk(ctx->mu);
  cudaSetDevice(ctx->device);
  return forward_residues_locked(ctx, dtype, nlines, x, L, m, q, X, (cudaStream_t)stream);
}

hd_status_t hd_backward_residues(hd_ctx_t ctx, hd_dtype_t dtype, int64_t nlines, const void* X,
                                 int32_t m, int32_t q, void* x, int64_t Lout, void* stream) {
  if (!ctx) return fail(nullptr, HD_ERR_INVALID, "null context");
  if (!x || !X || nlines < 1 || Lout < 1) return fail(ctx, HD_ERR_INVALID, "bad arguments");
  if (!is_pow2(m) || m < 2 || m > 4096 || q < 1 || (int64_t)q * m < Lout)
    return fail(ctx, HD_ERR_INVALID, "need m a power of two in [2,4096] and q*m >= Lout");
  std::lock_guard<std::recursive_mutex> lk(ctx->mu);
  cudaSetDevice(ctx->device);
  return backward_residues_locked(ctx, dtype, nlines, X, m, q, x, Lout, (cudaStream_t)stream);
}

// Row f1: short f with size-m residues (q_f = Lambda q_g), long g
// with size-(Lambda m) residues (q_g), matched product, size-(Lambda m) inverse.
static hd_status_t lambda_locked(hd_ctx_t ctx, hd_dtype_t dtype, int64_t batch, const void* f, int64_t Lf,
                                 const void* g, int64_t Lg, void* h, int32_t m, int32_t Lambda, int32_t Lm,
                                 int32_t qg, int32_t qf, int64_t M1, int64_t Lout, cudaStream_t st);

hd_status_t hd_conv1d_lambda(hd_ctx_t ctx, hd_dtype_t dtype, int64_t batch, const void* f, int64_t Lf,
                             const void* g, int64_t Lg, void* h, int64_t M, int32_t m, int32_t Lambda,
                             void* stream) {
  if (!ctx) return fail(nullptr, HD_ERR_INVALID, "null context");
  if (dtype != HD_C64 && dtype != HD_C128) return fail(ctx, HD_ERR_INVALID, "dtype must be HD_C64 or HD_C128");
  if (!f || !g || !h || batch < 1 || Lf < 1 || Lg < 1) return fail(ctx, HD_ERR_INVALID, "bad arguments");
  if (Lf > Lg) return fail(ctx, HD_ERR_INVALID, "hd_conv1d_lambda needs L_f <= L_g (PAPER.md:682)");
  if (!is_pow2(m) || m < 2 || !is_pow2(Lambda) || Lambda < 1 || (int64_t)m * Lambda > 4096)
    return fail(ctx, HD_ERR_INVALID, "m and Lambda must be powers of two with Lambda*m <= 4096");
  const int64_t Lout = Lf + Lg - 1;
  if (M <= 0) M = Lout;
  if (M < Lout) return fail(ctx, HD_ERR_INVALID, "M < L_f + L_g - 1 would alias (PAPER.md:592)");
  const int32_t Lm = m * Lambda;
  const int64_t qg64 = cdiv(M, Lm);
  if (qg64 * Lambda > (1 << 20)) return fail(ctx, HD_ERR_UNSUPPORTED, "too many residues");
  const int32_t qg = (int32_t)qg64, qf = Lambda * qg;
  const int64_t M1 = (int64_t)qg * Lm;
  std::lock_guard<std::recursive_mutex> lk(ctx->mu);
  cudaSetDevice(ctx->device);
  const size_t eb = elem_bytes(dtype);
  const size_t need = 2 * align256((size_t)batch * M1 * eb);
  hd_status_t sg = grow_scratch(ctx, &ctx->ws, &ctx->ws_size, need, "cudaMalloc(workspace)");
  if (sg != HD_OK) return sg;
  cudaStream_t st = (cudaStream_t)stream;
  sg = scratch_acquire(ctx, st);
  if (sg != HD_OK) return sg;
  sg = lambda_locked(ctx, dtype, batch, f, Lf, g, Lg, h, m, Lambda, Lm, qg, qf, M1, Lout, st);
  hd_status_t r = scratch_release(ctx, st);
  return sg != HD_OK ? sg : r;
}

static hd_status_t lambda_locked(hd_ctx_t ctx, hd_dtype_t dtype, int64_t batch, const void* f, int64_t Lf,
                                 const void* g, int64_t Lg, void* h, int32_t m, int32_t Lambda, int32_t Lm,
                                 int32_t qg, int32_t qf, int64_t M1, int64_t Lout, cudaStream_t st) {
  const size_t eb = elem_bytes(dtype);
  char* Xf = (char*)ctx->ws;
  char* Xg = Xf + align256((size_t)batch * M1 * eb);
  const int32_t *perm_g = nullptr, *iperm_f = nullptr;
  hd_status_t s = get_perm(ctx, Lm, false, &perm_g);
  if (s != HD_OK) return s;
  s = get_perm(ctx, m, true, &iperm_f);
  if (s != HD_OK) return s;
  s = forward_residues_locked(ctx, dtype, batch, f, Lf, m, qf, Xf, st);
  if (s != HD_OK) return s;
  s = forward_residues_locked(ctx, dtype, batch, g, Lg, Lm, qg, Xg, st);
  if (s != HD_OK) return s;
  cudaError_t e = hd::launch_lambda_product(dtype == HD_C128, Xf, Xg, perm_g, iperm_f, batch, m, Lambda, qg,
                                            1.0 / (double)M1, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "lambda_product");
  ctx->launches += 1;
  return backward_residues_locked(ctx, dtype, batch, Xg, Lm, qg, h, Lout, st);
}

hd_status_t hd_profile_enable(hd_ctx_t ctx, int32_t enable) {
  if (!ctx) return fail(nullptr, HD_ERR_INVALID, "null context");
  ctx->profiling = enable != 0;
  return HD_OK;
}

int32_t hd_profile_read(hd_ctx_t ctx, int32_t max, double* ms, int64_t* launches, char* names) {
  if (!ctx) return -1;
  int32_t n = 0;
  for (auto& p : ctx->prof) {
    for (auto& ev : p.pending) {
      float t = 0;
      if (cudaEventElapsedTime(&t, ev.first, ev.second) == cudaSuccess) p.ms += t;
      cudaEventDestroy(ev.first);
      cudaEventDestroy(ev.second);
    }
    p.pending.clear();
    if (n < max) {
      if (ms) ms[n] = p.ms;
      if (launches) launches[n] = p.launches;
      if (names) { std::strncpy(names + 32 * n, p.name.c_str(), 31); names[32 * n + 31] = 0; }
    }
    ++n;
  }
  return n;
}

hd_status_t hd_profile_reset(hd_ctx_t ctx) {
  if (!ctx) return fail(nullptr, HD_ERR_INVALID, "null context");
  for (auto& p : ctx->prof)
    for (auto& ev : p.pending) { cudaEventDestroy(ev.first); cudaEventDestroy(ev.second); }
  ctx->prof.clear();
  return HD_OK;
}

int64_t hd_launch_count(hd_ctx_t ctx) { return ctx ? ctx->launches : -1; }

int64_t hd_graph_replays(hd_ctx_t ctx) { return ctx ? ctx->graph_replays : -1; }

int64_t hd_engine_launches(hd_ctx_t ctx, int32_t engine) {
  if (!ctx || engine < 0 || engine > HD_ENGINE_S4096R) return -1;
  return ctx->engine_launches[engine];
}

static bool conv_lines_in(const hd_lines_t& d, LineIn& in, int64_t nbatch, int n, bool need_ptr) {
  for (int k = 0; k < n; ++k) {
    if (need_ptr && !d.ptr[k]) return false;
    in.ptr[k] = d.ptr[k];
  }
  if (d.L < 1) return false;
  in.L = d.L;
  in.nbi = d.nbi > 0 ? d.nbi : nbatch;
  in.s_bo = d.s_bo; in.s_b = d.s_b;
  in.tl = d.tl; in.s_t = d.s_t; in.s_l = d.s_l;
  in.jd = d.jd > 0 ? d.jd : 0; in.s_jt = d.s_jt; in.s_j = d.s_j;
  return true;
}
static bool conv_lines_out(const hd_lines_t& d, LineOut& o, int64_t nbatch, int n) {
  for (int k = 0; k < n; ++k) {
    if (!d.ptr[k]) return false;
    o.ptr[k] = d.ptr[k];
  }
  if (d.L < 1) return false;
  o.L = d.L;
  o.nbi = d.nbi > 0 ? d.nbi : nbatch;
  o.s_bo = d.s_bo; o.s_b = d.s_b;
  o.tl = d.tl; o.s_t = d.s_t; o.s_l = d.s_l;
  if (d.jd > 0 && is_pow2(d.jd) && d.jd < (int64_t(1) << 29)) {
    o.so_log2 = ilog2(d.jd); o.jd = 0;
  } else if (d.jd > 0) {
    if (d.jd > 0x7fffffff) return false;
    o.so_log2 = 40; o.jd = d.jd;
  } else {
    o.so_log2 = 40; o.jd = 0;
  }
  o.s_jt = d.s_jt; o.s_js = d.s_j;
  return true;
}

hd_status_t hd_pass(hd_ctx_t ctx, hd_dtype_t dtype, const hd_pass_desc_t* d, void* stream) {
  if (!ctx || !d) return fail(ctx, HD_ERR_INVALID, "null argument");
  if (dtype != HD_C64 && dtype != HD_C128) return fail(ctx, HD_ERR_INVALID, "bad dtype");
  if (d->mode < HD_PASS_FWD || d->mode > HD_PASS_CONV) return fail(ctx, HD_ERR_INVALID, "bad pass mode");
  if (d->npairs < 1 || d->npairs > HD_MAX_PAIRS) return fail(ctx, HD_ERR_INVALID, "npairs must be in [1, 16]");
  if (d->nlines < 1 || d->nbatch < 1 || d->M < 1) return fail(ctx, HD_ERR_INVALID, "nlines, nbatch, M must be >= 1");
  const hd_axis_plan_t& ap = d->axis;
  if (!is_pow2(ap.m) || ap.m < 2 || ap.m > 4096) return fail(ctx, HD_ERR_INVALID, "m must be a power of two in [2, 4096]");
  const int C = ap.C ? ap.C : 1;
  if (!valid_lines(C)) return fail(ctx, HD_ERR_INVALID, "C must be 1, 2, 4, 8 or 16");
  const int q = (int)cdiv(d->M, ap.m);
  int D = ap.D ? ap.D : q;
  if (D < 1 || D > q) return fail(ctx, HD_ERR_INVALID, "D must be in [1, q]");
  if (ap.threads && !valid_threads(ap.threads)) return fail(ctx, HD_ERR_INVALID, "bad threads");
  // a D whose residue group does not fit the generic engine's shared memory is lowered
  // (the engine walks the groups of D residues in turn and the results do not depend on
  // D; e.g. the residue-sharded 1-D pass of hd_conv1d_dist at m = 4096, D = q = 3)
  {
    const int nb = d->mode == HD_PASS_CONV ? conv_nbuf(d->npairs) : 1;
    while (D > 1 && pass_smem(elem_bytes(dtype), q, C, D, ap.m, nb) > hd::kMaxSmem) --D;
  }
  const bool rrange = d->r_begin != 0 || (d->r_end != 0 && d->r_end != q);
  if (d->r_begin < 0 || d->r_end < 0 || d->r_end > q || (d->r_end != 0 && d->r_begin >= d->r_end) ||
      (d->r_end == 0 && d->r_begin != 0))
    return fail(ctx, HD_ERR_INVALID, "residue range must satisfy 0 <= r_begin < r_end <= q");
  if (rrange && d->mode != HD_PASS_CONV) return fail(ctx, HD_ERR_INVALID, "a residue range needs HD_PASS_CONV");
  std::lock_guard<std::recursive_mutex> lk(ctx->mu);
  cudaSetDevice(ctx->device);
  const bool dbl = dtype == HD_C128;
  const int64_t M1 = (int64_t)q * ap.m;
  const void *twm, *twM1, *twst;
  hd_status_t s = get_table(ctx, ap.m, dbl, &twm);
  if (s != HD_OK) return s;
  s = get_table(ctx, M1, dbl, &twM1);
  if (s != HD_OK) return s;
  s = get_stage_table(ctx, ap.m, dbl, &twst);
  if (s != HD_OK) return s;
  Launch L;
  std::memset(&L, 0, sizeof(L));
  L.flags = d->flags | (rrange ? HD_FLAG_GENERIC_FFT : 0u);  // residue subsets: generic engine
  L.mode = d->mode;
  L.name = d->mode == HD_PASS_FWD ? "pass_fwd" : (d->mode == HD_PASS_INV ? "pass_inv" : "pass_conv");
  // forward / inverse keep the documented spectral order unless the caller opts into
  // the staged engines' own order (HD_FLAG_STAGED_ORDER, the same for both passes)
  const bool staged_order = (d->flags & HD_FLAG_STAGED_ORDER) != 0;
  L.s512_axis = d->mode == HD_PASS_CONV || staged_order;
  L.s128_axis = d->mode == HD_PASS_CONV || staged_order;
  L.m = ap.m;
  L.lines = C;
  L.threads = ap.threads ? ap.threads : default_threads(C, D, ap.m);
  L.auto_engine = ap.threads == 0;
  L.nbuf = d->mode == HD_PASS_CONV ? conv_nbuf(d->npairs) : 1;
  init_in(L.a.in_f);
  init_in(L.a.in_g);
  init_out(L.a.out);
  const int narr = d->mode == HD_PASS_CONV ? d->npairs : (d->mode == HD_PASS_FWD ? d->npairs : 1);
  if (!conv_lines_in(d->in_f, L.a.in_f, d->nbatch, narr, true))
    return fail(ctx, HD_ERR_INVALID, "bad in_f description");
  if (d->mode == HD_PASS_CONV && !conv_lines_in(d->in_g, L.a.in_g, d->nbatch, narr, true))
    return fail(ctx, HD_ERR_INVALID, "bad in_g description");
  if (!conv_lines_out(d->out, L.a.out, d->nbatch, d->mode == HD_PASS_FWD ? narr : 1))
    return fail(ctx, HD_ERR_INVALID, "bad out description");
  L.a.in_f.p = (int)cdiv(L.a.in_f.L, ap.m);
  L.a.in_g.p = (int)cdiv(L.a.in_g.L, ap.m);
  L.a.out.T = (int)cdiv(std::min<int64_t>(L.a.out.L, M1), ap.m);
  if (d->mode != HD_PASS_FWD && L.a.out.L > M1) return fail(ctx, HD_ERR_INVALID, "out.L exceeds q*m");
  L.a.tw_m = twm; L.a.tw_M1 = twM1; L.a.tw_st = twst;
  L.a.q = q; L.a.D = D; L.a.C = C; L.a.c_log2 = ilog2(C); L.a.M1 = M1;
  L.a.npairs = d->mode == HD_PASS_CONV ? d->npairs : 1;
  L.a.scale = d->mode == HD_PASS_CONV ? d->scale : 1.0;
  L.a.nlines = d->nlines; L.a.nbatch = d->nbatch; L.a.batch_fastest = d->batch_fastest ? 1 : 0;
  L.a.r_lo = rrange ? d->r_begin : 0;
  L.a.r_hi = rrange ? d->r_end : 0;
  L.narrays = d->mode == HD_PASS_FWD ? narr : 1;
  L.ngroups = cdiv(d->nlines, C); L.nbatch = d->nbatch;
  if (staged_order && d->mode != HD_PASS_CONV && !use_s512(dtype, L) && !use_s128(dtype, L))
    return fail(ctx, HD_ERR_UNSUPPORTED, "HD_FLAG_STAGED_ORDER: no staged engine for this pass");
  return launch(ctx, dtype, L, (cudaStream_t)stream);
}

}  // extern "C"

// ===========================================================================
// On-device tuning sweep: the paper's "experience" search,
// per dimension independently, scored by measured time of
// the whole convolution (CUDA events, median of reps after 2 warm-ups), first
// strict minimum wins with a lexicographic (m, C, S, D) tie-break
// (SPEC.md:350).
// ===========================================================================
namespace {

struct AxisCand { int m, C, S, D, threads; };

bool cand_less(const AxisCand& a, const AxisCand& b) {
  if (a.m != b.m) return a.m < b.m;
  if (a.C != b.C) return a.C < b.C;
  if (a.S != b.S) return a.S < b.S;
  if (a.D != b.D) return a.D < b.D;
  return a.threads < b.threads;
}

// The documented per-axis search space (include/hdconv.h hd_tune):
// m a power of two in [16, 4096] with q = ceil(M/m) <= 1024; C in {1, 2, 4, 8};
// D in {q, ceil(q/2), ceil(q/4), ..., 1}; S in {1, 2, 4, 8, 16} (1 in 1-D); threads in
// {automatic, the sweep-matched default, 256} plus {768, 1024} for passes whose shared
// memory leaves one CTA per SM and whose butterfly sweep has >= 512 items; a candidate
// whose generic pass exceeds the shared memory is not in the space.
std::vector<AxisCand> axis_candidates(const hd_plan_t& base, int i, int ndim, int npairs,
                                      const int64_t* Lf, const int64_t* Lg, const int64_t* M,
                                      size_t eb) {
  (void)base;
  std::vector<AxisCand> out;
  const int64_t Lout = Lf[i] + Lg[i] - 1;
  const int64_t Mi = (M && M[i] > 0) ? M[i] : Lout;
  const int nbuf = (i == 0) ? conv_nbuf(npairs) : 1;
  const std::vector<int> Ss = (ndim == 1) ? std::vector<int>{1} : std::vector<int>{1, 2, 4, 8, 16};
  for (int m = 16; m <= 4096; m *= 2) {
    const int64_t q64 = cdiv(Mi, m);
    if (q64 > 1024) continue;
    const int q = (int)q64;
    std::vector<int> Ds;
    for (int D = q;; D = (D + 1) / 2) {
      Ds.push_back(D);
      if (D == 1) break;
    }
    for (int C : {1, 2, 4, 8}) {
      for (int D : Ds) {
        if (pass_smem(eb, q, C, D, m, nbuf) > hd::kMaxSmem) continue;
        const int dt = default_threads(C, D, m);
        std::vector<int> ths = {0, dt};  // 0: automatic engine (warp engine where it applies)
        if (dt != 256) ths.push_back(256);
        const int64_t bflies = (int64_t)C * D * (m / 8);
        if (bflies >= 512 && pass_smem(eb, q, C, D, m, nbuf) > hd::kMaxSmem / 2)
          for (int t : {768, 1024}) if (t != dt) ths.push_back(t);
        for (int S : Ss)
          for (int th : ths) out.push_back(AxisCand{m, C, S, D, th});
      }
    }
  }
  return out;
}

void apply_cand(hd_plan_t& p, int i, int ndim, const AxisCand& c) {
  (void)ndim;
  p.axis[i].m = c.m; p.axis[i].C = c.C; p.axis[i].S = c.S; p.axis[i].D = c.D;
  p.axis[i].threads = c.threads;
}

}  // namespace

extern "C" {

// The paper's tuning "experience": A0 grid search over the cross
// product, per-axis search (separability), A1 random search
// and the skinny-rectangle proxy heuristic.
hd_status_t hd_tune_ex(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N, int64_t batch,
                       const int64_t* Lf, const int64_t* Lg, const int64_t* M, const hd_tune_opts_t* opts,
                       void* stream, hd_plan_t* out) {
  if (!ctx || !out || !opts) return fail(ctx, HD_ERR_INVALID, "null argument");
  const uint32_t flags = opts->flags;
  const bool random = (flags & HD_TUNE_RANDOM) != 0;
  if (random && opts->n1 < 1) return fail(ctx, HD_ERR_INVALID, "HD_TUNE_RANDOM needs n1 >= 1");
  if (opts->proxy_rows < 0) return fail(ctx, HD_ERR_INVALID, "proxy_rows must be >= 0");
  Problem P0;
  hd_status_t s = setup(ctx, P0, dtype, ndim, N, batch, nullptr, Lf, nullptr, Lg, nullptr, M, nullptr, false);
  if (s != HD_OK) return s;
  hd_plan_t base;
  s = default_plan(ctx, dtype, ndim, N, Lf, Lg, M, &base);
  if (s != HD_OK) return s;
  const int reps = opts->reps > 0 ? opts->reps : 5;
  const bool fake = opts->fake_cost != 0;
  std::lock_guard<std::recursive_mutex> lk(ctx->mu);
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  if (!fake) {
    s = scratch_acquire(ctx, st);
    if (s != HD_OK) return s;
  }
  const size_t eb = elem_bytes(dtype);
  // synthetic scratch operands of the problem's shape (timing is value independent)
  int64_t nf = batch, ng = batch, nh = batch;
  for (int i = 0; i < ndim; ++i) { nf *= Lf[i]; ng *= Lg[i]; nh *= Lf[i] + Lg[i] - 1; }
  const size_t bf = align256((size_t)nf * eb), bg = align256((size_t)ng * eb), bh = align256((size_t)nh * eb);
  char* scratch = nullptr;
  if (!fake) {
    cudaError_t e = cudaMalloc(&scratch, N * (bf + bg) + bh);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(tune scratch)");
    cudaMemsetAsync(scratch, 0, N * (bf + bg) + bh, st);
  }
  const void* fp[HD_MAX_PAIRS];
  const void* gp[HD_MAX_PAIRS];
  for (int k = 0; k < N; ++k) { fp[k] = scratch + k * bf; gp[k] = scratch + N * bf + k * bg; }
  void* hp = scratch + N * (bf + bg);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (!fake) { cudaEventCreate(&e0); cudaEventCreate(&e1); }
  ctx->tune_log.clear();
  const bool prof_was = ctx->profiling;
  ctx->profiling = false;

  // skinny proxy: the same problem with at most proxy_rows lines along axis 0
  int64_t Lfp[HD_MAX_DIM], Lgp[HD_MAX_DIM], Mp[HD_MAX_DIM];
  const bool proxy = opts->proxy_rows > 0 && ndim >= 2;
  for (int i = 0; i < ndim; ++i) {
    Lfp[i] = Lf[i]; Lgp[i] = Lg[i]; Mp[i] = M ? M[i] : 0;
  }
  if (proxy) {
    Lfp[0] = std::min<int64_t>(Lf[0], opts->proxy_rows);
    Lgp[0] = std::min<int64_t>(Lg[0], opts->proxy_rows);
    Mp[0] = 0;
  }

  // testing hook: a deterministic cost of the candidate instead of a timing
  auto fake_cost = [&](const hd_plan_t& pl) -> double {
    if (opts->fake_cost == 2) return 1.0;  // every candidate ties
    uint64_t h = 0x9E3779B97F4A7C15ull ^ (uint64_t)opts->seed;
    for (int i = 0; i < ndim; ++i) {
      const hd_axis_plan_t& a = pl.axis[i];
      for (int64_t v : {(int64_t)a.m, (int64_t)a.C, (int64_t)a.S, (int64_t)a.D, (int64_t)a.threads}) {
        h ^= (uint64_t)v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 31;
      }
    }
    return 1.0 + (double)(h >> 11) * (1.0 / 9007199254740992.0);
  };

  double abort_ref = 1e300;  // best time so far (early-abort reference)
  auto time_plan_on = [&](hd_plan_t pl, const int64_t* lf, const int64_t* lg, const int64_t* mm,
                          double* secs) -> bool {
    Problem P;
    P.dt = dtype; P.ndim = ndim; P.N = N; P.batch = batch; P.shared_g = false;
    for (int k = 0; k < N; ++k) { P.f[k] = fp[k]; P.g[k] = gp[k]; }
    P.h = hp;
    if (complete_plan(ctx, dtype, ndim, N, lf, lg, mm, &pl, P.ax) != HD_OK) return false;
    P.plan = pl;
    choose_engines(P);
    if (fake) {
      *secs = fake_cost(pl);
      ctx->tune_log.push_back({pl, *secs});
      return true;
    }
    // first warm-up timed: a candidate > 3x the best time so far is recorded with that
    // time and not repeated (documented pruning: it cannot win)
    {
      cudaEventRecord(e0, st);
      if (run_pipeline(ctx, P, nullptr, 0, st) != HD_OK) return false;
      cudaEventRecord(e1, st);
      if (cudaEventSynchronize(e1) != cudaSuccess) return false;
      float ms0 = 0;
      cudaEventElapsedTime(&ms0, e0, e1);
      if (abort_ref < 1e299 && ms0 * 1e-3 > 3.0 * abort_ref) {
        *secs = ms0 * 1e-3;
        ctx->tune_log.push_back({pl, *secs});
        return true;
      }
    }
    if (run_pipeline(ctx, P, nullptr, 0, st) != HD_OK) return false;
    std::vector<double> ts;
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(e0, st);
      if (run_pipeline(ctx, P, nullptr, 0, st) != HD_OK) return false;
      cudaEventRecord(e1, st);
      if (cudaEventSynchronize(e1) != cudaSuccess) return false;
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ts.push_back(ms * 1e-3);
    }
    std::sort(ts.begin(), ts.end());
    *secs = ts[ts.size() / 2];
    ctx->tune_log.push_back({pl, *secs});
    return true;
  };
  auto time_plan = [&](hd_plan_t pl, double* secs) { return time_plan_on(pl, Lf, Lg, M, secs); };
  // lexicographic order of whole plans (axis by axis on (m, C, S, D, threads))
  auto plan_less = [&](const hd_plan_t& x, const hd_plan_t& y) {
    for (int i = 0; i < ndim; ++i) {
      const AxisCand a{x.axis[i].m, x.axis[i].C, x.axis[i].S, x.axis[i].D, x.axis[i].threads};
      const AxisCand b{y.axis[i].m, y.axis[i].C, y.axis[i].S, y.axis[i].D, y.axis[i].threads};
      if (cand_less(a, b)) return true;
      if (cand_less(b, a)) return false;
    }
    return false;
  };

  hd_plan_t best = base;
  double best_t = 1e300;
  if (flags & (HD_TUNE_EXHAUSTIVE | HD_TUNE_RANDOM)) {
    std::vector<std::vector<AxisCand>> lists;
    size_t combos = 1;
    for (int i = 0; i < ndim; ++i) {
      lists.push_back(axis_candidates(base, i, ndim, N, Lf, Lg, M, eb));
      combos *= std::max<size_t>(1, lists.back().size());
    }
    if (combos > ((size_t)1 << 22)) {
      ctx->profiling = prof_was;
      if (!fake) scratch_release(ctx, st);
      if (e0) cudaEventDestroy(e0);
      if (e1) cudaEventDestroy(e1);
      if (scratch) cudaFree(scratch);
      return fail(ctx, HD_ERR_UNSUPPORTED, "search space of " + std::to_string(combos) +
                                               " plans exceeds 2^22: use the per-axis or random search");
    }
    std::vector<size_t> order(combos);
    for (size_t c = 0; c < combos; ++c) order[c] = c;
    size_t count = combos;
    if (random && (size_t)opts->n1 < combos) {
      // partial Fisher-Yates with splitmix64: n1 candidates uniformly without replacement
      uint64_t x = opts->seed;
      auto next = [&]() {
        uint64_t z = (x += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
      };
      count = (size_t)opts->n1;
      for (size_t k = 0; k < count; ++k) {
        const size_t j = k + (size_t)(next() % (uint64_t)(combos - k));
        std::swap(order[k], order[j]);
      }
    }
    for (size_t k = 0; k < count; ++k) {
      hd_plan_t pl = base;
      size_t r = order[k];
      for (int i = 0; i < ndim; ++i) {
        if (lists[i].empty()) continue;
        apply_cand(pl, i, ndim, lists[i][r % lists[i].size()]);
        r /= lists[i].size();
      }
      double t;
      if (!time_plan(pl, &t)) continue;
      const bool tie = std::fabs(t - best_t) <= 1e-12 * best_t;
      if ((t < best_t && !tie) || (tie && plan_less(pl, best))) { best_t = t; best = pl; }
      abort_ref = std::min(abort_ref, best_t);
    }
  } else {
    if (!time_plan(best, &best_t)) best_t = 1e300;
    for (int i = 0; i < ndim; ++i) {
      abort_ref = (proxy && i > 0) ? 1e300 : best_t;
      const bool on_proxy = proxy && i > 0;
      std::vector<AxisCand> cands = axis_candidates(best, i, ndim, N, on_proxy ? Lfp : Lf, on_proxy ? Lgp : Lg,
                                                    on_proxy ? Mp : M, eb);
      AxisCand bc{best.axis[i].m, best.axis[i].C, best.axis[i].S, best.axis[i].D, best.axis[i].threads};
      double ref_t = best_t;
      if (on_proxy && !time_plan_on(best, Lfp, Lgp, Mp, &ref_t)) ref_t = 1e300;
      if (on_proxy) abort_ref = ref_t;
      // candidates come in groups of equal (m, C); the group's first member is timed
      // first and, if it is more than 3x slower than the best so far, the rest of the
      // group is logged as pruned (time +inf) without being timed
      int gm = -1, gC = -1;
      bool gpruned = false;
      for (const AxisCand& c : cands) {
        hd_plan_t pl = best;
        apply_cand(pl, i, ndim, c);
        const bool first = c.m != gm || c.C != gC;
        if (!first && gpruned && !fake) {
          ctx->tune_log.push_back({pl, std::numeric_limits<double>::infinity()});
          continue;
        }
        double t;
        if (!(on_proxy ? time_plan_on(pl, Lfp, Lgp, Mp, &t) : time_plan(pl, &t))) {
          if (first) { gm = c.m; gC = c.C; gpruned = true; }
          continue;
        }
        if (first) {
          gm = c.m; gC = c.C;
          gpruned = ref_t < 1e299 && t > 3.0 * ref_t;
        }
        const bool tie = std::fabs(t - ref_t) <= 1e-12 * ref_t;
        if (t < ref_t && !tie) { ref_t = t; best = pl; bc = c; }
        else if (tie && cand_less(c, bc)) { best = pl; bc = c; }
        abort_ref = std::min(abort_ref, ref_t);
      }
      if (on_proxy) best_t = 1e300;  // the full problem's time of the final plan is taken below
      else best_t = ref_t;
    }
    if (best_t >= 1e300) time_plan(best, &best_t);
  }
  ctx->profiling = prof_was;
  if (!fake) scratch_release(ctx, st);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (scratch) cudaFree(scratch);
  AxisInfo ax[HD_MAX_DIM];
  s = complete_plan(ctx, dtype, ndim, N, Lf, Lg, M, &best, ax);
  if (s != HD_OK) return s;
  best.tuned_seconds = best_t;
  ctx->plan_cache[problem_key(dtype, ndim, N, batch, Lf, Lg, M, 0)] = best;
  *out = best;
  return HD_OK;
}

// Size (and optionally the list) of the per-axis search space of hd_tune for axis i.
int32_t hd_tune_space(hd_dtype_t dtype, int32_t ndim, int32_t N, const int64_t* Lf, const int64_t* Lg,
                      const int64_t* M, int32_t axis, hd_axis_plan_t* out, int32_t cap) {
  if (!Lf || !Lg || ndim < 1 || ndim > HD_MAX_DIM || axis < 0 || axis >= ndim || N < 1) return -1;
  if (dtype != HD_C64 && dtype != HD_C128) return -1;
  hd_plan_t base;
  std::memset(&base, 0, sizeof(base));
  const std::vector<AxisCand> c = axis_candidates(base, axis, ndim, N, Lf, Lg, M, elem_bytes(dtype));
  for (int32_t k = 0; out && k < cap && k < (int32_t)c.size(); ++k) {
    std::memset(&out[k], 0, sizeof(out[k]));
    out[k].m = c[k].m; out[k].C = c[k].C; out[k].S = c[k].S; out[k].D = c[k].D; out[k].threads = c[k].threads;
  }
  return (int32_t)c.size();
}

// The explicit-padding baseline's own plan (PAPER.md:602-605 with the tuner's search,
// PAPER.md:758-766): per axis of the padded problem (M_exp = next power of two >= L_out,
// p = q), m in {64, ..., min(4096, M_exp)}, C in {1, 2, 4} (C > 1 for m <= 256), S in
// {1, 2, 4, 8} (ndim > 1), timed as whole hd_conv_explicit calls on zero operands.
hd_status_t hd_tune_explicit(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N, const int64_t* Lf,
                             const int64_t* Lg, int32_t reps, void* stream, hd_plan_t* out) {
  if (!ctx || !Lf || !Lg || !out) return fail(ctx, HD_ERR_INVALID, "null argument");
  if (ndim < 1 || ndim > HD_MAX_DIM || N < 1 || N > HD_MAX_PAIRS) return fail(ctx, HD_ERR_INVALID, "bad ndim or N");
  std::lock_guard<std::recursive_mutex> lk(ctx->mu);
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t eb = elem_bytes(dtype);
  int64_t nf = 1, ng = 1, nh = 1, Me[HD_MAX_DIM];
  for (int i = 0; i < ndim; ++i) {
    nf *= Lf[i]; ng *= Lg[i]; nh *= Lf[i] + Lg[i] - 1;
    Me[i] = 1;
    while (Me[i] < Lf[i] + Lg[i] - 1) Me[i] *= 2;
  }
  const size_t bf = align256((size_t)nf * eb), bg = align256((size_t)ng * eb), bh = align256((size_t)nh * eb);
  char* buf = nullptr;
  if (cudaMalloc(&buf, N * (bf + bg) + bh) != cudaSuccess) return fail(ctx, HD_ERR_CUDA, "cudaMalloc(tune scratch)");
  cudaMemsetAsync(buf, 0, N * (bf + bg) + bh, st);
  const void* fp[HD_MAX_PAIRS];
  const void* gp[HD_MAX_PAIRS];
  for (int k = 0; k < N; ++k) { fp[k] = buf + k * bf; gp[k] = buf + N * bf + k * bg; }
  void* hp = buf + N * (bf + bg);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int nrep = reps > 0 ? reps : 3;
  auto time_plan = [&](hd_plan_t pl, double* secs) -> bool {
    pl.flags = HD_FLAG_EXPLICIT_PLAN;
    if (hd_conv_explicit(ctx, dtype, ndim, N, fp, Lf, gp, Lg, hp, &pl, st) != HD_OK) return false;
    std::vector<double> ts;
    for (int r = 0; r < nrep; ++r) {
      cudaEventRecord(e0, st);
      if (hd_conv_explicit(ctx, dtype, ndim, N, fp, Lf, gp, Lg, hp, &pl, st) != HD_OK) return false;
      cudaEventRecord(e1, st);
      if (cudaEventSynchronize(e1) != cudaSuccess) return false;
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ts.push_back(ms * 1e-3);
    }
    std::sort(ts.begin(), ts.end());
    *secs = ts[ts.size() / 2];
    ctx->tune_log.push_back({pl, *secs});
    return true;
  };
  ctx->tune_log.clear();
  hd_plan_t best;
  std::memset(&best, 0, sizeof(best));
  best.ndim = ndim;
  for (int i = 0; i < ndim; ++i) {
    best.axis[i].m = (int)std::min<int64_t>(512, Me[i]);
    best.axis[i].C = 1;
    best.axis[i].S = ndim > 1 ? 2 : 1;
  }
  double best_t = 1e300;
  if (!time_plan(best, &best_t)) best_t = 1e300;
  for (int i = 0; i < ndim; ++i) {
    for (int m = 64; m <= std::min<int64_t>(4096, Me[i]); m *= 2)
      for (int C : {1, 2, 4}) {
        if (C > 1 && m > 256) continue;
        for (int S : {1, 2, 4, 8}) {
          if (ndim == 1 && S > 1) continue;
          hd_plan_t pl = best;
          pl.axis[i].m = m; pl.axis[i].C = C; pl.axis[i].S = S; pl.axis[i].D = 0;
          double t;
          if (time_plan(pl, &t) && t < best_t) { best_t = t; best = pl; }
        }
      }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  if (best_t >= 1e300) return fail(ctx, HD_ERR_UNSUPPORTED, "no explicit plan could be timed");
  best.flags = HD_FLAG_EXPLICIT_PLAN;
  best.tuned_seconds = best_t;
  ctx->plan_cache[problem_key(dtype, ndim, N, 1, Lf, Lg, nullptr, HD_FLAG_EXPLICIT_PLAN)] = best;
  *out = best;
  return HD_OK;
}

hd_status_t hd_tune(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N, int64_t batch,
                    const int64_t* Lf, const int64_t* Lg, const int64_t* M, uint32_t flags,
                    int32_t reps, void* stream, hd_plan_t* out) {
  hd_tune_opts_t o;
  std::memset(&o, 0, sizeof(o));
  o.flags = flags & HD_TUNE_EXHAUSTIVE;
  o.reps = reps;
  return hd_tune_ex(ctx, dtype, ndim, N, batch, Lf, Lg, M, &o, stream, out);
}

int32_t hd_tune_log(hd_ctx_t ctx, int32_t max, hd_plan_t* plans, double* seconds) {
  if (!ctx) return -1;
  const int32_t n = (int32_t)ctx->tune_log.size();
  for (int32_t i = 0; i < n && i < max; ++i) {
    if (plans) plans[i] = ctx->tune_log[i].first;
    if (seconds) seconds[i] = ctx->tune_log[i].second;
  }
  return n;
}

}  // extern "C"
