// hd_dist.cu -- multi-GPU entry points of libhdconv.so: one
// process per GPU, NCCL over NVLink for the exchange steps the method has.
//
//  * 1-D (BASELINE config 2, "residue sharding across GPUs"): the batch of independent
//    pairs shards with no collective (HD_SHARD_BATCH); HD_SHARD_RESIDUE splits the q
//    residues of every line over the ranks -- each residue's transform, product and
//    backward contribution are independent (the q residues of the
//    Forward Eq. PAPER.md:528) -- and the partial backward sums meet in
//    an NCCL reduce-scatter that leaves each rank its batch slice of h.
//  * 2-D / 3-D (configs 3-5): slab decomposition along axis 0 with one all-to-all
//    transpose each way (the axes are separable passes).  2-D: rank k
//    holds rows of f (g replicated) -> forward along x -> all-to-all to spectral-column
//    slabs -> convolution along y -> all-to-all to output-row slabs -> inverse along x.
//    Both exchanges run per chunk on a communication stream while the pass producing
//    the next chunk runs on the caller's stream (rows chunks for exchange 1, column
//    chunks for exchange 2), so the NVLink transfer overlaps the compute.
//
// Every arithmetic step is an hd_pass launch (hd_api.cu); this file only computes
// partitions and layouts (integers) and orders launches and NCCL calls.  NCCL is
// resolved at run time (dlopen of libnccl.so.2: the copy torch already loaded, else
// the system one), so the library loads without it.
#include "hdconv.h"
#include "hd_internal.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

hd_status_t derr(hd_status_t st, const std::string& m) {
  g_err = m;
  return st;
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- NCCL (run-time bound)
struct Nccl {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclReduceScatter) ReduceScatter = nullptr;
  decltype(&ncclGetErrorString) ErrorString = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { n.why = std::string("libnccl.so.2 not found: ") + dlerror(); return; }
    bool all = true;
    auto get = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      if (!fp) all = false;
    };
    get(n.GetUniqueId, "ncclGetUniqueId");
    get(n.CommInitRank, "ncclCommInitRank");
    get(n.CommDestroy, "ncclCommDestroy");
    get(n.GroupStart, "ncclGroupStart");
    get(n.GroupEnd, "ncclGroupEnd");
    get(n.Send, "ncclSend");
    get(n.Recv, "ncclRecv");
    get(n.ReduceScatter, "ncclReduceScatter");
    get(n.ErrorString, "ncclGetErrorString");
    n.ok = all;
    if (!all) n.why = "libnccl.so.2 lacks a required symbol";
  });
  return n;
}

hd_status_t nccl_fail(ncclResult_t r, const char* what) {
  return derr(HD_ERR_NCCL, std::string(what) + ": " + (nccl().ErrorString ? nccl().ErrorString(r) : "nccl error"));
}

// ---------------------------------------------------------------- per-context state
struct Dist {
  ncclComm_t comm = nullptr;
  int n = 1, rank = 0, device = 0;
  cudaStream_t cs = nullptr;             // communication stream
  std::vector<cudaEvent_t> ev;            // compute -> communication hand-over, per chunk
  cudaEvent_t evx = nullptr;              // communication -> compute
  void* buf = nullptr;                    // exchange buffers (grown on demand)
  size_t buf_size = 0;
};
std::mutex g_mu;
std::map<hd_ctx_t, Dist*> g_dist;

Dist* find(hd_ctx_t ctx) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_dist.find(ctx);
  return it == g_dist.end() ? nullptr : it->second;
}

hd_status_t ensure_events(Dist* d, size_t n) {
  while (d->ev.size() < n) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return derr(HD_ERR_CUDA, "cudaEventCreate");
    d->ev.push_back(e);
  }
  if (!d->evx && cudaEventCreateWithFlags(&d->evx, cudaEventDisableTiming) != cudaSuccess)
    return derr(HD_ERR_CUDA, "cudaEventCreate");
  return HD_OK;
}

hd_status_t ensure_buf(Dist* d, size_t bytes) {
  if (d->buf_size >= bytes) return HD_OK;
  cudaDeviceSynchronize();  // the old buffer may still be in flight on either stream
  if (d->buf) cudaFree(d->buf);
  d->buf = nullptr;
  d->buf_size = 0;
  if (cudaMalloc(&d->buf, bytes) != cudaSuccess) return derr(HD_ERR_CUDA, "cudaMalloc(exchange buffers)");
  d->buf_size = bytes;
  return HD_OK;
}

size_t a256(size_t b) { return (b + 255) & ~size_t(255); }

hd_lines_t lines(void* p, int64_t L, int64_t s_l) {
  hd_lines_t x;
  std::memset(&x, 0, sizeof(x));
  x.ptr[0] = p;
  x.L = L;
  x.tl = 40;
  x.s_l = s_l;
  x.s_j = 1;
  return x;
}
void elem_tiled(hd_lines_t& x, int64_t jd, int64_t s_jt, int64_t s_j) {
  x.jd = jd;
  x.s_jt = s_jt;
  x.s_j = s_j;
}
void line_tiled(hd_lines_t& x, int64_t T, int64_t s_t) {  // line l at (l / T) s_t + l % T
  if (T <= 1) { x.s_l = s_t; return; }
  int tl = 0;
  while ((int64_t(1) << tl) < T) ++tl;
  x.tl = tl;
  x.s_t = s_t;
  x.s_l = 1;
}
hd_pass_desc_t pass(int mode, int64_t nlines, int64_t nbatch, int64_t M, const hd_axis_plan_t& ax, int C) {
  hd_pass_desc_t d;
  std::memset(&d, 0, sizeof(d));
  d.mode = mode;
  d.npairs = 1;
  d.nlines = nlines;
  d.nbatch = nbatch;
  d.M = M;
  d.axis.m = ax.m;
  d.axis.C = C;
  d.axis.D = 0;
  d.axis.threads = 0;
  return d;
}
void* off(void* p, int64_t elems, size_t eb) { return static_cast<char*>(p) + elems * (int64_t)eb; }
const void* off(const void* p, int64_t elems, size_t eb) { return static_cast<const char*>(p) + elems * (int64_t)eb; }

// one chunk of an all-to-all of equal blocks: rank d's piece at send + d * block + c_off
// goes to d's recv + rank * block + c_off (self included)
// piece p of the send buffer at send_off + p * send_stride, piece p of the receive
// buffer (from rank p) at recv_off + p * recv_stride, `count` elements each
hd_status_t exchange_pieces(Dist* D, void* send, int64_t send_off, int64_t send_stride, void* recv,
                            int64_t recv_off, int64_t recv_stride, int64_t count, size_t eb) {
  if (count <= 0) return HD_OK;
  Nccl& N = nccl();
  const ncclDataType_t ty = eb == 16 ? ncclFloat64 : ncclFloat32;  // complex = 2 reals
  const size_t cnt = (size_t)count * 2;
  ncclResult_t r = N.GroupStart();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
  for (int p = 0; p < D->n; ++p) {
    r = N.Send(off(send, send_off + p * send_stride, eb), cnt, ty, p, D->comm, D->cs);
    if (r != ncclSuccess) { N.GroupEnd(); return nccl_fail(r, "ncclSend"); }
    r = N.Recv(off(recv, recv_off + p * recv_stride, eb), cnt, ty, p, D->comm, D->cs);
    if (r != ncclSuccess) { N.GroupEnd(); return nccl_fail(r, "ncclRecv"); }
  }
  r = N.GroupEnd();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
  return HD_OK;
}

hd_status_t exchange_chunk(Dist* D, void* send, void* recv, int64_t block, int64_t c_off, int64_t count,
                           size_t eb) {
  if (count <= 0) return HD_OK;
  Nccl& N = nccl();
  const ncclDataType_t ty = eb == 16 ? ncclFloat64 : ncclFloat32;  // complex = 2 reals
  const size_t cnt = (size_t)count * 2;
  ncclResult_t r = N.GroupStart();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
  for (int p = 0; p < D->n; ++p) {
    r = N.Send(off(send, p * block + c_off, eb), cnt, ty, p, D->comm, D->cs);
    if (r != ncclSuccess) { N.GroupEnd(); return nccl_fail(r, "ncclSend"); }
    r = N.Recv(off(recv, p * block + c_off, eb), cnt, ty, p, D->comm, D->cs);
    if (r != ncclSuccess) { N.GroupEnd(); return nccl_fail(r, "ncclRecv"); }
  }
  r = N.GroupEnd();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
  return HD_OK;
}

hd_status_t ctx_fail(hd_ctx_t ctx, hd_status_t st) {
  if (st != HD_OK) g_err = std::string(hd_last_error(ctx));
  return st;
}

}  // namespace

namespace hd {
void dist_release(hd_ctx_t ctx) {
  Dist* d = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_dist.find(ctx);
    if (it == g_dist.end()) return;
    d = it->second;
    g_dist.erase(it);
  }
  if (d->cs) cudaStreamSynchronize(d->cs);
  if (d->comm && nccl().CommDestroy) nccl().CommDestroy(d->comm);
  for (auto e : d->ev) cudaEventDestroy(e);
  if (d->evx) cudaEventDestroy(d->evx);
  if (d->cs) cudaStreamDestroy(d->cs);
  if (d->buf) cudaFree(d->buf);
  delete d;
}
}  // namespace hd

extern "C" {

const char* hd_dist_last_error(void) { return g_err.c_str(); }

hd_status_t hd_dist_unique_id(void* id) {
  if (!id) return derr(HD_ERR_INVALID, "null id");
  Nccl& N = nccl();
  if (!N.ok) return derr(HD_ERR_NCCL, N.why);
  ncclUniqueId u;
  ncclResult_t r = N.GetUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof(u));
  return HD_OK;
}

hd_status_t hd_dist_init(hd_ctx_t ctx, const void* id, int32_t nranks, int32_t rank) {
  if (!ctx) return derr(HD_ERR_INVALID, "null context");
  if (nranks < 1 || rank < 0 || rank >= nranks) return derr(HD_ERR_INVALID, "need 0 <= rank < nranks");
  if (nranks > 1 && !id) return derr(HD_ERR_INVALID, "null NCCL unique id");
  hd::dist_release(ctx);
  int dev = 0;
  cudaGetDevice(&dev);
  Dist* d = new Dist();
  d->n = nranks;
  d->rank = rank;
  d->device = dev;
  if (cudaStreamCreateWithFlags(&d->cs, cudaStreamNonBlocking) != cudaSuccess) {
    delete d;
    return derr(HD_ERR_CUDA, "cudaStreamCreate(comm)");
  }
  if (nranks > 1) {
    Nccl& N = nccl();
    if (!N.ok) {
      cudaStreamDestroy(d->cs);
      delete d;
      return derr(HD_ERR_NCCL, N.why);
    }
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ncclResult_t r = N.CommInitRank(&d->comm, nranks, u, rank);
    if (r != ncclSuccess) {
      cudaStreamDestroy(d->cs);
      delete d;
      return nccl_fail(r, "ncclCommInitRank");
    }
  }
  std::lock_guard<std::mutex> lk(g_mu);
  g_dist[ctx] = d;
  return HD_OK;
}

hd_status_t hd_dist_partition(int64_t extent, int32_t nranks, int32_t rank, int64_t* lo, int64_t* hi) {
  if (!lo || !hi || extent < 0 || nranks < 1 || rank < 0 || rank >= nranks)
    return derr(HD_ERR_INVALID, "bad partition arguments");
  const int64_t per = cdiv(extent, nranks);
  *lo = std::min<int64_t>(rank * per, extent);
  *hi = std::min<int64_t>((rank + 1) * per, extent);
  return HD_OK;
}

// The slab layout of a 2-D / 3-D problem (host only): see include/hdconv.h.
hd_status_t hd_dist_slab_plan(hd_dtype_t dtype, int32_t ndim, int32_t nranks, int32_t rank, int32_t nchunks,
                              const int64_t* Lf, const int64_t* Lg, const hd_plan_t* plan, hd_slab_plan_t* out) {
  if (!Lf || !Lg || !out) return derr(HD_ERR_INVALID, "null argument");
  if (ndim != 2 && ndim != 3) return derr(HD_ERR_INVALID, "slab decomposition needs ndim 2 or 3");
  if (nranks < 1 || rank < 0 || rank >= nranks) return derr(HD_ERR_INVALID, "need 0 <= rank < nranks");
  if (nchunks < 0) return derr(HD_ERR_INVALID, "nchunks must be >= 0");
  hd_plan_t p;
  hd_status_t s;
  if (plan) {
    p = *plan;
    s = hd_plan_complete(dtype, ndim, 1, Lf, Lg, nullptr, &p);
  } else {
    s = hd_plan_default(dtype, ndim, 1, Lf, Lg, nullptr, &p);
    if (s == HD_OK) s = hd_plan_complete(dtype, ndim, 1, Lf, Lg, nullptr, &p);
  }
  if (s != HD_OK) return derr(s, "plan: " + std::string(hd_last_error(nullptr)));
  hd_slab_plan_t o;
  std::memset(&o, 0, sizeof(o));
  o.ndim = ndim;
  o.nranks = nranks;
  o.rank = rank;
  o.scale = 1.0;
  for (int i = 0; i < ndim; ++i) o.scale /= (double)p.axis[i].M1;
  const size_t eb = dtype == HD_C128 ? 16 : 8;
  const int64_t O0 = Lf[0] + Lg[0] - 1;
  if (ndim == 2) {
    const int C = nchunks > 0 ? nchunks : (nranks > 1 ? 2 : 1);  // 2 balances launch count and overlap
    o.nchunks = C;
    const int64_t Kx = p.axis[1].M1;
    o.chunk_rows = cdiv(cdiv(Lf[0], nranks), C);
    o.R = C * o.chunk_rows;
    o.chunk_cols = cdiv(cdiv(cdiv(Kx, nranks), C), 16) * 16;  // 16-wide kx tiles (send1)
    o.Ks = C * o.chunk_cols;
    o.Ro = cdiv(O0, nranks);
    o.block1 = o.Ks * o.R;
    o.block2 = o.Ks * o.Ro;
    o.spec_lo = std::min<int64_t>(rank * o.Ks, Kx);
    o.spec_hi = std::min<int64_t>((rank + 1) * o.Ks, Kx);
  } else {
    o.nchunks = 1;
    const int64_t Ky = p.axis[1].M1, Kx = p.axis[2].M1;
    o.chunk_rows = o.R = cdiv(Lf[0], nranks);    // f planes per rank
    o.Ro = cdiv(O0, nranks);                     // output planes per rank
    o.Ks = cdiv(Ky, nranks);                     // spectral y rows per rank
    o.chunk_cols = (Kx % 4 == 0) ? 4 : 1;        // kx tile T of the exchange blocks
    o.block1 = o.Ks * Kx * o.R;
    o.block2 = o.Ks * Kx * o.Ro;
    o.spec_lo = std::min<int64_t>(rank * o.Ks, Ky);
    o.spec_hi = std::min<int64_t>((rank + 1) * o.Ks, Ky);
  }
  o.in_lo = std::min<int64_t>(rank * o.R, Lf[0]);
  o.in_hi = std::min<int64_t>((rank + 1) * o.R, Lf[0]);
  o.out_lo = std::min<int64_t>(rank * o.Ro, O0);
  o.out_hi = std::min<int64_t>((rank + 1) * o.Ro, O0);
  o.bytes_sent = (int64_t)(nranks - 1) * (o.block1 + o.block2) * (int64_t)eb;
  o.plan = p;
  *out = o;
  return HD_OK;
}

// ---------------------------------------------------------------- 1-D
hd_status_t hd_conv1d_dist(hd_ctx_t ctx, hd_dtype_t dtype, int64_t batch, const void* f, int64_t Lf, const void* g,
                           int64_t Lg, void* h, const hd_plan_t* plan, uint32_t shard, void* stream) {
  if (!ctx || !f || !g || !h) return derr(HD_ERR_INVALID, "null argument");
  if (batch < 1 || Lf < 1 || Lg < 1) return derr(HD_ERR_INVALID, "bad extents");
  Dist* D = find(ctx);
  if (!D) return derr(HD_ERR_INVALID, "hd_dist_init has not been called on this context");
  const size_t eb = dtype == HD_C128 ? 16 : 8;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t b0, b1;
  hd_dist_partition(batch, D->n, D->rank, &b0, &b1);
  if (shard == HD_SHARD_BATCH) {
    // f, g, h hold this rank's batch slice [b0, b1) only: independent pairs, no collective
    if (b1 <= b0) return HD_OK;
    return ctx_fail(ctx, hd_conv1d(ctx, dtype, b1 - b0, f, Lf, g, Lg, h, 0, plan, nullptr, 0, stream));
  }
  if (shard != HD_SHARD_RESIDUE) return derr(HD_ERR_INVALID, "shard must be HD_SHARD_BATCH or HD_SHARD_RESIDUE");
  // f, g: the whole batch on every rank; this rank convolves residues [r0, r1) of every
  // line, and the partial sums are reduce-scattered: h = rows [b0, b1) of the result
  const int64_t Lout = Lf + Lg - 1;
  hd_plan_t p;
  hd_status_t s;
  if (plan) { p = *plan; s = hd_plan_complete(dtype, 1, 1, &Lf, &Lg, nullptr, &p); }
  else {
    s = hd_plan_default(dtype, 1, 1, &Lf, &Lg, nullptr, &p);
    if (s == HD_OK) s = hd_plan_complete(dtype, 1, 1, &Lf, &Lg, nullptr, &p);
  }
  if (s != HD_OK) return derr(s, "plan: " + std::string(hd_last_error(nullptr)));
  const hd_axis_plan_t& ax = p.axis[0];
  int64_t r0, r1;
  hd_dist_partition(ax.q, D->n, D->rank, &r0, &r1);
  const int64_t Bc = cdiv(batch, D->n);
  void* part = h;
  void* slice = nullptr;  // reduce-scatter target: Bc rows (the last rank may own fewer)
  if (D->n > 1) {
    const size_t bp = a256((size_t)D->n * Bc * Lout * eb);
    s = ensure_buf(D, bp + a256((size_t)Bc * Lout * eb));
    if (s != HD_OK) return s;
    part = D->buf;
    slice = static_cast<char*>(D->buf) + bp;
    if (r1 <= r0 && cudaMemsetAsync(part, 0, (size_t)D->n * Bc * Lout * eb, st) != cudaSuccess)
      return derr(HD_ERR_CUDA, "cudaMemsetAsync");
  }
  if (r1 > r0) {
    hd_pass_desc_t d = pass(HD_PASS_CONV, batch, 1, ax.M1, ax, ax.C ? ax.C : 1);
    d.axis.D = ax.D;
    d.in_f = lines(const_cast<void*>(f), Lf, Lf);
    d.in_g = lines(const_cast<void*>(g), Lg, Lg);
    d.out = lines(part, Lout, Lout);
    d.scale = 1.0 / (double)ax.M1;
    d.r_begin = (int32_t)r0;
    d.r_end = (int32_t)r1;
    s = hd_pass(ctx, dtype, &d, stream);
    if (s != HD_OK) return ctx_fail(ctx, s);
  }
  if (D->n == 1) return HD_OK;
  s = ensure_events(D, 1);
  if (s != HD_OK) return s;
  cudaEventRecord(D->ev[0], st);
  cudaStreamWaitEvent(D->cs, D->ev[0], 0);
  Nccl& N = nccl();
  const size_t cnt = (size_t)Bc * Lout * 2;
  ncclResult_t r = N.ReduceScatter(part, slice, cnt, eb == 16 ? ncclFloat64 : ncclFloat32, ncclSum, D->comm, D->cs);
  if (r != ncclSuccess) return nccl_fail(r, "ncclReduceScatter");
  cudaEventRecord(D->evx, D->cs);
  cudaStreamWaitEvent(st, D->evx, 0);
  if (b1 > b0 && cudaMemcpyAsync(h, slice, (size_t)(b1 - b0) * Lout * eb, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return derr(HD_ERR_CUDA, "cudaMemcpyAsync(h slice)");
  return HD_OK;
}

// ---------------------------------------------------------------- 2-D slabs
// Layouts (elements; R, Ks padded to chunk multiples, Rc = R / C, Kc = Ks / C, Kc a
// multiple of 16; P1 = Ks Rc, one (rank, chunk) piece of the first exchange):
//   xg    [kx][y]                                   g forward along x (replicated)
//   send1 [row chunk][kx / 16][y % Rc][kx % 16]     pass A output, chunk c = rows [c Rc, (c+1) Rc):
//                                                   the 16-wide kx tiles of the pipeline's X, so the
//                                                   pass stores 256-byte pieces by TMA; the piece for
//                                                   dest d of chunk c is contiguous, at (c nranks + d) P1
//   recv1 [src ][row chunk][kx_local / 16][y % Rc][kx_local % 16]
//                                                   piece (src, c) at (src C + c) P1: element (kx_local, y)
//                                                   at (y / Rc) P1 + (kx_local / 16) 16 Rc + (y % Rc) 16 + kx_local % 16
//   send2 [col chunk][yo][kx % Kc]                  pass B output, chunk cc = local columns [cc Kc, (cc+1) Kc):
//                                                   chunk-major (P2 = Ro Kc; the piece for dest d of chunk cc
//                                                   is rows [d Ro, (d+1) Ro), at (cc nranks + d) P2), so a
//                                                   column is one line of element stride Kc (TMA stores)
//   recv2 [src ][col chunk][yo_local][kx % Kc]      piece (src, cc) at (src C + cc) P2: element (yo_local, kx)
//                                                   at (kx / Kc) Ro Kc + yo_local Kc + kx % Kc (plain rows
//                                                   at one rank: pass C loads each by one bulk copy)
// One chunk of one stage (c < 0: every chunk of the stage).
static hd_status_t slab2d_stage(hd_ctx_t ctx, hd_dtype_t dtype, const hd_slab_plan_t& S, const int64_t* Lf,
                                const int64_t* Lg, int stage, int c, const void* in, const void* xg, void* out,
                                void* stream) {
  const size_t eb = dtype == HD_C128 ? 16 : 8;
  const hd_axis_plan_t &ay = S.plan.axis[0], &ax = S.plan.axis[1];
  const int64_t Kx = ax.M1, Oy = Lf[0] + Lg[0] - 1, Ox = Lf[1] + Lg[1] - 1;
  const int C = S.nchunks;
  const int64_t Rc = S.chunk_rows, Kc = S.chunk_cols, Ks = S.Ks, Ro = S.Ro;
  const int64_t nrows = S.in_hi - S.in_lo, ncols = S.spec_hi - S.spec_lo, nro = S.out_hi - S.out_lo;
  // x passes in the staged engine's own spectral order when both qualify (forward and
  // inverse of the same axis must agree, hd_pass HD_FLAG_STAGED_ORDER)
  const uint32_t xflags = (dtype == HD_C128 && ax.m == 512 && ax.q <= 11 && ax.p_f <= 8 && ax.p_g <= 8)
                              ? HD_FLAG_STAGED_ORDER : 0u;
  hd_status_t s = HD_OK;
  const int c0 = c < 0 ? 0 : c, c1 = c < 0 ? C : c + 1;
  if (stage == 0) {  // g forward along x: xg[kx][y]
    hd_pass_desc_t d = pass(HD_PASS_FWD, Lg[0], 1, Kx, ax, 1);
    d.flags = xflags;
    d.in_f = lines(const_cast<void*>(in), Lg[1], Lg[1]);
    d.out = lines(out, Kx, 1);
    d.out.s_j = Lg[0];
    return hd_pass(ctx, dtype, &d, stream);
  }
  for (int cc = c0; cc < c1; ++cc) {
    if (stage == 1) {  // pass A: rows of chunk cc -> send1
      const int64_t y0 = cc * Rc, y1 = std::min<int64_t>((cc + 1) * Rc, nrows);
      if (y1 <= y0) continue;
      hd_pass_desc_t d = pass(HD_PASS_FWD, y1 - y0, 1, Kx, ax, 1);
      d.flags = xflags;
      d.in_f = lines(const_cast<void*>(off(in, y0 * Lf[1], eb)), Lf[1], Lf[1]);
      d.out = lines(off(out, cc * S.nranks * Ks * Rc, eb), Kx, 16);
      elem_tiled(d.out, 16, 16 * Rc, 1);
      s = hd_pass(ctx, dtype, &d, stream);
    } else if (stage == 2) {  // pass B: columns of chunk cc, recv1 + xg -> send2
      const int64_t k0 = cc * Kc, k1 = std::min<int64_t>((cc + 1) * Kc, ncols);
      if (k1 <= k0) continue;
      hd_pass_desc_t d = pass(HD_PASS_CONV, k1 - k0, 1, ay.M1, ay, 1);
      d.in_f = lines(const_cast<void*>(off(in, k0 * Rc, eb)), Lf[0], 1);
      line_tiled(d.in_f, 16, 16 * Rc);
      elem_tiled(d.in_f, Rc, Ks * Rc, 16);
      d.in_g = lines(const_cast<void*>(off(xg, (S.spec_lo + k0) * Lg[0], eb)), Lg[0], Lg[0]);
      d.out = lines(off(out, cc * S.nranks * Ro * Kc, eb), Oy, 1);
      d.out.tl = 0;  // lines as tiles of width 1 (same addresses): TMA stores of the
      d.out.s_t = 1; // 16-byte pieces, element stride Kc (hd_api.cu)
      d.out.s_j = Kc;
      d.scale = S.scale;
      s = hd_pass(ctx, dtype, &d, stream);
    } else if (stage == 3) {  // pass C: recv2 -> output rows (all chunks at once)
      if (cc != c0 || nro <= 0) continue;
      hd_pass_desc_t d = pass(HD_PASS_INV, nro, 1, Kx, ax, 1);
      d.flags = xflags;
      d.in_f = lines(const_cast<void*>(in), Kx, Kc);
      elem_tiled(d.in_f, Kc, Ro * Kc, 1);
      d.out = lines(out, Ox, Ox);
      s = hd_pass(ctx, dtype, &d, stream);
    } else {
      return derr(HD_ERR_INVALID, "stage must be 0..3");
    }
    if (s != HD_OK) return s;
  }
  return HD_OK;
}

// ---------------------------------------------------------------- 3-D slabs
// z-slabs (S.R planes of f per rank, g replicated); T = S.chunk_cols kx tile.
//   X1    [z][kx/T][y][kx%T]                    x forward of the planes (scratch)
//   xyg   [ky][kx/T][z][kx%T]                   g's x and y forward (stage 0)
//   send1 [dest][kyl][kx/T][zl][kx%T]           y forward (ky = dest Ks + kyl)       (stage 1)
//   recv1 [src][kyl][kx/T][zl][kx%T]            -> lines (kyl, kx) of z = src R + zl
//   send2 [dest][zol][kx/T][kyl][kx%T]          convolution along z (zo = dest Ro + zol) (stage 2)
//   recv2 [src][zol][kx/T][kyl][kx%T]           -> lines (zol, kx) of ky = src Ks + kyl
//   W     [zol][y/T][kx][y%T]                   y inverse (scratch), then x inverse -> h (stage 3)
static hd_status_t slab3d_stage(hd_ctx_t ctx, hd_dtype_t dtype, const hd_slab_plan_t& S, const int64_t* Lf,
                                const int64_t* Lg, int stage, const void* in, const void* xyg, void* out,
                                void* scratch, void* stream) {
  const size_t eb = dtype == HD_C128 ? 16 : 8;
  const hd_axis_plan_t &az = S.plan.axis[0], &ay = S.plan.axis[1], &ax = S.plan.axis[2];
  const int64_t Ky = ay.M1, Kx = ax.M1;
  const int64_t O0 = Lf[0] + Lg[0] - 1, O1 = Lf[1] + Lg[1] - 1, O2 = Lf[2] + Lg[2] - 1;
  const int64_t T = S.chunk_cols, Rz = S.R, Roz = S.Ro, Kys = S.Ks;
  const int64_t nz = S.in_hi - S.in_lo, nzo = S.out_hi - S.out_lo, nky = S.spec_hi - S.spec_lo;
  const int64_t Oyp = cdiv(O1, T) * T;
  auto staged = [&](const hd_axis_plan_t& a) {
    return dtype == HD_C64 && a.m == 128 && a.q <= 8 && std::max(a.p_f, a.p_g) <= 8;
  };
  auto desc = [&](int mode, const hd_axis_plan_t& a, int64_t nl, int64_t nb) {
    const bool stg = T == 4 && staged(a);
    hd_pass_desc_t d = pass(mode, nl, nb, a.M1, a, stg ? 4 : 1);
    if (stg && mode != HD_PASS_CONV) d.flags = HD_FLAG_STAGED_ORDER;
    return d;
  };
  // x then y forward of nzz planes [z][y][x] (Ly, Lx); element (z, ky, kx) of the result
  // at out + ky-part + (kx / T) s_t + kx % T + z s_z (ky-part: ky s_ky, or
  // (ky / jd) s_jt + (ky % jd) s_ky when jd > 0); X1 in `scratch`
  auto xy = [&](const void* src, int64_t nzz, int64_t Ly, int64_t Lx, void* o, int64_t s_ky, int64_t s_t,
                int64_t s_z, int64_t jd, int64_t s_jt) -> hd_status_t {
    hd_pass_desc_t d = desc(HD_PASS_FWD, ax, Ly, nzz);
    d.in_f = lines(const_cast<void*>(src), Lx, Lx);
    d.in_f.s_b = Ly * Lx;
    d.in_f.nbi = nzz;
    d.out = lines(scratch, Kx, T);
    if (T > 1) elem_tiled(d.out, T, Ly * T, 1);
    else d.out.s_j = Ly;
    d.out.s_b = Kx * Ly;
    d.out.nbi = nzz;
    hd_status_t r = hd_pass(ctx, dtype, &d, stream);
    if (r != HD_OK) return r;
    hd_pass_desc_t e = desc(HD_PASS_FWD, ay, Kx, nzz);
    e.in_f = lines(scratch, Ly, 0);
    line_tiled(e.in_f, T, Ly * T);
    e.in_f.s_j = T;
    e.in_f.s_b = Kx * Ly;
    e.in_f.nbi = nzz;
    e.out = lines(o, Ky, 0);
    line_tiled(e.out, T, s_t);
    e.out.s_j = s_ky;
    if (jd > 0) { e.out.jd = jd; e.out.s_jt = s_jt; }
    e.out.s_b = s_z;
    e.out.nbi = nzz;
    e.batch_fastest = 1;
    return hd_pass(ctx, dtype, &e, stream);
  };
  if (stage == 0) return xy(in, Lg[0], Lg[1], Lg[2], out, Kx * Lg[0], Lg[0] * T, T, 0, 0);
  if (stage == 1) {
    if (nz <= 0) return HD_OK;
    const bool tiled = Kys < Ky;
    return xy(in, nz, Lf[1], Lf[2], out, Kx * Rz, Rz * T, T, tiled ? Kys : 0, tiled ? S.block1 : 0);
  }
  if (stage == 2) {
    if (nky <= 0) return HD_OK;
    hd_pass_desc_t d = desc(HD_PASS_CONV, az, Kx, nky);
    d.in_f = lines(const_cast<void*>(in), Lf[0], 0);
    line_tiled(d.in_f, T, Rz * T);
    d.in_f.s_j = T;
    if (Rz < Lf[0]) { d.in_f.jd = Rz; d.in_f.s_jt = S.block1; }
    d.in_f.s_b = Kx * Rz;
    d.in_f.nbi = nky;
    d.in_g = lines(const_cast<void*>(off(xyg, S.spec_lo * Kx * Lg[0], eb)), Lg[0], 0);
    line_tiled(d.in_g, T, Lg[0] * T);
    d.in_g.s_j = T;
    d.in_g.s_b = Kx * Lg[0];
    d.in_g.nbi = nky;
    d.out = lines(out, O0, 0);
    line_tiled(d.out, T, Kys * T);
    d.out.s_j = Kx * Kys;
    if (Roz < O0) { d.out.jd = Roz; d.out.s_jt = S.block2; }
    d.out.s_b = T;
    d.out.nbi = nky;
    d.scale = S.scale;
    d.batch_fastest = 1;
    return hd_pass(ctx, dtype, &d, stream);
  }
  if (stage == 3) {
    if (nzo <= 0) return HD_OK;
    hd_pass_desc_t d = desc(HD_PASS_INV, ay, Kx, nzo);
    d.in_f = lines(const_cast<void*>(in), Ky, 0);
    line_tiled(d.in_f, T, Kys * T);
    d.in_f.s_j = T;
    if (Kys < Ky) { d.in_f.jd = Kys; d.in_f.s_jt = S.block2; }
    d.in_f.s_b = Kx * Kys;
    d.in_f.nbi = nzo;
    d.out = lines(scratch, O1, T);
    if (T > 1) elem_tiled(d.out, T, Kx * T, 1);
    else d.out.s_j = Kx;
    d.out.s_b = Oyp * Kx;
    d.out.nbi = nzo;
    hd_status_t r = hd_pass(ctx, dtype, &d, stream);
    if (r != HD_OK) return r;
    hd_pass_desc_t e = desc(HD_PASS_INV, ax, O1, nzo);
    e.in_f = lines(scratch, Kx, 0);
    line_tiled(e.in_f, T, Kx * T);
    e.in_f.s_j = T;
    e.in_f.s_b = Oyp * Kx;
    e.in_f.nbi = nzo;
    e.out = lines(out, O2, O2);
    e.out.s_b = O1 * O2;
    e.out.nbi = nzo;
    return hd_pass(ctx, dtype, &e, stream);
  }
  return derr(HD_ERR_INVALID, "stage must be 0..3");
}

// scratch elements stage 1 / 3 of a 3-D slab need (X1 / W)
static int64_t slab3d_scratch(const hd_slab_plan_t& S, const int64_t* Lf, const int64_t* Lg) {
  const int64_t Kx = S.plan.axis[2].M1, T = S.chunk_cols;
  const int64_t zmax = std::max<int64_t>(std::max<int64_t>(S.in_hi - S.in_lo, Lg[0]), 1);
  const int64_t x1 = zmax * Kx * std::max(Lf[1], Lg[1]);
  const int64_t w = std::max<int64_t>(S.out_hi - S.out_lo, 1) * cdiv(Lf[1] + Lg[1] - 1, T) * T * Kx;
  return std::max(x1, w);
}

hd_status_t hd_slab_stage(hd_ctx_t ctx, hd_dtype_t dtype, const hd_slab_plan_t* S, const int64_t* Lf,
                          const int64_t* Lg, int32_t stage, const void* in, const void* gt, void* out,
                          void* scratch, void* stream) {
  if (!ctx || !S || !Lf || !Lg) return derr(HD_ERR_INVALID, "null argument");
  if (stage < 0 || stage > 3) return derr(HD_ERR_INVALID, "stage must be 0..3");
  if (!out || (!in && !(stage == 1 && S->in_hi <= S->in_lo))) return derr(HD_ERR_INVALID, "null buffer");
  if (stage == 2 && !gt) return derr(HD_ERR_INVALID, "stage 2 needs the transformed g");
  if (S->ndim == 3 && (stage == 0 || stage == 1 || stage == 3) && !scratch)
    return derr(HD_ERR_INVALID, "3-D stages 0, 1, 3 need scratch (hd_slab_scratch_bytes)");
  hd_status_t s = S->ndim == 2 ? slab2d_stage(ctx, dtype, *S, Lf, Lg, stage, -1, in, gt, out, stream)
                               : slab3d_stage(ctx, dtype, *S, Lf, Lg, stage, in, gt, out, scratch, stream);
  return ctx_fail(ctx, s);
}

size_t hd_slab_scratch_bytes(hd_dtype_t dtype, const hd_slab_plan_t* S, const int64_t* Lf, const int64_t* Lg) {
  if (!S || !Lf || !Lg || S->ndim != 3) return 0;
  return (size_t)slab3d_scratch(*S, Lf, Lg) * (dtype == HD_C128 ? 16 : 8);
}

size_t hd_slab_g_bytes(hd_dtype_t dtype, const hd_slab_plan_t* S, const int64_t* Lg) {
  if (!S || !Lg) return 0;
  const size_t eb = dtype == HD_C128 ? 16 : 8;
  if (S->ndim == 2) return (size_t)S->plan.axis[1].M1 * Lg[0] * eb;
  return (size_t)S->plan.axis[1].M1 * S->plan.axis[2].M1 * Lg[0] * eb;
}

// The distributed convolutions: stages on the caller's stream, all-to-alls on the
// communication stream (2-D: per chunk, right after the chunk is produced).
static hd_status_t slab_dist(hd_ctx_t ctx, hd_dtype_t dtype, int ndim, const void* f, const int64_t* Lf,
                             const void* g, const int64_t* Lg, void* h, const hd_plan_t* plan, int32_t nchunks,
                             void* stream) {
  if (!ctx || !g || !h || !Lf || !Lg) return derr(HD_ERR_INVALID, "null argument");
  Dist* D = find(ctx);
  if (!D) return derr(HD_ERR_INVALID, "hd_dist_init has not been called on this context");
  hd_slab_plan_t S;
  hd_status_t s = hd_dist_slab_plan(dtype, ndim, D->n, D->rank, ndim == 2 ? nchunks : 1, Lf, Lg, plan, &S);
  if (s != HD_OK) return s;
  if (S.in_hi > S.in_lo && !f) return derr(HD_ERR_INVALID, "null f slab");
  const size_t eb = dtype == HD_C128 ? 16 : 8;
  cudaStream_t st = (cudaStream_t)stream;
  const bool one = D->n == 1;
  const size_t bg = a256(hd_slab_g_bytes(dtype, &S, Lg));
  const size_t b1 = a256((size_t)D->n * S.block1 * eb), b2 = a256((size_t)D->n * S.block2 * eb);
  const size_t bsc = ndim == 3 ? a256((size_t)slab3d_scratch(S, Lf, Lg) * eb) : 0;
  s = ensure_buf(D, bg + bsc + (one ? 1 : 2) * (b1 + b2));
  if (s != HD_OK) return s;
  const int C = S.nchunks;
  s = ensure_events(D, (size_t)2 * C);
  if (s != HD_OK) return s;
  char* base = static_cast<char*>(D->buf);
  void* gt = base;
  void* scratch = base + bg;
  void* send1 = base + bg + bsc;
  void* send2 = base + bg + bsc + b1;
  void* recv1 = one ? send1 : base + bg + bsc + b1 + b2;
  void* recv2 = one ? send2 : base + bg + bsc + 2 * b1 + b2;
  auto stage = [&](int stg, int c, const void* in, const void* x, void* out) {
    return ndim == 2 ? slab2d_stage(ctx, dtype, S, Lf, Lg, stg, c, in, x, out, stream)
                     : slab3d_stage(ctx, dtype, S, Lf, Lg, stg, in, x, out, scratch, stream);
  };
  // one exchange: chunk c of the block (2-D: pieces of `piece` elements at c * piece)
  auto exchange = [&](int evi, void* send, void* recv, int64_t block, int64_t c_off, int64_t count) {
    if (one) return HD_OK;
    cudaEventRecord(D->ev[evi], st);
    cudaStreamWaitEvent(D->cs, D->ev[evi], 0);
    return exchange_chunk(D, send, recv, block, c_off, count, eb);
  };
  // the first 2-D exchange: send1 is chunk-major (piece for dest d of chunk c at
  // (c n + d) P1), recv1 source-major (piece from src s of chunk c at (s C + c) P1)
  // 2-D exchanges: send chunk-major (piece for dest d of chunk c at (c n + d) P), recv
  // source-major (piece from src s of chunk c at s block + c P)
  auto exchange_cm = [&](int evi, void* send, void* recv, int64_t block, int c, int64_t P) {
    if (one) return HD_OK;
    cudaEventRecord(D->ev[evi], st);
    cudaStreamWaitEvent(D->cs, D->ev[evi], 0);
    return exchange_pieces(D, send, c * D->n * P, P, recv, c * P, block, P, eb);
  };
  auto join = [&]() {
    if (one) return;
    cudaEventRecord(D->evx, D->cs);
    cudaStreamWaitEvent(st, D->evx, 0);
  };
  const int64_t piece1 = ndim == 2 ? S.Ks * S.chunk_rows : S.block1;
  const int64_t piece2 = ndim == 2 ? S.Ro * S.chunk_cols : S.block2;
  // 3-D: stage 1 reads the transformed g (the y forward of g's planes happens there)
  if (ndim == 3 && (s = stage(0, -1, g, nullptr, gt)) != HD_OK) return ctx_fail(ctx, s);
  for (int c = 0; c < C; ++c) {
    if ((s = stage(1, c, f, nullptr, send1)) != HD_OK) return ctx_fail(ctx, s);
    if ((s = ndim == 2 ? exchange_cm(c, send1, recv1, S.block1, c, piece1)
                       : exchange(c, send1, recv1, S.block1, c * piece1, piece1)) != HD_OK)
      return s;
  }
  // 2-D: g's forward pass (needed from pass B on) runs while the last exchanges fly
  if (ndim == 2 && (s = stage(0, -1, g, nullptr, gt)) != HD_OK) return ctx_fail(ctx, s);
  join();
  for (int c = 0; c < C; ++c) {
    if ((s = stage(2, c, recv1, gt, send2)) != HD_OK) return ctx_fail(ctx, s);
    if ((s = ndim == 2 ? exchange_cm(C + c, send2, recv2, S.block2, c, piece2)
                       : exchange(C + c, send2, recv2, S.block2, c * piece2, piece2)) != HD_OK)
      return s;
  }
  join();
  if ((s = stage(3, -1, recv2, nullptr, h)) != HD_OK) return ctx_fail(ctx, s);
  return HD_OK;
}

hd_status_t hd_conv2d_dist(hd_ctx_t ctx, hd_dtype_t dtype, const void* f_rows, const int64_t Lf[2], const void* g,
                           const int64_t Lg[2], void* h_rows, const hd_plan_t* plan, int32_t nchunks, void* stream) {
  return slab_dist(ctx, dtype, 2, f_rows, Lf, g, Lg, h_rows, plan, nchunks, stream);
}

hd_status_t hd_conv3d_dist(hd_ctx_t ctx, hd_dtype_t dtype, const void* f_planes, const int64_t Lf[3], const void* g,
                           const int64_t Lg[3], void* h_planes, const hd_plan_t* plan, void* stream) {
  return slab_dist(ctx, dtype, 3, f_planes, Lf, g, Lg, h_planes, plan, 1, stream);
}

}  // extern "C"
