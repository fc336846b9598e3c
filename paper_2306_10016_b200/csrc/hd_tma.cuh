// hd_tma.cuh -- TMA / mbarrier / bulk-copy primitives (inline PTX) shared by the
// staged engines (hd_s512.cuh: m = 512 complex double; hd_s128.cuh: m = 128
// complex float).
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "hd_device.cuh"

namespace hd {

// ---------------------------------------------------------------------------
// TMA / mbarrier / bulk-copy primitives (PTX)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(bar)), "r"(bytes) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps until the phase completes
// (or ~1 ms passes) instead of re-issuing the probe, leaving issue slots to the
// compute warps of its SM sub-partition
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = su32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n}" :: "r"(a), "r"(parity), "r"(1000000u) : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, const int* c, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      :: "r"(su32(dst)), "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap* map, const int* c, const void* src) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
      :: "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(su32(src)) : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(dst), "r"(su32(src)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void compute_sync(int n) { asm volatile("bar.sync 1, %0;" :: "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(su32(bar)) : "memory");
}

// TMA coordinates of element j0 of line l, batch entry b (see TmaLine in hd_device.cuh)
__device__ __forceinline__ void tma_coords(const TmaLine& t, int64_t b, int64_t l, int j0, int* c) {
  const uint32_t ub = (uint32_t)b, un = (uint32_t)t.nbi;
  const uint32_t bo = ub / un;
  c[3] = (t.bcast & 1) ? 0 : (int)(ub - bo * un);
  c[4] = (t.bcast & 2) ? 0 : (int)bo;
  if (t.kind == TMA_LINE_TILED) {  // dims {2S (line in tile), j, line tile, b % nbi, b / nbi}
    c[0] = 2 * (int)(l & ((1 << t.slog) - 1));
    c[1] = j0;
    c[2] = (int)(l >> t.slog);
  } else if (t.kind == TMA_ELEM2) {  // dims {2S (line in tile), j % jd, j / jd, line tile, batch}
    const int jd = (int)t.jd;
    c[0] = 2 * (int)(l & ((1 << t.slog) - 1));
    c[1] = j0 % jd;
    c[2] = j0 / jd;
    c[3] = (int)(l >> t.slog);
    c[4] = (t.bcast & 1) ? 0 : (int)b;
  } else {                          // TMA_ELEM_TILED: dims {2S (j in tile), line, j tile, ...}
    c[0] = 0;
    c[1] = (int)l;
    c[2] = j0 >> t.slog;
  }
}

}  // namespace hd
