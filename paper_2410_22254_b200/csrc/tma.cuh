// TMA tensor maps (host) and tiled tensor loads (device) for the plain-layout
// GEMM operands.  Packs stack their lanes as the outermost tensor dimension,
// so one CUtensorMap serves every lane of a grouped launch (coordinate 2 =
// lane).  cuTensorMapEncodeTiled is resolved through the runtime's driver
// entry point (no link-time libcuda dependency).
#pragma once
#include <cuda.h>

#include "tlk_common.cuh"
#include "tlk_ptx.cuh"

namespace tlk {

// bf16 3-D tensor [d2][d1][d0] (d0 contiguous) -> tensor map with box
// {b0, b1, 1} and 128-byte swizzle (b0 * 2 must be 128).
int make_tmap_bf16_3d(CUtensorMap* out, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                      uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1);

// bf16 5-D tensor (dims[0] contiguous, byte strides of dims 1..4) -> tensor
// map with box {b0, b1, 1, 1, 1}, 128-byte swizzle.  Size-1 dims may pass
// any stride (it is replaced by a valid one).
int make_tmap_bf16_5d(CUtensorMap* out, const void* base, const uint64_t dims[5],
                      const uint64_t strides_bytes[4], uint32_t b0, uint32_t b1, uint32_t b2 = 1,
                      uint32_t b3 = 1);

TLK_DEV void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

// Box load: smem (swizzled) <- tensor[c2][c1 .. c1+b1)[c0 .. c0+b0), completing
// the box's bytes on `bar`.  Out-of-range elements are zero-filled.
TLK_DEV void tma_load_3d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

TLK_DEV void tma_load_5d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4,
                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"(smem_u32(bar))
      : "memory");
}

// L2 prefetch of the same box (no shared-memory destination, no completion)
TLK_DEV void tma_prefetch_l2_5d(const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
               : "memory");
}

// Generic 5-D tensor map (dims[0] contiguous, byte strides of dims 1..4),
// box {b0, b1, 1, 1, 1}, given element type and swizzle (epilogue tiles).
int make_tmap_5d(CUtensorMap* out, CUtensorMapDataType dt, const void* base, const uint64_t dims[5],
                 const uint64_t strides_bytes[4], uint32_t b0, uint32_t b1, CUtensorMapSwizzle sw);

// Generic 3-D tensor map (dims[0] contiguous), box {b0, b1, 1}, given element
// type and swizzle; used for the fp32 optimizer-state tiles and the bf16
// shadow tile of the CNN's fused fc1 wgrad + Adam kernel.
int make_tmap_3d(CUtensorMap* out, CUtensorMapDataType dt, const void* base, uint64_t d0, uint64_t d1,
                 uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1,
                 CUtensorMapSwizzle sw);

// Box store: tensor[c2][c1 ..][c0 ..] <- smem (same layout/swizzle as a load),
// tracked by the issuing thread's bulk async-group.
TLK_DEV void tma_store_3d(const CUtensorMap* m, uint32_t src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
TLK_DEV void tma_store_5d(const CUtensorMap* m, uint32_t src, int c0, int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(m)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
TLK_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N bulk groups still READ their shared-memory source
template <int N>
TLK_DEV void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
TLK_DEV void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace tlk
