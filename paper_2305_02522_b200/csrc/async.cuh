// Bulk asynchronous copies (global -> shared) completing on mbarriers: the
// TMA path of the streaming kernels (window.cu, bmm.cu).  sm_90+ PTX.
#pragma once

#include <stdint.h>

namespace bg {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// The same wait, but a thread whose phase is not complete yet is suspended
// until it completes (or the hint, in ns, runs out) instead of re-polling:
// a ring consumer waiting behind the slowest warp then costs no issue slots.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
// Four fp32 values -> four +-1 bytes for a kind::i8 operand (x >= 0 -> 0x01,
// else 0xFF; -0.0 -> 0x01, NaN -> 0xFF, the oracle's comparison): one
// FSET.BF per value (1.0f / 0.0f: byte 2 is 0x80 / 0x00), byte 2 of each
// gathered sign-replicated (PRMT selector nibble 8 + 2, 8 + 6) into a 0xFF /
// 0x00 mask per byte by three byte permutes, then ~(mask & 0xFE) -- 8
// instructions per 4 values (a compare-and-select build takes 13).
__device__ __forceinline__ uint32_t ge0_bf(float x) {
  float m;
  asm("set.ge.f32.f32 %0, %1, 0f00000000;" : "=f"(m) : "f"(x));
  return __float_as_uint(m);
}
__device__ __forceinline__ uint32_t prmt_sx(uint32_t a, uint32_t b) {  // bytes: sx(a.b2), sx(b.b2), 0, 0
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x00EA;" : "=r"(r) : "r"(a), "r"(b));  // __byte_perm drops the nibbles' sign bit
  return r;
}
__device__ __forceinline__ uint32_t pm1_bytes4(float x0, float x1, float x2, float x3) {
  const uint32_t lo = prmt_sx(ge0_bf(x0), ge0_bf(x1)), hi = prmt_sx(ge0_bf(x2), ge0_bf(x3));
  return ~(__byte_perm(lo, hi, 0x5410u) & 0xFEFEFEFEu);
}
// 8-byte shared-memory load by shared-window address
__device__ __forceinline__ float2 lds_f2(uint32_t saddr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(saddr));
  return v;
}
// 16-byte shared-memory load by shared-window address
__device__ __forceinline__ float4 lds_f4(uint32_t saddr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(saddr));
  return v;
}

// global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// 4-byte global -> shared copy (LDGSTS): the issuing thread does not wait,
// so a staging loop keeps every copy in flight; cp_async_wait_all() then a
// barrier before the data is read.
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Bulk prefetch of [src, src + bytes) into L2 (16-byte aligned, multiple of 16).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

}  // namespace bg
