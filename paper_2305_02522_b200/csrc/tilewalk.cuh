// Warp-cooperative walk of one FRDC tile row (ref: bitsparse.hpp:22-25 tile
// layout; kernels.cpp:277-330 consumes the same bits one by one on the CPU).
//
// The 32 lanes stream the tile row's col_ind/tiles with coalesced
// non-allocating loads (one tile per lane per 32-tile chunk).  Every set bit
// (local row n, local column c) of a lane's tile becomes an entry j = 4*col+c
// in the shared-memory ring of node row n; a packed 4x8-bit warp scan gives
// each lane its slots and each lane loops once per set bit of its own tile
// (about once: synthetic graphs carry ~1 bit per tile).  After every chunk the
// caller's drain(n, head, count) consumes full batches of B entries per row;
// at the end the partial batches.  fill[n] ends as the degree of node row n.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "ops.cuh"

namespace bg {

constexpr int kRing = 256;  // ring entries per node row per warp (power of two)

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t ld_nc_u32(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));  // read-only data: no volatile
  return v;
}

__device__ __forceinline__ uint32_t ld_nc_u16(const uint16_t* p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}

// SWAR per-byte modular add of two packed 4x8-bit counters.
__device__ __forceinline__ uint32_t add_bytes(uint32_t a, uint32_t b) {
  return ((a & 0x7F7F7F7Fu) + (b & 0x7F7F7F7Fu)) ^ ((a ^ b) & 0x80808080u);
}

template <int n, class Drain>
__device__ __forceinline__ void drain_row(Drain& d, uint32_t h, uint32_t c) {
  d(std::integral_constant<int, n>{}, h, c);
}

// B: entries per drained batch.  Drain is called as drain(integral_constant<n>, head, count).
template <int B, class Drain>
__device__ __forceinline__ void walk_tile_row(const uint64_t* __restrict__ rp,
                                              const uint32_t* __restrict__ ci,
                                              const uint16_t* __restrict__ ti, int64_t tr,
                                              uint32_t (*ring)[kRing], uint32_t (&fill)[4],
                                              Drain& drain) {
  const int lane = threadIdx.x & 31;
  uint32_t head[4] = {0, 0, 0, 0};
  fill[0] = fill[1] = fill[2] = fill[3] = 0;
  uint32_t fillp = 0;  // fill[n] mod 256 packed in byte n
  const uint64_t t0 = rp[tr];
  const uint32_t cnt = static_cast<uint32_t>(rp[tr + 1] - t0);
  const uint16_t* tib = ti + t0;
  const uint32_t* cib = ci + t0;
  uint32_t* ring_base = &ring[0][0];
  for (uint32_t o = 0; o < cnt; o += 32) {
    __syncwarp();
    const uint32_t k = o + static_cast<uint32_t>(lane);
    uint32_t tile = 0, col = 0;
    if (k < cnt) {
      tile = ld_nc_u16(tib + k);
      col = ld_nc_u32(cib + k);
    }
    // per-row bit counts of this lane's tile, row n in byte n
    const uint32_t packed = __popc(tile & 0xF000u) | (__popc(tile & 0x0F00u) << 8) |
                            (__popc(tile & 0x00F0u) << 16) | (__popc(tile & 0x000Fu) << 24);
    uint32_t incl = packed;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += v;  // byte fields never exceed 128: no carries
    }
    const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    uint32_t slot = add_bytes(fillp, incl - packed);  // ring slot of this lane's next entry per row
    const uint32_t colx4 = 4 * col;
    uint32_t bits = tile;
    while (bits) {
      const int b = 31 - __clz(bits);  // bit b <-> (r, c) index 15 - b
      bits ^= 1u << b;
      const int rc = 15 - b;
      const int sh = 8 * (rc >> 2);
      ring_base[(rc >> 2) * kRing + ((slot >> sh) & (kRing - 1))] =
          colx4 + static_cast<uint32_t>(rc & 3);
      slot = add_bytes(slot, 1u << sh);
    }
    fill[0] += total & 0xFFu;
    fill[1] += (total >> 8) & 0xFFu;
    fill[2] += (total >> 16) & 0xFFu;
    fill[3] += total >> 24;
    fillp = add_bytes(fillp, total);
    __syncwarp();
    while (fill[0] - head[0] >= static_cast<uint32_t>(B)) { drain_row<0>(drain, head[0], B); head[0] += B; }
    while (fill[1] - head[1] >= static_cast<uint32_t>(B)) { drain_row<1>(drain, head[1], B); head[1] += B; }
    while (fill[2] - head[2] >= static_cast<uint32_t>(B)) { drain_row<2>(drain, head[2], B); head[2] += B; }
    while (fill[3] - head[3] >= static_cast<uint32_t>(B)) { drain_row<3>(drain, head[3], B); head[3] += B; }
  }
  __syncwarp();
  if (fill[0] > head[0]) drain_row<0>(drain, head[0], fill[0] - head[0]);
  if (fill[1] > head[1]) drain_row<1>(drain, head[1], fill[1] - head[1]);
  if (fill[2] > head[2]) drain_row<2>(drain, head[2], fill[2] - head[2]);
  if (fill[3] > head[3]) drain_row<3>(drain, head[3], fill[3] - head[3]);
}

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) {
  return (a & b) | (c & (a ^ b));
}

// Harley-Seal: add 8 words into bit-sliced planes P[0..NP) (P[q] weighs 2^q).
template <int NP>
__device__ __forceinline__ void hs_add8(uint32_t (&P)[NP], const uint32_t (&x)[8]) {
  uint32_t t1, t2, f1, f2, e, s;
  s = P[0] ^ x[0] ^ x[1]; t1 = maj3(P[0], x[0], x[1]); P[0] = s;
  s = P[0] ^ x[2] ^ x[3]; t2 = maj3(P[0], x[2], x[3]); P[0] = s;
  s = P[1] ^ t1 ^ t2;     f1 = maj3(P[1], t1, t2);     P[1] = s;
  s = P[0] ^ x[4] ^ x[5]; t1 = maj3(P[0], x[4], x[5]); P[0] = s;
  s = P[0] ^ x[6] ^ x[7]; t2 = maj3(P[0], x[6], x[7]); P[0] = s;
  s = P[1] ^ t1 ^ t2;     f2 = maj3(P[1], t1, t2);     P[1] = s;
  s = P[2] ^ f1 ^ f2;     e = maj3(P[2], f1, f2);      P[2] = s;
#pragma unroll
  for (int q = 3; q < NP; ++q) {
    const uint32_t nq = P[q] ^ e;
    e &= P[q];
    P[q] = nq;
  }
}

// Sum the bit-sliced counters of the S slot lanes that share word lane g
// (lanes g, g+G, g+2G, ...): every one of them ends with the total.
template <int G, int NP, int NQ>
__device__ __forceinline__ void slot_reduce(const uint32_t (&P)[NP], uint32_t (&Q)[NQ]) {
#pragma unroll
  for (int q = 0; q < NQ; ++q) Q[q] = q < NP ? P[q] : 0u;
#pragma unroll
  for (int d = G; d < 32; d <<= 1) {
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const uint32_t a = Q[q], b = __shfl_xor_sync(0xFFFFFFFFu, Q[q], d);
      Q[q] = a ^ b ^ c;
      c = maj3(a, b, c);
    }
  }
}

// Plane-wise comparison: bit b set iff count_b >= T (T uniform).
template <int NQ>
__device__ __forceinline__ uint32_t planes_ge(const uint32_t (&Q)[NQ], uint32_t T) {
  if (T >> NQ) return 0u;
  uint32_t gt = 0, eq = 0xFFFFFFFFu;
#pragma unroll
  for (int q = NQ - 1; q >= 0; --q) {
    if ((T >> q) & 1u) {
      eq &= Q[q];
    } else {
      gt |= eq & Q[q];
      eq &= ~Q[q];
    }
  }
  return gt | eq;
}

template <int NQ>
__device__ __forceinline__ uint32_t plane_count(const uint32_t (&Q)[NQ], int b) {
  uint32_t cnt = 0;
#pragma unroll
  for (int q = 0; q < NQ; ++q) cnt |= ((Q[q] >> (31 - b)) & 1u) << q;
  return cnt;
}

// Calls fn(col) for every adjacency bit of node row i in ascending column
// order (sliver entries are sorted; padding sentinels close the row).
template <class Fn>
__device__ __forceinline__ void for_each_col(const uint64_t* srp, const uint32_t* sl, int64_t i, Fn&& fn) {
  for (uint64_t e = srp[i]; e < srp[i + 1]; ++e) {
    const uint32_t ent = sl[e];
    if (ent == kSliverSentinel) break;
    const uint32_t first = ent >> 3;
    fn(first);
    for (uint32_t more = ent & 7u; more; more &= more - 1) fn(first + __ffs(more));
  }
}

}  // namespace bg
