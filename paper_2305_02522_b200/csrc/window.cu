// Column-windowed bit-SpMM (BSpMM.BBB / BBF, ref kernels.cpp:254-333 and the
// emit loop :438-465): out(i,k) = 2*#{j in N(i): x_jk = 1} - deg_i.
//
// Why: the per-edge gather of a 16-byte packed neighbour row from L2 costs one
// L1TEX wavefront per edge (ncu: the gather kernel k_sl_bb runs at 87% of
// L1TEX throughput), so a dense graph is bound at ~1 edge/clk/SM however the
// loads are shaped.  Here the packed operand streams through shared memory
// instead, one half-window of Wh node rows at a time (cp.async.bulk +
// mbarrier, a ring of three 64 KB slots), and each edge becomes one 16-byte
// LDS.  The CTA owns a block of T node rows, one per thread, whose
// bit-sliced counters stay in registers for the whole sweep.  Counting is
// order-free integer work, so the result equals the reference's
// TwoAndMinusPopc / IfElse / AndAndNot strategies bit for bit.
//
// Two-choice schedule: at step k the ring holds half-windows k and k+1, so an
// edge into half k may be counted at step k-1 or k.  A warp's 32 rows share
// one loop count per step (ELL segment), which would otherwise be the maximum
// of 32 Poisson counts; the build-time schedule finishes half k at step k and
// tops every lane up to that step's length with edges of half k+1, which
// evens the lanes out (simulated slot fill 56% -> ~80% on Reddit-like graphs).
//
// Entry encoding: u16 = slot * kSlotRec + (column - half*Wh), slot = half %
// kSlots, so the shared address is base + entry * 16 with the slots
// contiguous; padding is kWinPad (slot 0's last record: a zero record that no
// bulk copy ever overwrites).  BG_WIN_SLOTS=4 (4 x 56 KB: a refill may land
// while the slowest warp is two steps behind) measured slower on Reddit,
// 0.244 vs 0.228 ms: 68 smaller steps instead of 57 cost more in per-step
// work and padding than the extra slack saves.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "async.cuh"
#include "ops.cuh"
#include "tilewalk.cuh"

namespace bg {
namespace {

constexpr int kWinRec = 16;             // bytes per packed node row (4 u32 words)
#ifndef BG_WIN_SLOTS
#define BG_WIN_SLOTS 3
#endif
constexpr int kSlots = BG_WIN_SLOTS;    // ring slots; half h lives in slot h % kSlots
#ifndef BG_WIN_CHOICES
#define BG_WIN_CHOICES (BG_WIN_SLOTS >= 4 ? 3 : 2)
#endif
// halves a step may count: step k finishes half k and tops its lanes up with
// the first edges of halves k+1 .. k+kChoices-1 (in column order)
constexpr int kChoices = BG_WIN_CHOICES;
static_assert(kSlots > kChoices && kChoices >= 2, "the ring holds the step's halves plus one refill");
// records per ring slot: 4 x 56 KB (or 3 x 64 KB) of shared memory
constexpr int kSlotRec = kSlots == 4 ? 3584 : 4096;  // 64 KB slots by default
constexpr int kWinHalf = kSlotRec - 1;  // node rows per half-window (the last record stays zero)
constexpr uint16_t kWinPad = kWinHalf;  // slot 0's zero record
constexpr int kWinQ = 8;                // ELL groups in flight per lane (4 or 8)
constexpr int kWinPrefetch = 24;        // groups ahead the stream is bulk-prefetched into L2
constexpr int kWinMaxThreads = 576;     // 18 warps (5 per SMSP): <= 96 registers per thread
constexpr size_t kWinSmem = static_cast<size_t>(kSlots) * kSlotRec * kWinRec;  // 192 KB (224 KB with 4 slots)

__device__ __forceinline__ uint2 ld_nc_v2(const uint2* p) {
  uint2 v;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// ---- view construction (build once) -----------------------------------------

// Thread per node row: entries per half-window (u16, row-major rows x nh).
__global__ void k_win_count(const uint64_t* __restrict__ srp, const uint32_t* __restrict__ sl,
                            int64_t rows, int Wh, int nh, const int32_t* __restrict__ deg,
                            uint16_t* __restrict__ cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows || deg[i] >= kHubDeg) return;  // hub rows: no entries (hubs.cu)
  uint16_t* c = cnt + i * nh;
  int cur = -1;
  uint32_t run = 0;
  for_each_col(srp, sl, i, [&](uint32_t col) {
    const int h = static_cast<int>(col / static_cast<uint32_t>(Wh));
    if (h != cur) {
      if (cur >= 0) c[cur] = static_cast<uint16_t>(run);
      cur = h;
      run = 0;
    }
    ++run;
  });
  if (cur >= 0) c[cur] = static_cast<uint16_t>(run);
}

// Warp per (row block, warp of the block), lane per row: the two-choice
// schedule.  Step k must finish what is left of half k; its length K is the
// lanes' maximum of that, rounded up to a batch of 8 entries (two ELL
// groups), and every lane fills the rest of K with the first edges of half
// k+1.  Writes the per-step entry counts of each row (u16, rows x nh), the
// step lengths in groups (u16, warp-major: [b][v][k]) and each warp stream's
// total (for the scan of stream bases), padded to a multiple of 8 groups: the
// kernel consumes a stream 32 entries per lane at a time.
__global__ void k_win_sched(const uint16_t* __restrict__ cnt, int64_t rows, int RB, int RW, int nh, int64_t nbv,
                            uint16_t* __restrict__ nk, uint16_t* __restrict__ steplen,
                            uint32_t* __restrict__ total) {
  const int64_t wv = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (wv >= nbv) return;
  const int lane = threadIdx.x & 31, streams = RB / RW;  // RW rows per warp stream
  const int64_t b = wv / streams;
  const int v = static_cast<int>(wv % streams);
  const int64_t i = b * RB + v * RW + lane;
  const bool ok = lane < RW && i < rows;
  uint32_t left[kChoices];  // entries of halves k .. k+kChoices-1 not yet scheduled
#pragma unroll
  for (int c = 0; c < kChoices; ++c) left[c] = (ok && c < kChoices - 1 && c < nh) ? cnt[i * nh + c] : 0u;
  uint32_t sum = 0;
  for (int k = 0; k < nh; ++k) {
    uint32_t m = left[0];
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    const uint32_t K = (m + 7) & ~7u;
    left[kChoices - 1] = (ok && k + kChoices - 1 < nh) ? cnt[i * nh + k + kChoices - 1] : 0u;
    uint32_t room = K - left[0], n = left[0];
#pragma unroll
    for (int c = 1; c < kChoices; ++c) {  // in column order: half k+1 before k+2
      const uint32_t t = min(room, left[c]);
      left[c] -= t;
      room -= t;
      n += t;
    }
    if (ok) nk[i * nh + k] = static_cast<uint16_t>(n);
#pragma unroll
    for (int c = 0; c + 1 < kChoices; ++c) left[c] = left[c + 1];
    if (lane == 0) steplen[wv * nh + k] = static_cast<uint16_t>(K / 4);
    sum += K / 4;
  }
  if (lane == 0) total[wv] = (sum + 7) & ~7u;
}

__global__ void k_fill_u16(uint16_t* __restrict__ p, int64_t n, uint16_t v) {
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[t] = v;
}

// Thread per node row: its columns in order, nk[k] of them into step k's
// segment (the step's share of half k, then of half k+1).  A warp's segments
// are consecutive in its stream: stream base + the lengths of earlier steps.
__global__ void k_win_fill(const uint64_t* __restrict__ srp, const uint32_t* __restrict__ sl,
                           int64_t rows, int RW, int Wh, int nh, const uint16_t* __restrict__ nk,
                           const uint32_t* __restrict__ sbase, const uint16_t* __restrict__ steplen,
                           const int32_t* __restrict__ deg, uint16_t* __restrict__ ell) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows || deg[i] >= kHubDeg) return;
  const int64_t wv = i / RW;  // = b * (RB/RW) + v (RB is a multiple of RW)
  const int lane = static_cast<int>(i % RW);
  const uint16_t* n = nk + i * nh;
  const uint16_t* sll = steplen + wv * nh;
  int k = -1;
  uint32_t left = 0, pos = 0;
  uint64_t g = sbase[wv], base = 0;
  for_each_col(srp, sl, i, [&](uint32_t col) {
    while (left == 0) {
      if (k >= 0) g += sll[k];
      ++k;
      left = n[k];
      pos = 0;
      base = g * (4 * RW) + lane * 4;
    }
    const uint32_t h = col / static_cast<uint32_t>(Wh);
    ell[base + (pos >> 2) * (4 * RW) + (pos & 3)] =
        static_cast<uint16_t>((h % kSlots) * kSlotRec + (col - h * static_cast<uint32_t>(Wh)));
    ++pos;
    --left;
  });
}

// Bank-aware slot order (build once).  An LDS.128 is served per quarter warp
// (8 lanes, 128 bytes): lanes of a quarter whose records sit in the same
// 16-byte bank group (record index mod 8, the slots being 64 KB apart) and differ in
// address cost an extra wavefront each.  Counting is order-free, so each
// lane's entries within a segment may be permuted freely: position k is
// filled greedily with, per lane, an entry of a bank group no other lane of
// the quarter uses there (bounded look-ahead).  K entries per lane; q quarter.
__device__ void bank_order_segment(uint16_t* __restrict__ segp, uint32_t K, int q, int RW) {
  constexpr int kLook = 48;
  if (K == 0) return;
  auto bank = [](uint32_t e) { return e & 7u; };
  auto at = [&](int l, uint32_t k) -> uint16_t& { return segp[(k >> 2) * (4 * RW) + (8 * q + l) * 4 + (k & 3)]; };
  uint32_t cnt[8];
  for (int l = 0; l < 8; ++l) {
    uint32_t c = 0;
    while (c < K && at(l, c) != kWinPad) ++c;
    cnt[l] = c;
  }
  const uint32_t pad_bit = 1u << bank(kWinPad);
  for (uint32_t k = 0; k < K; ++k) {
    uint32_t used = 0;
    for (int l = 0; l < 8; ++l)
      if (cnt[l] <= k) used |= pad_bit;
    for (int l = 0; l < 8; ++l) {
      if (cnt[l] <= k) continue;
      const uint32_t end = min(cnt[l], k + kLook);
      uint32_t pick = k;
      for (uint32_t j = k; j < end; ++j)
        if (!((used >> bank(at(l, j))) & 1u)) {
          pick = j;
          break;
        }
      const uint16_t e = at(l, pick);
      if (pick != k) {
        at(l, pick) = at(l, k);
        at(l, k) = e;
      }
      used |= 1u << bank(e);
    }
  }
}

// Matching-based order for segments of at most kMatchK entries per lane.
// Per position, the lanes of the group are matched to distinct bank groups by
// augmenting paths (Kuhn), lanes with the most real entries left first and
// bank groups with the most entries left tried first (the max-degree rule of
// bipartite edge colouring, under which K positions suffice whenever no bank
// group holds more than K of the group's entries).  Padding entries all
// address the same zero record (bank group 7): any number of them at one
// position is one wavefront, but they block bank group 7 for real entries.
constexpr int kMatchK = 48;
__device__ void bank_match_segment(uint16_t* __restrict__ segp, uint32_t K, int q, int RW) {
  auto at = [&](int l, uint32_t k) -> uint16_t& { return segp[(k >> 2) * (4 * RW) + (8 * q + l) * 4 + (k & 3)]; };
  uint16_t ent[8][kMatchK];
  uint8_t cnt[8][8];
  int real[8], pads[8], bank_left[8];
  for (int b = 0; b < 8; ++b) bank_left[b] = 0;
  for (int l = 0; l < 8; ++l) {
    real[l] = pads[l] = 0;
    for (int b = 0; b < 8; ++b) cnt[l][b] = 0;
    for (uint32_t k = 0; k < K; ++k) {
      const uint16_t e = at(l, k);
      ent[l][k] = e;
      if (e == kWinPad) {
        ++pads[l];
      } else {
        ++real[l];
        ++cnt[l][e & 7];
        ++bank_left[e & 7];
      }
    }
  }
  for (uint32_t k = 0; k < K; ++k) {
    int order[8], n = 0;
    for (int l = 0; l < 8; ++l)
      if (real[l] > 0) order[n++] = l;
    for (int a = 1; a < n; ++a)  // most real entries left first
      for (int c = a; c > 0 && real[order[c]] > real[order[c - 1]]; --c) {
        const int t = order[c];
        order[c] = order[c - 1];
        order[c - 1] = t;
      }
    int border[8];
    for (int b = 0; b < 8; ++b) border[b] = b;
    for (int a = 1; a < 8; ++a)
      for (int c = a; c > 0 && bank_left[border[c]] > bank_left[border[c - 1]]; --c) {
        const int t = border[c];
        border[c] = border[c - 1];
        border[c - 1] = t;
      }
    bool pad_forced = false;  // a lane with only padding left places it here
    for (int l = 0; l < 8; ++l)
      if (real[l] == 0 && pads[l] > 0) pad_forced = true;
    int lane_bank[8], bank_lane[8];
    auto match = [&](bool allow7) {
      for (int b = 0; b < 8; ++b) bank_lane[b] = -1;
      for (int l = 0; l < 8; ++l) lane_bank[l] = -1;
      for (int a = 0; a < n; ++a) {
        // iterative augmenting-path search from lane order[a]
        int prev_bank[8], via_lane[8];
        bool seen[8] = {false, false, false, false, false, false, false, false};
        int queue[8], qh = 0, qt = 0, found = -1;
        queue[qt++] = order[a];
        int from_bank_of_lane[8];
        for (int l = 0; l < 8; ++l) from_bank_of_lane[l] = -1;
        while (qh < qt && found < 0) {
          const int l = queue[qh++];
          for (int bi = 0; bi < 8 && found < 0; ++bi) {
            const int b = border[bi];
            if (seen[b] || cnt[l][b] == 0 || (b == 7 && !allow7)) continue;
            seen[b] = true;
            via_lane[b] = l;
            prev_bank[b] = from_bank_of_lane[l];
            if (bank_lane[b] < 0) {
              found = b;
            } else {
              const int l2 = bank_lane[b];
              from_bank_of_lane[l2] = b;
              queue[qt++] = l2;
            }
          }
        }
        for (int b = found; b >= 0;) {  // flip the path
          const int l = via_lane[b], pb = prev_bank[b];
          bank_lane[b] = l;
          lane_bank[l] = b;
          b = pb;
        }
      }
    };
    match(!pad_forced);
    bool any_pad = pad_forced;
    for (int a = 0; a < n; ++a)
      if (lane_bank[order[a]] < 0 && pads[order[a]] > 0) any_pad = true;
    if (any_pad && !pad_forced && bank_lane[7] >= 0) {
      // padding will be placed: see whether giving up bank group 7 costs a lane
      int lb[8], bl[8];
      for (int i = 0; i < 8; ++i) lb[i] = lane_bank[i], bl[i] = bank_lane[i];
      int m1 = 0;
      for (int l = 0; l < 8; ++l) m1 += lane_bank[l] >= 0;
      match(false);
      int m2 = 0;
      for (int l = 0; l < 8; ++l) m2 += lane_bank[l] >= 0;
      // a real entry in bank group 7 next to padding costs one wavefront, as
      // does one lane fewer matched: keep bank 7 only if that saves more
      if (m2 + 1 < m1)
        for (int i = 0; i < 8; ++i) lane_bank[i] = lb[i], bank_lane[i] = bl[i];
    }
    // place: matched lanes an entry of their bank group, the rest padding if
    // they have any, else any real entry (a conflict)
    for (int l = 0; l < 8; ++l) {
      int want = lane_bank[l];
      bool pad = false;
      if (want < 0) {
        if (pads[l] > 0) pad = true;
        else
          for (int b = 0; b < 8 && want < 0; ++b)
            if (cnt[l][b]) want = b;
      }
      // find a remaining entry at positions >= k and swap it to k
      uint32_t pick = k;
      for (uint32_t j = k; j < K; ++j) {
        const uint16_t e = ent[l][j];
        if (pad ? e == kWinPad : (e != kWinPad && (e & 7) == static_cast<uint32_t>(want))) {
          pick = j;
          break;
        }
      }
      const uint16_t e = ent[l][pick];
      ent[l][pick] = ent[l][k];
      ent[l][k] = e;
      if (e == kWinPad) {
        --pads[l];
      } else {
        --real[l];
        --cnt[l][e & 7];
        --bank_left[e & 7];
      }
    }
  }
  for (int l = 0; l < 8; ++l)
    for (uint32_t k = 0; k < K; ++k) at(l, k) = ent[l][k];
}

// Thread per (warp stream, conflict group of 8 rows): every step segment of
// the stream in turn.  (An LDS.128 is served per 8 lanes; with two threads
// per row an LDS.64 is served per 16 lanes = 8 rows: a group is 8 rows either way.)
__global__ void k_win_bankorder(const uint32_t* __restrict__ sbase, const uint16_t* __restrict__ steplen,
                                int64_t nbv, int nh, int RW, uint16_t* __restrict__ ell) {
  const int cg = RW / 8;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nbv * cg) return;
  const int64_t wv = t / cg;
  uint64_t g = sbase[wv];
  for (int k = 0; k < nh; ++k) {
    const uint32_t len = steplen[wv * nh + k];
    if (len * 4 <= kMatchK) bank_match_segment(ell + g * (4 * RW), len * 4, static_cast<int>(t % cg), RW);
    else bank_order_segment(ell + g * (4 * RW), len * 4, static_cast<int>(t % cg), RW);
    g += len;
  }
}

// ---- the aggregation kernel ---------------------------------------------------

// Harley-Seal over 8 words into planes P[0..2]; returns the weight-8 carry.
template <int NP>
__device__ __forceinline__ uint32_t hs8_low(uint32_t (&P)[NP], const uint32_t (&x)[8]) {
  uint32_t t1, t2, f1, f2, e, s;
  s = P[0] ^ x[0] ^ x[1]; t1 = maj3(P[0], x[0], x[1]); P[0] = s;
  s = P[0] ^ x[2] ^ x[3]; t2 = maj3(P[0], x[2], x[3]); P[0] = s;
  s = P[1] ^ t1 ^ t2;     f1 = maj3(P[1], t1, t2);     P[1] = s;
  s = P[0] ^ x[4] ^ x[5]; t1 = maj3(P[0], x[4], x[5]); P[0] = s;
  s = P[0] ^ x[6] ^ x[7]; t2 = maj3(P[0], x[6], x[7]); P[0] = s;
  s = P[1] ^ t1 ^ t2;     f2 = maj3(P[1], t1, t2);     P[1] = s;
  s = P[2] ^ f1 ^ f2;     e = maj3(P[2], f1, f2);      P[2] = s;
  return e;
}

// Harley-Seal over 4 words into planes P[0..1]; returns the weight-4 carry.
template <int NP>
__device__ __forceinline__ uint32_t hs4_low(uint32_t (&P)[NP], const uint32_t (&x)[4]) {
  uint32_t t1, t2, f, s;
  s = P[0] ^ x[0] ^ x[1]; t1 = maj3(P[0], x[0], x[1]); P[0] = s;
  s = P[0] ^ x[2] ^ x[3]; t2 = maj3(P[0], x[2], x[3]); P[0] = s;
  s = P[1] ^ t1 ^ t2;     f = maj3(P[1], t1, t2);      P[1] = s;
  return f;
}

// Ripple a carry word of weight 2^q0 into planes q0.. (counts stay < 2^NP).
template <int NP>
__device__ __forceinline__ void ripple(uint32_t (&P)[NP], uint32_t c, int q0) {
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    if (q < q0) continue;
    const uint32_t nq = P[q] ^ c;
    c &= P[q];
    P[q] = nq;
  }
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// TPR threads per node row: each owns W = 4/TPR of the row's words (TPR = 2
// halves the per-thread state, so ~1.5x the warps fit at the same register
// file, and a warp stream covers 16 rows).
//
// A warp walks its stream of the current row block as one sequence of
// groups (4 entries per lane), 32 entries per lane per iteration: the step
// boundaries (release half S, wait for half S+2) are checked between 8-entry
// batches, so the ELL prefetch queue sits at fixed registers and the carry
// tree is static -- four weight-8 carries per iteration fold through planes 3
// and 4 and ripple from plane 5.  Streams are padded to whole iterations with
// zero-record entries, and the ELL array is padded past its end, so the
// prefetch needs no bounds checks.
template <int NP, bool OUTB, int TPR>
__global__ void __launch_bounds__(TPR == 1 ? (NP <= 10 ? kWinMaxThreads : 480) : 800, 1)
    k_win_bb(const uint32_t* __restrict__ sbase, const uint16_t* __restrict__ steplen,
             const uint16_t* __restrict__ ell, int nh, int Wh,
             int64_t xrows, int64_t row0, int64_t row1, int b0, int b1,
             const int32_t* __restrict__ degree, const uint4* __restrict__ x, int64_t f,
             uint32_t* __restrict__ out_bits, float* __restrict__ out_f, const FEpi ep) {
  static_assert(NP >= 6, "three-level Harley-Seal needs planes 0..5");
  constexpr int W = 4 / TPR, RW = 32 / TPR;  // words per thread, rows per warp stream
  extern __shared__ __align__(16) uint4 sbuf[];  // kSlots x kSlotRec records
  __shared__ __align__(8) uint64_t full[kSlots];
  __shared__ uint32_t done[kSlots];  // warps finished with each slot (monotone)
  const int tid = threadIdx.x, T = blockDim.x, nwarps = T >> 5, warp = tid >> 5, lane = tid & 31;
  if (tid < kSlots) {
    sbuf[tid * kSlotRec + kWinHalf] = make_uint4(0u, 0u, 0u, 0u);  // zero record (padding target)
    done[tid] = 0;
    mbar_init(&full[tid], 1);
  }
  if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int mine = b1 - b0 - static_cast<int>(blockIdx.x);
  const int nblk = mine > 0 ? (mine + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x) : 0;
  const int nsteps = nblk * nh;  // one half-window per step; nh % kSlots == 0
  auto issue = [&](int H) {      // half H of this CTA's sequence into slot H % kSlots
    const int64_t n0 = static_cast<int64_t>(H % nh) * Wh;
    const int64_t nodes = min(static_cast<int64_t>(Wh), xrows - n0);
    uint64_t* bar = &full[H % kSlots];
#if defined(BG_WIN_PROBE) && BG_WIN_PROBE >= 2
    if (false) {  // timing probe: no refills, results are wrong
#else
    if (nodes > 0) {
#endif
      const uint32_t bytes = static_cast<uint32_t>(nodes) * kWinRec;
      mbar_expect_tx(bar, bytes);
      bulk_g2s(sbuf + (H % kSlots) * kSlotRec, x + n0, bytes, bar);
    } else {
      mbar_arrive(bar);  // padding half: nothing to load
    }
  };
  if (tid == 0)
    for (int H = 0; H < kSlots && H < nsteps; ++H) issue(H);
  const int part = threadIdx.x % TPR;  // which W words of the row
  const uint2* ell2 = reinterpret_cast<const uint2*>(ell) + lane / TPR;  // this row's 4 entries per group
  const uint32_t sbw = smem_addr(sbuf) + part * (4 * W);  // + entry * 16 = this thread's words of a record
  uint32_t P[W][NP];
  // 8 entries: 8 shared loads (W words each), Harley-Seal into planes 0..2 of
  // each word -> weight-8 carries
  auto batch8 = [&](const uint2& a, const uint2& c, uint32_t (&e)[W]) {
    const uint32_t pk[4] = {a.x, a.y, c.x, c.y};
    uint32_t v[8][W];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      // entry -> byte address: extract + one shift-add (LOP3/SHF + LEA)
      const uint32_t ent = (m & 1) ? (pk[m >> 1] >> 16) : (pk[m >> 1] & 0xFFFFu);
      const uint32_t addr = sbw + (ent << 4);
      if (W == 4) {
        const uint4 t = lds128(addr);
        v[m][0] = t.x, v[m][1] = t.y, v[m][W > 2 ? 2 : 0] = t.z, v[m][W > 3 ? 3 : 0] = t.w;
      } else {
        const uint2 t = lds64(addr);
        v[m][0] = t.x, v[m][1] = t.y;
      }
    }
#pragma unroll
    for (int q = 0; q < W; ++q) {
      uint32_t xw[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) xw[m] = v[m][q];
      e[q] = hs8_low<NP>(P[q], xw);
    }
  };
  int S = 0, slot = 0;  // step (half-window) counter of this CTA, S % kSlots
  uint32_t use = 0;     // S / kSlots
  // release half S; the last warp out refills its slot with half S + 3
  auto finish = [&]() {
    __syncwarp();
    if (lane == 0) {
      const uint32_t prev = atomicAdd(&done[slot], 1u);
      if (prev + 1 == static_cast<uint32_t>(nwarps) * (use + 1) && S + kSlots < nsteps) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(S + kSlots);
      }
    }
    ++S;
    if (++slot == kSlots) slot = 0, ++use;
  };
  // step S may count entries of halves S .. S+kChoices-1: all but the last
  // were waited for at earlier steps (a slot cannot be refilled before every
  // warp has finished the step of its half)
  auto wait_half = [&](int H) {
#if defined(BG_WIN_PROBE) && BG_WIN_PROBE == 3
    return;  // timing probe: no ring waits, results are wrong
#endif
    if (H < nsteps) mbar_wait_sleep(&full[H % kSlots], static_cast<uint32_t>(H / kSlots) & 1u);
  };
  auto wait_next = [&]() { wait_half(S + kChoices - 1); };
  for (int H = 0; H + 1 < kChoices; ++H) wait_half(H);
  for (int bi = 0; bi < nblk; ++bi) {
#pragma unroll
    for (int q = 0; q < W; ++q)
#pragma unroll
      for (int p = 0; p < NP; ++p) P[q][p] = 0u;
    const int b = b0 + static_cast<int>(blockIdx.x) + bi * static_cast<int>(gridDim.x);
    const int64_t wv = static_cast<int64_t>(b) * nwarps + warp;
    const uint32_t gp = __ldg(sbase + wv), total = __ldg(sbase + wv + 1) - gp;  // groups, multiple of 8
    const uint2* es = ell2 + static_cast<size_t>(gp) * RW;
    if (lane == 0 && total > kWinQ)
      bulk_prefetch_l2(es + kWinQ * RW, min(static_cast<uint32_t>(kWinPrefetch - kWinQ), total - kWinQ) * RW *
                                            static_cast<uint32_t>(sizeof(uint2)));
    uint2 fq[kWinQ];  // groups g .. g+kWinQ-1 in flight
#pragma unroll
    for (int u = 0; u < kWinQ; ++u) fq[u] = ld_nc_v2(es + u * RW);
    int kk = 0;  // step of this block
    // step lengths, lane-parallel: lenA = steps 32c.., lenB = the next 32
    // (loaded a whole chunk ahead of use)
    const uint16_t* sl = steplen + wv * nh;
    uint32_t lenA = lane < nh ? __ldg(sl + lane) : 0u;
    uint32_t lenB = 32 + lane < nh ? __ldg(sl + 32 + lane) : 0u;
    uint32_t step_end = __shfl_sync(0xFFFFFFFFu, lenA, 0);  // group index where step kk ends
    wait_next();
    auto boundary = [&](uint32_t at) {  // finish every step that ends at group `at`
      while (at == step_end && kk < nh) {
        finish();
        if (++kk < nh) {
          if ((kk & 31) == 0) {
            lenA = lenB;
            const int k2 = kk + 32 + lane;
            lenB = k2 < nh ? __ldg(sl + k2) : 0u;
          }
          step_end += __shfl_sync(0xFFFFFFFFu, lenA, kk & 31);
          wait_next();
        }
      }
    };
    for (uint32_t g = 0; g < total; g += 8) {
      // the stream's groups g+24 .. g+31 into L2 (one bulk prefetch per 8
      // groups), so the register queue only has to cover L2 latency
      if (lane == 0 && g + kWinPrefetch < total)
        bulk_prefetch_l2(es + static_cast<size_t>(g + kWinPrefetch) * RW,
                         min(8u, total - g - kWinPrefetch) * RW * static_cast<uint32_t>(sizeof(uint2)));
      uint32_t e0[W], c1[W];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        boundary(g + 2 * u);
        const uint2 a = fq[(2 * u) % kWinQ], c = fq[(2 * u + 1) % kWinQ];
        fq[(2 * u) % kWinQ] = ld_nc_v2(es + static_cast<size_t>(g + 2 * u + kWinQ) * RW);
        fq[(2 * u + 1) % kWinQ] = ld_nc_v2(es + static_cast<size_t>(g + 2 * u + kWinQ + 1) * RW);
        uint32_t e[W];
#if defined(BG_WIN_PROBE) && BG_WIN_PROBE == 1
#pragma unroll
        for (int q = 0; q < W; ++q) e[q] = a.x ^ c.y ^ q;  // timing probe: no counting, results are wrong
#else
        batch8(a, c, e);
#endif
#pragma unroll
        for (int q = 0; q < W; ++q) {
          if (u == 0 || u == 2) {
            e0[q] = e[q];
          } else {  // two weight-8 carries: CSA into plane 3 -> weight-16 carry
            const uint32_t s3 = P[q][3] ^ e0[q] ^ e[q], cy = maj3(P[q][3], e0[q], e[q]);
            P[q][3] = s3;
            if (u == 1) {
              c1[q] = cy;
            } else {  // two weight-16 carries: CSA into plane 4, ripple from plane 5
              const uint32_t s4 = P[q][4] ^ c1[q] ^ cy, d = maj3(P[q][4], c1[q], cy);
              P[q][4] = s4;
              ripple<NP>(P[q], d, 5);
            }
          }
        }
      }
    }
    boundary(total);
    const int64_t i = static_cast<int64_t>(b) * (T / TPR) + tid / TPR;
    if (i >= row0 && i < row1) {
      const uint32_t deg = static_cast<uint32_t>(__ldg(degree + i));
      if (OUTB) {
#pragma unroll
        for (int q = 0; q < W; ++q) {
          const int wd = part * W + q;
          // cnt >= ceil(deg/2)  <=>  2*cnt - deg >= 0   (kernels.cpp:440-454)
          uint32_t ge = planes_ge<NP>(P[q], (deg + 1) >> 1);
          if (32 * (wd + 1) > f) ge &= (32 * wd >= f) ? 0u : tail_mask32(f);
          out_bits[i * 4 + wd] = ge;
        }
      } else {
#pragma unroll
        for (int q = 0; q < W; ++q)
          fepi_store_word(ep, out_f, i, f, part * W + q, [&](int bb) {
            return static_cast<float>(2 * static_cast<int64_t>(plane_count<NP>(P[q], bb)) - static_cast<int64_t>(deg));
          });
      }
    }
  }
}

bool window_forced() { return aggregation_mode() == BG_AGG_WINDOW; }

// Largest block (multiple of 32 threads) the kernel instance can run with the
// given dynamic shared memory, one CTA per SM.
template <class K>
int max_threads(K kern, size_t smem) {
  BG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int t = 1024;
  for (; t >= 32; t -= 32) {
    int nb = 0;
    BG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, t, smem));
    if (nb >= 1) break;
  }
  if (t < 32) fail("window_bb: kernel does not fit on an SM");
  return t;
}

// RB node rows per block, RW rows per warp stream (32 / threads per row).
void build_windows(bg_frdc& A, int RB, int RW, int Wh, cudaStream_t s) {
  auto& W = A.win;
  if (W.T == RB && W.Wn == Wh && W.rw == RW) return;
  frdc_slivers(A, s);
  const int64_t rows = A.rows;
  const int nh = static_cast<int>(cdiv(cdiv(A.cols, Wh), kSlots) * kSlots);
  const int nb = static_cast<int>(cdiv(rows, RB));
  const int64_t nbv = static_cast<int64_t>(nb) * (RB / RW);  // warp streams
  DevBuf cnt(static_cast<size_t>(std::max<int64_t>(rows * nh, 1)) * 2);
  DevBuf nk(static_cast<size_t>(std::max<int64_t>(rows * nh, 1)) * 2);
  DevBuf total(static_cast<size_t>(nbv + 1) * 4);
  W.seg.alloc(static_cast<size_t>(nbv + 1) * 4);
  W.steplen.alloc(static_cast<size_t>(std::max<int64_t>(nbv * nh, 1)) * 2);
  BG_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes, s));
  BG_CUDA(cudaMemsetAsync(total.p, 0, total.bytes, s));
  if (rows > 0)
    k_win_count<<<static_cast<unsigned>(cdiv(rows, 256)), 256, 0, s>>>(A.srp(), A.sl(), rows, Wh, nh,
                                                                       A.deg(), cnt.as<uint16_t>());
  BG_LAUNCH_CHECK();
  if (nbv > 0)
    k_win_sched<<<static_cast<unsigned>(cdiv(nbv * 32, 256)), 256, 0, s>>>(
        cnt.as<uint16_t>(), rows, RB, RW, nh, nbv, nk.as<uint16_t>(), W.steplen.as<uint16_t>(), total.as<uint32_t>());
  BG_LAUNCH_CHECK();
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, total.as<uint32_t>(), W.seg.as<uint32_t>(),
                                static_cast<int>(nbv + 1), s);
  DevBuf tmp(std::max<size_t>(tmp_bytes, 1));
  cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, total.as<uint32_t>(), W.seg.as<uint32_t>(),
                                static_cast<int>(nbv + 1), s);
  BG_LAUNCH_CHECK();
  uint32_t groups = 0;
  BG_CUDA(cudaMemcpyAsync(&groups, W.seg.as<uint32_t>() + nbv, 4, cudaMemcpyDeviceToHost, s));
  BG_CUDA(cudaStreamSynchronize(s));
  // + 8 groups past the end: the kernel's prefetch runs up to 8 groups ahead
  const int64_t n16 = (static_cast<int64_t>(groups) + 8) * 4 * RW;
  W.ell.alloc(static_cast<size_t>(n16) * 2);
  k_fill_u16<<<static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(cdiv(n16, 256), 65536))), 256, 0, s>>>(
      W.ell.as<uint16_t>(), n16, kWinPad);
  BG_LAUNCH_CHECK();
  if (rows > 0)
    k_win_fill<<<static_cast<unsigned>(cdiv(rows, 256)), 256, 0, s>>>(
        A.srp(), A.sl(), rows, RW, Wh, nh, nk.as<uint16_t>(), W.seg.as<uint32_t>(), W.steplen.as<uint16_t>(),
        A.deg(), W.ell.as<uint16_t>());
  BG_LAUNCH_CHECK();
  if (nbv > 0)
    k_win_bankorder<<<static_cast<unsigned>(cdiv(nbv * (RW / 8), 128)), 128, 0, s>>>(
        W.seg.as<uint32_t>(), W.steplen.as<uint16_t>(), nbv, nh, RW, W.ell.as<uint16_t>());
  BG_LAUNCH_CHECK();
  BG_CUDA(cudaStreamSynchronize(s));
  W.T = RB;
  ++A.gen;
  W.rw = RW;
  W.Wn = Wh;
  W.nw = nh;
  W.nb = nb;
}

// Threads per row: 1 (default; measured faster on Reddit: 0.235 vs 0.286 ms --
// TPR 2 needs 4 waves of streaming instead of 3 and twice the shared loads,
// which outweighs its ~1.5x resident warps).  BG_WINDOW_TPR=2 selects the other.
int win_tpr() {
  const char* e = std::getenv("BG_WINDOW_TPR");
  return e && std::atoi(e) == 2 ? 2 : 1;
}

template <int NP, bool OUTB, int TPR>
bool launch_win(bg_frdc& A, const uint32_t* x, int64_t f, uint32_t* ob, float* of, int64_t r0,
                int64_t r1, cudaStream_t s) {
  constexpr int RW = 32 / TPR;
  auto kern = k_win_bb<NP, OUTB, TPR>;
  const int sms = sm_count();
  const int Wh = std::max(1, std::min<int>(window_nodes_setting() > 0 ? std::min(window_nodes_setting(), kWinHalf)
                                                                       : kWinHalf,
                                           static_cast<int>(A.cols)));
  static const int tmax = max_threads(kern, kWinSmem);  // per instance
  const int64_t rmax = tmax / TPR;                      // rows per block at most
  // blocks sized for the rows this call produces (a rank's shard under
  // multi-GPU), so every SM gets a block
  const int64_t nrows = r1 - r0;
  const int64_t waves = std::max<int64_t>(1, cdiv(nrows, static_cast<int64_t>(sms) * rmax));
  const int RB = static_cast<int>(std::max<int64_t>(RW, std::min<int64_t>(
      rmax / RW * RW, cdiv(cdiv(nrows, static_cast<int64_t>(sms) * waves), RW) * RW)));
  if (!window_forced()) {
    // cost model: bytes streamed into shared memory per adjacency bit of the
    // rows produced (every block streams the whole operand) vs the ~32-byte L2
    // sector an edge gather costs; range bits estimated from the mean degree
    const double bits = static_cast<double>(A.nnz_bits) * static_cast<double>(nrows) / static_cast<double>(A.rows);
    const double streamed = static_cast<double>(waves) * std::min<int64_t>(sms, cdiv(nrows, RB)) *
                            static_cast<double>(A.cols) * kWinRec;
    // 48 bytes per bit: at 8 Reddit shards (38.5 bytes streamed per bit) the
    // windowed kernel still beats the sliver gather by 17% (scripts/shard_probe.py)
    if (bits < static_cast<double>(int64_t{1} << 22) || streamed > 48.0 * bits) return false;
  }
  build_windows(A, RB, RW, Wh, s);
  const auto& W = A.win;
  const int b0 = static_cast<int>(r0 / RB), b1 = static_cast<int>(cdiv(r1, RB));
  const int grid = std::min(sms, b1 - b0);
  kern<<<grid, RB * TPR, kWinSmem, s>>>(W.seg.as<uint32_t>(), W.steplen.as<uint16_t>(), W.ell.as<uint16_t>(), W.nw,
                                        W.Wn, A.cols, r0, r1, b0, b1, A.deg(), reinterpret_cast<const uint4*>(x), f,
                                        ob, of, current_fepi());
  BG_LAUNCH_CHECK();
  return true;
}

template <bool OUTB>
bool launch_win_np(bg_frdc& A, const uint32_t* x, int64_t f, uint32_t* ob, float* of, int64_t r0,
                   int64_t r1, cudaStream_t s) {
  const int64_t d = light_max_deg(A, s);  // hub rows: hubs.cu
  auto go = [&](auto tpr) {
    constexpr int TPR = decltype(tpr)::value;
    if (d < (1 << 6)) return launch_win<6, OUTB, TPR>(A, x, f, ob, of, r0, r1, s);
    if (d < (1 << 8)) return launch_win<8, OUTB, TPR>(A, x, f, ob, of, r0, r1, s);
    if (d < (1 << 10)) return launch_win<10, OUTB, TPR>(A, x, f, ob, of, r0, r1, s);
    if (d < (1 << 12)) return launch_win<12, OUTB, TPR>(A, x, f, ob, of, r0, r1, s);
    return false;
  };
  return win_tpr() == 1 ? go(std::integral_constant<int, 1>{}) : go(std::integral_constant<int, 2>{});
}

}  // namespace

bool window_bb(bg_frdc& A, const uint32_t* x, int64_t f, int wb, uint32_t* out_bits, float* out_f,
               cudaStream_t s, int64_t r0, int64_t r1) {
  // A may be a rank's row slice (rows < cols): blocks index its rows, the
  // streamed operand has A.cols rows
  if (spw(f, wb) != 4 || A.rows == 0 || A.cols == 0 || r1 <= r0) return false;
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0) return false;
  const int mode = aggregation_mode();
  if (mode == BG_AGG_SLIVERS || mode == BG_AGG_TILES) return false;
  if (out_bits) return launch_win_np<true>(A, x, f, out_bits, nullptr, r0, r1, s);
  return launch_win_np<false>(A, x, f, nullptr, out_f, r0, r1, s);
}

}  // namespace bg
