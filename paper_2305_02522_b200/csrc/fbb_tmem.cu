// MM.FBB / FFB for a wide fp32 input (Reddit: K = 602) on the 5th-generation
// tensor cores with the A operand in TENSOR MEMORY (ref: bmm B-output path,
// kernels.cpp:140-176; binarize x >= 0, bitdense.cpp:83).
//
// fbb_tc.cu keeps A (the +-1 bytes of a 128-row tile) in shared memory next
// to the weights; at K = 602 the two take 156 KB and leave room for only
// ~58 KB of fp32 row pieces in flight, below the per-SM bandwidth-latency
// product of HBM (~44 KB/us x ~2 us), so that kernel runs at 0.26-0.29 ms
// where the stream needs 86 us.  Here A never touches shared memory: the
// converters write each row's +-1 bytes straight into TMEM with tcgen05.st
// (four K values per 32-bit column; TMEM lane = row of the tile) and
// tcgen05.mma reads A from TMEM.  Shared memory holds the weights (Reddit 78
// KB, Flickr's 256 columns 128 KB) and a ring of fp32 row pieces.
//
// One CTA per SM walks 128-row tiles.  Roles:
//   * producer (warp 0, one lane): pieces of PR = 16 consecutive rows
//     (contiguous in HBM) into a ring of 3 slots by cp.async.bulk (full /
//     empty mbarrier per slot);
//   * MMA issuer (warp 1, one lane): ceil(K/32) tcgen05.mma.kind::i8 per tile
//     (M = 128, N = the product's columns rounded to 32, A from TMEM buffer
//     tile % 2, B = the weights in shared memory) into the TMEM accumulator,
//     then tcgen05.commit to the accumulator-full and A-empty barriers;
//   * epilogue (warps 4..7, TMEM lane quarter warp % 4): tcgen05.ld of the
//     accumulator, dot >= 0 -> bit, MSB-first words, one row per thread;
//   * converters (warps 8..23): warp (quarter q, part j) converts K steps
//     [j*S/4, (j+1)*S/4) of the two pieces of lane quarter q with 16-lane
//     stores (tcgen05.st.16x256b), so a piece is released as soon as it is
//     converted -- a 32-lane store would hold a piece until its sibling
//     landed too (measured: one piece in flight, 0.213 ms on Reddit).
// Integer dots are exact: the bits equal the reference's for any order.
//
// The default form is the 2-CTA one (PAIR below: tcgen05.mma.cta_group::2,
// each CTA holding half of the weight columns, four ring slots); a paired
// product (a SAGE / GraphConv layer's W1 and W2 on one input) runs two MMA
// rounds per tile into the same accumulator, the input read once.
// Measured (1 B200, in-graph CUDA events): Reddit 0.136 (mma.sync) -> 0.122
// ms (ncu 0.115 ms, 4.9 TB/s); Flickr's 256-column pair 2 x 0.139 (warp per
// row) -> one pass, forward 0.526 -> 0.142 ms over the round.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "async.cuh"
#include "ops.cuh"

namespace bg {
namespace {

constexpr int kTmM = 128;
constexpr int kTmPR = 16;                              // rows per fp32 piece
constexpr int kTmParts = 4;                            // converter warps per TMEM lane quarter
constexpr int kTmConv = 4 * kTmParts;                  // 16 converter warps
constexpr int kTmThreads = (8 + kTmConv) * 32;         // 24 warps
constexpr int kTmPieces = kTmM / kTmPR;                // pieces per tile
constexpr int kTmMaxSlots = 4;

__device__ __forceinline__ uint32_t tm_sign4(float x0, float x1, float x2, float x3) {
  return pm1_bytes4(x0, x1, x2, x3);
}

__device__ __forceinline__ void tm_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// a wait that traps instead of hanging if a phase never completes
__device__ __forceinline__ void tm_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  for (uint32_t it = 0; it < (1u << 26) && !ok; ++it)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  if (!ok) __trap();
}

// the same wait with cluster-scope acquire (barriers the peer CTA arrives on)
__device__ __forceinline__ void tm_wait_cl(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  for (uint32_t it = 0; it < (1u << 26) && !ok; ++it)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  if (!ok) __trap();
}

// arrive on the barrier at the same shared-memory offset in CTA `cta` of the cluster
__device__ __forceinline__ void tm_arrive_cta(uint64_t* bar, uint32_t cta) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_addr(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint64_t tm_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // sm_100 descriptor version; no swizzle, base offset 0
  return d;
}

struct TmArgs {
  const float* x;
  const uint32_t* wt;  // n x kspw transposed weight bits
  int64_t rows;
  int k, kspw, kpad, n, N, ospw;
  uint32_t a_cols;     // TMEM columns per A buffer (multiple of 32)
  uint32_t a_col0;     // first A buffer's column (after the N accumulator columns)
  int64_t span;        // rows per CTA (multiple of 16): CTA b owns [b*span, min(rows, (b+1)*span))
  int slots;           // fp32 ring slots (<= kTmMaxSlots)
  int stage_slots;     // trailing slots that hold the packed weights until they are expanded
  int wcols;           // rows of wt (a pair: W1 | zero pad | W2)
  int half;            // a pair: the second product's first weight row (0: single product)
  int rounds;          // MMA rounds per tile: 1, or 2 for a pair (W1 then W2 into the same accumulator)
  uint32_t* out2;      // a pair: the second product's bits
  uint32_t* out;
};

// PAIR: a 2-CTA cluster runs tcgen05.mma.cta_group::2 (M = 256, one 128-row
// tile per CTA): each CTA holds half of the weight columns, so the freed 39 KB
// (Reddit) buy a fourth ring slot; the leader CTA issues the MMAs, the peer's
// converters and epilogue warps arrive on the leader's barriers remotely, and
// the leader's commits are multicast to both CTAs.
template <bool PAIR>
__global__ void __launch_bounds__(kTmThreads, 1) k_fbb_tmem(const TmArgs a) {
  const int kTmSlots = a.slots;
  constexpr int kTile = PAIR ? 2 * kTmM : kTmM;  // rows per (pair) tile
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[kTmMaxSlots], empty[kTmMaxSlots], a_full[2], a_empty[2], acc_full, acc_empty;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const bool leader = rank == 0;
  const int kpad = a.kpad, N = a.N, NB = PAIR ? a.N / 2 : a.N;  // N per MMA round; NB: columns held here per round
  const uint32_t bchunk = static_cast<uint32_t>(NB) * 16u;
  uint8_t* B = sm;  // kpad/16 chunks x NB rows x 16 B (canonical K-major, no swizzle)
  const uint32_t slot_floats = static_cast<uint32_t>(kTmPR * a.k) + 32;  // + pad: the last row's last step reads past
  float* ring = reinterpret_cast<float*>(B + static_cast<size_t>(a.rounds) * kpad * NB);
  // this CTA's rows: one contiguous, 16-aligned range per CTA (per pair: the
  // pair's tiles of 256 rows, the leader taking the first 128 of each); all
  // ranges finish together, the last tile of a range is partial
  const int64_t unit = PAIR ? blockIdx.x >> 1 : blockIdx.x;
  const int64_t rb0 = unit * a.span, rb1 = std::min(a.rows, rb0 + a.span);
  const int64_t my = rb1 > rb0 ? (rb1 - rb0 + kTile - 1) / kTile : 0;
  const int64_t npieces = my * kTmPieces;
  auto tile_row0 = [&](int64_t j) { return rb0 + j * kTile + static_cast<int64_t>(kTmM) * rank; };
  // piece u of this CTA: rows [r0, r0 + nr); bulk-copied when its byte
  // count is a multiple of 16 (every full piece), else read from HBM
  auto piece = [&](int64_t u, int64_t* r0) {
    *r0 = tile_row0(u / kTmPieces) + kTmPR * (u % kTmPieces);
    const int64_t left = rb1 - *r0;
    return static_cast<int>(left <= 0 ? 0 : left < kTmPR ? left : kTmPR);
  };
  auto staged_piece = [&](int nr) { return nr > 0 && (static_cast<uint32_t>(nr) * a.k * 4u) % 16 == 0; };
  auto issue = [&](int64_t u, int s) {  // piece u into slot s (= u % slots)
    int64_t r0;
    const int nr = piece(u, &r0);
    if (staged_piece(nr)) {
      const uint32_t bytes = static_cast<uint32_t>(nr) * static_cast<uint32_t>(a.k) * 4u;
      mbar_expect_tx(&full[s], bytes);
      bulk_g2s(ring + s * slot_floats, a.x + r0 * a.k, bytes, &full[s]);
    } else {
      tm_arrive(&full[s]);  // empty or unaligned piece: the converters read HBM
    }
  };
  if (tid == 0) {
    for (int s = 0; s < kTmSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmConv);  // every converter warp releases every piece
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&a_full[b], PAIR ? 2 * kTmConv : kTmConv);  // (leader) both CTAs' converters
      mbar_init(&a_empty[b], 1);
    }
    mbar_init(&acc_full, 1);
    mbar_init(&acc_empty, PAIR ? 8 : 4);  // (leader) both CTAs' epilogue warps
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the first two pieces go out before the weights are set up
    for (int64_t u = 0; u < std::min<int64_t>(kTmSlots - a.stage_slots, npieces); ++u) issue(u, static_cast<int>(u));
  }
  // weights as +-1 bytes (0 past K and for columns >= n): the packed words
  // are staged in the last (still idle) ring slot by asynchronous copies
  // first, so the expansion below does not wait one L2 round trip per
  // iteration
  const uint32_t* wst = reinterpret_cast<const uint32_t*>(ring + (kTmSlots - a.stage_slots) * slot_floats);
  for (int t = tid; t < a.wcols * a.kspw; t += blockDim.x) cp_async4(const_cast<uint32_t*>(wst) + t, a.wt + t);
  cp_async_wait_all();
  __syncthreads();
  for (int t = tid; t < a.rounds * NB * (kpad / 4); t += blockDim.x) {
    const int ro = t / (NB * (kpad / 4)), tr = t - ro * NB * (kpad / 4);  // round, item in it
    const int o = tr / (kpad / 4), p4 = (tr % (kpad / 4)) * 4;
    const int pc = o + static_cast<int>(rank) * NB;  // the column in its product
    const int oc = ro ? a.half + pc : pc;           // the weight row (a pair: W1 | pad | W2)
    uint32_t v = 0;
    if (pc < a.n && p4 < a.k) {
      const uint32_t word = wst[oc * a.kspw + (p4 >> 5)];
      const uint32_t nib = (word >> (28 - (p4 & 31))) & 0xFu;
      const uint32_t spread = ((nib >> 3) & 1u) | (((nib >> 2) & 1u) << 8) | (((nib >> 1) & 1u) << 16) | ((nib & 1u) << 24);
      v = 0xFFFFFFFFu - 0xFEu * spread;
      if (p4 + 4 > a.k) v &= 0xFFFFFFFFu >> (8 * (p4 + 4 - a.k));
    }
    *reinterpret_cast<uint32_t*>(B + static_cast<size_t>(ro) * kpad * NB + (p4 >> 4) * bchunk + o * 16 + (p4 & 15)) = v;
  }
  if (warp == 1) {  // TMEM: two A buffers + one accumulator
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_base)),
                   "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_base)),
                   "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }

  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // weights -> tensor core
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR) cluster_sync_all();  // the peer's weights, barriers and TMEM are ready
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t acc_col = 0, a_col0 = a.a_col0;  // accumulator at column 0, A buffers after it

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      // slot s and use count k of piece u (u = k * slots + s) kept incrementally
      int s = kTmSlots - a.stage_slots;
      uint32_t k = 0;
      for (int64_t u = s; u < npieces; ++u) {  // the first slots - stage_slots pieces went out in the prologue
        if (k > 0) tm_wait(&empty[s], (k - 1) & 1u);
        // the generic reads of the slot (converters; for the last slot's first
        // piece, the weight expansion) before the bulk copy's async-proxy writes
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(u, s);
        if (++s == kTmSlots) s = 0, ++k;
      }
    }
  } else if (warp == 1 && leader) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
                           (static_cast<uint32_t>(kTile >> 4) << 24);  // kind::i8, s32 += s8 x s8, K-major
    for (int64_t j = 0; j < my; ++j) {
      const int b = static_cast<int>(j & 1);
      tm_wait_cl(&a_full[b], static_cast<uint32_t>((j >> 1) & 1));
      for (int ro = 0; ro < a.rounds; ++ro) {
        const int64_t R = j * a.rounds + ro;  // accumulator use
        if (R >= 1) tm_wait_cl(&acc_empty, static_cast<uint32_t>((R - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const uint32_t bbase = smem_addr(B) + static_cast<uint32_t>(ro * kpad * NB);
          const uint32_t acol = tmem + a_col0 + static_cast<uint32_t>(b) * a.a_cols, dcol = tmem + acc_col;
          for (int ks = 0; ks < kpad / 32; ++ks) {
            const uint64_t bd = tm_desc(bbase + 2 * ks * bchunk, bchunk, 128);
            const uint32_t accum = ks > 0 ? 1u : 0u;
            if (PAIR)
              asm volatile(
                  "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                  " tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dcol),
                  "r"(acol + 8u * ks), "l"(bd), "r"(idesc), "r"(accum)
                  : "memory");
            else
              asm volatile(
                  "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                  " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dcol),
                  "r"(acol + 8u * ks), "l"(bd), "r"(idesc), "r"(accum)
                  : "memory");
          }
          const bool last = ro + 1 == a.rounds;
          if (PAIR) {  // both CTAs' barriers
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    smem_addr(&acc_full)),
                "h"(static_cast<uint16_t>(3))
                : "memory");
            if (last)
              asm volatile(
                  "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                      smem_addr(&a_empty[b])),
                  "h"(static_cast<uint16_t>(3))
                  : "memory");
          } else {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_addr(&acc_full))
                         : "memory");
            if (last)
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                               smem_addr(&a_empty[b]))
                           : "memory");
          }
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- epilogue: TMEM lanes 32*(warp-4) .. +31 ----------------
    const int q = warp - 4;
    for (int64_t j = 0; j < my; ++j) {
     for (int ro = 0; ro < a.rounds; ++ro) {  // round ro's product: out, or the pair's out2
      const int64_t R = j * a.rounds + ro;
      tm_wait(&acc_full, static_cast<uint32_t>(R & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t row = tile_row0(j) + 32 * q + lane;
      uint32_t* o = (ro ? a.out2 : a.out) + row * a.ospw;
      const bool live = row < rb1;
      for (int cw = 0; cw < N / 32; ++cw) {
        uint32_t d[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
              "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]),
              "=r"(d[15]), "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]),
              "=r"(d[22]), "=r"(d[23]), "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]),
              "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
            : "r"(tmem + (static_cast<uint32_t>(32 * q) << 16) + acc_col + static_cast<uint32_t>(32 * cw)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // the sign bits shift in one funnel shift each (MSB-first); bit = dot >= 0
        uint32_t m = 0;
#pragma unroll
        for (int t = 0; t < 32; ++t) m = __funnelshift_l(d[t], m, 1);
        m = ~m;
        if (32 * cw + 32 > a.n) m &= 32 * cw >= a.n ? 0u : tail_mask32(a.n);  // columns >= n stay 0
        if (live && cw < a.ospw) o[cw] = m;
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (PAIR) tm_arrive_cta(&acc_empty, 0);  // the leader's
        else tm_arrive(&acc_empty);
      }
      if (live)
        for (int w = N / 32; w < a.ospw; ++w) o[w] = 0u;  // 64-bit word padding
     }
    }
  } else if (warp >= 8) {
    // ---------------- converters ----------------
    // Warp (quarter q, part j) converts K steps [j*S/4, (j+1)*S/4) of the two
    // 16-row pieces of lane quarter q (TMEM lanes 32q .. 32q+15 and +16 ..
    // +31) with 16-lane stores (tcgen05.st.16x256b: thread t holds lanes t/4
    // and t/4 + 8, columns 2(t%4) and 2(t%4)+1 of an 8-column K step, i.e.
    // floats 8(t%4) .. 8(t%4)+7 of two rows), so each piece is released as
    // soon as it is converted.  Every converter warp waits for EVERY piece of
    // the tile in order and releases the ones it does not read at once: a
    // warp that skipped a slot's earlier phases could take that phase's
    // parity for the one it wants (an mbarrier parity wait only tells the
    // current phase from the previous one), and the producer refills a slot
    // only when all 16 warps have released it.
    const int q = warp & 3, part = (warp - 8) >> 2;  // TMEM lane quarter, K part
    const int steps = kpad / 32;
    const int s0 = steps * part / kTmParts, s1 = steps * (part + 1) / kTmParts;
    const int pq = 32 / kTmPR;  // pieces per lane quarter
    const int tr = lane >> 2, tc = lane & 3;  // rows tr and tr+8 of a piece, floats 8tc .. 8tc+7 of a step
    int cs = 0;        // slot of the next piece (pieces are consumed in order)
    uint32_t ck = 0;   // its use count
    for (int64_t j = 0; j < my; ++j) {
      const int b = static_cast<int>(j & 1);
      if (j >= 2) tm_wait(&a_empty[b], static_cast<uint32_t>(((j >> 1) - 1) & 1));
      for (int p = 0; p < kTmPieces; ++p) {
        const int64_t v = j * kTmPieces + p;
        const int s = cs;
        tm_wait(&full[s], ck & 1u);
        if (++cs == kTmSlots) cs = 0, ++ck;
        if (p / pq == q) {
          const int h = p % pq;  // which 16 lanes of the quarter
          int64_t pr0;
          const bool staged = staged_piece(piece(v, &pr0));  // rows past the range read stale floats: never stored
          const float* slot = ring + s * slot_floats;
          const uint32_t tcol = tmem + (static_cast<uint32_t>(32 * q + 16 * h) << 16) + a_col0 +
                                static_cast<uint32_t>(b) * a.a_cols;
          for (int ks = s0; ks < s1; ++ks) {
            const int k0 = 32 * ks + 8 * tc;
            uint32_t c[4];
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
              const int ri = tr + 8 * rr;  // row in the piece
              if (staged && (a.k & 1) == 0) {
                // rows are 8-byte aligned in the slot; floats past K (the last
                // step) read the next row or the slot pad and meet zero weights
                const uint32_t p2 = smem_addr(slot) + 4u * static_cast<uint32_t>(ri * a.k + k0);
                const float2 x0 = lds_f2(p2), x1 = lds_f2(p2 + 8), x2 = lds_f2(p2 + 16), x3 = lds_f2(p2 + 24);
                c[2 * rr] = tm_sign4(x0.x, x0.y, x1.x, x1.y);
                c[2 * rr + 1] = tm_sign4(x2.x, x2.y, x3.x, x3.y);
              } else {
                const int64_t r = pr0 + ri;
                const float* src = staged ? slot + static_cast<int64_t>(ri) * a.k : a.x + r * a.k;
                float e[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                  const int kk = k0 + t;
                  e[t] = r < rb1 && kk < a.k ? (staged ? src[kk] : __ldg(src + kk)) : 0.0f;  // slot or HBM
                }
                c[2 * rr] = tm_sign4(e[0], e[1], e[2], e[3]);
                c[2 * rr + 1] = tm_sign4(e[4], e[5], e[6], e[7]);
              }
            }
            asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1,%2,%3,%4};" ::"r"(
                             tcol + 8u * static_cast<uint32_t>(ks)),
                         "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3])
                         : "memory");
          }
        }
        __syncwarp();
        if (lane == 0) tm_arrive(&empty[s]);  // the slot's floats are in registers / TMEM now
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (PAIR) tm_arrive_cta(&a_full[b], 0);  // the leader's
        else tm_arrive(&a_full[b]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR) cluster_sync_all();  // the leader's MMAs have read this CTA's TMEM for the last time
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1) {
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

}  // namespace

// FBB on k_fbb_tmem: false (nothing launched) when not eligible.  Products
// (or pairs, BmmArgs::out_bits2) with <= 256 output columns each whose A tile
// fits two TMEM buffers next to the accumulator (N <= 128: K <= 768; N = 256:
// K <= 512) and whose weights and ring fit in shared memory.  pair: the 2-CTA
// cta_group::2 form (N >= 64).
bool fbb_tmem(const BmmArgs& a, cudaStream_t s, bool pair) {
  if (!a.a_f || !a.out_bits || a.n == 0 || a.n > 256 || a.k <= 0 || a.rows == 0) return false;
  const bool paired = a.out_bits2 != nullptr;
  if (paired && a.n2 != a.n) return false;
  if (reinterpret_cast<uintptr_t>(a.a_f) % 16 != 0) return false;
  TmArgs t{};
  t.x = a.a_f;
  t.wt = a.wt;
  t.rows = a.rows;
  t.k = static_cast<int>(a.k);
  t.kspw = static_cast<int>(spw(a.k, a.wb));
  t.kpad = static_cast<int>(32 * cdiv(a.k, 32));
  t.n = static_cast<int>(a.n);
  // a pair runs two MMA rounds per tile (W1, then W2) into one accumulator
  t.half = paired ? static_cast<int>(32 * cdiv(a.n, 32)) : 0;
  t.rounds = paired ? 2 : 1;
  t.N = static_cast<int>(32 * cdiv(a.n, 32));
  t.wcols = paired ? t.half + t.n : t.n;
  t.ospw = static_cast<int>(spw(a.n, a.wb));
  t.out = a.out_bits;
  t.out2 = a.out_bits2;
  t.a_cols = static_cast<uint32_t>(32 * cdiv(t.kpad / 4, 32));
  t.a_col0 = static_cast<uint32_t>(std::max(128, t.N));
  if (t.a_col0 + 2 * t.a_cols > 512) return false;
  if (pair && t.N < 64) return false;
  // as many 16-row fp32 slots as the shared memory left by the weights
  // holds, at least three and at most four (Reddit: 3, or 4 as a pair;
  // Flickr as a pair: 4 slots of 32 KB 94.6 us, 5 slots 98.5 us;
  // BG_TMEM_SLOTS caps lower)
  const int nb = pair ? t.N / 2 : t.N;
  const size_t cap = 227 * 1024 - 1024;  // static shared memory (barriers, TMEM base) counts too
  const size_t wbytes = static_cast<size_t>(t.rounds) * t.kpad * nb, sbytes = (static_cast<size_t>(kTmPR) * a.k + 32) * 4;
  if (wbytes + 3 * sbytes > cap) return false;
  t.slots = static_cast<int>(std::min<size_t>(4, (cap - wbytes) / sbytes));
  if (const char* e = std::getenv("BG_TMEM_SLOTS")) t.slots = std::max(3, std::min(t.slots, std::atoi(e)));
  // the packed weights are staged in the last slot(s) before the ring starts
  t.stage_slots = static_cast<int>(cdiv(static_cast<int64_t>(t.wcols) * t.kspw * 4, static_cast<int64_t>(sbytes)));
  if (t.stage_slots >= t.slots) return false;
  const size_t smem = wbytes + static_cast<size_t>(t.slots) * sbytes;
  static int attr_done[2] = {0, 0};
  auto kern = pair ? k_fbb_tmem<true> : k_fbb_tmem<false>;
  if (!attr_done[pair]) {
    BG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cap)));
    attr_done[pair] = 1;
  }
  if (!pair) {
    // one contiguous 16-aligned row range per CTA, as even as 16 rows allow
    t.span = 16 * cdiv(cdiv(a.rows, sm_count()), 16);
    const int64_t blocks = cdiv(a.rows, t.span);
    kern<<<static_cast<unsigned>(blocks), kTmThreads, smem, s>>>(t);
  } else {
    // one contiguous range of 256-row tiles per CTA pair (2-CTA clusters);
    // 32-row ranges that use every pair of the chip but end in a partial
    // tile measured 4 % slower (Reddit 162 vs 156 us, Flickr 97 vs 93 us)
    const int64_t pairs = std::max<int64_t>(1, std::min<int64_t>(sm_count() / 2, cdiv(a.rows, 256)));
    t.span = 256 * cdiv(cdiv(a.rows, pairs), 256);
    const int64_t used = cdiv(a.rows, t.span);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * used));
    cfg.blockDim = dim3(kTmThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    BG_CUDA(cudaLaunchKernelEx(&cfg, kern, t));
  }
  BG_LAUNCH_CHECK();
  return true;
}

}  // namespace bg
