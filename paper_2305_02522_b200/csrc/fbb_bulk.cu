// MM.FBB / MM.FBF for graphs with few node rows (Cora 2.7 K, PubMed 20 K):
// every row of X is requested from HBM at kernel start (ref: bmm F-input
// path kernels.cpp:140-191, binarize x >= 0 bitdense.cpp:83).
//
// Each warp owns a ring of D row slots in shared memory; lane 0 fills a slot
// with ONE cp.async.bulk of the whole row (the 16-byte-aligned byte range
// that covers it) completing on the slot's mbarrier, and keeps D rows of its
// stripe in flight, so a CTA of 16 warps has 32-64 rows requested before the
// first one is consumed (Cora: the whole matrix across the 148 SMs).
//
// Opt-in (BG_FBB=bulk), measured (ncu launch durations, 1 B200): Cora 10 us
// vs 9.5 us for the warp-per-row kernel (bmm.cu k_bmm), PubMed 8.1 vs 7.5 us;
// the data movement alone (BG_BULK_PROBE=1) takes 6.2 / 5.7 us, and the
// per-row ballot + XOR-POPC chain after the last rows land is not hidden at
// 16 warps per SM.  Kept as a tested alternative (tests/test_gpu_umma.py).
//
// Consuming a row: word m of the packed row is one conflict-free LDS per
// lane (floats 32m .. 32m+31) and a ballot (bit = x >= 0, LSB-first: the
// weight words are staged bit-reversed against the MSB-first layout of
// bitdense.hpp:61-107); the ballot result is warp-uniform, so
// every lane immediately XOR-POPCs it against its output columns' weight
// words (transposed weight bits in shared memory, odd row stride so the 32
// lanes hit 32 banks).  The packed row never exists in memory.
//   B output: bit = K - 2*popc >= 0 (kernels.cpp:159-176), words by ballot;
//   F output: float((alpha*dot)*beta) in double in that order (:179-190).
// Integer dots are exact, so the results are the reference's bit for bit.
#include <algorithm>
#include <cstdlib>

#include "async.cuh"
#include "ops.cuh"

namespace bg {
namespace {

constexpr int kBkWarps = 16;  // warps per CTA (one CTA per SM)

struct BulkArgs {
  const float* x;
  int64_t rows;
  int k;          // logical inner dimension (floats per row)
  int nwk;        // ceil(k / 32): packed words that can be non-zero
  int kspw;       // storage words per weight row (global)
  int ld;         // shared weight row stride (odd, >= nwk)
  int n, n2;      // result columns (n2 > 0: paired product, second result)
  int nw1;        // words of the first result
  int ntot;       // combined columns (32*nw1 + n2 when paired, else n)
  int ospw;       // storage words per output row
  const uint32_t* wt;
  const float* alpha;  // F output: row scales or null
  const float* beta;   // F output: column scales or null
  uint32_t* out_bits;
  uint32_t* out_bits2;
  float* out_f;
  int d;               // row slots per warp
  uint32_t slot_bytes;
  uintptr_t x_end;     // one past the last float of X (bytes)
  int probe;           // skip the products (timing probe)
};

template <int M, bool OUTB>
__global__ void __launch_bounds__(kBkWarps * 32, 1) k_fbb_bulk(const BulkArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t* sw = reinterpret_cast<uint32_t*>(smem);
  const uint32_t wbytes = (static_cast<uint32_t>(32 * M * a.ld) * 4u + 127u) & ~127u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + wbytes);
  unsigned char* ring = smem + wbytes + ((kBkWarps * a.d * 8 + 127) & ~127);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* mybar = bars + warp * a.d;
  unsigned char* myring = ring + static_cast<size_t>(warp) * a.d * a.slot_bytes;

  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kBkWarps + warp;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kBkWarps;
  const int nrows = gw < a.rows ? static_cast<int>((a.rows - gw + nwarps - 1) / nwarps) : 0;  // this warp's stripe

  // The byte range [a0, a1) a bulk copy can fetch for row r: 16-byte aligned,
  // never past the end of X (a last row that ends off alignment leaves up to
  // three floats to plain loads).
  auto issue = [&](int t) {
    const int64_t r = gw + static_cast<int64_t>(t) * nwarps;
    const uintptr_t b0 = reinterpret_cast<uintptr_t>(a.x + r * a.k);
    const uintptr_t a0 = b0 & ~static_cast<uintptr_t>(15);
    uintptr_t a1 = (b0 + 4u * static_cast<uint32_t>(a.k) + 15u) & ~static_cast<uintptr_t>(15);
    a1 = std::min(a1, a.x_end & ~static_cast<uintptr_t>(15));
    const int s = t % a.d;
    mbar_expect_tx(mybar + s, static_cast<uint32_t>(a1 - a0));
    bulk_g2s(myring + static_cast<size_t>(s) * a.slot_bytes, reinterpret_cast<const void*>(a0),
             static_cast<uint32_t>(a1 - a0), mybar + s);
  };
  if (lane == 0) {
    for (int s = 0; s < a.d; ++s) mbar_init(mybar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int t = 0; t < std::min(a.d, nrows); ++t) issue(t);
  }
  // transposed weight words -> shared memory (row stride ld; rows past ntot
  // and words past nwk stay zero so unused lanes read defined values), bit
  // reversed: a ballot puts float 32w + l at bit l (LSB-first), so the
  // reversed weight word pairs with it without a BREV per activation word.
  // Asynchronous copies: every word in flight at once, not one L2 round
  // trip per loop iteration; each thread reverses the words it copied.
  for (int j = warp; j < 32 * M; j += kBkWarps)
    for (int w = lane; w < a.ld; w += 32) {
      if (j < a.ntot && w < a.nwk) cp_async4(sw + j * a.ld + w, a.wt + static_cast<int64_t>(j) * a.kspw + w);
      else sw[j * a.ld + w] = 0u;
    }
  cp_async_wait_all();
  for (int j = warp; j < 32 * M; j += kBkWarps)
    for (int w = lane; w < a.ld; w += 32) sw[j * a.ld + w] = __brev(sw[j * a.ld + w]);
  __syncthreads();

  const uint32_t* swl = sw + lane * a.ld;
  const int kfull = a.k >> 5, krem = a.k & 31;
  int s = 0;
  uint32_t phase = 0;
  for (int t = 0; t < nrows; ++t) {
    const int64_t r = gw + static_cast<int64_t>(t) * nwarps;
    mbar_wait(mybar + s, phase);
    const float* xrow = a.x + r * a.k;
    const uintptr_t b0 = reinterpret_cast<uintptr_t>(xrow);
    float* xs = reinterpret_cast<float*>(myring + static_cast<size_t>(s) * a.slot_bytes) + ((b0 & 15u) >> 2);
    // a row ending at an unaligned end of X lacks its last < 4 floats in the
    // slot (the bulk copy stops at the aligned end): patch them in
    const uintptr_t cend = std::min((b0 + 4u * static_cast<uint32_t>(a.k) + 15u) & ~static_cast<uintptr_t>(15),
                                    a.x_end & ~static_cast<uintptr_t>(15));
    const int have = static_cast<int>(std::min<uintptr_t>(a.k, (cend - b0) >> 2));
    if (have < a.k) {
      if (lane < a.k - have) xs[have + lane] = __ldg(xrow + have + lane);
      __syncwarp();
    }
    int diff[M];
#pragma unroll
    for (int m = 0; m < M; ++m) diff[m] = 0;
    const float* xl = xs + lane;
    int w = 0;
    if (a.probe) w = kfull;  // BG_BULK_PROBE: the data movement alone
    for (; w + 4 <= kfull; w += 4) {
      uint32_t aw[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) aw[q] = __ballot_sync(0xFFFFFFFFu, xl[32 * (w + q)] >= 0.0f);
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int m = 0; m < M; ++m) diff[m] += __popc(aw[q] ^ swl[32 * m * a.ld + w + q]);
    }
    for (; w < kfull; ++w) {
      const uint32_t aw = __ballot_sync(0xFFFFFFFFu, xl[32 * w] >= 0.0f);
#pragma unroll
      for (int m = 0; m < M; ++m) diff[m] += __popc(aw ^ swl[32 * m * a.ld + w]);
    }
    if (krem) {  // the last, partial word: bits past k are 0 like the weights'
      const uint32_t aw = __ballot_sync(0xFFFFFFFFu, lane < krem && xl[32 * w] >= 0.0f);
#pragma unroll
      for (int m = 0; m < M; ++m) diff[m] += __popc(aw ^ swl[32 * m * a.ld + w]);
    }
    __syncwarp();
    if (lane == 0 && t + a.d < nrows) {  // every lane has read slot s
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the async-proxy refill
      issue(t + a.d);
    }
    if (++s == a.d) s = 0, phase ^= 1u;
    if (OUTB) {
      uint32_t mine = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int j = 32 * m + lane;
        const bool second = m >= a.nw1;
        const int col = second ? j - 32 * a.nw1 : j;
        const bool bit = col < (second ? a.n2 : a.n) && (a.k - 2 * diff[m]) >= 0;
        const uint32_t word = __brev(__ballot_sync(0xFFFFFFFFu, bit));
        if (lane == m) mine = word;
      }
      // lane m stores word m (padding words of 64-bit rows are zero)
      if (a.out_bits2 == nullptr) {
        if (lane < a.ospw) a.out_bits[r * a.ospw + lane] = lane < M ? mine : 0u;
      } else {
        // the second result's word w is combined word nw1 + w
        const int nw2 = (a.n2 + 31) / 32;
        const uint32_t v2 = __shfl_sync(0xFFFFFFFFu, mine, (lane + a.nw1) & 31);
        if (lane < a.ospw) {
          a.out_bits[r * a.ospw + lane] = lane < a.nw1 ? mine : 0u;
          a.out_bits2[r * a.ospw + lane] = lane < nw2 ? v2 : 0u;
        }
      }
    } else {
      const double al = a.alpha ? static_cast<double>(__ldg(a.alpha + r)) : 1.0;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int j = 32 * m + lane;
        if (j < a.n) {
          const double be = a.beta ? static_cast<double>(__ldg(a.beta + j)) : 1.0;
          const double dot = static_cast<double>(a.k - 2 * diff[m]);
          a.out_f[r * a.n + j] = __double2float_rn(__dmul_rn(__dmul_rn(al, dot), be));
        }
      }
    }
  }
}

}  // namespace

// Eligible: fp32 input, at most 128 combined output columns, a row of at
// least 64 bytes, and the rings fit in shared memory.
bool fbb_bulk(const BmmArgs& a, cudaStream_t s) {
  if (!a.a_f || a.rows == 0) return false;
  if (a.k < 16 || a.k > 16384) return false;
  const bool paired = a.out_bits2 != nullptr;
  if (paired && !a.out_bits) return false;
  const int nw1 = static_cast<int>(cdiv(a.n, 32));
  const int ntot = paired ? 32 * nw1 + static_cast<int>(a.n2) : static_cast<int>(a.n);
  if (ntot > 128 || ntot <= 0) return false;
  const int ospw = static_cast<int>(spw(a.out_bits ? (paired ? std::max(a.n, a.n2) : a.n) : 0, a.wb));
  if (a.out_bits && (ospw > 32 || (paired && spw(a.n2, a.wb) != ospw))) return false;

  BulkArgs b{};
  b.x = a.a_f;
  b.rows = a.rows;
  b.k = static_cast<int>(a.k);
  b.nwk = static_cast<int>(cdiv(a.k, 32));
  b.kspw = static_cast<int>(spw(a.k, a.wb));
  b.ld = b.nwk | 1;
  b.n = static_cast<int>(a.n);
  b.n2 = paired ? static_cast<int>(a.n2) : 0;
  b.nw1 = nw1;
  b.ntot = ntot;
  b.ospw = a.out_bits ? static_cast<int>(spw(a.n, a.wb)) : 0;
  b.wt = a.wt;
  b.alpha = a.alpha;
  b.beta = a.beta;
  b.out_bits = a.out_bits;
  b.out_bits2 = a.out_bits2;
  b.out_f = a.out_f;
  b.slot_bytes = static_cast<uint32_t>(((4 * a.k + 15) / 16) * 16 + 16 + 128);
  b.x_end = reinterpret_cast<uintptr_t>(a.a_f + a.rows * a.k);
  b.probe = std::getenv("BG_BULK_PROBE") != nullptr;

  const int M = ntot <= 32 ? 1 : ntot <= 64 ? 2 : 4;
  const size_t wbytes = (static_cast<size_t>(32 * M * b.ld) * 4 + 127) & ~static_cast<size_t>(127);
  const size_t cap = 210 * 1024;
  // ~160 KB of row slots per SM: Cora 16 warps x 2 rows of 5.7 KB (the
  // whole matrix is in flight across the SMs), PubMed 16 x 4 rows of 2 KB
  int d = static_cast<int>(std::min<int64_t>(8, std::max<int64_t>(2, (160 * 1024) / (kBkWarps * b.slot_bytes))));
  auto smem_of = [&](int dd) {
    return wbytes + ((kBkWarps * dd * 8 + 127) & ~127) + static_cast<size_t>(kBkWarps) * dd * b.slot_bytes;
  };
  while (d > 2 && smem_of(d) > cap) --d;
  if (smem_of(d) > cap) return false;
  b.d = d;
  const size_t smem = smem_of(d);
  auto go = [&](auto kern) {
    BG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 0;
    BG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBkWarps * 32, smem));
    const int64_t blocks = std::max<int64_t>(
        1, std::min<int64_t>(cdiv(a.rows, kBkWarps), static_cast<int64_t>(sm_count()) * std::max(per_sm, 1)));
    kern<<<static_cast<unsigned>(blocks), kBkWarps * 32, smem, s>>>(b);
  };
  if (a.out_bits) {
    if (M == 1) go(k_fbb_bulk<1, true>);
    else if (M == 2) go(k_fbb_bulk<2, true>);
    else go(k_fbb_bulk<4, true>);
  } else {
    if (M == 1) go(k_fbb_bulk<1, false>);
    else if (M == 2) go(k_fbb_bulk<2, false>);
    else go(k_fbb_bulk<4, false>);
  }
  BG_LAUNCH_CHECK();
  return true;
}

}  // namespace bg
