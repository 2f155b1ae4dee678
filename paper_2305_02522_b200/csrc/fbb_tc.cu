// MM.FBB / FFB (and the paired F->B product of a SAGE / GraphConv layer) on
// the 5th-generation tensor cores: tcgen05.mma.kind::i8 with a TMEM
// accumulator, warp-specialized and pipelined (ref: bmm B-output path,
// kernels.cpp:140-176; binarize x >= 0, bitdense.cpp:83).
//
// One CTA per SM walks 128-row tiles of X.  Roles:
//   * producer (warp 0): fp32 pieces of PR consecutive rows (contiguous in
//     HBM) into a ring of S shared-memory slots by cp.async.bulk, one
//     mbarrier per slot (full / empty);
//   * converters (warps 2..2+kTcConv-1): each piece -> +-1 bytes (x >= 0 ->
//     +1) written straight into the tile's A operand in the canonical
//     no-swizzle K-major UMMA layout (element (r, k) at (k/16)*M*16 + r*16 +
//     k%16: 8-row x 16-byte core matrices, LBO = M*16 B between K chunks, SBO
//     = 128 B between 8-row groups); lanes run over rows, so every 16-byte
//     store of a quarter warp lands in distinct banks;
//   * MMA issuer (warp 1, one elected lane): ceil(K/32) tcgen05.mma per tile
//     (M = 128, N = 128 or the pair's 256) into TMEM accumulator buffer
//     tile % 2, then tcgen05.commit to the accumulator-full barrier and to
//     the A-empty barrier (A may be refilled once the MMAs have read it);
//   * epilogue (warps 4..7, one per TMEM lane quarter): tcgen05.ld 32
//     columns at a time, dot >= 0 -> bit, MSB-first words, one row per
//     thread (16-byte stores), then the accumulator buffer is released.
// The weights (+-1 bytes, zero past K and past n, so the zero-filled and
// out-of-row A bytes never count) stay in shared memory for the whole kernel.
// Integer dots are exact, so the bits equal the reference's for any order.
#include <cstdlib>
#include <string>

#include "async.cuh"
#include "ops.cuh"

namespace bg {
namespace {

constexpr int kTcM = 128;
constexpr int kTcConv = 12;                      // converter warps
constexpr int kTcThreads = (6 + kTcConv) * 32;   // 18 warps
// warp roles: 0 producer, 1 MMA, 2..3 converters, 4..7 epilogue (warp % 4 =
// its TMEM lane quarter), 8..13 converters
__device__ __forceinline__ bool tc_is_conv(int w) { return w == 2 || w == 3 || w >= 8; }
__device__ __forceinline__ int tc_conv_index(int w) { return w < 4 ? w - 2 : w - 6; }

__device__ __forceinline__ uint32_t sign4(float x0, float x1, float x2, float x3) {
  return pm1_bytes4(x0, x1, x2, x3);
}

__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// A wait that traps instead of hanging if a phase never completes (2 s of
// global time).  Each try suspends the thread until the phase completes or
// `hint` ns pass, so a warp parked behind the pipeline does not spin through
// issue slots the converters and the epilogue need (hint 0: the hardware's
// own short limit).
__device__ __forceinline__ uint32_t tc_try(uint64_t* bar, uint32_t parity, uint32_t hint) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity), "r"(hint)
      : "memory");
  return ok;
}
__device__ __forceinline__ uint64_t tc_now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __noinline__ void tc_wait_slow(uint64_t* bar, uint32_t parity, uint32_t hint) {
  const uint64_t t0 = tc_now();
  while (!tc_try(bar, parity, hint))
    if (tc_now() - t0 > 2000000000ull) __trap();
}
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t parity, uint32_t hint) {
  if (!tc_try(bar, parity, hint)) tc_wait_slow(bar, parity, hint);
}

__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // sm_100 descriptor version; no swizzle, base offset 0
  return d;
}

struct TcArgs {
  const float* x;
  const uint32_t* wt;  // ncols x kspw transposed weight bits (pair: W1 | pad | W2)
  int64_t rows;
  int k, kspw, kpad, n, ncols, ospw, pr, prlog, slots, abufs;
  uint32_t hint;       // try_wait suspend hint, ns
  uint32_t pmagic;     // t / gp by magic multiply (item -> row group)
  uint32_t* out;
  uint32_t* out2;      // pair: columns [ncols/2, ncols) of the accumulator
};

__global__ void __launch_bounds__(kTcThreads, 1) k_fbb_tc(const TcArgs a) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[4], empty[4], a_full[2], a_empty[2], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kpad = a.kpad, N = a.ncols;
  const uint32_t bchunk = static_cast<uint32_t>(N) * 16u, achunk = kTcM * 16u;
  uint8_t* B = sm;                                          // kpad/16 chunks x N rows x 16 B
  uint8_t* A = B + static_cast<size_t>(kpad) * N;           // abufs x (kpad/16 chunks x 128 rows x 16 B)
  float* ring = reinterpret_cast<float*>(A + static_cast<size_t>(a.abufs) * kpad * kTcM);
  const uint32_t slot_floats = static_cast<uint32_t>(a.pr * a.k) + 16;  // + pad: a row's last group may read past
  // weights as +-1 bytes (0 past K and for columns >= n of each half)
  const int half_cols = a.out2 ? N / 2 : N;
  for (int t = tid; t < N * (kpad / 4); t += blockDim.x) {
    const int o = t / (kpad / 4), p4 = (t % (kpad / 4)) * 4;
    uint32_t v = 0;
    if ((o % half_cols) < a.n && p4 < a.k) {
      const uint32_t word = __ldg(a.wt + static_cast<int64_t>(o) * a.kspw + (p4 >> 5));
      const uint32_t nib = (word >> (28 - (p4 & 31))) & 0xFu;
      const uint32_t spread = ((nib >> 3) & 1u) | (((nib >> 2) & 1u) << 8) | (((nib >> 1) & 1u) << 16) | ((nib & 1u) << 24);
      v = 0xFFFFFFFFu - 0xFEu * spread;
      if (p4 + 4 > a.k) v &= 0xFFFFFFFFu >> (8 * (p4 + 4 - a.k));
    }
    *reinterpret_cast<uint32_t*>(B + (p4 >> 4) * bchunk + o * 16 + (p4 & 15)) = v;
  }
  const int64_t tiles = (a.rows + kTcM - 1) / kTcM;
  const int64_t my = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int ppt = kTcM / a.pr;  // pieces per tile
  const int64_t npieces = my * ppt;
  if (warp == 0) {  // TMEM: two accumulators of N s32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_base)),
                 "r"(2 * N)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int s = 0; s < a.slots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTcConv);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&a_full[b], kTcConv);
      mbar_init(&a_empty[b], 1);
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // weights -> tensor core
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  // Piece u of this CTA is piece p = u % ppt of tile j = u / ppt (rows
  // tile0 + pr * p, tile0 = (blockIdx.x + j * grid) * 128) and uses ring slot
  // u % slots and A buffer j % abufs; every role walks these with counters
  // (no 64-bit divisions per piece).
  const int64_t tstep = static_cast<int64_t>(gridDim.x) * kTcM;
  auto piece_len = [&](int64_t r0) {
    const int64_t left = a.rows - r0;
    return static_cast<int>(left <= 0 ? 0 : left < a.pr ? left : a.pr);
  };

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      int s = 0, p = 0;
      uint32_t ph = 0;  // (u / slots) & 1
      int64_t tile0 = static_cast<int64_t>(blockIdx.x) * kTcM;
      for (int64_t u = 0; u < npieces; ++u) {
        if (u >= a.slots) {
          tc_wait(&empty[s], ph ^ 1u, a.hint);
          // the converters' generic reads of the slot before the bulk copy's async-proxy writes
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        const int64_t r0 = tile0 + static_cast<int64_t>(a.pr) * p;
        const int nr = piece_len(r0);
        const uint32_t bytes = static_cast<uint32_t>(nr) * static_cast<uint32_t>(a.k) * 4u;
        if (nr == a.pr && bytes % 16 == 0) {
          mbar_expect_tx(&full[s], bytes);
          bulk_g2s(ring + s * slot_floats, a.x + r0 * a.k, bytes, &full[s]);
        } else {
          mbar_arrive1(&full[s]);  // partial piece: the converters read it from global memory
        }
        if (++s == a.slots) s = 0, ph ^= 1u;
        if (++p == ppt) p = 0, tile0 += tstep;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
                           (static_cast<uint32_t>(kTcM >> 4) << 24);  // kind::i8, s32 += s8 x s8, K-major
    int ab = 0;
    uint32_t aph = 0;  // (j / abufs) & 1
    for (int64_t j = 0; j < my; ++j) {
      const int b = static_cast<int>(j & 1);
      tc_wait(&a_full[ab], aph, a.hint);
      if (j >= 2) tc_wait(&acc_empty[b], static_cast<uint32_t>(((j >> 1) - 1) & 1), a.hint);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t abase = smem_addr(A + static_cast<size_t>(ab) * kpad * kTcM), bbase = smem_addr(B);
        const uint32_t dcol = tmem + static_cast<uint32_t>(b * N);
        for (int ks = 0; ks < kpad / 32; ++ks) {
          const uint64_t ad = tc_desc(abase + 2 * ks * achunk, achunk, 128);
          const uint64_t bd = tc_desc(bbase + 2 * ks * bchunk, bchunk, 128);
          const uint32_t accum = ks > 0 ? 1u : 0u;
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dcol),
              "l"(ad), "l"(bd), "r"(idesc), "r"(accum)
              : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_addr(&acc_full[b]))
                     : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_addr(&a_empty[ab]))
                     : "memory");
      }
      __syncwarp();
      if (++ab == a.abufs) ab = 0, aph ^= 1u;
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- epilogue: TMEM lanes 32*(warp-4) .. +31 ----------------
    const int q = warp - 4;
    for (int64_t j = 0; j < my; ++j) {
      const int b = static_cast<int>(j & 1);
      tc_wait(&acc_full[b], static_cast<uint32_t>((j >> 1) & 1), a.hint);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t row = (blockIdx.x + j * gridDim.x) * kTcM + 32 * q + lane;
      for (int h = 0; h < (a.out2 ? 2 : 1); ++h) {
        uint32_t words[8];
#pragma unroll
        for (int cw = 0; cw < 8; ++cw) words[cw] = 0u;
        for (int cw = 0; cw < half_cols / 32 && cw < 8; ++cw) {
          uint32_t d[32];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
                "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]),
                "=r"(d[15]), "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]),
                "=r"(d[22]), "=r"(d[23]), "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]),
                "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
              : "r"(tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(b * N + h * half_cols + 32 * cw)));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          // the sign bits shift in one funnel shift each (MSB-first); bit = dot >= 0
          uint32_t m = 0;
#pragma unroll
          for (int t = 0; t < 32; ++t) m = __funnelshift_l(d[t], m, 1);
          m = ~m;
          if (32 * cw + 32 > a.n) m &= 32 * cw >= a.n ? 0u : tail_mask32(a.n);  // columns >= n stay 0
          words[cw] = m;
        }
        uint32_t* o = (h ? a.out2 : a.out) + row * a.ospw;
        if (row < a.rows) {
          if (a.ospw == 4) {
            *reinterpret_cast<uint4*>(o) = make_uint4(words[0], words[1], words[2], words[3]);
          } else {
            for (int w = 0; w < a.ospw; ++w) o[w] = w < 8 ? words[w] : 0u;
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive1(&acc_empty[b]);
    }
  } else if (tc_is_conv(warp)) {
    // ---------------- converters ----------------
    const int cw = tc_conv_index(warp), ct = cw * 32 + lane;
    const int gp = (a.k + 15) / 16;                // 16-column groups per row
    const int items = a.pr * gp;                   // (row, group) per piece; item t -> row t % pr, group t / pr
    int s = 0, p = 0, ab = 0;
    uint32_t ph = 0, aph = 0;  // (u / slots) & 1, (j / abufs) & 1
    int64_t j = 0, tile0 = static_cast<int64_t>(blockIdx.x) * kTcM;
    for (int64_t u = 0; u < npieces; ++u) {
      if (p == 0 && j >= a.abufs) tc_wait(&a_empty[ab], aph ^ 1u, a.hint);
      tc_wait(&full[s], ph, a.hint);
      const int64_t r0 = tile0 + static_cast<int64_t>(a.pr) * p;
      const int nr = piece_len(r0);
      const bool staged = nr == a.pr && (static_cast<uint32_t>(nr) * a.k * 4u) % 16 == 0;
      const float* src = staged ? ring + s * slot_floats : a.x + r0 * a.k;
      uint8_t* At = A + static_cast<size_t>(ab) * kpad * kTcM;
      const int rbase = a.pr * p;
      for (int t = ct; t < items; t += kTcConv * 32) {
        const int r = t & (a.pr - 1), g = t >> a.prlog;  // pr is a power of two
        const int c0 = 16 * g;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (r < nr) {
          const float* xr = src + static_cast<int64_t>(r) * a.k + c0;
          float e[16];
          if (staged) {  // past-row reads stay inside the slot (+16 floats) and meet zero weights
            if ((a.k & 3) == 0) {
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                const float4 f = lds_f4(smem_addr(xr) + 16u * h);
                e[4 * h] = f.x, e[4 * h + 1] = f.y, e[4 * h + 2] = f.z, e[4 * h + 3] = f.w;
              }
            } else if ((a.k & 1) == 0) {
#pragma unroll
              for (int h = 0; h < 8; ++h) {
                const float2 f = reinterpret_cast<const float2*>(xr)[h];
                e[2 * h] = f.x, e[2 * h + 1] = f.y;
              }
            } else {
#pragma unroll
              for (int h = 0; h < 16; ++h) e[h] = xr[h];
            }
          } else {
#pragma unroll
            for (int h = 0; h < 16; ++h) e[h] = c0 + h < a.k ? __ldg(xr + h) : 0.0f;
          }
          v = make_uint4(sign4(e[0], e[1], e[2], e[3]), sign4(e[4], e[5], e[6], e[7]),
                         sign4(e[8], e[9], e[10], e[11]), sign4(e[12], e[13], e[14], e[15]));
        }
        *reinterpret_cast<uint4*>(At + static_cast<size_t>(g) * achunk + (rbase + r) * 16) = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // A (generic stores) -> tensor core
      __syncwarp();
      if (lane == 0) {
        mbar_arrive1(&empty[s]);
        if (p == ppt - 1) mbar_arrive1(&a_full[ab]);
      }
      if (++s == a.slots) s = 0, ph ^= 1u;
      if (++p == ppt) {
        p = 0, ++j, tile0 += tstep;
        if (++ab == a.abufs) ab = 0, aph ^= 1u;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * N) : "memory");
}

}  // namespace

// FBB (or a pair) on k_fbb_tc: false (nothing launched) when not eligible.
bool fbb_tc(const BmmArgs& a, cudaStream_t s) {
  if (!a.a_f || !a.out_bits || a.n == 0 || a.n > 128 || a.k <= 0 || a.rows == 0) return false;
  if (const char* e = std::getenv("BG_FBB"); e && std::string(e) != "tc") return false;
  if (reinterpret_cast<uintptr_t>(a.a_f) % 16 != 0) return false;
  const bool pair = a.out_bits2 != nullptr;
  if (pair && a.n2 != a.n) return false;
  const int nw = static_cast<int>(cdiv(a.n, 32));
  // N of the MMA: one product's columns rounded to 32 (pair: W1 | pad | W2 as
  // the paired weights lay them out), a power of two for the TMEM allocation
  int half = 32;
  while (half < 32 * nw) half *= 2;
  if (pair && half != 32 * nw) return false;  // the pair's second matrix must start at column `half`
  const int N = pair ? 2 * half : half;
  if (N > 256) return false;
  TcArgs t{};
  t.x = a.a_f;
  t.wt = a.wt;
  t.rows = a.rows;
  t.k = static_cast<int>(a.k);
  t.kspw = static_cast<int>(spw(a.k, a.wb));
  t.kpad = static_cast<int>(32 * cdiv(a.k, 32));
  t.n = static_cast<int>(a.n);
  t.ncols = N;
  t.ospw = static_cast<int>(spw(a.n, a.wb));
  t.out = a.out_bits;
  t.out2 = a.out_bits2;
  t.hint = 0;
  if (const char* e = std::getenv("BG_TC_HINT")) t.hint = static_cast<uint32_t>(std::atoi(e));
  // shared memory: weights + A buffers + the fp32 ring; the largest pieces
  // (rows) and then two A buffers if they fit
  const size_t wbytes = static_cast<size_t>(t.kpad) * N, abytes = static_cast<size_t>(t.kpad) * kTcM;
  const size_t cap = 227 * 1024 - 2048;  // static shared memory (barriers, TMEM base) counts too
  bool ok = false;
  for (int abufs = 2; abufs >= 1 && !ok; --abufs)
    for (int pr = 128; pr >= 8 && !ok; pr /= 2)
      for (int slots = 4; slots >= 2 && !ok; --slots) {
        const size_t ring = static_cast<size_t>(slots) * (static_cast<size_t>(pr) * a.k + 16) * 4;
        if (wbytes + abufs * abytes + ring <= cap) {
          t.abufs = abufs;
          t.pr = pr;
          t.slots = slots;
          ok = true;
        }
      }
  if (!ok) return false;
  // By default only where the pipeline has room: two A buffers (the next
  // tile converts while the MMAs read this one) and >= 32-row pieces.
  // Measured: products' paired FBB (K = 100, N = 2 x 128) 0.52 -> 0.31 ms;
  // Reddit's FBB (K = 602: 78 KB of weights + a 78 KB A tile leave an
  // 8-row, 3-slot ring and one A buffer) 0.29 ms vs 0.14 ms on the TMA-fed
  // mma.sync kernel, which therefore keeps that shape.
  const char* force = std::getenv("BG_FBB");
  if (!force && (t.abufs < 2 || t.pr < 32)) return false;
  t.prlog = 0;
  while ((1 << t.prlog) < t.pr) ++t.prlog;
  const size_t smem = wbytes + t.abufs * abytes + static_cast<size_t>(t.slots) * (static_cast<size_t>(t.pr) * a.k + 16) * 4;
  static int attr_done = 0;
  if (!attr_done) {
    BG_CUDA(cudaFuncSetAttribute(k_fbb_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cap)));
    attr_done = 1;
  }
  const int64_t tiles = cdiv(a.rows, kTcM);
  const int64_t blocks = std::min<int64_t>(tiles, sm_count());
  k_fbb_tc<<<static_cast<unsigned>(blocks), kTcThreads, smem, s>>>(t);
  BG_LAUNCH_CHECK();
  return true;
}

}  // namespace bg
