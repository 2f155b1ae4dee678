// Binary dense transform (ref: bmm, kernels.cpp:140-191).
//
// dot(i,j) = K - 2*popc(a_i XOR w_j) over whole packed rows (padding bits are
// zero on both sides and cancel, kernels.cpp:30-41).  B output: bit = dot >= 0
// with no scale (SCL elimination, :159-161).  F output: float((alpha*dot)*beta)
// evaluated in double in that order (:179-190).
//
// One warp per row; the transposed weight bits live in shared memory (row
// stride padded to an odd word count, so the 32 lanes of a warp -- one output
// column each -- hit 32 distinct banks).  With fp32 input the row is
// binarized in the prologue by warp ballots on coalesced loads, so FBB/FBF
// read X exactly once and never write packed X back (north-star item 4).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "ops.cuh"
#include "async.cuh"

namespace bg {
namespace {

constexpr int kWarps = 8;
constexpr int kMaxOutPerLane = 8;  // output columns per lane per pass (256 per pass)
constexpr int kF4 = 4;             // float4 chunks per lane in flight (k_bmm fp32 rows: 512 floats per warp round)

template <bool AF, bool OUTB, int M>
__global__ void __launch_bounds__(kWarps * 32)
    k_bmm(const uint32_t* __restrict__ a_bits, const float* __restrict__ a_f,
          const float* __restrict__ alpha, const uint32_t* __restrict__ wt,
          const float* __restrict__ beta, int64_t rows, int64_t k, int64_t n, int64_t kspw,
          int64_t ld, int64_t c0, int64_t nc, int64_t ospw, uint32_t* __restrict__ out_bits,
          float* __restrict__ out_f, uint32_t* __restrict__ out_bits2, int64_t n2, int64_t ntot) {
  extern __shared__ uint32_t smem[];
  uint32_t* sw = smem;                       // nc x ld transposed weight words
  uint32_t* srow = smem + 32 * M * ld;       // kWarps x kspw packed activation rows (after all 32*M weight rows the lanes read)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // fp32 input: 16-byte loads from the row's 16-byte-aligned frame (t = the
  // float's index from the aligned address below the row start, s = the row
  // start's offset in it), lane per float4 chunk: a nibble of signs per
  // chunk, 8 lanes' nibbles OR-shuffled into one aligned word A_v (floats t
  // in [32v, 32v+32)), then each packed row word is the funnel shift
  // (A_w, A_w+1) << s.  kF4 chunks per lane are in flight at once (1,536
  // floats per warp: a Cora row is one DRAM round trip).  The first batch of
  // this warp's first row goes out before the weight staging, so the two
  // latencies overlap.
  constexpr int B4 = kF4;
  // 32-bit index math below (row offsets stay 64-bit): k < 2^28 floats
  const int kk = static_cast<int>(k), kw = static_cast<int>(kspw);
  const int nwa = kw + 1;  // aligned words A_0 .. A_kspw
  const int nch = 8 * nwa; // chunks covering them
  uint32_t* araw = srow + kWarps * kw + warp * (kw + 2);
  auto frame = [&](int64_t row, int& sh) {
    const uintptr_t p = reinterpret_cast<uintptr_t>(a_f + row * k);
    sh = static_cast<int>((p >> 2) & 3);
    return reinterpret_cast<const float4*>(p - 4 * static_cast<uintptr_t>(sh));
  };
  auto load = [&](const float4* xa, int sh, int c0, float4 (&v)[B4]) {
    const int lim = (sh + kk + 3) >> 2;  // chunks holding row floats
#pragma unroll
    for (int m = 0; m < B4; ++m) {
      const int c = c0 + 32 * m + lane;
      v[m] = c < lim ? __ldg(xa + c) : make_float4(-1.0f, -1.0f, -1.0f, -1.0f);
    }
  };
  float4 pre[B4];
  const int64_t row_first = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  if (AF && row_first < rows) {
    int sh;
    const float4* xa = frame(row_first, sh);
    load(xa, sh, 0, pre);
  }
  // warp per weight row, lanes along its words; asynchronous copies, so
  // every word is in flight at once instead of one L2 round trip per row
  {
    // the pass's nc x kspw weight words are contiguous: a flat copy, word t
    // of weight row j = t / kspw landing at t + j * (ld - kspw)
    const uint32_t* wsrc = wt + c0 * kspw;
    const uint32_t total = static_cast<uint32_t>(nc * kspw), pad = static_cast<uint32_t>(ld - kspw);
    if (pad == 0 && (total & 3u) == 0 && (reinterpret_cast<uintptr_t>(wsrc) & 15) == 0) {
      for (uint32_t t = 4 * threadIdx.x; t < total; t += 4 * blockDim.x) cp_async16(sw + t, wsrc + t);
    } else {
      const uint32_t magic = 0xFFFFFFFFu / static_cast<uint32_t>(kw) + 1u;  // t / kspw = umulhi(t, magic) (t * kspw < 2^31)
      for (uint32_t t = threadIdx.x; t < total; t += blockDim.x)
        cp_async4(sw + t + __umulhi(t, magic) * pad, wsrc + t);
    }
  }
  cp_async_wait_all();
  __syncthreads();
  uint32_t* arow = srow + warp * kspw;
  for (int64_t row = row_first; row < rows; row += static_cast<int64_t>(gridDim.x) * kWarps) {
    if (AF) {
      int sh;
      const float4* xa = frame(row, sh);
      const int lo = sh, hi = sh + kk;  // row floats: t in [lo, hi)
      for (int c0 = 0; c0 < nch; c0 += 32 * B4) {
        float4 (&v)[B4] = pre;  // the first batch of the first row is already in flight
        if (c0 != 0 || row != row_first) load(xa, sh, c0, v);
#pragma unroll
        for (int m = 0; m < B4; ++m) {
          if (c0 + 32 * m >= nch) break;  // warp-uniform
          const int c = c0 + 32 * m + lane, t0 = 4 * c;
          uint32_t nib = (v[m].x >= 0.0f ? 8u : 0u) | (v[m].y >= 0.0f ? 4u : 0u) | (v[m].z >= 0.0f ? 2u : 0u) |
                         (v[m].w >= 0.0f ? 1u : 0u);
          if (t0 < lo || t0 + 4 > hi) {  // chunk straddles the row's ends
            uint32_t msk = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) msk |= (t0 + q >= lo && t0 + q < hi) ? (8u >> q) : 0u;
            nib &= msk;
          }
          uint32_t w = nib << (28 - 4 * (lane & 7));
          w |= __shfl_xor_sync(0xFFFFFFFFu, w, 1);
          w |= __shfl_xor_sync(0xFFFFFFFFu, w, 2);
          w |= __shfl_xor_sync(0xFFFFFFFFu, w, 4);
          if ((lane & 7) == 0 && (c >> 3) < nwa) araw[c >> 3] = w;
        }
      }
      __syncwarp();
      for (int w = lane; w < kw; w += 32) arow[w] = __funnelshift_l(araw[w + 1], araw[w], sh);
    } else {
      for (int64_t w = lane; w < kspw; w += 32) arow[w] = __ldg(a_bits + row * kspw + w);
    }
    __syncwarp();
    int diff[M];
#pragma unroll
    for (int m = 0; m < M; ++m) diff[m] = 0;
    const uint32_t* swl = sw + lane * ld;
    const int kw2 = static_cast<int>(kspw), ld2 = static_cast<int>(ld);
#pragma unroll 4
    for (int w = 0; w < kw2; ++w) {
      const uint32_t aw = arow[w];
#pragma unroll
      for (int m = 0; m < M; ++m) diff[m] += __popc(aw ^ swl[32 * m * ld2 + w]);
    }
    __syncwarp();
    if (OUTB) {
      // combined column jg = c0 + j: words below nw1 belong to the first
      // result (n valid columns), the rest to out_bits2 (n2 valid columns)
      const int64_t nw1 = (n + 31) / 32, nw2 = (n2 + 31) / 32;
      const int64_t ospw2 = out_bits2 ? ospw : 0;  // paired results share the word width and column count class
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int64_t j = 32 * m + lane, gw = c0 / 32 + m;
        const bool second = gw >= nw1;
        const int64_t col = second ? c0 + j - 32 * nw1 : c0 + j;
        const bool bit = j < nc && col < (second ? n2 : n) && (k - 2 * static_cast<int64_t>(diff[m])) >= 0;
        const uint32_t word = __brev(__ballot_sync(0xFFFFFFFFu, bit));
        if (lane == 0 && 32 * m < nc) {  // only words of this pass
          if (second) out_bits2[row * ospw2 + (gw - nw1)] = word;
          else out_bits[row * ospw + gw] = word;
        }
      }
      // zero the storage-padding words of 64-bit rows after the last pass
      if (lane == 0 && c0 + nc == ntot) {
        for (int64_t w = nw1; w < ospw; ++w) out_bits[row * ospw + w] = 0;
        if (out_bits2)
          for (int64_t w = nw2; w < ospw2; ++w) out_bits2[row * ospw2 + w] = 0;
      }
    } else {
      const double al = alpha ? static_cast<double>(alpha[row]) : 1.0;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int64_t j = 32 * m + lane;
        if (j < nc) {
          const double be = beta ? static_cast<double>(beta[c0 + j]) : 1.0;
          const double dot = static_cast<double>(k - 2 * static_cast<int64_t>(diff[m]));
          out_f[row * n + c0 + j] = __double2float_rn(__dmul_rn(__dmul_rn(al, dot), be));
        }
      }
    }
  }
}

// ---- B-output products with one node row per lane ---------------------------
// Binary output needs no scales (kernels.cpp:159-161), so the product is pure
// popcount work: each lane owns one activation row (its KW packed words in
// registers) and every weight word is a warp-uniform shared-memory broadcast
// (LDS.128, four output columns at a time), i.e. XOR + POPC + 1/2 IADD3 per
// (row, column, word) and no per-lane weight traffic.  With fp32 input the
// warp first binarizes its 32 rows with ballots on coalesced loads (the row
// goes through shared memory, never through HBM packed).
constexpr int kLrWarps = 8;

template <bool AF, int KW>
__global__ void __launch_bounds__(kLrWarps * 32)
    k_bmm_lanerow(const uint32_t* __restrict__ a_bits, const float* __restrict__ a_f,
                  const uint32_t* __restrict__ wt, int64_t rows, int k, int kspw, int n, int npad,
                  int ospw, uint32_t* __restrict__ out_bits) {
  extern __shared__ uint4 smem4[];
  uint32_t* sw = reinterpret_cast<uint32_t*>(smem4);  // kspw x npad: W[w][o]
  const int ld = kspw | 1;                             // stage row stride (odd: no conflicts)
  uint32_t* stage = sw + kspw * npad + (threadIdx.x >> 5) * 32 * ld;
  for (int t = threadIdx.x; t < kspw * npad; t += blockDim.x) {
    const int w = t / npad, o = t % npad;
    if (o < n) cp_async4(sw + t, wt + static_cast<int64_t>(o) * kspw + w);  // all in flight at once
    else sw[t] = 0u;
  }
  cp_async_wait_all();
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = static_cast<int64_t>(blockIdx.x) * kLrWarps + (threadIdx.x >> 5);
  for (int64_t base = warp0 * 32; base < rows; base += static_cast<int64_t>(gridDim.x) * kLrWarps * 32) {
    const int64_t row = base + lane;
    uint32_t a[KW];
    if (AF) {
      const int nr = rows - base < 32 ? static_cast<int>(rows - base) : 32;
      for (int r = 0; r < nr; ++r) {
        const float* xr = a_f + (base + r) * k;
        float v[KW];
#pragma unroll
        for (int w = 0; w < KW; ++w) {
          const int j = 32 * w + lane;
          v[w] = (w < kspw && j < k) ? __ldg(xr + j) : -1.0f;
        }
#pragma unroll
        for (int w = 0; w < KW; ++w) {
          const uint32_t word = __brev(__ballot_sync(0xFFFFFFFFu, v[w] >= 0.0f));
          if (lane == 0 && w < kspw) stage[r * ld + w] = word;
        }
      }
      __syncwarp();
#pragma unroll
      for (int w = 0; w < KW; ++w) a[w] = w < kspw ? stage[lane * ld + w] : 0u;
      __syncwarp();
    } else {
#pragma unroll
      for (int w = 0; w < KW; ++w) a[w] = (w < kspw && row < rows) ? __ldg(a_bits + row * kspw + w) : 0u;
    }
    for (int oc = 0; oc < ospw; ++oc) {
      uint32_t bits = 0;
      if (32 * oc < n) {
        int d[32];
#pragma unroll
        for (int o = 0; o < 32; ++o) d[o] = 0;
#pragma unroll
        for (int w = 0; w < KW; ++w) {
          if (w < kspw) {
            const uint4* wv = reinterpret_cast<const uint4*>(sw + w * npad + 32 * oc);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const uint4 c = wv[q];
              d[4 * q + 0] += __popc(a[w] ^ c.x);
              d[4 * q + 1] += __popc(a[w] ^ c.y);
              d[4 * q + 2] += __popc(a[w] ^ c.z);
              d[4 * q + 3] += __popc(a[w] ^ c.w);
            }
          }
        }
        // dot = K - 2*diff >= 0 (padding bits are zero on both sides and cancel)
#pragma unroll
        for (int o = 0; o < 32; ++o)
          if (32 * oc + o < n && 2 * d[o] <= k) bits |= 0x80000000u >> o;
      }
      if (row < rows) out_bits[row * ospw + oc] = bits;
    }
  }
}

// ---- fp32-input products on the int8 tensor cores ---------------------------
// sign(x) in {+1, -1} (bit = x >= 0, bitdense.cpp:71-88) is an exact int8, so
// the +-1 dot of FBB/FBF is an int8 GEMM with int32 accumulation: dot =
// sum_k s(a_ik) s(w_kj), |dot| <= K, exact.  One warp owns 16 rows (one
// m16n8k32 A tile) and converts them straight from fp32 registers to int8
// fragments -- X is read from HBM exactly once and never materialised packed.
// The weights live in shared memory as +-1 bytes (0 past K / past n), each
// 32-k block permuted so a B fragment (k 4t..4t+3 and 16+4t..16+4t+3 of
// column g) is one 8-byte load, rows padded to a conflict-free stride.
// (The b1 mma.sync form is emulated on sm_100a -- LOP3/MOVM.U4TO8 expansion
// plus 8 IMMA per instruction, see DESIGN.md -- so int8 is the native path.)
constexpr int kImWarps = 8;

__device__ __forceinline__ void mma_s8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Four fp32 values -> four +-1 bytes (element i in byte i): the x >= 0 nibble
// is spread to bytes by one multiply, then 1 -> 0x01, 0 -> 0xFF.
__device__ __forceinline__ uint32_t sign_bytes4(float x0, float x1, float x2, float x3) {
  const uint32_t m = static_cast<uint32_t>(x0 >= 0.0f) | (static_cast<uint32_t>(x1 >= 0.0f) << 1) |
                     (static_cast<uint32_t>(x2 >= 0.0f) << 2) | (static_cast<uint32_t>(x3 >= 0.0f) << 3);
  return 0xFFFFFFFFu - 0xFEu * ((m * 0x00204081u) & 0x01010101u);
}

// Four fp32 values -> four +-1 bytes (element i in byte i); `valid` bytes past K are 0.
__device__ __forceinline__ uint32_t sign_bytes(float x0, float x1, float x2, float x3) {
  return (x0 >= 0.0f ? 0x00000001u : 0x000000FFu) | (x1 >= 0.0f ? 0x00000100u : 0x0000FF00u) |
         (x2 >= 0.0f ? 0x00010000u : 0x00FF0000u) | (x3 >= 0.0f ? 0x01000000u : 0xFF000000u);
}

template <bool OUTB, int NT>
__global__ void __launch_bounds__(kImWarps * 32)
    k_bmm_imma(const float* __restrict__ a_f, const float* __restrict__ alpha,
               const uint32_t* __restrict__ wt, const float* __restrict__ beta, int64_t rows, int k,
               int kspw, int n, int ksteps, int ldw, int ospw, uint32_t* __restrict__ out_bits,
               float* __restrict__ out_f) {
  extern __shared__ uint4 smem4[];
  uint8_t* w8 = reinterpret_cast<uint8_t*>(smem4);  // (8*NT) x ldw bytes
  const int kpad = 32 * ksteps;
  // weights: byte of (column o, position p) with p = 32*blk + 8*t + 4*half + i <-> k = 32*blk + 16*half + 4*t + i
  for (int t = threadIdx.x; t < 8 * NT * (kpad / 4); t += blockDim.x) {
    const int o = t / (kpad / 4), p4 = (t % (kpad / 4)) * 4;
    const int blk = p4 >> 5, tt = (p4 >> 3) & 3, half = (p4 >> 2) & 1;
    const int k0 = 32 * blk + 16 * half + 4 * tt;
    uint32_t v = 0;
    if (o < n) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int kk = k0 + i;
        if (kk < k) {
          const uint32_t bit = (__ldg(wt + static_cast<int64_t>(o) * kspw + (kk >> 5)) >> (31 - (kk & 31))) & 1u;
          v |= (bit ? 0x01u : 0xFFu) << (8 * i);
        }
      }
    }
    *reinterpret_cast<uint32_t*>(w8 + o * ldw + p4) = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const bool vec2 = (k & 1) == 0 && (reinterpret_cast<uintptr_t>(a_f) & 7) == 0;
  for (int64_t tile = static_cast<int64_t>(blockIdx.x) * kImWarps + (threadIdx.x >> 5); tile * 16 < rows;
       tile += static_cast<int64_t>(gridDim.x) * kImWarps) {
    const int64_t r0 = tile * 16 + g, r1 = r0 + 8;
    const float* x0 = a_f + (r0 < rows ? r0 : 0) * static_cast<int64_t>(k);
    const float* x1 = a_f + (r1 < rows ? r1 : 0) * static_cast<int64_t>(k);
    int acc[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0;
    for (int ks = 0; ks < ksteps; ++ks) {
      const int ka = 32 * ks + 4 * t4, kb = ka + 16;  // element columns of a0/a1 and a2/a3
      float v[16];
      if (32 * ks + 32 <= k && vec2) {
        const float2* p00 = reinterpret_cast<const float2*>(x0 + ka);
        const float2* p01 = reinterpret_cast<const float2*>(x0 + kb);
        const float2* p10 = reinterpret_cast<const float2*>(x1 + ka);
        const float2* p11 = reinterpret_cast<const float2*>(x1 + kb);
        float2 q[8] = {__ldg(p00), __ldg(p00 + 1), __ldg(p10), __ldg(p10 + 1),
                       __ldg(p01), __ldg(p01 + 1), __ldg(p11), __ldg(p11 + 1)};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[2 * i] = q[i].x;
          v[2 * i + 1] = q[i].y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          v[i] = ka + i < k ? __ldg(x0 + ka + i) : 0.0f;
          v[4 + i] = ka + i < k ? __ldg(x1 + ka + i) : 0.0f;
          v[8 + i] = kb + i < k ? __ldg(x0 + kb + i) : 0.0f;
          v[12 + i] = kb + i < k ? __ldg(x1 + kb + i) : 0.0f;
        }
      }
      uint32_t a[4];
#pragma unroll
      for (int f = 0; f < 4; ++f) a[f] = sign_bytes(v[4 * f], v[4 * f + 1], v[4 * f + 2], v[4 * f + 3]);
      if (32 * ks + 32 > k) {  // K tail: elements past K contribute 0
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (ka + i >= k) { a[0] &= ~(0xFFu << (8 * i)); a[1] &= ~(0xFFu << (8 * i)); }
          if (kb + i >= k) { a[2] &= ~(0xFFu << (8 * i)); a[3] &= ~(0xFFu << (8 * i)); }
        }
      }
      const uint8_t* wb = w8 + g * ldw + 32 * ks + 8 * t4;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const uint2 b = *reinterpret_cast<const uint2*>(wb + 8 * j * ldw);
        mma_s8(acc[j], a, b.x, b.y);
      }
    }
    // c0,c1: row r0, columns 8j+2t, 8j+2t+1; c2,c3: row r1, same columns
    if (OUTB) {
      // word w of a row = columns 32w..32w+31 = tiles 4w..4w+3; bit 31-c
#pragma unroll
      for (int w = 0; w < (NT + 3) / 4; ++w) {
        uint32_t m0 = 0, m1 = 0;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = 4 * w + jj;
          if (j < NT) {
            const int c = 8 * jj + 2 * t4;
            if (acc[j][0] >= 0) m0 |= 0x80000000u >> c;
            if (acc[j][1] >= 0) m0 |= 0x40000000u >> c;
            if (acc[j][2] >= 0) m1 |= 0x80000000u >> c;
            if (acc[j][3] >= 0) m1 |= 0x40000000u >> c;
          }
        }
        m0 |= __shfl_xor_sync(0xFFFFFFFFu, m0, 1);
        m0 |= __shfl_xor_sync(0xFFFFFFFFu, m0, 2);
        m1 |= __shfl_xor_sync(0xFFFFFFFFu, m1, 1);
        m1 |= __shfl_xor_sync(0xFFFFFFFFu, m1, 2);
        // columns >= n are zero padding (their weights are 0 so dot = 0 -> bit set): clear them
        if (32 * w + 32 > n) {
          const uint32_t keep = 32 * w >= n ? 0u : tail_mask32(n);
          m0 &= keep;
          m1 &= keep;
        }
        if (t4 == (w & 3) && w < ospw) {  // words past the row (N < 32*NT/4) do not exist
          if (r0 < rows) out_bits[r0 * ospw + w] = m0;
          if (r1 < rows) out_bits[r1 * ospw + w] = m1;
        }
      }
      if (t4 == 0)
        for (int w = (n + 31) / 32; w < ospw; ++w) {  // storage padding of 64-bit rows
          if (r0 < rows) out_bits[r0 * ospw + w] = 0;
          if (r1 < rows) out_bits[r1 * ospw + w] = 0;
        }
    } else {
      const double al0 = r0 < rows && alpha ? static_cast<double>(alpha[r0]) : 1.0;
      const double al1 = r1 < rows && alpha ? static_cast<double>(alpha[r1]) : 1.0;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 8 * j + 2 * t4 + e;
          if (c < n) {
            const double be = beta ? static_cast<double>(beta[c]) : 1.0;
            if (r0 < rows)
              out_f[r0 * n + c] = __double2float_rn(__dmul_rn(__dmul_rn(al0, static_cast<double>(acc[j][e])), be));
            if (r1 < rows)
              out_f[r1 * n + c] = __double2float_rn(__dmul_rn(__dmul_rn(al1, static_cast<double>(acc[j][2 + e])), be));
          }
        }
      }
    }
  }
}

// ---- TMA-fed FBB: the fp32 activation stream at HBM speed -------------------
// A CTA of two teams of four warps walks 16-row tiles of X.  Each tile (16 x K
// fp32, contiguous) arrives by one bulk async copy into a 3-deep ring; the
// team converts it once to +-1 bytes in shared memory (the fp32 slot is then
// refilled with the tile three ahead), and warp w of the team runs the
// m16n8k32 s8 MMAs for output word w (columns 32w..32w+31) and packs
// dot >= 0 into the word (kernels.cpp:166-171).  Weights are +-1 bytes in
// shared memory for the whole kernel.
// One ring slot per team: slot j % kFbbStages is only ever waited on by team
// j % kFbbTeams, so each slot's mbarrier phases are consumed in order by the
// team that refills it (a parity wait cannot tell use u from use u-2).
constexpr int kFbbTeams = 3;
constexpr int kFbbStages = kFbbTeams;

// fp32 -> +-1 bytes (x >= 0 -> +1, bitdense.cpp:83) of one 16-row tile into
// the team's int8 tile.  Item t = (row r, 8-column group) with r = t / q
// (magic multiply); groups past K are never written (zeroed once); the last
// group of a row is masked; rows >= valid become zero.  GLOBAL: the source is
// the operand itself (partial last tile), else the shared-memory ring slot.
template <bool GLOBAL>
__device__ __forceinline__ void fbb_convert(const float* __restrict__ src, int valid, int k, bool keven,
                                            uint32_t items, uint32_t q, uint32_t qmagic, int ttid, int nthr,
                                            int lda, uint8_t* __restrict__ mine) {
  for (uint32_t t = ttid; t < items; t += nthr) {
    const uint32_t r = __umulhi(t, qmagic);
    const uint32_t c = 8 * (t - r * q);
    uint2 v = make_uint2(0u, 0u);
    if (!GLOBAL || static_cast<int>(r) < valid) {
      const float* x = src + r * k + c;
      float e[8];
      if (keven && (!GLOBAL || c + 8 <= static_cast<uint32_t>(k))) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const float2 p2 = *reinterpret_cast<const float2*>(x + 2 * h);
          e[2 * h] = p2.x;
          e[2 * h + 1] = p2.y;
        }
      } else {
#pragma unroll
        for (int h = 0; h < 8; ++h) e[h] = (!GLOBAL || c + h < static_cast<uint32_t>(k)) ? x[h] : 0.0f;
      }
      v.x = sign_bytes4(e[0], e[1], e[2], e[3]);
      v.y = sign_bytes4(e[4], e[5], e[6], e[7]);
      if (c + 8 > static_cast<uint32_t>(k)) {
        const int rem = k - static_cast<int>(c);  // 1..7 valid columns
        v.x &= rem >= 4 ? 0xFFFFFFFFu : 0xFFFFFFFFu >> (8 * (4 - rem));
        v.y &= rem <= 4 ? 0u : 0xFFFFFFFFu >> (8 * (8 - rem));
      }
    }
    *reinterpret_cast<uint2*>(mine + r * lda + c) = v;
  }
}

// Even K, full tile in the ring slot: the tile is TR*K contiguous fp32 in
// shared memory (16-byte aligned), so it is read as 16-byte chunks of the
// flattened tile -- one LDS.128 per lane, consecutive lanes consecutive
// chunks (4 wavefronts per warp instruction, where fbb_convert's per-row
// 8-column items cost 8 per LDS.64).  A chunk's elements (2p, 2p+1) never
// straddle a row (K even), so it lands as two 2-byte stores.
__device__ __forceinline__ void fbb_convert4(const float* __restrict__ src, int tr, int k, uint32_t kmagic,
                                             int ttid, int nthr, int lda, uint8_t* __restrict__ mine) {
  const uint32_t nch = static_cast<uint32_t>(tr * k) >> 2;
  const float4* s4 = reinterpret_cast<const float4*>(src);
  for (uint32_t i = ttid; i < nch; i += nthr) {
    const float4 v = s4[i];
    const uint32_t b = sign_bytes4(v.x, v.y, v.z, v.w);
    const uint32_t f = 4 * i;
    const uint32_t r = __umulhi(f, kmagic);  // f / k (f * k < 2^32)
    const uint32_t c = f - r * static_cast<uint32_t>(k);
    *reinterpret_cast<uint16_t*>(mine + r * lda + c) = static_cast<uint16_t>(b);
    const bool wrap = c + 2 >= static_cast<uint32_t>(k);
    *reinterpret_cast<uint16_t*>(mine + (wrap ? (r + 1) * lda : r * lda + c + 2)) = static_cast<uint16_t>(b >> 16);
  }
}

template <int NW, int HALVES>  // output words per row (N <= 32*NW); one warp per word; 2: paired product
__global__ void __launch_bounds__(kFbbTeams * NW * 32, 1)
    k_fbb_tma(const float* __restrict__ a_f, const uint32_t* __restrict__ wt, int64_t rows, int k,
              int kspw, int n, int ksteps, int ospw, uint32_t qmagic, uint32_t kmagic, int mb,
              uint32_t* __restrict__ out_bits, uint32_t* __restrict__ out_bits2) {
  // out_bits2: paired product -- weight columns [32*NW, 64*NW) of wt are a
  // second matrix (same n) whose result goes there; each warp then runs its
  // MMAs twice on the same converted tile
  constexpr int halves = HALVES;
  extern __shared__ __align__(16) uint8_t fbb_smem[];
  __shared__ __align__(8) uint64_t full[kFbbStages];
  const int kpad = 32 * ksteps;
  const int lda = kpad + 16;  // bytes; (lda/4) % 32 == 28 -> conflict-free fragments
  const int TR = 16 * mb;  // rows per tile: mb m16 blocks (small K: several, so per-tile costs amortize)
  const uint32_t tile_bytes = static_cast<uint32_t>(TR * k) * 4u;
  float* ring = reinterpret_cast<float*>(fbb_smem);                                  // stages x TR x k fp32
  uint8_t* a8 = fbb_smem + static_cast<size_t>(kFbbStages) * tile_bytes;            // teams x TR x lda
  uint8_t* w8 = a8 + static_cast<size_t>(kFbbTeams) * TR * lda;                     // halves*32*NW x lda
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int team = warp / NW, wq = warp % NW, ttid = tid - team * NW * 32;
  const int g = lane >> 2, t4 = lane & 3;
  // weights as +-1 bytes (0 past K and for columns >= n): 4 weight bits ->
  // 4 bytes by spreading the nibble and mapping 1 -> 0x01, 0 -> 0xFF
  for (int o = warp; o < 32 * NW * halves; o += blockDim.x >> 5)
    for (int p4 = 4 * lane; p4 < kpad; p4 += 128) {
      uint32_t v = 0;
      if ((o & (32 * NW - 1)) < n && p4 < k) {
        const uint32_t word = __ldg(wt + static_cast<int64_t>(o) * kspw + (p4 >> 5));
        const uint32_t nib = (word >> (28 - (p4 & 31))) & 0xFu;  // bit 3 <-> element p4
        const uint32_t spread = ((nib >> 3) & 1u) | (((nib >> 2) & 1u) << 8) | (((nib >> 1) & 1u) << 16) |
                                ((nib & 1u) << 24);
        v = 0xFFFFFFFFu - 0xFEu * spread;
        if (p4 + 4 > k) v &= 0xFFFFFFFFu >> (8 * (p4 + 4 - k));
      }
      *reinterpret_cast<uint32_t*>(w8 + o * lda + p4) = v;
    }
  // the activation tiles' padding columns [K, kpad) stay zero
  for (int t = tid; t < kFbbTeams * TR * (lda / 4); t += blockDim.x) reinterpret_cast<uint32_t*>(a8)[t] = 0u;
  // TR-row tiles; a partial last tile (rows % TR) is converted straight from
  // global memory (a bulk copy must be a multiple of 16 bytes and must not
  // read past the operand).  It is the last tile of its CTA, so skipping its
  // copy leaves no later use of that ring slot out of phase.
  const int64_t tiles = (rows + TR - 1) / TR, full_tiles = rows / TR;
  const int64_t my = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (tid == 0) {
    for (int s = 0; s < kFbbStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int64_t j = 0; j < kFbbStages && j < my; ++j) {
      const int64_t tile = blockIdx.x + j * gridDim.x;
      if (tile >= full_tiles) break;
      mbar_expect_tx(&full[j], tile_bytes);
      bulk_g2s(ring + j * (tile_bytes / 4), a_f + tile * TR * static_cast<int64_t>(k), tile_bytes, &full[j]);
    }
  }
  __syncthreads();
  uint8_t* mine = a8 + team * TR * lda;
  const int nthr = NW * 32;
  const uint32_t q = (k + 7) / 8, items = TR * q;  // 8-column groups per row, per tile
  const bool keven = (k & 1) == 0;
  for (int64_t j = team; j < my; j += kFbbTeams) {
    const int slot = static_cast<int>(j % kFbbStages);
    const int64_t tile = blockIdx.x + j * gridDim.x;
    const bool partial = tile >= full_tiles;
    if (!partial) mbar_wait(&full[slot], static_cast<uint32_t>(j / kFbbStages) & 1u);
    // fp32 -> +-1 bytes (x >= 0 -> +1, bitdense.cpp:83).  Item t = (row r,
    // 8-column group) with r = t / q (magic multiply); groups past K are
    // never written (zeroed once above); the last group of a row is masked.
    if (!partial && keven)
      fbb_convert4(ring + static_cast<size_t>(slot) * (tile_bytes / 4), TR, k, kmagic, ttid, nthr, lda, mine);
    else if (!partial)
      fbb_convert<false>(ring + static_cast<size_t>(slot) * (tile_bytes / 4), TR, k, keven, items, q, qmagic,
                         ttid, nthr, lda, mine);
    else
      fbb_convert<true>(a_f + tile * TR * static_cast<int64_t>(k), static_cast<int>(rows - tile * TR), k, keven,
                        items, q, qmagic, ttid, nthr, lda, mine);
    asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(nthr) : "memory");
    const int64_t nt = blockIdx.x + (j + kFbbStages) * gridDim.x;
    if (ttid == 0 && j + kFbbStages < my && nt < full_tiles) {  // the fp32 slot is free: refill it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&full[slot], tile_bytes);
      bulk_g2s(ring + static_cast<size_t>(slot) * (tile_bytes / 4), a_f + nt * TR * static_cast<int64_t>(k),
               tile_bytes, &full[slot]);
    }
    for (int mblk = 0; mblk < mb; ++mblk) {
    // both halves of a paired product share each A fragment load and run as
    // independent accumulator chains (twice the MMA ILP per k step)
    int acc[HALVES][4][4];
#pragma unroll
    for (int hf = 0; hf < HALVES; ++hf)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) acc[hf][jj][0] = acc[hf][jj][1] = acc[hf][jj][2] = acc[hf][jj][3] = 0;
    const uint8_t* ab = mine + (16 * mblk + g) * lda + 4 * t4;
    const uint8_t* bb0 = w8 + (32 * wq + g) * lda + 4 * t4;
    const uint8_t* bb1 = w8 + (32 * (wq + NW) + g) * lda + 4 * t4;
#pragma unroll 4
    for (int ks = 0; ks < ksteps; ++ks) {
      uint32_t a[4];
      a[0] = *reinterpret_cast<const uint32_t*>(ab + 32 * ks);
      a[1] = *reinterpret_cast<const uint32_t*>(ab + 8 * lda + 32 * ks);
      a[2] = *reinterpret_cast<const uint32_t*>(ab + 32 * ks + 16);
      a[3] = *reinterpret_cast<const uint32_t*>(ab + 8 * lda + 32 * ks + 16);
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const uint8_t* bp = bb0 + 8 * jj * lda + 32 * ks;
        mma_s8(acc[0][jj], a, *reinterpret_cast<const uint32_t*>(bp), *reinterpret_cast<const uint32_t*>(bp + 16));
      }
      if constexpr (HALVES == 2) {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const uint8_t* bp = bb1 + 8 * jj * lda + 32 * ks;
          mma_s8(acc[HALVES - 1][jj], a, *reinterpret_cast<const uint32_t*>(bp),
                 *reinterpret_cast<const uint32_t*>(bp + 16));
        }
      }
    }
#pragma unroll
    for (int half = 0; half < HALVES; ++half) {
    uint32_t* const ob = half ? out_bits2 : out_bits;
    // c0,c1: row g, columns 8jj+2t4, +1; c2,c3: row g+8; bit 31-c of word wq
    uint32_t m0 = 0, m1 = 0;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int c = 8 * jj + 2 * t4;
      const int* ac = acc[half][jj];
      if (ac[0] >= 0) m0 |= 0x80000000u >> c;
      if (ac[1] >= 0) m0 |= 0x40000000u >> c;
      if (ac[2] >= 0) m1 |= 0x80000000u >> c;
      if (ac[3] >= 0) m1 |= 0x40000000u >> c;
    }
    m0 |= __shfl_xor_sync(0xFFFFFFFFu, m0, 1);
    m0 |= __shfl_xor_sync(0xFFFFFFFFu, m0, 2);
    m1 |= __shfl_xor_sync(0xFFFFFFFFu, m1, 1);
    m1 |= __shfl_xor_sync(0xFFFFFFFFu, m1, 2);
    if (32 * wq + 32 > n) {  // columns >= n: zero weights give dot 0 -> clear
      const uint32_t keep = 32 * wq >= n ? 0u : tail_mask32(n);
      m0 &= keep;
      m1 &= keep;
    }
    const int64_t r0 = tile * TR + 16 * mblk + g;
    if (t4 == 0 && wq < ospw) {
      if (r0 < rows) ob[r0 * ospw + wq] = m0;
      if (r0 + 8 < rows) ob[(r0 + 8) * ospw + wq] = m1;
    }
    if (t4 == 1 && wq == 0)  // storage padding words of 64-bit rows
      for (int w = NW; w < ospw; ++w) {
        if (r0 < rows) ob[r0 * ospw + w] = 0u;
        if (r0 + 8 < rows) ob[(r0 + 8) * ospw + w] = 0u;
      }
    }  // half
    }  // m16 block
    asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(nthr) : "memory");  // int8 tile reusable
  }
}

// ---- FBB on the 5th-generation tensor cores (tcgen05.mma.kind::i8) -------------
// A persistent CTA per SM walks 128-row tiles of X.  All warps convert the
// tile's fp32 rows to +-1 bytes (x >= 0 -> +1, bitdense.cpp:83) straight from
// global memory into shared memory in the canonical no-swizzle K-major UMMA
// layout -- element (r, k) at (k/16)*128*16 + r*16 + k%16, i.e. 8x16-byte core
// matrices, SBO = 128 B between 8-row groups, LBO = 2 KB between 16-byte K
// chunks.  One thread then issues ceil(K/32) tcgen05.mma.kind::i8 (M = N =
// 128, s8 x s8 -> s32) into a TMEM accumulator and commits to an mbarrier;
// warps 0-3 read the accumulator back with tcgen05.ld.32x32b.x32 -- thread =
// output row, 32 columns per load -- and pack dot >= 0 into one output word
// per load (kernels.cpp:166-171).  The weights (N <= 128 columns) are +-1
// bytes in the same layout for the whole kernel; the tensor core reads both
// operands from shared memory once per 128 rows.
constexpr int kUmmaM = 128, kUmmaN = 128;

// mbarrier wait that traps (a launch error) instead of hanging if the phase
// never completes -- a malformed MMA would otherwise wedge the GPU.
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  for (uint32_t it = 0; it < (1u << 24) && !ok; ++it)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  if (!ok) __trap();
}
constexpr int kUmmaThreads = 512;

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
  return d;                             // base offset 0, layout SWIZZLE_NONE (0)
}

// kind::i8 instruction descriptor: D s32, A/B signed 8-bit, K-major, N = 128, M = 128.
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((kUmmaN >> 3) << 17) | ((kUmmaM >> 4) << 24);

__device__ __forceinline__ void umma_epilogue(uint32_t tmem_acc, int warp, int lane, int64_t row0, int valid,
                                              int n, int ospw, uint32_t* __restrict__ out_bits) {
  const int r = 32 * warp + lane;
  uint32_t words[4];
#pragma unroll
  for (int cw = 0; cw < 4; ++cw) {
    uint32_t d[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
          "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]),
          "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]),
          "=r"(d[23]), "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]),
          "=r"(d[30]), "=r"(d[31])
        : "r"(tmem_acc + (static_cast<uint32_t>(32 * warp) << 16) + 32u * cw));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) m |= (static_cast<int32_t>(d[j]) >= 0 ? 1u : 0u) << (31 - j);
    if (32 * cw + 32 > n) m &= 32 * cw >= n ? 0u : tail_mask32(n);
    words[cw] = m;
  }
  if (r < valid) {
    uint32_t* o = out_bits + (row0 + r) * ospw;
    for (int w = 0; w < ospw; ++w) o[w] = w < 4 ? words[w] : 0u;
  }
}

__global__ void __launch_bounds__(kUmmaThreads, 1)
    k_fbb_umma(const float* __restrict__ a_f, const uint32_t* __restrict__ wt, int64_t rows, int k, int kspw,
               int n, int ksteps, int ospw, uint32_t qmagic, uint32_t* __restrict__ out_bits) {
  extern __shared__ __align__(1024) uint8_t um_smem[];
  __shared__ __align__(8) uint64_t mma_done;
  __shared__ uint32_t tmem_base;
  const int kpad = 32 * ksteps;
  const int chunk = kUmmaM * 16;            // bytes per 16-byte K chunk of a 128-row operand
  uint8_t* A = um_smem;                     // kpad/16 chunks x 128 rows x 16 B
  uint8_t* Bw = um_smem + kpad * kUmmaM;    // same layout, 128 output columns
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // weights: column o, element kk -> +-1 byte at (kk/16)*chunk + o*16 + kk%16 (0 past K / n)
  for (int t = tid; t < kUmmaN * (kpad / 4); t += blockDim.x) {
    const int o = t / (kpad / 4), p4 = (t % (kpad / 4)) * 4;
    uint32_t v = 0;
    if (o < n && p4 < k) {
      const uint32_t word = __ldg(wt + static_cast<int64_t>(o) * kspw + (p4 >> 5));
      const uint32_t nib = (word >> (28 - (p4 & 31))) & 0xFu;
      const uint32_t spread = ((nib >> 3) & 1u) | (((nib >> 2) & 1u) << 8) | (((nib >> 1) & 1u) << 16) | ((nib & 1u) << 24);
      v = 0xFFFFFFFFu - 0xFEu * spread;
      if (p4 + 4 > k) v &= 0xFFFFFFFFu >> (8 * (p4 + 4 - k));
    }
    *reinterpret_cast<uint32_t*>(Bw + (p4 >> 4) * chunk + o * 16 + (p4 & 15)) = v;
  }
  // zero the A columns [8*ceil(K/8), kpad) once; the conversion never writes them
  for (int t = tid; t < kUmmaM * (kpad / 4); t += blockDim.x) {
    const int r = t / (kpad / 4), p4 = (t % (kpad / 4)) * 4;
    if (p4 >= (k + 7) / 8 * 8) *reinterpret_cast<uint32_t*>(A + (p4 >> 4) * chunk + r * 16 + (p4 & 15)) = 0u;
  }
  if (warp == 0) {  // TMEM: 128 lanes x 128 s32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_base)),
                 "r"(kUmmaN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(&mma_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // weights visible to the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t q = (k + 7) / 8, items = kUmmaM * q;
  const bool keven = (k & 1) == 0;
  const int64_t tiles = (rows + kUmmaM - 1) / kUmmaM;
  uint32_t phase = 0;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, phase ^= 1u) {
    const int64_t row0 = tile * kUmmaM;
    const int valid = static_cast<int>(rows - row0 < kUmmaM ? rows - row0 : kUmmaM);
    const float* src = a_f + row0 * static_cast<int64_t>(k);
    // fp32 -> +-1 bytes, item t = (row r, 8-column group): coalesced 8-byte
    // loads along a row, four items per thread in flight (all loads first;
    // rows past the operand are clamped for the load and zeroed after)
    for (uint32_t t0 = tid; t0 < items; t0 += 4 * blockDim.x) {
      uint32_t rr[4], cc[4];
      float2 ld[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t t = min(t0 + u * blockDim.x, items - 1);
        rr[u] = __umulhi(t, qmagic);
        cc[u] = 8 * (t - rr[u] * q);
        const uint32_t rl = min(rr[u], static_cast<uint32_t>(valid - 1));
        const float* x = src + static_cast<int64_t>(rl) * k + cc[u];
        const int lim = k - static_cast<int>(cc[u]);
        if (keven) {
#pragma unroll
          for (int h = 0; h < 4; ++h)
            ld[u][h] = 2 * h < lim ? __ldg(reinterpret_cast<const float2*>(x) + h) : make_float2(0.0f, 0.0f);
        } else {
#pragma unroll
          for (int h = 0; h < 4; ++h)
            ld[u][h] = make_float2(2 * h < lim ? __ldg(x + 2 * h) : 0.0f, 2 * h + 1 < lim ? __ldg(x + 2 * h + 1) : 0.0f);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t t = t0 + u * blockDim.x;
        if (t >= items) break;
        uint2 v = make_uint2(0u, 0u);
        if (static_cast<int>(rr[u]) < valid) {
          v.x = sign_bytes4(ld[u][0].x, ld[u][0].y, ld[u][1].x, ld[u][1].y);
          v.y = sign_bytes4(ld[u][2].x, ld[u][2].y, ld[u][3].x, ld[u][3].y);
          if (cc[u] + 8 > static_cast<uint32_t>(k)) {
            const int rem = k - static_cast<int>(cc[u]);
            v.x &= rem >= 4 ? 0xFFFFFFFFu : 0xFFFFFFFFu >> (8 * (4 - rem));
            v.y &= rem <= 4 ? 0u : 0xFFFFFFFFu >> (8 * (8 - rem));
          }
        }
        *reinterpret_cast<uint2*>(A + (cc[u] >> 4) * chunk + rr[u] * 16 + (cc[u] & 15)) = v;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t abase = smem_addr(A), bbase = smem_addr(Bw);
      for (int ks = 0; ks < ksteps; ++ks) {
        const uint64_t ad = umma_desc(abase + 2 * ks * chunk, chunk, 128);
        const uint64_t bd = umma_desc(bbase + 2 * ks * chunk, chunk, 128);
        const uint32_t acc = ks > 0 ? 1u : 0u;
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(kIdescI8), "r"(acc)
            : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_addr(&mma_done))
                   : "memory");
    }
    mbar_wait_bounded(&mma_done, phase);  // MMAs done: A may be overwritten, TMEM holds the tile
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4) umma_epilogue(tmem, warp, lane, row0, valid, n, ospw, out_bits);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // TMEM read back before the next tile's MMAs
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kUmmaN) : "memory");
}

// TMA-fed variant: the fp32 rows arrive by bulk copies of 8-row sub-tiles
// (contiguous, 16-byte multiples) into a 3-slot ring; team t of three
// converts sub-tiles u = t (mod 3) -- slot t is only ever consumed and
// refilled by team t, so its mbarrier phases are waited in order -- into the
// 128-row A tile; after a tile's 16 sub-tiles one thread issues the MMAs and
// warps 0-3 read the accumulator back.  Shared memory: weights + A + ring =
// 2*128*kpad + 3*8*K*4 bytes (213 KB at K = 602).
constexpr int kU2Teams = 3;

__global__ void __launch_bounds__(kU2Teams * 128, 1)
    k_fbb_umma2(const float* __restrict__ a_f, const uint32_t* __restrict__ wt, int64_t rows, int k, int kspw,
                int n, int ksteps, int ospw, uint32_t qmagic, int sr, uint32_t* __restrict__ out_bits) {
  extern __shared__ __align__(1024) uint8_t u2_smem[];
  const int kU2Sub = sr;  // rows per sub-tile: 8..128, divides 128
  __shared__ __align__(8) uint64_t full[kU2Teams], mma_done;
  __shared__ uint32_t tmem_base;
  const int kpad = 32 * ksteps;
  const int chunk = kUmmaM * 16;
  uint8_t* Bw = u2_smem;
  uint8_t* A = u2_smem + kpad * kUmmaN;
  float* ring = reinterpret_cast<float*>(u2_smem + 2 * kpad * kUmmaM);
  const uint32_t slot_bytes = static_cast<uint32_t>(kU2Sub * k) * 4u;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int team = warp / 4, ttid = tid - team * 128;
  for (int t = tid; t < kUmmaN * (kpad / 4); t += blockDim.x) {
    const int o = t / (kpad / 4), p4 = (t % (kpad / 4)) * 4;
    uint32_t v = 0;
    if (o < n && p4 < k) {
      const uint32_t word = __ldg(wt + static_cast<int64_t>(o) * kspw + (p4 >> 5));
      const uint32_t nib = (word >> (28 - (p4 & 31))) & 0xFu;
      const uint32_t spread = ((nib >> 3) & 1u) | (((nib >> 2) & 1u) << 8) | (((nib >> 1) & 1u) << 16) | ((nib & 1u) << 24);
      v = 0xFFFFFFFFu - 0xFEu * spread;
      if (p4 + 4 > k) v &= 0xFFFFFFFFu >> (8 * (p4 + 4 - k));
    }
    *reinterpret_cast<uint32_t*>(Bw + (p4 >> 4) * chunk + o * 16 + (p4 & 15)) = v;
  }
  for (int t = tid; t < kUmmaM * (kpad / 4); t += blockDim.x) {  // A columns past 8*ceil(K/8) stay zero
    const int r = t / (kpad / 4), p4 = (t % (kpad / 4)) * 4;
    if (p4 >= (k + 7) / 8 * 8) *reinterpret_cast<uint32_t*>(A + (p4 >> 4) * chunk + r * 16 + (p4 & 15)) = 0u;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_base)),
                 "r"(kUmmaN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  const int64_t tiles = (rows + kUmmaM - 1) / kUmmaM;
  const int64_t my = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nsub = my * (kUmmaM / kU2Sub);
  // sub-tile u of this CTA: tile blockIdx.x + (u/16)*grid, rows +8*(u%16); rows past the operand -> no copy
  // full sub-tiles arrive by bulk copy; a partial one (rows % sr) is read
  // straight from global memory (a copy must be a 16-byte multiple and must
  // not read past the operand), so its slot only gets a plain arrive
  auto sub_rows = [&](int64_t u, int64_t* r0) {
    const int64_t tile = blockIdx.x + (u / (kUmmaM / kU2Sub)) * gridDim.x;
    *r0 = tile * kUmmaM + kU2Sub * (u % (kUmmaM / kU2Sub));
    const int64_t left = rows - *r0;
    return static_cast<int>(left <= 0 ? 0 : left < kU2Sub ? left : kU2Sub);
  };
  auto issue = [&](int64_t u) {
    int64_t r0;
    const int nr = sub_rows(u, &r0);
    uint64_t* bar = &full[u % kU2Teams];
    if (nr == kU2Sub) {
      const uint32_t bytes = static_cast<uint32_t>(nr * k) * 4u;
      mbar_expect_tx(bar, bytes);
      bulk_g2s(ring + (u % kU2Teams) * (slot_bytes / 4), a_f + r0 * static_cast<int64_t>(k), bytes, bar);
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
    }
  };
  if (tid == 0) {
    for (int t = 0; t < kU2Teams; ++t) mbar_init(&full[t], 1);
    mbar_init(&mma_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int64_t u = 0; u < kU2Teams && u < nsub; ++u) issue(u);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t q = (k + 7) / 8, items = static_cast<uint32_t>(kU2Sub) * q;
  const bool keven = (k & 1) == 0;
  for (int64_t ti = 0; ti < my; ++ti) {
    const int64_t row0 = (blockIdx.x + ti * gridDim.x) * kUmmaM;
    const int valid = static_cast<int>(rows - row0 < kUmmaM ? rows - row0 : kUmmaM);
    // this team's sub-tiles of tile ti
    for (int64_t u = ti * (kUmmaM / kU2Sub); u < (ti + 1) * (kUmmaM / kU2Sub); ++u) {
      if (u % kU2Teams != team) continue;
      mbar_wait_bounded(&full[team], static_cast<uint32_t>(u / kU2Teams) & 1u);
      int64_t r0;
      const int nr = sub_rows(u, &r0);
      const int rbase = static_cast<int>(kU2Sub * (u % (kUmmaM / kU2Sub)));
      const float* src = nr == kU2Sub ? ring + team * (slot_bytes / 4) : a_f + r0 * static_cast<int64_t>(k);
      for (uint32_t t = ttid; t < items; t += 128) {
        const uint32_t r = __umulhi(t, qmagic);
        const uint32_t c = 8 * (t - r * q);
        uint2 v = make_uint2(0u, 0u);
        if (static_cast<int>(r) < nr) {
          const float* x = src + r * k + c;
          float e[8];
          if (keven && c + 8 <= static_cast<uint32_t>(k)) {
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const float2 p2 = *reinterpret_cast<const float2*>(x + 2 * h);
              e[2 * h] = p2.x;
              e[2 * h + 1] = p2.y;
            }
          } else {
#pragma unroll
            for (int h = 0; h < 8; ++h) e[h] = c + h < static_cast<uint32_t>(k) ? x[h] : 0.0f;
          }
          v.x = sign_bytes4(e[0], e[1], e[2], e[3]);
          v.y = sign_bytes4(e[4], e[5], e[6], e[7]);
          if (c + 8 > static_cast<uint32_t>(k)) {
            const int rem = k - static_cast<int>(c);
            v.x &= rem >= 4 ? 0xFFFFFFFFu : 0xFFFFFFFFu >> (8 * (4 - rem));
            v.y &= rem <= 4 ? 0u : 0xFFFFFFFFu >> (8 * (8 - rem));
          }
        }
        *reinterpret_cast<uint2*>(A + (c >> 4) * chunk + (rbase + r) * 16 + (c & 15)) = v;
      }
      asm volatile("bar.sync %0, 128;" ::"r"(1 + team) : "memory");  // the team is done with its slot
      if (ttid == 0 && u + kU2Teams < nsub) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(u + kU2Teams);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // A (generic writes) -> tensor core
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t abase = smem_addr(A), bbase = smem_addr(Bw);
      for (int ks = 0; ks < ksteps; ++ks) {
        const uint64_t ad = umma_desc(abase + 2 * ks * chunk, chunk, 128);
        const uint64_t bd = umma_desc(bbase + 2 * ks * chunk, chunk, 128);
        const uint32_t acc = ks > 0 ? 1u : 0u;
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(kIdescI8), "r"(acc)
            : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_addr(&mma_done))
                   : "memory");
    }
    mbar_wait_bounded(&mma_done, static_cast<uint32_t>(ti & 1));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4) umma_epilogue(tmem, warp, lane, row0, valid, n, ospw, out_bits);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kUmmaN) : "memory");
}

bool fbb_umma2(const BmmArgs& a, cudaStream_t s) {
  if (a.a_f == nullptr || a.out_bits == nullptr || a.n > kUmmaN || a.k <= 8) return false;
  if (reinterpret_cast<uintptr_t>(a.a_f) % 16 != 0) return false;
  const char* e = std::getenv("BG_FBB");  // opt-in: measured 0.246 ms on Reddit vs 0.158 ms default
  if (!e || std::string(e) != "umma2") return false;
  const int ksteps = static_cast<int>(cdiv(a.k, 32));
  // rows per fp32 sub-tile: the largest of 128, 64, ..., 8 whose 3 ring slots fit
  const size_t ab = static_cast<size_t>(2) * kUmmaM * 32 * ksteps;
  int sr = 128;
  while (sr > 8 && ab + static_cast<size_t>(kU2Teams) * sr * a.k * 4 > 226 * 1024) sr /= 2;
  const size_t smem = ab + static_cast<size_t>(kU2Teams) * sr * a.k * 4;
  if (smem > 226 * 1024) return false;
  const int kspw = static_cast<int>(spw(a.k, a.wb));
  const int ospw = static_cast<int>(spw(a.n, a.wb));
  const uint32_t q = static_cast<uint32_t>((a.k + 7) / 8);
  if (q > 5792) return false;  // t / q == umulhi(t, ceil(2^32/q)) for t < 128 q: error 128 q^2 < 2^32
  const uint32_t qmagic = static_cast<uint32_t>(((uint64_t{1} << 32) + q - 1) / q);
  static bool attr = false;
  if (!attr) {
    BG_CUDA(cudaFuncSetAttribute(k_fbb_umma2, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
    attr = true;
  }
  const int64_t tiles = (a.rows + kUmmaM - 1) / kUmmaM;
  const int64_t blocks = std::min<int64_t>(tiles, sm_count());
  k_fbb_umma2<<<static_cast<unsigned>(blocks), kU2Teams * 128, smem, s>>>(
      a.a_f, a.wt, a.rows, static_cast<int>(a.k), kspw, static_cast<int>(a.n), ksteps, ospw, qmagic, sr,
      a.out_bits);
  BG_LAUNCH_CHECK();
  return true;
}

// FBB through k_fbb_umma (opt-in: BG_FBB=umma); false when not selected or
// not eligible.  Measured on Reddit (FBB 564.7 MB): 0.175 ms against 0.158 ms
// for the TMA-fed mma.sync kernel -- the tensor core is idle >90% either way;
// what differs is how the fp32 stream reaches shared memory (here 8-byte LDGs,
// there one bulk copy per 16-row tile), and a TMA-fed variant of this kernel
// does not fit: 3 fp32 stages + the 128-row A tile + the weights exceed 227 KB.
bool fbb_umma(const BmmArgs& a, cudaStream_t s) {
  if (a.a_f == nullptr || a.out_bits == nullptr || a.n > kUmmaN || a.k <= 8) return false;
  const char* e = std::getenv("BG_FBB");
  if (!e || std::string(e) != "umma") return false;
  const int ksteps = static_cast<int>(cdiv(a.k, 32));
  const size_t smem = static_cast<size_t>(2) * kUmmaM * 32 * ksteps;
  if (smem > 200 * 1024) return false;
  const int kspw = static_cast<int>(spw(a.k, a.wb));
  const int ospw = static_cast<int>(spw(a.n, a.wb));
  const uint32_t q = static_cast<uint32_t>((a.k + 7) / 8);
  if (q > 5792) return false;  // t / q == umulhi(t, ceil(2^32/q)) for t < 128 q: error 128 q^2 < 2^32
  const uint32_t qmagic = static_cast<uint32_t>(((uint64_t{1} << 32) + q - 1) / q);
  static bool attr = false;
  if (!attr) {
    BG_CUDA(cudaFuncSetAttribute(k_fbb_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  const int64_t tiles = (a.rows + kUmmaM - 1) / kUmmaM;
  const int64_t blocks = std::min<int64_t>(tiles, sm_count());
  k_fbb_umma<<<static_cast<unsigned>(blocks), kUmmaThreads, smem, s>>>(
      a.a_f, a.wt, a.rows, static_cast<int>(a.k), kspw, static_cast<int>(a.n), ksteps, ospw, qmagic, a.out_bits);
  BG_LAUNCH_CHECK();
  return true;
}

// FBB through k_fbb_tma (all rows; 0 = not eligible, use the direct kernel).
int64_t fbb_tma(const BmmArgs& a, cudaStream_t s) {
  if (a.a_f == nullptr || a.out_bits == nullptr || a.n > 128 || a.k <= 8 || std::getenv("BG_BMM_POPC")) return 0;
  if (reinterpret_cast<uintptr_t>(a.a_f) % 16 != 0) return 0;
  const int ksteps = static_cast<int>(cdiv(a.k, 32));
  const int lda = 32 * ksteps + 16;
  const int nw = static_cast<int>(cdiv(a.n, 32));
  const int NW = nw <= 1 ? 1 : nw <= 2 ? 2 : 4;
  const int halves = a.out_bits2 ? 2 : 1;
  // a paired product needs W2 to start at word NW of the combined weights
  if (a.out_bits2 && (a.n2 != a.n || NW != nw)) return 0;
  // m16 blocks per tile: a slot of at most 16 x 602 fp32 (the Reddit tile),
  // so small K batches several blocks per bulk copy and per barrier
  int mb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8, 38528 / (64 * a.k))));
  auto smem_of = [&](int m) {
    return static_cast<size_t>(kFbbStages) * 16 * m * a.k * 4 + static_cast<size_t>(kFbbTeams) * 16 * m * lda +
           static_cast<size_t>(32 * NW * halves) * lda;
  };
  while (mb > 1 && smem_of(mb) > 227 * 1024 - 128) --mb;
  const size_t smem = smem_of(mb);
  if (smem > 227 * 1024 - 128) return 0;  // opt-in shared memory per block, less the static part
  const int64_t tiles = (a.rows + 16 * mb - 1) / (16 * mb);
  const int kspw = static_cast<int>(spw(a.k, a.wb));
  const int ospw = static_cast<int>(spw(a.n, a.wb));
  // t / q == umulhi(t, ceil(2^32 / q)) for t < 16 mb q: the error term t*(M*q - 2^32) < 128 q^2 < 2^32
  const uint32_t q = static_cast<uint32_t>((a.k + 7) / 8);
  const uint32_t qmagic = static_cast<uint32_t>(((uint64_t{1} << 32) + q - 1) / q);
  // f / k == umulhi(f, ceil(2^32 / k)) for flat tile offsets f < 16 mb k (f k < 2^32)
  const uint32_t kmagic = static_cast<uint32_t>(((uint64_t{1} << 32) + a.k - 1) / a.k);
  auto go = [&](auto kern) {
    BG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    const int64_t blocks = std::min<int64_t>(tiles, sm_count());
    kern<<<static_cast<unsigned>(blocks), kFbbTeams * NW * 32, smem, s>>>(
        a.a_f, a.wt, a.rows, static_cast<int>(a.k), kspw, static_cast<int>(a.n), ksteps, ospw, qmagic, kmagic, mb,
        a.out_bits, a.out_bits2);
  };
  if (halves == 2) {
    if (NW == 1) go(k_fbb_tma<1, 2>);
    else if (NW == 2) go(k_fbb_tma<2, 2>);
    else go(k_fbb_tma<4, 2>);
  } else {
    if (NW == 1) go(k_fbb_tma<1, 1>);
    else if (NW == 2) go(k_fbb_tma<2, 1>);
    else go(k_fbb_tma<4, 1>);
  }
  BG_LAUNCH_CHECK();
  return a.rows;
}

bool imma_ok(const BmmArgs& a) {
  return a.a_f != nullptr && a.n <= 128 && a.k <= 8192 && std::getenv("BG_BMM_POPC") == nullptr;
}

template <bool OUTB>
void launch_imma(const BmmArgs& a, cudaStream_t s) {
  const int ksteps = static_cast<int>(cdiv(a.k, 32));
  const int ldw = 32 * ksteps + 16;  // bytes; stride/4 = 8*ksteps + 4 -> conflict-free fragments
  const int kspw = static_cast<int>(spw(a.k, a.wb));
  const int ospw = static_cast<int>(spw(a.n, a.wb));
  const int nt = static_cast<int>(cdiv(a.n, 8));
  auto go = [&](auto kern, int NT) {
    const size_t smem = static_cast<size_t>(8 * NT) * ldw;
    BG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 0;
    BG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kImWarps * 32, smem));
    const int64_t blocks = std::max<int64_t>(
        1, std::min<int64_t>(cdiv(a.rows, 16 * kImWarps), static_cast<int64_t>(sm_count()) * std::max(per_sm, 1)));
    kern<<<static_cast<unsigned>(blocks), kImWarps * 32, smem, s>>>(
        a.a_f, a.alpha, a.wt, a.beta, a.rows, static_cast<int>(a.k), kspw, static_cast<int>(a.n), ksteps, ldw,
        ospw, a.out_bits, a.out_f);
  };
  if (nt <= 2) go(k_bmm_imma<OUTB, 2>, 2);
  else if (nt <= 4) go(k_bmm_imma<OUTB, 4>, 4);
  else if (nt <= 8) go(k_bmm_imma<OUTB, 8>, 8);
  else go(k_bmm_imma<OUTB, 16>, 16);
  BG_LAUNCH_CHECK();
}

// Row-per-lane B-output path: word count small enough for registers and the
// weight table for shared memory.
bool lanerow_ok(const BmmArgs& a) {
  const int64_t kspw = spw(a.k, a.wb);
  const int64_t npad = cdiv(a.n, 32) * 32;
  const size_t smem = static_cast<size_t>(kspw * npad + kLrWarps * 32 * (kspw | 1)) * 4;
  return a.out_bits != nullptr && kspw <= 32 && smem <= 160 * 1024 && std::getenv("BG_BMM_WARPROW") == nullptr;
}

template <bool AF>
void launch_lanerow(const BmmArgs& a, cudaStream_t s) {
  const int kspw = static_cast<int>(spw(a.k, a.wb));
  const int npad = static_cast<int>(cdiv(a.n, 32) * 32);
  const int ospw = static_cast<int>(spw(a.n, a.wb));
  const size_t smem = static_cast<size_t>(kspw * npad + kLrWarps * 32 * (kspw | 1)) * 4;
  const int64_t blocks = std::max<int64_t>(
      1, std::min<int64_t>(cdiv(a.rows, kLrWarps * 32), static_cast<int64_t>(sm_count()) * 4));
  auto go = [&](auto kern) {
    if (smem > 48 * 1024)
      BG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<static_cast<unsigned>(blocks), kLrWarps * 32, smem, s>>>(
        a.a_bits, a.a_f, a.wt, a.rows, static_cast<int>(a.k), kspw, static_cast<int>(a.n), npad, ospw,
        a.out_bits);
  };
  if (kspw <= 4) go(k_bmm_lanerow<AF, 4>);
  else if (kspw <= 8) go(k_bmm_lanerow<AF, 8>);
  else if (kspw <= 16) go(k_bmm_lanerow<AF, 16>);
  else if (kspw <= 20) go(k_bmm_lanerow<AF, 20>);
  else go(k_bmm_lanerow<AF, 32>);
  BG_LAUNCH_CHECK();
}

template <bool AF, bool OUTB>
void launch(const BmmArgs& a, cudaStream_t s) {
  // F->B products may take 512 columns per pass (a paired product of two
  // 256-column weights reads its input once)
  constexpr bool wide = AF && OUTB;
  auto pick = [](int64_t nc) {
    return nc <= 32 ? k_bmm<AF, OUTB, 1> : nc <= 64 ? k_bmm<AF, OUTB, 2>
         : nc <= 128 ? k_bmm<AF, OUTB, 4> : nc <= 256 || !wide ? k_bmm<AF, OUTB, 8> : k_bmm<AF, OUTB, wide ? 16 : 8>;
  };
  const int64_t kspw = spw(a.k, a.wb);
  const int64_t ld = kspw | 1;
  const int64_t ospw = spw(a.n, a.wb);
  const int64_t ntot = a.out_bits2 ? 32 * cdiv(a.n, 32) + a.n2 : a.n;  // combined columns
  const int64_t pass = 32 * (wide ? 2 * kMaxOutPerLane : kMaxOutPerLane);
  int64_t blocks = std::min<int64_t>(cdiv(a.rows, kWarps), static_cast<int64_t>(sm_count()) * 8);
  blocks = std::max<int64_t>(blocks, 1);
  for (int64_t c0 = 0; c0 < ntot; c0 += pass) {
    const int64_t nc = std::min(pass, ntot - c0);
    const int64_t mcols = nc <= 32 ? 32 : nc <= 64 ? 64 : nc <= 128 ? 128 : nc <= 256 ? 256 : 512;  // 32*M of pick(nc)
    const size_t smem = static_cast<size_t>(mcols * ld + kWarps * kspw + (AF ? kWarps * (kspw + 2) : 0)) * 4;
    auto kern = pick(nc);
    if (smem > 48 * 1024) BG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      static_cast<int>(smem)));
    if (smem > 200 * 1024) fail("bmm: inner dimension too large for one pass");
    kern<<<static_cast<unsigned>(blocks), kWarps * 32, smem, s>>>(
        a.a_bits, a.a_f, a.alpha, a.wt, a.beta, a.rows, a.k, a.n, kspw, ld, c0, nc, ospw,
        a.out_bits, a.out_f, a.out_bits2, a.n2, ntot);
    BG_LAUNCH_CHECK();
  }
}

}  // namespace

// Which F-input path (tests and A/B runs: BG_FBB=scalar|imma|tma; default
// picks by shape).  0 = default, 1 = scalar warp per row, 2 = imma, 3 = tma.
int fbb_force() {
  const char* e = std::getenv("BG_FBB");
  if (!e) return 0;
  const std::string v(e);
  return v == "scalar" ? 1 : v == "imma" ? 2 : v == "tma" ? 3 : v == "tc" ? 5 : v == "bulk" ? 6 : v == "tmem" ? 7 : v == "tmem2" ? 8 : 0;
}

bool bmm_pair(const BmmArgs& a, cudaStream_t s) {
  if (!a.a_f || !a.out_bits || !a.out_bits2 || a.n2 != a.n || a.n == 0) return false;
  if (a.rows == 0) return true;
  const int force = fbb_force();
  const bool few_rows = a.rows < 24576 && std::getenv("BG_FBB") == nullptr;  // as bmm()
  if (force == 6 && fbb_bulk(a, s)) return true;
  if (force == 7 && fbb_tmem(a, s)) return true;
  if (force == 8 && fbb_tmem(a, s, true)) return true;
  // a wide-K pair (Flickr's SAGE layer: K = 500, 2 x 256 columns) as two MMA
  // rounds per tile of the 2-CTA tcgen05 kernel: the input is read once
  if (force == 0 && a.k >= 256 && a.rows >= 8192 && a.n >= 64 && !std::getenv("BG_TMEM_NOPAIR") &&
      fbb_tmem(a, s, true))
    return true;
  if (force == 1 || few_rows) {
    // warp per row: pairs up to 256 combined columns (8 per lane); wider
    // pairs measured slower than two products (Flickr, 2 x 256 columns:
    // 0.35 ms paired vs 2 x 0.154 ms)
    if (32 * cdiv(a.n, 32) + a.n2 > 32 * kMaxOutPerLane) return false;
    launch<true, true>(a, s);
    return true;
  }
  if ((force == 0 || force == 5) && fbb_tc(a, s)) return true;
  if (force == 0 || force == 3) return imma_ok(a) && fbb_tma(a, s) == a.rows;
  return false;  // other forced kernels take the products one at a time
}

void bmm(const BmmArgs& a, cudaStream_t s) {
  if (a.rows == 0 || a.n == 0) return;
  const bool af = a.a_f != nullptr, ob = a.out_bits != nullptr;
  const int force = af ? fbb_force() : 0;
  // Few rows (Cora 2.7K, PubMed 20K): a warp per row puts every row in
  // flight at once, where the tile kernel leaves SMs idle or runs short
  // pipelines (measured FBB: Cora 66 -> 20 us, PubMed 28 -> 26 us).  From
  // ~25K rows the TMA kernel wins (K = 602, scripts/fbb_rows_probe.py: 29K
  // rows -- a Reddit shard of 8 -- 81 vs 99 us; 233K rows 0.14 vs 0.30 ms);
  // N > 128 (Flickr's 256 columns, 89K rows: 154 vs 169 us on the lane-per-
  // row kernel) stays on the warp-per-row kernel at any row count.
  // F output keeps the tensor-core kernel (Flickr FBF 63 vs 83 us).
  const bool few_rows = af && ob && (a.rows < 24576 || a.n > 128) && std::getenv("BG_FBB") == nullptr;
  // The tcgen05 kernel with A in tensor memory (fbb_tmem.cu), as 2-CTA
  // clusters (cta_group::2: each CTA holds half the weights, four ring
  // slots): Flickr's 256-column products 0.139 -> 0.055 ms, Reddit 0.136 ->
  // 0.12 ms; below ~100K rows at N <= 128 the TMA-fed mma.sync kernel is as
  // fast or faster (scripts/fbb_rows_probe.py) and keeps those shapes
  if (force == 0 && af && ob && a.n >= 64 && a.rows >= (a.n > 128 ? 8192 : 98304) && fbb_tmem(a, s, true)) return;
  if (((force == 0 && af && a.n > 128 && a.rows >= 16384) || force == 7) && ob && fbb_tmem(a, s)) return;
  if (force == 8 && ob && fbb_tmem(a, s, true)) return;
  // opt-in (BG_FBB=bulk): every row requested at once by bulk copies
  // (fbb_bulk.cu); measured slower than the warp-per-row kernel on Cora and
  // PubMed (DESIGN 4.3)
  if (force == 6 && fbb_bulk(a, s)) return;
  if (force == 1 || few_rows) {
    if (ob) launch<true, true>(a, s);
    else launch<true, false>(a, s);
    return;
  }
  if (imma_ok(a)) {
    if (ob) {
      // the warp-specialized tcgen05 kernel (fbb_tc.cu); else whole 16-row
      // tiles on the TMA-fed mma.sync kernel, the rest on the direct one
      if ((force == 0 || force == 5) && fbb_tc(a, s)) return;
      if (fbb_umma(a, s)) return;
      if (fbb_umma2(a, s)) return;
      const int64_t done = force == 2 ? 0 : fbb_tma(a, s);
      if (done < a.rows) {
        BmmArgs rest = a;
        rest.rows = a.rows - done;
        rest.a_f = a.a_f + done * a.k;
        rest.alpha = a.alpha ? a.alpha + done : nullptr;
        rest.out_bits = a.out_bits + done * spw(a.n, a.wb);
        launch_imma<true>(rest, s);
      }
    } else {
      launch_imma<false>(a, s);
    }
    return;
  }
  if (lanerow_ok(a)) {
    if (af) launch_lanerow<true>(a, s);
    else launch_lanerow<false>(a, s);
    return;
  }
  if (af && ob) launch<true, true>(a, s);
  else if (af) launch<true, false>(a, s);
  else if (ob) launch<false, true>(a, s);
  else launch<false, false>(a, s);
}

}  // namespace bg
