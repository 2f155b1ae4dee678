// Aggregation kernels over the node-major sliver view of the FRDC bit tiles
// (ops.cuh bg_frdc::slivers): one warp per node row reads its nonzero 1x4
// nibbles with coalesced 4-byte loads -- no per-forward routing of tile bits
// to rows.  Same results as the tile-row walker kernels (bspmm.cu,
// gcn_fused.cu) and the reference (kernels.cpp:254-555).
//
//   k_sl_bb        BSpMM.BBB / BBF: lanes (word g, slot s) gather word g of the
//                  neighbour rows of 8 slivers per slot and count them with
//                  Harley-Seal planes; epilogue as in bspmm.cu.
//   k_bv_gcn1      fused layer-1 GCN (gcn_fused.cu) over the bit-entry view
//                  (one column per adjacency bit): 64-byte records laid out so
//                  every lane owns one h word and three q words -- all lanes
//                  run the same Harley-Seal + SWAR code, no divergence.
//   k_sl_f         real-valued walk in ascending column order (exact double
//                  accumulation order of the reference).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <string>

#include <cub/cub.cuh>

#include "async.cuh"
#include "ops.cuh"
#include "tilewalk.cuh"

namespace bg {
namespace {

constexpr int kSlWarps = 8;

// base + a * b with one IMAD.WIDE.U32 (gather address of node a, row stride b bytes).
__device__ __forceinline__ uint4 ld_nc_v4(const uint4* p) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t mad_wide(uint32_t a, uint32_t b, uint64_t base) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(base));
  return r;
}

template <int G, int NP, bool OUTB>
__global__ void __launch_bounds__(kSlWarps * 32)
    k_sl_bb(const uint64_t* __restrict__ srp, const uint32_t* __restrict__ sl, int64_t row0,
            int64_t row1, const int32_t* __restrict__ degree, const uint32_t* __restrict__ x,
            int64_t xspw, int64_t f, uint32_t* __restrict__ out_bits, float* __restrict__ out_f, const FEpi ep) {
  constexpr int S = 32 / G, B = 8 * S;
  constexpr int LOGS = S == 1 ? 0 : S == 2 ? 1 : S == 4 ? 2 : S == 8 ? 3 : S == 16 ? 4 : 5;
  constexpr int NQ = NP + LOGS;
  const int lane = threadIdx.x & 31;
  const int g = lane % G, slot = lane / G;
  const int64_t word = static_cast<int64_t>(blockIdx.y) * G + g;
  const bool word_ok = word < xspw;
  const uint64_t xbase = reinterpret_cast<uint64_t>(x + (word_ok ? word : 0));
  const uint32_t xsb = static_cast<uint32_t>(xspw) * 4;  // row stride in bytes
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = row0 + wid; i < row1; i += nw) {
    uint32_t P[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) P[q] = 0;
    const uint64_t e0 = srp[i];
    const uint32_t deg = static_cast<uint32_t>(__ldg(degree + i));
    // multiple of kSliverPad; hub rows are counted by hub_bb (hubs.cu)
    const uint32_t len = deg < kHubDeg ? static_cast<uint32_t>(srp[i + 1] - e0) : 0u;
    const uint32_t* rowp = sl + e0 + slot;
    for (uint32_t off = 0; off < len; off += B) {
      const uint32_t mcount = min(8u, (len - off) / S);  // warp-uniform (len % 8 == 0, S | 8)
      uint32_t ent[8], xv[8], ex = 0;
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        ent[m] = m < mcount ? ld_nc_u32(rowp + off + S * m) : kSliverSentinel;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(mad_wide(ent[m] >> 3, xsb, xbase));
        xv[m] = 0u;
        if (ent[m] != kSliverSentinel) xv[m] = __ldg(src);
        ex |= ent[m];
      }
      hs_add8<NP>(P, xv);
      // nibbles holding several bits: at most three further rounds (rare)
      if (__any_sync(0xFFFFFFFFu, (ex & 7u) != 0)) {
#pragma unroll 1
        for (int round = 0; round < 3; ++round) {
          uint32_t left = 0;
#pragma unroll
          for (int m = 0; m < 8; ++m) {
            const uint32_t more = ent[m] & 7u;
            const uint32_t k = __ffs(more);  // column first + k
            const uint32_t* src = reinterpret_cast<const uint32_t*>(mad_wide((ent[m] >> 3) + k, xsb, xbase));
            xv[m] = more ? __ldg(src) : 0u;
            ent[m] &= ~(more & (0u - more));
            left |= ent[m] & 7u;
          }
          hs_add8<NP>(P, xv);
          if (!__any_sync(0xFFFFFFFFu, left != 0)) break;
        }
      }
    }
    __syncwarp();
    uint32_t Q[NQ];
    slot_reduce<G, NP, NQ>(P, Q);
    if (!word_ok) {
    } else if (OUTB) {
      // cnt >= ceil(deg/2)  <=>  2*cnt - deg >= 0   (kernels.cpp:440-454)
      uint32_t ge = planes_ge<NQ>(Q, (deg + 1) >> 1);
      if (32 * (word + 1) > f) ge &= (32 * word >= f) ? 0u : tail_mask32(f);
      if (slot == 0) out_bits[i * xspw + word] = ge;
    } else if (ep.bits) {  // every slot lane holds the totals: one packs the word
      if (slot == 0)
        fepi_store_word(ep, out_f, i, f, word, [&](int b) {
          return static_cast<float>(2 * static_cast<int64_t>(plane_count<NQ>(Q, b)) - static_cast<int64_t>(deg));
        });
    } else {
      for (int b = slot; b < 32; b += S) {
        const int64_t k = 32 * word + b;
        if (k >= f) break;
        out_f[i * f + k] = fepi_apply(
            ep, static_cast<float>(2 * static_cast<int64_t>(plane_count<NQ>(Q, b)) - static_cast<int64_t>(deg)), k);
      }
    }
  }
}

// ---- BSpMM.BBB / BBF for low-degree graphs over the bit-entry view ----------
// Lane (row r, word g): R = 32/G rows per warp, each lane walks its own row's
// columns and counts word g of the neighbours with Harley-Seal planes; no
// slot reduction, no padding beyond the warp's longest row.  The sliver
// kernel's 8-slot split pays off for rows of hundreds of edges; for degrees
// in the tens it mostly counts padding (ncu, products shape: 780 M
// instructions, ALU 79 %).
template <int G, int NP, bool OUTB>
__global__ void __launch_bounds__(256)
    k_bv_bb(const uint64_t* __restrict__ bp, const uint32_t* __restrict__ bc, int64_t row0, int64_t row1,
            const int32_t* __restrict__ degree, const uint32_t* __restrict__ x, int64_t xspw, int64_t f,
            uint32_t* __restrict__ out_bits, float* __restrict__ out_f, const FEpi ep) {
  constexpr int R = 32 / G;
  const int lane = threadIdx.x & 31, r = lane / G, g = lane % G;
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const bool word_ok = g < xspw;
  // gather address = base + col * row stride: one IMAD.WIDE.U32 per load (a
  // 64-bit col * xspw product costs several IMADs)
  const uint64_t xbase = reinterpret_cast<uint64_t>(x + (word_ok ? g : 0));
  const uint32_t xsb = static_cast<uint32_t>(xspw) * 4u;
  for (int64_t i0 = row0 + wid * R; i0 < row1; i0 += nw * R) {
    const int64_t i = i0 + r;
    const bool ok = i < row1;
    const uint32_t deg = ok ? static_cast<uint32_t>(__ldg(degree + i)) : 0u;
    const uint32_t walk = deg < kHubDeg ? deg : 0u;  // hub rows: hub_bb (hubs.cu)
    uint32_t mx = walk;
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    const uint32_t* cols = bc + (ok ? bp[i] : 0);
    uint32_t P[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) P[q] = 0u;
    const uint32_t padded = (walk + kBitPad - 1) / kBitPad * kBitPad;  // this row's view length
    for (uint32_t j = 0; j < mx; j += 8) {
      // the row's next 8 column indices as two 16-byte loads (the 4 lanes of
      // a row read the same address: one request), not 8 scalar loads per
      // lane that re-fetch the same sector from L2
      uint4 c0 = make_uint4(0u, 0u, 0u, 0u), c1 = c0;
      if (j < padded) {
        c0 = __ldg(reinterpret_cast<const uint4*>(cols + j));
        c1 = __ldg(reinterpret_cast<const uint4*>(cols + j + 4));
      }
      const uint32_t cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      uint32_t v[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        v[m] = 0u;
        if (j + m < walk && word_ok) v[m] = __ldg(reinterpret_cast<const uint32_t*>(mad_wide(cc[m], xsb, xbase)));
      }
      hs_add8<NP>(P, v);
    }
    if (!ok || !word_ok) continue;
    if (OUTB) {
      // cnt >= ceil(deg/2)  <=>  2*cnt - deg >= 0   (kernels.cpp:440-454)
      uint32_t ge = planes_ge<NP>(P, (deg + 1) >> 1);
      if (32 * (g + 1) > f) ge &= (32 * g >= f) ? 0u : tail_mask32(f);
      out_bits[i * xspw + g] = ge;
    } else {
      fepi_store_word(ep, out_f, i, f, g, [&](int b) {
        return static_cast<float>(2 * static_cast<int64_t>(plane_count<NP>(P, b)) - static_cast<int64_t>(deg));
      });
    }
  }
}

// ---- fused layer-1 GCN over the bit-entry view -----------------------------
// float(beta*sdot - 2u*q) with 2u = 2^(exp(beta)-22) (gcn_fused.cu), exactly.
__device__ __forceinline__ float logit_of(float beta, int64_t sdot, int qsum) {
  const uint32_t bb = __float_as_uint(beta);
  const int e = static_cast<int>((bb >> 23) & 0xFF);
  if (e == 0 || e == 0xFF) {  // zero/subnormal/inf/nan scale: plain double path
    const double two_u = ldexp(1.0, e - 127 - 22);
    return __double2float_rn(__dsub_rn(__dmul_rn(static_cast<double>(beta), static_cast<double>(sdot)),
                                       __dmul_rn(two_u, static_cast<double>(qsum))));
  }
  const int64_t m = static_cast<int64_t>((bb & 0x7FFFFFu) | 0x800000u) * ((bb >> 31) ? -1 : 1);
  const int64_t X = m * sdot - 2 * static_cast<int64_t>(qsum);
  // float(X) * 2^(e-150): exact scaling unless the result leaves the normal range
  const int sc = e - 150;
  if (sc >= -126 && sc <= 127) return __ll2float_rn(X) * __int_as_float((sc + 127) << 23);
  return __double2float_rn(ldexp(static_cast<double>(X), sc));
}

// Record of node j (16 words): word 4g = h word g, words 4g+1..4g+3 = bytes
// q_jk + 32 of classes 12g .. 12g+11 (4 per word, little-endian).  Record
// `cols` (one past the last node) is all zero: the view's padding entries
// point there, so every load is unconditional and adds nothing.
constexpr int kRec = 16;

template <int NP>
__global__ void __launch_bounds__(kSlWarps * 32, 5)
    k_bv_gcn1(const uint64_t* __restrict__ bp, const uint32_t* __restrict__ bc, int64_t row0,
              int64_t row1, const int32_t* __restrict__ degree, const uint32_t* __restrict__ rec,
              const uint32_t* __restrict__ wt, int hspw, int K, const float* __restrict__ beta,
              int C, float* __restrict__ logits, float* __restrict__ probs) {
  constexpr int G = 4, S = 8, B = 8 * S, NQ = NP + 3;
  __shared__ int qsum_all[kSlWarps][48];
  __shared__ int sw_all[kSlWarps][48];
  __shared__ uint32_t wt_s[48 * 4];
  __shared__ int wpop_s[48];
  for (int t = threadIdx.x; t < 48 * 4; t += blockDim.x) {
    const int k = t >> 2, w = t & 3;
    wt_s[t] = (k < C && w < hspw) ? wt[k * hspw + w] : 0u;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 48; k += blockDim.x)
    wpop_s[k] = __popc(wt_s[4 * k]) + __popc(wt_s[4 * k + 1]) + __popc(wt_s[4 * k + 2]) + __popc(wt_s[4 * k + 3]);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane % G, slot = lane / G;
  const uint64_t rbase = reinterpret_cast<uint64_t>(reinterpret_cast<const uint4*>(rec) + g);
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = row0 + wid; i < row1; i += nw) {
    uint32_t P[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) P[q] = 0;
    uint32_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    const uint64_t e0 = bp[i];
    const uint32_t len = static_cast<uint32_t>(bp[i + 1] - e0);  // multiple of kBitPad
    // slot s takes entries 8s .. 8s+7 of each 64-entry block: two 16-byte
    // loads per lane (a warp instruction covers one 128-byte line) instead
    // of eight 4-byte ones (eight lines); the sums are order-free integers
    const uint4* rowp = reinterpret_cast<const uint4*>(bc + e0) + 2 * slot;
    for (uint32_t off = 0; off < len; off += B) {
      const uint4 ca = ld_nc_v4(rowp + off / 4), cb = ld_nc_v4(rowp + off / 4 + 1);
      const uint32_t cols[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
      uint4 v[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) v[m] = __ldg(reinterpret_cast<const uint4*>(mad_wide(cols[m], kRec * 4, rbase)));
      uint32_t h[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) h[m] = v[m].x;
      hs_add8<NP>(P, h);
      // q bytes are <= 64: three words add byte-wise without carries
#pragma unroll
      for (int w = 0; w < 3; ++w) {
        auto qw = [&](int m) { return w == 0 ? v[m].y : w == 1 ? v[m].z : v[m].w; };
        const uint32_t a = qw(0) + qw(1) + qw(2), b = qw(3) + qw(4) + qw(5), c = qw(6) + qw(7);
        lo[w] += (a & 0x00FF00FFu) + (b & 0x00FF00FFu) + (c & 0x00FF00FFu);
        hi[w] += ((a >> 8) & 0x00FF00FFu) + ((b >> 8) & 0x00FF00FFu) + ((c >> 8) & 0x00FF00FFu);
      }
    }
    // slot reductions: h planes (bit-sliced butterfly; every lane of word g
    // ends with the row's planes of word g) and q sums (16-bit lanes)
    uint32_t Q[NQ];
    slot_reduce<G, NP, NQ>(P, Q);
#pragma unroll
    for (int w = 0; w < 3; ++w)
      for (int d = G; d < 32; d <<= 1) {
        lo[w] += __shfl_xor_sync(0xFFFFFFFFu, lo[w], d);
        hi[w] += __shfl_xor_sync(0xFFFFFFFFu, hi[w], d);
      }
    const int deg = __ldg(degree + i);
    if (slot == 0) {
      const int bias = 32 * deg;
#pragma unroll
      for (int w = 0; w < 3; ++w) {
        const int k0 = 12 * g + 4 * w;
        qsum_all[warp][k0 + 0] = static_cast<int>(lo[w] & 0xFFFFu) - bias;
        qsum_all[warp][k0 + 1] = static_cast<int>(hi[w] & 0xFFFFu) - bias;
        qsum_all[warp][k0 + 2] = static_cast<int>(lo[w] >> 16) - bias;
        qsum_all[warp][k0 + 3] = static_cast<int>(hi[w] >> 16) - bias;
      }
    }
    // sum_b cnt_b over this lane's word, then over the four words
    int sall = 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) sall += __popc(Q[q]) << q;
    sall += __shfl_xor_sync(0xFFFFFFFFu, sall, 1);
    sall += __shfl_xor_sync(0xFFFFFFFFu, sall, 2);
    // sum_b [w_kb] cnt_b = sum_q 2^q popc(w_k & Q_q): (class, word) pairs over
    // the lanes -- lane (k%8, g) of pass k/8 -- then a sum over the 4 words
    for (int k0 = 0; k0 < C; k0 += 8) {
      const int k = k0 + (lane >> 2);
      const uint32_t wk = wt_s[4 * min(k, 47) + g];
      int t = 0;
#pragma unroll
      for (int q = 0; q < NQ; ++q) t += __popc(wk & Q[q]) << q;
      t += __shfl_xor_sync(0xFFFFFFFFu, t, 1);
      t += __shfl_xor_sync(0xFFFFFFFFu, t, 2);
      if (g == 0 && k < C) sw_all[warp][k] = t;
    }
    __syncwarp();
    // Per class: sum_j dot_jk = 2*(2*sw - sall) - deg*(2*popc(w_k) - K); then
    // the exact combination of gcn_fused.cu and the fused softmax.
    float lg[2];
    double mx = -INFINITY;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      const int k = lane + 32 * pass;
      lg[pass] = -INFINITY;
      if (k < C) {
        const int64_t sdot = 2 * (2 * static_cast<int64_t>(sw_all[warp][k]) - sall) -
                             static_cast<int64_t>(deg) * (2 * wpop_s[k] - K);
        // beta*sdot - 2u*qsum = 2^(e-23) * (m_beta*sdot - 2*qsum): an exact
        // integer below 2^41 (the reference's double sum is exact too), so one
        // int64 -> float rounding reproduces float(d); the scale is exact.
        lg[pass] = logit_of(beta[k], sdot, qsum_all[warp][k]);
        if (logits) logits[i * C + k] = lg[pass];
        mx = fmax(mx, static_cast<double>(lg[pass]));
      }
    }
    if (probs) {  // kernel parameter: warp-uniform (the model path runs softmax as a layer)
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
      const double x0 = lane < C ? exp_nonpos(static_cast<double>(lg[0]) - mx) : 0.0;
      const double x1 = lane + 32 < C ? exp_nonpos(static_cast<double>(lg[1]) - mx) : 0.0;
      double sum = x0 + x1;
#pragma unroll
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
      if (lane < C) probs[i * C + lane] = __double2float_rn(x0 / sum);
      if (lane + 32 < C) probs[i * C + lane + 32] = __double2float_rn(x1 / sum);
    }
    __syncwarp();
  }
}

// Bit-entry view construction (frdc_bitview).
__global__ void k_bv_count(const int32_t* __restrict__ deg, int64_t rows, unsigned long long* __restrict__ cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < rows) cnt[i] = (static_cast<unsigned long long>(deg[i]) + kBitPad - 1) / kBitPad * kBitPad;
}

__global__ void k_bv_fill(const uint64_t* __restrict__ srp, const uint32_t* __restrict__ sl, int64_t rows,
                          uint32_t pad, const unsigned long long* __restrict__ bp, uint32_t* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  uint64_t p = bp[i];
  for_each_col(srp, sl, i, [&](uint32_t col) { out[p++] = col; });
  for (; p < bp[i + 1]; ++p) out[p] = pad;
}

// Record producer for k_bv_gcn1 (layout above): thread per (node, word group
// g), which holds the node's h words and writes its 16-byte quarter -- h word
// g and the q bytes of classes 12g .. 12g+11 -- with one store; plus the zero
// record after the last node.  The weight bits and scales are staged in
// shared memory once per block.
__global__ void __launch_bounds__(256)
    k_sl_gcn1_records(const uint32_t* __restrict__ h, int64_t rows, int hspw, int K,
                      const uint32_t* __restrict__ wt, const float* __restrict__ beta, int C,
                      uint32_t* __restrict__ rec, bool h_v4) {
  __shared__ uint4 wt_s[48];
  __shared__ float beta_s[48], inv2u_s[48];
  for (int t = threadIdx.x; t < 48 * 4; t += blockDim.x) {
    const int k = t >> 2, w = t & 3;
    reinterpret_cast<uint32_t*>(wt_s)[t] = (k < C && w < hspw) ? wt[k * hspw + w] : 0u;
  }
  for (int k = threadIdx.x; k < 48; k += blockDim.x) {
    const float bk = k < C ? beta[k] : 1.0f;
    beta_s[k] = bk;
    const int ex = ((__float_as_int(bk) >> 23) & 0xFF) - 127;
    inv2u_s[k] = __int_as_float((127 + 22 - ex) << 23);  // 1 / (2u): u = the ulp unit of beta
  }
  __syncthreads();
  uint4* rec4 = reinterpret_cast<uint4*>(rec);
  // grid-stride over (node, word group) items: each block stages the weights once
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < (rows + 1) * 4;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (t >= rows * 4) {
      rec4[t] = make_uint4(0u, 0u, 0u, 0u);
      continue;
    }
    const int64_t j = t >> 2;
    const int g = static_cast<int>(t & 3);
    uint32_t hw[4] = {0, 0, 0, 0};
    if (h_v4) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(h) + j);
      hw[0] = v.x, hw[1] = v.y, hw[2] = v.z, hw[3] = v.w;
    } else {
      for (int q = 0; q < hspw; ++q) hw[q] = __ldg(h + j * hspw + q);
    }
    uint32_t out[3] = {0u, 0u, 0u};
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int k = 12 * g + 4 * p + b;
        if (k >= C) continue;
        const uint4 wk = wt_s[k];
        const int diff = __popc(hw[0] ^ wk.x) + __popc(hw[1] ^ wk.y) + __popc(hw[2] ^ wk.z) + __popc(hw[3] ^ wk.w);
        // int <-> float through the 2^23 magic instead of I2F / F2I (those
        // share the quarter-rate pipe with the 164 POPCs of a node)
        const float fd = __int_as_float(0x4B000000 + K - 2 * diff + 0x400000) - 12582912.0f;  // exact (|dot| <= 2^21)
        const float bk = beta_s[k];
        const float x = __fmul_rn(fd, bk);
        const float e = __fmaf_rn(fd, bk, -x);  // exact rounding error of the product
        // q = e / (2u), an integer in [-32, 32]: exact in fp32, rounded by the magic add
        const int q = __float_as_int(__fmaf_rn(e, inv2u_s[k], 12582912.0f)) - 0x4B400000;
        out[p] |= static_cast<uint32_t>(q + 32) << (8 * b);
      }
    rec4[t] = make_uint4(hw[g], out[0], out[1], out[2]);
  }
}

// ---- real-valued walk in ascending column order ------------------------------
template <int M, bool XBITS, bool OUTB>
__global__ void __launch_bounds__(256)
    k_sl_f(const uint64_t* __restrict__ srp, const uint32_t* __restrict__ sl, int64_t row0,
           int64_t row1, const float* __restrict__ xf, const uint32_t* __restrict__ xb,
           int64_t xspw, const float* __restrict__ rs, const float* __restrict__ cs, int64_t f,
           int64_t ospw, uint32_t* __restrict__ out_bits, float* __restrict__ out_f, const FEpi ep) {
  const int64_t i = row0 + ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  if (i >= row1) return;
  const int lane = threadIdx.x & 31;
  const int64_t fbase = static_cast<int64_t>(blockIdx.y) * 32 * M;
  double d[M];
#pragma unroll
  for (int m = 0; m < M; ++m) d[m] = 0.0;
  // operand row address = base + col * row bytes by one IMAD.WIDE.U32
  const uint32_t xrs = XBITS ? static_cast<uint32_t>(xspw) * 4u : static_cast<uint32_t>(f) * 4u;
  const uint64_t xrow0 = XBITS ? reinterpret_cast<uint64_t>(xb) : reinterpret_cast<uint64_t>(xf);
  const uint64_t e0 = srp[i];
  const uint32_t len = static_cast<uint32_t>(srp[i + 1] - e0);
  for (uint32_t base = 0; base < len; base += 32) {
    const uint32_t mine = base + lane < len ? ld_nc_u32(sl + e0 + base + lane) : kSliverSentinel;
    const int cnt = static_cast<int>(min(32u, len - base));
    for (int L = 0; L < cnt; ++L) {  // slivers in order, then columns in order
      const uint32_t ent = __shfl_sync(0xFFFFFFFFu, mine, L);
      if (ent == kSliverSentinel) continue;  // row padding (warp-uniform)
      const uint32_t first = ent >> 3;
      uint32_t more = ent & 7u, col = first;
      for (;;) {
        const int64_t j = col;
        const double w = cs ? static_cast<double>(__ldg(cs + j)) : 1.0;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const int64_t k = fbase + 32 * m + lane;
          if (k < f) {
            if (XBITS) {
              const uint32_t* xr = reinterpret_cast<const uint32_t*>(mad_wide(col, xrs, xrow0));
              const uint32_t bit = (__ldg(xr + (k >> 5)) >> (31 - (k & 31))) & 1u;
              d[m] = __dadd_rn(d[m], bit ? w : -w);
            } else {
              const float* xr = reinterpret_cast<const float*>(mad_wide(col, xrs, xrow0));
              d[m] = __dadd_rn(d[m], __dmul_rn(w, static_cast<double>(__ldg(xr + k))));
            }
          }
        }
        if (!more) break;
        col = first + __ffs(more);
        more &= more - 1;
      }
    }
  }
  const double si = rs ? static_cast<double>(rs[i]) : 1.0;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int64_t k = fbase + 32 * m + lane;
    const double v = __dmul_rn(si, d[m]);
    if (OUTB) {
      const uint32_t word = __brev(__ballot_sync(0xFFFFFFFFu, k < f && v >= 0.0));
      const int64_t w = (fbase >> 5) + m;
      if (lane == 0 && w < ospw) out_bits[i * ospw + w] = word;
    } else {
      fepi_store_lane(ep, out_f, i, f, k, __double2float_rn(v));
    }
  }
  if (OUTB && lane == 0 && blockIdx.y == gridDim.y - 1)
    for (int64_t w = (f + 31) / 32; w < ospw; ++w) out_bits[i * ospw + w] = 0;
}

int64_t grid_warps(int64_t rows) {
  return std::max<int64_t>(1, std::min<int64_t>(cdiv(rows, kSlWarps), static_cast<int64_t>(sm_count()) * 32));
}

// Most bits a slot lane can count: its share of the row's (padded) entries
// (batches of 8 per slot) plus every extra bit of multi-bit nibbles.
int64_t lane_bound(const bg_frdc& A, int S) {
  return (A.max_sl_row + 8 * S - 1) / (8 * S) * 8 + A.max_extra_bits;
}

template <int G, bool OUTB>
void launch_sl_bb(const bg_frdc& A, const uint32_t* x, int64_t f, int64_t xspw, uint32_t* ob,
                  float* of, int64_t r0, int64_t r1, cudaStream_t s) {
  const int64_t per_lane = lane_bound(A, 32 / G);
  dim3 grid(static_cast<unsigned>(grid_warps(r1 - r0)), static_cast<unsigned>(cdiv(xspw, G)));
  auto go = [&](auto kern) {
    kern<<<grid, kSlWarps * 32, 0, s>>>(A.srp(), A.sl(), r0, r1, A.deg(), x, xspw, f, ob, of, current_fepi());
  };
  if (per_lane < (1 << 7)) go(k_sl_bb<G, 7, OUTB>);
  else if (per_lane < (1 << 10)) go(k_sl_bb<G, 10, OUTB>);
  else if (per_lane < (1 << 13)) go(k_sl_bb<G, 13, OUTB>);
  else if (per_lane < (1 << 16)) go(k_sl_bb<G, 16, OUTB>);
  else if (per_lane < (1 << 20)) go(k_sl_bb<G, 20, OUTB>);  // hub rows (power-law graphs)
  else if (per_lane < (1 << 26)) go(k_sl_bb<G, 26, OUTB>);
  else fail("bspmm: node degree " + std::to_string(A.max_deg) + " exceeds the counter range");
  BG_LAUNCH_CHECK();
}

// Narrow F outputs (f <= 16: Flickr's 7 classes): G = 8 or 16 lanes per row,
// 32/G rows per warp, so the lanes that a warp per row would leave idle past
// column f walk other rows.  Each lane group walks its row's slivers in the
// same ascending order with the same double accumulation (bit-identical to
// k_sl_f); the entry loop runs to the longest row of the warp, shorter rows
// idle through the rest.
template <int G, bool XBITS>
__global__ void __launch_bounds__(256)
    k_sl_f_sub(const uint64_t* __restrict__ srp, const uint32_t* __restrict__ sl, int64_t row0,
               int64_t row1, const float* __restrict__ xf, const uint32_t* __restrict__ xb,
               int64_t xspw, const float* __restrict__ rs, const float* __restrict__ cs, int64_t f,
               float* __restrict__ out_f, const FEpi ep) {
  const int lane = threadIdx.x & 31, grp = lane / G, t = lane % G;
  const int64_t i = row0 + ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * (32 / G) + grp;
  if (row0 + ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * (32 / G) >= row1) return;
  const bool live = i < row1;
  double d = 0.0;
  // operand row address = base + col * row bytes by one IMAD.WIDE.U32
  const uint32_t xrs = XBITS ? static_cast<uint32_t>(xspw) * 4u : static_cast<uint32_t>(f) * 4u;
  const uint64_t xrow0 = XBITS ? reinterpret_cast<uint64_t>(xb) : reinterpret_cast<uint64_t>(xf);
  const uint64_t e0 = live ? srp[i] : 0;
  const uint32_t len = live ? static_cast<uint32_t>(srp[i + 1] - e0) : 0u;
  uint32_t lmax = len;  // the warp's longest row
#pragma unroll
  for (int o = G; o < 32; o <<= 1) lmax = max(lmax, __shfl_xor_sync(0xFFFFFFFFu, lmax, o));
  for (uint32_t base = 0; base < lmax; base += G) {
    const uint32_t mine = base + t < len ? ld_nc_u32(sl + e0 + base + t) : kSliverSentinel;
    const int cnt = static_cast<int>(min(static_cast<uint32_t>(G), lmax - base));
    for (int L = 0; L < cnt; ++L) {  // slivers in order, then columns in order
      const uint32_t ent = __shfl_sync(0xFFFFFFFFu, mine, L, G);
      if (ent == kSliverSentinel) continue;  // row padding or past this row's end (group-uniform)
      const uint32_t first = ent >> 3;
      uint32_t more = ent & 7u, col = first;
      for (;;) {
        const int64_t j = col;
        const double w = cs ? static_cast<double>(__ldg(cs + j)) : 1.0;
        if (t < f) {
          if (XBITS) {
            const uint32_t bit = (__ldg(reinterpret_cast<const uint32_t*>(mad_wide(col, xrs, xrow0))) >> (31 - t)) & 1u;
            d = __dadd_rn(d, bit ? w : -w);
          } else {
            d = __dadd_rn(d, __dmul_rn(w, static_cast<double>(__ldg(reinterpret_cast<const float*>(mad_wide(col, xrs, xrow0)) + t))));
          }
        }
        if (!more) break;
        col = first + __ffs(more);
        more &= more - 1;
      }
    }
  }
  const double si = rs && live ? static_cast<double>(rs[i]) : 1.0;
  const float v = __double2float_rn(__dmul_rn(si, d));
  const float y = live && t < f ? fepi_apply(ep, v, t) : 0.0f;
  if (ep.bits) {  // fused Binarize: the group's sign bits, MSB-first
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, live && t < f && y >= 0.0f);
    const uint32_t mine = (bal >> (grp * G)) & ((1u << G) - 1u);
    if (live && t == 0) ep.bits[i * ep.bspw] = __brev(mine);
  } else if (live && t < f) {
    out_f[i * f + t] = y;
  }
}

template <int M, bool XBITS, bool OUTB>
void launch_sl_f(const bg_frdc& A, const SpmmFArgs& a, int64_t r0, int64_t r1, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>(cdiv((r1 - r0) * 32, 256)), static_cast<unsigned>(cdiv(a.f, 32 * M)));
  const int64_t xspw = XBITS ? spw(a.f, a.xwb) : 0;
  const int64_t ospw = OUTB ? spw(a.f, a.owb) : 0;
  k_sl_f<M, XBITS, OUTB><<<grid, 256, 0, s>>>(A.srp(), A.sl(), r0, r1, a.x_f, a.x_bits, xspw,
                                              a.row_scale, a.col_scale, a.f, ospw, a.out_bits,
                                              a.out_f, current_fepi());
  BG_LAUNCH_CHECK();
}

template <bool XBITS, bool OUTB>
void launch_sl_f_m(const bg_frdc& A, const SpmmFArgs& a, int64_t r0, int64_t r1, cudaStream_t s) {
  if (!OUTB && a.f <= 16 && std::getenv("BG_SLF_WARP") == nullptr) {
    // narrow rows: G lanes per row (k_sl_f_sub)
    auto go = [&](auto kern, int G) {
      const int64_t warps = cdiv(r1 - r0, 32 / G);
      kern<<<static_cast<unsigned>(cdiv(warps * 32, 256)), 256, 0, s>>>(
          A.srp(), A.sl(), r0, r1, a.x_f, a.x_bits, XBITS ? spw(a.f, a.xwb) : 0, a.row_scale, a.col_scale, a.f,
          a.out_f, current_fepi());
      BG_LAUNCH_CHECK();
    };
    if (a.f <= 8) go(k_sl_f_sub<8, XBITS>, 8);
    else go(k_sl_f_sub<16, XBITS>, 16);
    return;
  }
  if (a.f <= 32) launch_sl_f<1, XBITS, OUTB>(A, a, r0, r1, s);
  else if (a.f <= 64) launch_sl_f<2, XBITS, OUTB>(A, a, r0, r1, s);
  else launch_sl_f<4, XBITS, OUTB>(A, a, r0, r1, s);
}

// Row-group path for graphs whose rows are short (average degree < 64): see k_bv_bb.
template <int G, bool OUTB>
bool launch_bv_bb(bg_frdc& A, const uint32_t* x, int64_t f, int64_t xspw, uint32_t* ob, float* of, int64_t r0,
                  int64_t r1, cudaStream_t s) {
  constexpr int R = 32 / G;
  frdc_bitview(A, s);
  const int64_t warps = std::max<int64_t>(
      1, std::min<int64_t>(cdiv(r1 - r0, R), static_cast<int64_t>(sm_count()) * 64));
  const unsigned blocks = static_cast<unsigned>(cdiv(warps * 32, 256));
  auto go = [&](auto kern) {
    kern<<<blocks, 256, 0, s>>>(A.bit_ptr.as<uint64_t>(), A.bit_cols.as<uint32_t>(), r0, r1, A.deg(), x, xspw,
                                f, ob, of, current_fepi());
  };
  const int64_t d = light_max_deg(A, s);
  if (d < (1 << 6)) go(k_bv_bb<G, 6, OUTB>);
  else if (d < (1 << 9)) go(k_bv_bb<G, 9, OUTB>);
  else if (d < (1 << 12)) go(k_bv_bb<G, 12, OUTB>);
  else go(k_bv_bb<G, 16, OUTB>);
  BG_LAUNCH_CHECK();
  return true;
}

}  // namespace

bool rowgroup_bb(bg_frdc& A, const uint32_t* x, int64_t f, int64_t xspw, uint32_t* out_bits, float* out_f,
                 cudaStream_t s, int64_t r0, int64_t r1) {
  // AUTO only: the SLIVERS / TILES / WINDOW modes keep their kernels (coverage)
  if (aggregation_mode() != BG_AGG_AUTO) return false;
  if (xspw > 8 || A.rows == 0) return false;
  if (A.nnz_bits >= 64 * A.rows) return false;  // long rows: the 8-slot sliver split balances better
  const bool ob = out_bits != nullptr;
  auto run = [&](auto gtag) {
    constexpr int G = decltype(gtag)::value;
    return ob ? launch_bv_bb<G, true>(A, x, f, xspw, out_bits, out_f, r0, r1, s)
              : launch_bv_bb<G, false>(A, x, f, xspw, out_bits, out_f, r0, r1, s);
  };
  if (xspw <= 1) return run(std::integral_constant<int, 1>{});
  if (xspw <= 2) return run(std::integral_constant<int, 2>{});
  if (xspw <= 4) return run(std::integral_constant<int, 4>{});
  return run(std::integral_constant<int, 8>{});
}

void sliver_bb(bg_frdc& A, const uint32_t* x, int64_t f, int wb, uint32_t* out_bits, float* out_f,
               cudaStream_t s, int64_t r0, int64_t r1) {
  if (r1 < 0) r1 = A.rows;
  const int64_t xspw = spw(f, wb);
  if (r1 <= r0 || xspw == 0) return;
  if (window_bb(A, x, f, wb, out_bits, out_f, s, r0, r1) || rowgroup_bb(A, x, f, xspw, out_bits, out_f, s, r0, r1))
    return hub_bb(A, x, f, xspw, out_bits, out_f, s, r0, r1);
  frdc_slivers(A, s);
  const bool ob = out_bits != nullptr;
  if (xspw <= 4) {
    if (ob) launch_sl_bb<4, true>(A, x, f, xspw, out_bits, out_f, r0, r1, s);
    else launch_sl_bb<4, false>(A, x, f, xspw, out_bits, out_f, r0, r1, s);
  } else if (xspw <= 8) {
    if (ob) launch_sl_bb<8, true>(A, x, f, xspw, out_bits, out_f, r0, r1, s);
    else launch_sl_bb<8, false>(A, x, f, xspw, out_bits, out_f, r0, r1, s);
  } else if (xspw <= 16) {
    if (ob) launch_sl_bb<16, true>(A, x, f, xspw, out_bits, out_f, r0, r1, s);
    else launch_sl_bb<16, false>(A, x, f, xspw, out_bits, out_f, r0, r1, s);
  } else {
    if (ob) launch_sl_bb<32, true>(A, x, f, xspw, out_bits, out_f, r0, r1, s);
    else launch_sl_bb<32, false>(A, x, f, xspw, out_bits, out_f, r0, r1, s);
  }
  hub_bb(A, x, f, xspw, out_bits, out_f, s, r0, r1);
}

void sliver_f(bg_frdc& A, const SpmmFArgs& a, cudaStream_t s, int64_t r0, int64_t r1) {
  if (r1 < 0) r1 = A.rows;
  if (r1 <= r0 || a.f == 0) return;
  frdc_slivers(A, s);
  const bool xb = a.x_bits != nullptr, ob = a.out_bits != nullptr;
  if (xb && ob) launch_sl_f_m<true, true>(A, a, r0, r1, s);
  else if (xb) launch_sl_f_m<true, false>(A, a, r0, r1, s);
  else if (ob) launch_sl_f_m<false, true>(A, a, r0, r1, s);
  else launch_sl_f_m<false, false>(A, a, r0, r1, s);
}

void sliver_gcn1_records(const uint32_t* h, int64_t n, int64_t K, int wb, const uint32_t* wt,
                         const float* beta, int64_t C, uint32_t* rec, cudaStream_t s) {
  const int hspw = static_cast<int>(spw(K, wb));
  const bool v4 = hspw == 4 && reinterpret_cast<uintptr_t>(h) % 16 == 0;
  k_sl_gcn1_records<<<static_cast<unsigned>(std::min<int64_t>(cdiv((n + 1) * 4, 256), sm_count() * 8)), 256, 0, s>>>(
      h, n, hspw, static_cast<int>(K), wt, beta, static_cast<int>(C), rec, v4);
  BG_LAUNCH_CHECK();
}

void sliver_gcn1_aggregate(bg_frdc& A, const uint32_t* rec, int64_t K, int wb, const uint32_t* wt,
                           const float* beta, int64_t C, float* logits, float* probs,
                           cudaStream_t s, int64_t r0, int64_t r1) {
  if (r1 < 0) r1 = A.rows;
  if (r1 <= r0) return;
  frdc_bitview(A, s);
  // a slot lane counts <= ceil(max_deg / 64) * 8 bits of its word
  const int64_t per_lane = (A.max_deg + kBitPad - 1) / kBitPad * 8;
  const int hspw = static_cast<int>(spw(K, wb));
  auto go = [&](auto kern) {
    kern<<<static_cast<unsigned>(grid_warps(r1 - r0)), kSlWarps * 32, 0, s>>>(
        A.bit_ptr.as<uint64_t>(), A.bit_cols.as<uint32_t>(), r0, r1, A.deg(), rec, wt, hspw,
        static_cast<int>(K), beta, static_cast<int>(C), logits, probs);
  };
  if (per_lane < (1 << 7)) go(k_bv_gcn1<7>);
  else if (per_lane < (1 << 10)) go(k_bv_gcn1<10>);
  else go(k_bv_gcn1<13>);
  BG_LAUNCH_CHECK();
}

void frdc_bitview(bg_frdc& m, cudaStream_t s) {
  if (m.nbits_view >= 0) return;
  frdc_slivers(m, s);
  const size_t n1 = static_cast<size_t>(m.rows) + 1;
  DevBuf cnt(n1 * 8);
  m.bit_ptr.alloc(n1 * 8);
  BG_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes, s));
  BG_CUDA(cudaMemsetAsync(m.bit_ptr.p, 0, m.bit_ptr.bytes, s));
  if (m.rows > 0)
    k_bv_count<<<static_cast<unsigned>(cdiv(m.rows, 256)), 256, 0, s>>>(m.deg(), m.rows,
                                                                        cnt.as<unsigned long long>());
  BG_LAUNCH_CHECK();
  size_t tmp_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, cnt.as<unsigned long long>(),
                                m.bit_ptr.as<unsigned long long>() + 1, static_cast<int>(m.rows), s);
  DevBuf tmp(std::max<size_t>(tmp_bytes, 1));
  if (m.rows > 0)
    cub::DeviceScan::InclusiveSum(tmp.p, tmp_bytes, cnt.as<unsigned long long>(),
                                  m.bit_ptr.as<unsigned long long>() + 1, static_cast<int>(m.rows), s);
  BG_LAUNCH_CHECK();
  unsigned long long total = 0;
  BG_CUDA(cudaMemcpyAsync(&total, m.bit_ptr.as<unsigned long long>() + m.rows, 8, cudaMemcpyDeviceToHost, s));
  BG_CUDA(cudaStreamSynchronize(s));
  m.bit_cols.alloc(std::max<size_t>(static_cast<size_t>(total) * 4, 4));
  if (m.rows > 0)
    k_bv_fill<<<static_cast<unsigned>(cdiv(m.rows, 256)), 256, 0, s>>>(
        m.srp(), m.sl(), m.rows, static_cast<uint32_t>(m.cols), m.bit_ptr.as<unsigned long long>(),
        m.bit_cols.as<uint32_t>());
  BG_LAUNCH_CHECK();
  BG_CUDA(cudaStreamSynchronize(s));
  m.nbits_view = static_cast<int64_t>(total);
  ++m.gen;
}

}  // namespace bg

namespace bg {
namespace {
int env_mode() {
  const char* e = std::getenv("BG_AGGREGATION");
  if (!e) return BG_AGG_AUTO;
  const std::string v(e);
  return v == "tiles" ? BG_AGG_TILES : v == "slivers" ? BG_AGG_SLIVERS : v == "window" ? BG_AGG_WINDOW : BG_AGG_AUTO;
}
int env_window_nodes() {
  const char* e = std::getenv("BG_WINDOW_NODES");
  return e && *e ? std::max(0, std::atoi(e)) : 0;
}
std::atomic<int> g_mode{env_mode()};
std::atomic<int> g_window_nodes{env_window_nodes()};
std::atomic<uint64_t> g_generation{0};
}  // namespace

int aggregation_mode() { return g_mode.load(std::memory_order_relaxed); }
int window_nodes_setting() { return g_window_nodes.load(std::memory_order_relaxed); }
uint64_t aggregation_generation() { return g_generation.load(std::memory_order_relaxed); }
void set_aggregation(int mode, int window_nodes) {
  if (mode < BG_AGG_AUTO || mode > BG_AGG_WINDOW) fail("aggregation mode must be one of BG_AGG_*");
  if (window_nodes < 0 || window_nodes > 65535) fail("window_nodes must be in [0, 65535]");
  g_mode.store(mode);
  g_window_nodes.store(window_nodes);
  g_generation.fetch_add(1);
}
}  // namespace bg
