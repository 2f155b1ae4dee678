// Fused second GCN layer of the default plan: MM.BBF + BSpMM.FBF (+ Softmax)
// (ref: modelconfig.cpp:51, gcn_layer graphops.cpp:270-285, bmm F-out
// kernels.cpp:179-190, bspmm F path :512-555, softmax_rows graphops.cpp:372-386).
//
// The reference materializes Y = float(dot * beta) (N x C fp32) and then sums
// Y over each node's neighbours in double.  Gathering 4*C bytes per edge makes
// that aggregation L2-gather bound, so this path never materializes Y:
//
//   x = fl(dot*b) is a product of an integer |dot| <= 128 (even when the
//   hidden width K is even) and a float b, so with u = ulp-unit of b
//   (b = M*u, 2^23 <= M < 2^24):
//     e = dot*b - x        is exact in fp32 (FFMA), a multiple of 2u,
//                          |e| <= 32*(2u)                 -> q = e/(2u) in [-32, 32]
//     sum_j x_j = b * sum_j dot_j - 2u * sum_j q_j         exactly, in double.
//   Every double partial sum of the reference is exact as well (all summands
//   are multiples of 2u below 2^53*2u), so the reference's ascending-order
//   double sum IS this exact value, and float() of it is bit-identical.
//
//   sum_j dot_jk = sum_b w+-_bk * sum_j h+-_jb is linear in the aggregated
//   sign bits, so it comes from bit-sliced counts of the gathered h rows.
//
// Producer (k_gcn1_records): one 64-byte record per node,
//   words 0..3   : the node's packed h bits (K <= 128)
//   words 4..15  : byte q_jk + 32 per class k (C <= 48), padding 0.
// Consumer (k_gcn1_aggregate): the tile-row walker (tilewalk.cuh) gathers one
// record per edge (two 32-byte sectors); lanes 0..3 count h bits with
// Harley-Seal planes, lanes 4..15 sum the q bytes in 16-bit SWAR lanes; the
// epilogue combines both per class, writes the logits and the fused softmax.
#include <algorithm>

#include "ops.cuh"
#include "tilewalk.cuh"

namespace bg {
namespace {

constexpr int kRecWords = 16;  // 64-byte record
constexpr int kFWarps = 8;

// Thread per (node, record word).
__global__ void k_gcn1_records(const uint32_t* __restrict__ h, int64_t rows, int hspw, int K,
                               const uint32_t* __restrict__ wt, const float* __restrict__ beta,
                               int C, uint32_t* __restrict__ rec) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * kRecWords) return;
  const int64_t j = t / kRecWords;
  const int w = static_cast<int>(t % kRecWords);
  uint32_t hw[4] = {0, 0, 0, 0};
  for (int q = 0; q < hspw; ++q) hw[q] = __ldg(h + j * hspw + q);
  if (w < 4) {  // h word w
    rec[t] = hw[w];
    return;
  }
  const int ew = w - 4;  // q word: classes 4ew .. 4ew+3
  uint32_t out = 0;
  for (int b = 0; b < 4; ++b) {
    const int k = 4 * ew + b;
    if (k >= C) break;
    int diff = 0;
    for (int q = 0; q < hspw; ++q) diff += __popc(hw[q] ^ __ldg(wt + k * hspw + q));
    const float fd = static_cast<float>(K - 2 * diff);  // exact
    const float bk = __ldg(beta + k);
    const float x = __fmul_rn(fd, bk);
    const float e = __fmaf_rn(fd, bk, -x);  // exact rounding error of the product
    // 2u = 2^(exponent(b) - 22): scale e to an exact integer in [-32, 32]
    const int ex = ((__float_as_int(bk) >> 23) & 0xFF) - 127;
    const float inv2u = __int_as_float((127 + 22 - ex) << 23);
    const int q = __float2int_rn(e * inv2u);
    out |= static_cast<uint32_t>(q + 32) << (8 * b);
  }
  rec[t] = out;
}

template <int NP>
__global__ void __launch_bounds__(kFWarps * 32)
    k_gcn1_aggregate(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                     const uint16_t* __restrict__ ti, int64_t tr0, int64_t trows, int64_t rows,
                     const int32_t* __restrict__ degree, const uint32_t* __restrict__ rec,
                     const uint32_t* __restrict__ wt, int hspw, int K,
                     const float* __restrict__ beta, int C, float* __restrict__ logits,
                     float* __restrict__ probs) {
  constexpr int G = 16, S = 2, B = 8 * S;
  constexpr int NQ = NP + 1;
  __shared__ uint32_t ring_all[kFWarps][4][kRing];
  __shared__ uint32_t planes_all[kFWarps][4][NQ];  // reduced h-count planes, 4 words
  __shared__ int esum_all[kFWarps][48];
  __shared__ uint32_t wt_s[48 * 4];
  for (int i = threadIdx.x; i < C * hspw; i += blockDim.x) wt_s[i] = wt[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane % G, slot = lane / G;
  uint32_t(*ring)[kRing] = ring_all[warp];
  const uint32_t* rw = rec + g;
  const bool hlane = g < 4;
  (void)degree;

  for (int64_t tr = tr0 + static_cast<int64_t>(blockIdx.x) * kFWarps + warp; tr < trows;
       tr += static_cast<int64_t>(gridDim.x) * kFWarps) {
    uint32_t P[4][NP];
    uint32_t alo[4], ahi[4];
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      alo[n] = ahi[n] = 0;
#pragma unroll
      for (int q = 0; q < NP; ++q) P[n][q] = 0;
    }
    auto drain = [&](auto nc, uint32_t hd, uint32_t cnt) {
      constexpr int n = decltype(nc)::value;
      uint32_t xv[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const uint32_t e = static_cast<uint32_t>(slot + S * m);
        xv[m] = 0;
        if (e < cnt) xv[m] = __ldg(rw + ring[n][(hd + e) & (kRing - 1)] * kRecWords);
      }
      if (hlane) {
        hs_add8<NP>(P[n], xv);
      } else {
        // q bytes are <= 64: three words add byte-wise without carries, then
        // bytes 0,2 and 1,3 go into 16-bit lanes.
        const uint32_t a = xv[0] + xv[1] + xv[2], b = xv[3] + xv[4] + xv[5], c = xv[6] + xv[7];
        alo[n] += (a & 0x00FF00FFu) + (b & 0x00FF00FFu) + (c & 0x00FF00FFu);
        ahi[n] += ((a >> 8) & 0x00FF00FFu) + ((b >> 8) & 0x00FF00FFu) + ((c >> 8) & 0x00FF00FFu);
      }
    };
    uint32_t fill[4];
    walk_tile_row<B>(rp, ci, ti, tr, ring, fill, drain);

#pragma unroll
    for (int n = 0; n < 4; ++n) {
      // h planes: sum the two slots; q sums: sum the two slots.
      uint32_t Q[NQ];
      slot_reduce<G, NP, NQ>(P[n], Q);
      const uint32_t lo = alo[n] + __shfl_xor_sync(0xFFFFFFFFu, alo[n], 16);
      const uint32_t hi = ahi[n] + __shfl_xor_sync(0xFFFFFFFFu, ahi[n], 16);
      const int64_t row = 4 * tr + n;
      const int deg = static_cast<int>(fill[n]);
      if (slot == 0) {
        if (hlane) {
#pragma unroll
          for (int q = 0; q < NQ; ++q) planes_all[warp][g][q] = Q[q];
        } else {
          const int k0 = 4 * (g - 4);
          const int bias = 32 * deg;
          esum_all[warp][k0 + 0] = static_cast<int>(lo & 0xFFFFu) - bias;
          esum_all[warp][k0 + 1] = static_cast<int>(hi & 0xFFFFu) - bias;
          esum_all[warp][k0 + 2] = static_cast<int>(lo >> 16) - bias;
          esum_all[warp][k0 + 3] = static_cast<int>(hi >> 16) - bias;
        }
      }
      __syncwarp();
      if (row >= rows) {
        __syncwarp();
        continue;
      }
      // Per class: sum_j dot_jk = sum_b w+-_bk (2 cnt_b - deg)
      //          = 2*(2*sum_b [w_bk] cnt_b - sum_b cnt_b) - deg*(2*popc(w_k) - K)
      // with sum_b [mask_b] cnt_b = sum_q 2^q popc(mask & Q_q).
      float lg[2];
      double mx = -INFINITY;
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        const int k = lane + 32 * pass;
        lg[pass] = -INFINITY;
        if (k < C) {
          int64_t sw = 0, sall = 0;
          int wpop = 0;
          for (int w = 0; w < hspw; ++w) {
            const uint32_t wk = wt_s[k * hspw + w];
            wpop += __popc(wk);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              const uint32_t pl = planes_all[warp][w][q];
              sw += static_cast<int64_t>(__popc(wk & pl)) << q;
              sall += static_cast<int64_t>(__popc(pl)) << q;
            }
          }
          // wt holds the transposed +-1 weight bits; padding bits are zero in
          // both wt and h, so only the K real features contribute.
          const int64_t sdot = 2 * (2 * sw - sall) - static_cast<int64_t>(deg) * (2 * wpop - K);
          const float bk = beta[k];
          const int ex = ((__float_as_int(bk) >> 23) & 0xFF) - 127;
          const double two_u = ldexp(1.0, ex - 22);
          const double v = __dsub_rn(__dmul_rn(static_cast<double>(bk), static_cast<double>(sdot)),
                                     __dmul_rn(two_u, static_cast<double>(esum_all[warp][k])));
          lg[pass] = __double2float_rn(v);
          if (logits) logits[row * C + k] = lg[pass];
          mx = fmax(mx, static_cast<double>(lg[pass]));
        }
      }
      if (probs) {
        for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
        double ex0 = lane < C ? exp(static_cast<double>(lg[0]) - mx) : 0.0;
        double ex1 = lane + 32 < C ? exp(static_cast<double>(lg[1]) - mx) : 0.0;
        double sum = ex0 + ex1;
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
        if (lane < C) probs[row * C + lane] = __double2float_rn(ex0 / sum);
        if (lane + 32 < C) probs[row * C + lane + 32] = __double2float_rn(ex1 / sum);
      }
      __syncwarp();
    }
  }
}

}  // namespace

bool gcn1_fused_supported(const bg_frdc& A, int64_t K, int wb, int64_t C) {
  const int64_t hspw = spw(K, wb);
  // 16-bit SWAR q sums hold 64*count; with 2 slots a lane sees <= deg/2+8 edges.
  return K % 2 == 0 && K <= 128 && hspw <= 4 && C >= 1 && C <= 48 &&
         (A.max_deg + 16) * 64 < 65536 && A.rows * kRecWords < (int64_t{1} << 32);
}

void gcn1_records(const uint32_t* h, int64_t n, int64_t K, int wb, const uint32_t* wt,
                  const float* beta, int64_t C, uint32_t* rec_buf, cudaStream_t s) {
  if (use_slivers()) return sliver_gcn1_records(h, n, K, wb, wt, beta, C, rec_buf, s);
  const int hspw = static_cast<int>(spw(K, wb));
  k_gcn1_records<<<static_cast<unsigned>(cdiv(n * kRecWords, 256)), 256, 0, s>>>(
      h, n, hspw, static_cast<int>(K), wt, beta, static_cast<int>(C), rec_buf);
  BG_LAUNCH_CHECK();
}

void gcn1_aggregate(const bg_frdc& A, const uint32_t* rec_buf, int64_t K, int wb,
                    const uint32_t* wt, const float* beta, int64_t C, float* logits, float* probs,
                    cudaStream_t s, int64_t row0, int64_t row1) {
  if (use_slivers())
    return sliver_gcn1_aggregate(const_cast<bg_frdc&>(A), rec_buf, K, wb, wt, beta, C, logits, probs, s, row0, row1);
  if (row1 < 0) row1 = A.rows;
  const int64_t t0 = row0 / 4, t1 = (row1 + 3) / 4;
  if (t1 <= t0) return;
  const int hspw = static_cast<int>(spw(K, wb));
  const int64_t blocks = std::max<int64_t>(
      1, std::min<int64_t>(cdiv(t1 - t0, kFWarps), static_cast<int64_t>(sm_count()) * 64));
  const int64_t per_lane = (A.max_deg + 15) / 16 * 8;  // ring deals edges to 2 slots
  auto go = [&](auto kern) {
    kern<<<static_cast<unsigned>(blocks), kFWarps * 32, 0, s>>>(
        A.rp(), A.ci(), A.ti(), t0, t1, A.rows, A.deg(), rec_buf, wt, hspw,
        static_cast<int>(K), beta, static_cast<int>(C), logits, probs);
  };
  if (per_lane < (1 << 7)) go(k_gcn1_aggregate<7>);
  else if (per_lane < (1 << 8)) go(k_gcn1_aggregate<8>);
  else if (per_lane < (1 << 10)) go(k_gcn1_aggregate<10>);
  else go(k_gcn1_aggregate<13>);
  BG_LAUNCH_CHECK();
}

}  // namespace bg
