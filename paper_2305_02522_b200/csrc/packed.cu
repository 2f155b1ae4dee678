// Two-valued activations kept packed (SURVEY.md §7 "hard parts" 7).
//
// A SAGE / GraphConv layer whose ADD is BBF with the layer's ReLU produces
// ReLU(2(a + b) - 2) with a, b in {0, 1} (kernels.cpp:619-624,
// graphops.cpp:319): exactly 2 where a AND b, else 0.  The engine keeps that
// F tensor as its bit pattern (an Op with pval = 2: value = bit ? 2 : 0,
// 1/32 of the fp32 bytes) and the consumers read the values from the bits:
//   * binarize (x >= 0, bitdense.cpp:83) of {0, 2} is all ones, so an
//     F-input product sees the all-ones row: dot_k = 2 popc(w_k) - K for
//     every row;
//   * its row scale (binarize_with_scale, bitdense.cpp:90-104) is the double
//     sum of the row's |x| = 2 c (c = set bits, exact), / K, floored at
//     1e-12, as float -- bit for bit the reference's value;
// so MM.FBB / FFB rows are one constant pattern and MM.FBF is
// float((alpha_i dot_k) beta_k) (kernels.cpp:179-190) from one popcount per
// row, optionally with the following row softmax (graphops.cpp:372-386) in
// the same pass.  Any other consumer materializes the fp32 tensor first.
#include <cstdlib>

#include "ops.cuh"

namespace bg {
namespace {

constexpr int kPackedMaxCols = 64;  // fused softmax: one row's logits in registers

__global__ void k_and_words(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, int64_t n,
                            uint32_t* __restrict__ o) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    o[t] = a[t] & b[t];
}

// value = bit ? pval : 0, row-major fp32 (packed rows of spw u32 words)
__global__ void k_expand(const uint32_t* __restrict__ bits, int64_t rows, int64_t cols, int64_t spw, float pval,
                         float* __restrict__ o) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < rows * cols;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = t / cols, j = t - i * cols;
    o[t] = (bits[i * spw + (j >> 5)] >> (31 - (j & 31))) & 1u ? pval : 0.0f;
  }
}

// The all-ones input row against the transposed weight bits: word w of the
// output pattern (dot_k = 2 popc(w_k) - K >= 0, kernels.cpp:166-171), then
// every row of the result gets the pattern (ospw <= 64 words).
__global__ void k_const_rows(const uint32_t* __restrict__ wt, int64_t k, int64_t n, int64_t kspw, int ospw,
                             int64_t rows, uint32_t* __restrict__ out) {
  __shared__ uint32_t pat[64];
  // lane per column, a warp per 32-column word: ballot + brev packs MSB-first
  const int lane = threadIdx.x & 31;
  for (int w = threadIdx.x >> 5; w < ospw; w += blockDim.x >> 5) {
    const int64_t col = 32 * static_cast<int64_t>(w) + lane;
    bool bit = false;
    if (col < n) {
      int64_t pc = 0;
      for (int64_t q = 0; q < kspw; ++q) pc += __popc(__ldg(wt + col * kspw + q));
      bit = 2 * pc - k >= 0;
    }
    const uint32_t word = __brev(__ballot_sync(0xFFFFFFFFu, bit));
    if (lane == 0) pat[w] = word;
  }
  __syncthreads();
  if ((ospw & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {  // 16-byte stores
    const int q4 = ospw >> 2;
    const int64_t total4 = rows * q4;
    uint4* o4 = reinterpret_cast<uint4*>(out);
    if (q4 == 1) {  // one 16-byte word per row (hidden 128)
      const uint4 v = make_uint4(pat[0], pat[1], pat[2], pat[3]);
      for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total4;
           t += static_cast<int64_t>(gridDim.x) * blockDim.x)
        o4[t] = v;
      return;
    }
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total4;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int w = 4 * static_cast<int>(t % q4);
      o4[t] = make_uint4(pat[w], pat[w + 1], pat[w + 2], pat[w + 3]);
    }
    return;
  }
  const int64_t total = rows * ospw;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[t] = pat[t % ospw];
}

// MM.FBF on a packed input.  A row's logits depend on the row only through
// its scale alpha, i.e. through c = popc(row) in [0, K]: the K+1 distinct
// logit rows (and their softmax rows) are computed once (one thread per c,
// the reference's arithmetic), and every output element is a table lookup --
// the pass is bound by writing the outputs.
// Warp per c: the lanes take the columns j = lane, lane + 32, ... of row c
// (logits in parallel; a column's popcount does not depend on c), the max by
// a warp reduction (order-free), then the softmax sum in the reference's
// sequential column order -- each exp broadcast from its lane and added in
// turn -- and the probabilities in parallel again.
constexpr int kTabWarps = 4;
__global__ void __launch_bounds__(kTabWarps * 32)
    k_fbf_table(int64_t k, double pval, const uint32_t* __restrict__ wt, int64_t kspw,
                const float* __restrict__ beta, int64_t n, int want_probs, float* __restrict__ tab_logits,
                float* __restrict__ tab_probs) {
  const int lane = threadIdx.x & 31;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * kTabWarps + (threadIdx.x >> 5);
  if (c > k) return;  // warp-uniform
  // binarize_with_scale row scale (bitdense.cpp:95-102): sum |x| in double
  // (pval c, exact for pval = 2), / cols, floor 1e-12, float
  double s = pval * static_cast<double>(c);
  s = s / static_cast<double>(k);
  const double a = static_cast<double>(static_cast<float>(s > 1e-12 ? s : 1e-12));
  float* yl = tab_logits + c * n;
  float mx = -INFINITY;
  for (int64_t j = lane; j < n; j += 32) {
    int64_t pc = 0;
    for (int64_t q = 0; q < kspw; ++q) pc += __popc(__ldg(wt + j * kspw + q));
    const double dot = static_cast<double>(2 * pc - k);  // the all-ones row against w_j
    // float((alpha dot) beta)  (kernels.cpp:179-190)
    yl[j] = __double2float_rn(__dmul_rn(__dmul_rn(a, dot), static_cast<double>(beta[j])));
    mx = fmaxf(mx, yl[j]);
  }
  if (!want_probs) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  // softmax_rows (graphops.cpp:372-386): double max, sequential double sum of
  // exp(x - max), float(exp(x - max) / sum)
  const double m = static_cast<double>(mx);
  double sum = 0.0;
  for (int64_t j0 = 0; j0 < n; j0 += 32) {
    const double ej = j0 + lane < n ? exp(static_cast<double>(yl[j0 + lane]) - m) : 0.0;
    const int cnt = static_cast<int>(n - j0 < 32 ? n - j0 : 32);
    for (int q = 0; q < cnt; ++q) sum = __dadd_rn(sum, __shfl_sync(0xFFFFFFFFu, ej, q));
  }
  for (int64_t j = lane; j < n; j += 32)
    tab_probs[c * n + j] = __double2float_rn(__ddiv_rn(exp(static_cast<double>(yl[j]) - m), sum));
}

// Block per kLookRows rows of [r0, r1): the rows' popcounts into shared
// memory as the offset of each row's table row from its output span
// (delta[r] = (popc_r - r) * n, so element e of the block's contiguous span
// reads table element e + delta[e / n]), then the span element by element
// (WL / WP: logits / probabilities wanted; V4: four consecutive elements and
// one 16-byte streaming store per output per thread).
constexpr int kLookRows = 256;
template <bool WL, bool WP, bool V4>
__global__ void __launch_bounds__(256) k_fbf_lookup(const uint32_t* __restrict__ bits, int64_t r0, int64_t r1,
                                                    int xspw, int n, uint32_t nmagic,
                                                    const float* __restrict__ tab_logits,
                                                    const float* __restrict__ tab_probs, float* __restrict__ logits,
                                                    float* __restrict__ probs) {
  __shared__ int delta[kLookRows];
  for (int64_t b0 = r0 + static_cast<int64_t>(blockIdx.x) * kLookRows; b0 < r1;
       b0 += static_cast<int64_t>(gridDim.x) * kLookRows) {
    const int nr = static_cast<int>(r1 - b0 < kLookRows ? r1 - b0 : kLookRows);
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < nr) {
      const uint32_t* row = bits + (b0 + threadIdx.x) * xspw;
      int c = 0;
      for (int q = 0; q < xspw; ++q) c += __popc(__ldg(row + q));
      delta[threadIdx.x] = (c - static_cast<int>(threadIdx.x)) * n;
    }
    __syncthreads();
    float* ol = logits + (WL ? b0 * n : 0);
    float* op = probs + (WP ? b0 * n : 0);
    const int total = nr * n;
    if (V4) {
      const int tail = total & ~3;  // the last (partial) block's 1-3 trailing elements: scalar, below
      if (static_cast<int>(threadIdx.x) < total - tail) {
        const int e = tail + threadIdx.x;
        const int src = e + delta[__umulhi(static_cast<uint32_t>(e), nmagic)];
        if (WL) ol[e] = __ldg(tab_logits + src);
        if (WP) op[e] = __ldg(tab_probs + src);
      }
      for (int e = 4 * static_cast<int>(threadIdx.x); e < tail; e += 4 * kLookRows) {
        int src[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)  // (e + i) / n by the magic multiply
          src[i] = e + i + delta[__umulhi(static_cast<uint32_t>(e + i), nmagic)];
        if (WL)
          __stcs(reinterpret_cast<float4*>(ol + e), make_float4(__ldg(tab_logits + src[0]), __ldg(tab_logits + src[1]),
                                                                __ldg(tab_logits + src[2]), __ldg(tab_logits + src[3])));
        if (WP)
          __stcs(reinterpret_cast<float4*>(op + e), make_float4(__ldg(tab_probs + src[0]), __ldg(tab_probs + src[1]),
                                                                __ldg(tab_probs + src[2]), __ldg(tab_probs + src[3])));
      }
    } else {
      for (int e = threadIdx.x; e < total; e += kLookRows) {
        const int src = e + delta[__umulhi(static_cast<uint32_t>(e), nmagic)];
        if (WL) ol[e] = __ldg(tab_logits + src);
        if (WP) op[e] = __ldg(tab_probs + src);
      }
    }
  }
}

int grid_n(int64_t n, int bs = 256) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cdiv(n, bs), 32LL * sm_count())));
}

}  // namespace

void and_words(const uint32_t* a, const uint32_t* b, int64_t n, uint32_t* out, cudaStream_t s) {
  if (n <= 0) return;
  k_and_words<<<grid_n(n), 256, 0, s>>>(a, b, n, out);
  BG_LAUNCH_CHECK();
}

void expand_packed(const uint32_t* bits, int64_t rows, int64_t cols, int wb, float pval, float* out, cudaStream_t s) {
  if (rows * cols <= 0) return;
  k_expand<<<grid_n(rows * cols), 256, 0, s>>>(bits, rows, cols, spw(cols, wb), pval, out);
  BG_LAUNCH_CHECK();
}

void packed_const_rows(const uint32_t* wt, int64_t k, int64_t n, int wb, int64_t rows, uint32_t* out,
                       cudaStream_t s) {
  if (spw(n, wb) > 64) fail("packed product: more than 2048 output columns");
  if (rows <= 0) return;
  k_const_rows<<<static_cast<unsigned>(std::min<int64_t>(cdiv(rows * spw(n, wb), 1024), 4LL * sm_count())), 256, 0,
                 s>>>(wt, k, n, spw(k, wb), static_cast<int>(spw(n, wb)), rows, out);
  BG_LAUNCH_CHECK();
}

bool packed_fbf_supported(int64_t n) { return n >= 1 && n <= kPackedMaxCols; }

size_t packed_fbf_table_bytes(int64_t k, int64_t n) { return static_cast<size_t>(2 * (k + 1) * n) * 4; }

void packed_fbf(const uint32_t* bits, int64_t r0, int64_t r1, int64_t k, int xwb, float pval, const uint32_t* wt,
                int wb, const float* beta, int64_t n, float* logits, float* probs, float* table, cudaStream_t s) {
  if (!packed_fbf_supported(n)) fail("packed product: unsupported output width");
  if (r1 <= r0) return;
  // the (K+1) x n tables (a few KB, caller's workspace) are rebuilt per call
  float* tl = table;
  float* tp = tl + (k + 1) * n;
  k_fbf_table<<<static_cast<unsigned>(cdiv(k + 1, kTabWarps)), kTabWarps * 32, 0, s>>>(
      k, static_cast<double>(pval), wt, spw(k, wb), beta, n, probs ? 1 : 0, tl, tp);
  BG_LAUNCH_CHECK();
  const int64_t blocks = std::min<int64_t>(cdiv(r1 - r0, kLookRows), 16LL * sm_count());
  // e / n == umulhi(e, ceil(2^32 / n)) for e < kLookRows * n (e * n < 2^32)
  const uint32_t nmagic = static_cast<uint32_t>(((uint64_t{1} << 32) + n - 1) / n);
  // 16-byte stores when every block's span starts 16-byte aligned (a full
  // block is kLookRows * n floats; the last block's 1-3 odd elements go scalar)
  auto al16 = [](const float* p) { return p == nullptr || reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  const bool v4 = al16(logits ? logits + r0 * n : nullptr) && al16(probs ? probs + r0 * n : nullptr);
  const unsigned g = static_cast<unsigned>(blocks);
  const int xs = static_cast<int>(spw(k, xwb)), nn = static_cast<int>(n);
#define BG_LOOKUP(WL, WP, V4) \
  k_fbf_lookup<WL, WP, V4><<<g, kLookRows, 0, s>>>(bits, r0, r1, xs, nn, nmagic, tl, tp, logits, probs)
  if (logits && probs) {
    if (v4) BG_LOOKUP(true, true, true); else BG_LOOKUP(true, true, false);
  } else if (probs) {
    if (v4) BG_LOOKUP(false, true, true); else BG_LOOKUP(false, true, false);
  } else if (logits) {
    if (v4) BG_LOOKUP(true, false, true); else BG_LOOKUP(true, false, false);
  }
#undef BG_LOOKUP
  BG_LAUNCH_CHECK();
}

}  // namespace bg
