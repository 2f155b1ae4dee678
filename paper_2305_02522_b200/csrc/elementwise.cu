// Small glue kernels of the layer chain: ADD variants, ReLU, softmax, SAGE
// mean fix-up, BatchNorm, SCL, dense MM.FFF and CONCAT.
// ref: kernels.cpp:193-212, :560-668; graphops.cpp:89-97, :304-314, :337-386.
#include <cstdlib>
#include <algorithm>

#include "ops.cuh"

namespace bg {
namespace {

unsigned grid1(int64_t n, int bs = 256) { return static_cast<unsigned>(cdiv(n, bs)); }

__device__ __forceinline__ uint32_t bit_of(const uint32_t* b, int64_t spw, int64_t i, int64_t j) {
  return (b[i * spw + (j >> 5)] >> (31 - (j & 31))) & 1u;
}

// ADD.BBB: (-1,-1) is the only negative sum, so the threshold is OR (:609-616).
__global__ void k_or(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, int64_t n,
                     uint32_t* __restrict__ o) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) o[t] = a[t] | b[t];
}

// ADD.BBF: 2*(a+b) - 2 over 0/1 bits (:618-624).
// ADD.BBF: 2*(a+b) - 2 per element (kernels.cpp:608-616), optionally with the
// layer's ReLU fused (graphops.cpp:89-97: x > 0 ? x : 0).  Thread per (row,
// 32-column word): two word loads, 32 floats out (float4 stores when the row
// start is 16-byte aligned).
template <bool RELU>
__global__ void k_add_bbf(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                          int64_t rows, int64_t cols, int64_t spw, float* __restrict__ o) {
  const int64_t wpr = (cols + 31) >> 5;  // 32-column words per row
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * wpr) return;
  const int64_t i = t / wpr, w = t - i * wpr;
  const uint32_t wa = a[i * spw + w], wb = b[i * spw + w];
  float* orow = o + i * cols;
  const int64_t c0 = 32 * w, n = cols - c0 < 32 ? cols - c0 : 32;
  auto val = [&](int q) {
    const float v = static_cast<float>(2 * static_cast<int>(((wa >> (31 - q)) & 1u) + ((wb >> (31 - q)) & 1u)) - 2);
    return RELU ? (v > 0.0f ? v : 0.0f) : v;
  };
  if (n == 32 && (reinterpret_cast<uintptr_t>(orow + c0) & 15) == 0) {
    float4* o4 = reinterpret_cast<float4*>(orow + c0);
#pragma unroll
    for (int q = 0; q < 8; ++q) o4[q] = make_float4(val(4 * q), val(4 * q + 1), val(4 * q + 2), val(4 * q + 3));
  } else {
    for (int q = 0; q < n; ++q) orow[c0 + q] = val(q);
  }
}

// ADD.FFF: float(double(a) + b) (:603-607), optionally with the ReLU fused;
// four elements per thread.
template <bool RELU>
__global__ void k_add_fff(const float* __restrict__ a, const float* __restrict__ b, int64_t n,
                          float* __restrict__ o) {
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  auto one = [](float x, float y) {
    const float v = __double2float_rn(__dadd_rn(static_cast<double>(x), static_cast<double>(y)));
    return RELU ? (v > 0.0f ? v : 0.0f) : v;
  };
  if (t + 4 <= n) {
    const float4 x = *reinterpret_cast<const float4*>(a + t), y = *reinterpret_cast<const float4*>(b + t);
    *reinterpret_cast<float4*>(o + t) = make_float4(one(x.x, y.x), one(x.y, y.y), one(x.z, y.z), one(x.w, y.w));
  } else {
    for (int64_t k = t; k < n; ++k) o[k] = one(a[k], b[k]);
  }
}

template <bool RELU>  // unaligned operands: element per thread
__global__ void k_add_fff1(const float* __restrict__ a, const float* __restrict__ b, int64_t n,
                           float* __restrict__ o) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const float v = __double2float_rn(__dadd_rn(static_cast<double>(a[t]), static_cast<double>(b[t])));
  o[t] = RELU ? (v > 0.0f ? v : 0.0f) : v;
}

__global__ void k_relu(float* __restrict__ x, int64_t n) {
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  auto r = [](float v) { return v > 0.0f ? v : 0.0f; };
  if (t + 4 <= n) {
    float4 v = *reinterpret_cast<float4*>(x + t);
    *reinterpret_cast<float4*>(x + t) = make_float4(r(v.x), r(v.y), r(v.z), r(v.w));
  } else {
    for (int64_t k = t; k < n; ++k) x[k] = r(x[k]);
  }
}

__global__ void k_relu1(float* __restrict__ x, int64_t n) {  // unaligned fallback
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) x[t] = x[t] > 0.0f ? x[t] : 0.0f;
}

// Row softmax in double, sequential column order (graphops.cpp:372-386).
// A warp owns kSmRows consecutive rows = one contiguous chunk of
// kSmRows*cols floats: it stages the chunk into shared memory with
// independent float4 loads, takes the row maxima lane per row, computes
// every exp(x - max) once element-parallel into a double buffer (row =
// element / cols by a magic multiply), sums each row lane per row in column
// order, and writes exp * (1/sum) back through float4 stores.
constexpr int kSmWarps = 2;  // 24 KB of staging per block
constexpr int kSmMaxCols = 64;
constexpr int kSmRows = 16;
__global__ void __launch_bounds__(kSmWarps * 32)
    k_softmax_staged(const float* __restrict__ x, int64_t rows, int cols, uint32_t cmagic, float* __restrict__ o) {
  __shared__ __align__(16) float buf[kSmWarps][kSmRows * kSmMaxCols];
  __shared__ double ebuf[kSmWarps][kSmRows * kSmMaxCols];
  __shared__ double rmx[kSmWarps][kSmRows], rinv[kSmWarps][kSmRows];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* b = buf[warp];
  double* e = ebuf[warp];
  for (int64_t r0 = (static_cast<int64_t>(blockIdx.x) * kSmWarps + warp) * kSmRows; r0 < rows;
       r0 += static_cast<int64_t>(gridDim.x) * kSmWarps * kSmRows) {
    const int nr = static_cast<int>(rows - r0 < kSmRows ? rows - r0 : kSmRows);
    const int n = nr * cols, n4 = n >> 2;
    const float* src = x + r0 * cols;  // 16-byte aligned: r0*cols is a multiple of 4*kSmRows
    const float4* src4 = reinterpret_cast<const float4*>(src);
    float4* b4 = reinterpret_cast<float4*>(b);
#pragma unroll 4
    for (int t = lane; t < n4; t += 32) b4[t] = __ldg(src4 + t);
    for (int t = 4 * n4 + lane; t < n; t += 32) b[t] = __ldg(src + t);
    __syncwarp();
    if (lane < nr) {
      const float* xr = b + lane * cols;
      float mx = -INFINITY;  // exact in float; NaN is skipped like std::max(mx, x) does
      for (int j = 0; j < cols; ++j) mx = fmaxf(mx, xr[j]);
      rmx[warp][lane] = static_cast<double>(mx);
    }
    __syncwarp();
#pragma unroll 4
    for (int t = lane; t < n; t += 32) {
      const uint32_t r = __umulhi(static_cast<uint32_t>(t), cmagic);  // t / cols
      e[t] = exp_nonpos(static_cast<double>(b[t]) - rmx[warp][r]);
    }
    __syncwarp();
    if (lane < nr) {
      const double* er = e + lane * cols;
      double sum = 0.0;
      for (int j = 0; j < cols; ++j) sum = __dadd_rn(sum, er[j]);
      rinv[warp][lane] = __drcp_rn(sum);
    }
    __syncwarp();
#pragma unroll 4
    for (int t = lane; t < n; t += 32) {
      const uint32_t r = __umulhi(static_cast<uint32_t>(t), cmagic);
      b[t] = __double2float_rn(__dmul_rn(e[t], rinv[warp][r]));
    }
    __syncwarp();
    float* dst = o + r0 * cols;
    float4* dst4 = reinterpret_cast<float4*>(dst);
#pragma unroll 4
    for (int t = lane; t < n4; t += 32) dst4[t] = b4[t];
    for (int t = 4 * n4 + lane; t < n; t += 32) dst[t] = b[t];
    __syncwarp();
  }
}

// Row softmax, lane per row with the row's exps in registers (cols <= CM):
// a warp stages 32 consecutive rows (one contiguous chunk) into shared memory
// with coalesced loads, each lane takes its row's maximum, its exps (kept in
// registers: independent, so they pipeline), their sum in column order and
// exp / sum -- the reference's operations and order (graphops.cpp:372-386)
// -- into the staging buffer, which goes out with coalesced stores.
constexpr int kSlRows = 32;
template <int CM>
__global__ void __launch_bounds__(128)
    k_softmax_lane(const float* __restrict__ x, int64_t rows, int cols, float* __restrict__ o) {
  __shared__ float buf[4][kSlRows * CM + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* b = buf[warp];
  for (int64_t r0 = (static_cast<int64_t>(blockIdx.x) * 4 + warp) * kSlRows; r0 < rows;
       r0 += static_cast<int64_t>(gridDim.x) * 4 * kSlRows) {
    const int nr = static_cast<int>(rows - r0 < kSlRows ? rows - r0 : kSlRows);
    const int n = nr * cols;
    const float* src = x + r0 * cols;
#pragma unroll 4
    for (int t = lane; t < n; t += 32) b[t] = __ldg(src + t);
    __syncwarp();
    if (lane < nr) {
      float* xr = b + lane * cols;  // stride cols words: conflict-free for odd cols
      double mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < CM; ++j)
        if (j < cols) mx = fmax(mx, static_cast<double>(xr[j]));  // NaN skipped, as std::max(mx, x)
      double e[CM];
#pragma unroll
      for (int j = 0; j < CM; ++j) e[j] = j < cols ? exp_nonpos(static_cast<double>(xr[j]) - mx) : 0.0;
      double sum = 0.0;
#pragma unroll
      for (int j = 0; j < CM; ++j)
        if (j < cols) sum = __dadd_rn(sum, e[j]);
#pragma unroll
      for (int j = 0; j < CM; ++j)
        if (j < cols) xr[j] = __double2float_rn(__ddiv_rn(e[j], sum));
    }
    __syncwarp();
    float* dst = o + r0 * cols;
#pragma unroll 4
    for (int t = lane; t < n; t += 32) dst[t] = b[t];
    __syncwarp();
  }
}

__global__ void k_softmax(const float* __restrict__ x, int64_t rows, int64_t cols,
                          float* __restrict__ o) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const float* xr = x + i * cols;
  double mx = -INFINITY;
  for (int64_t j = 0; j < cols; ++j) mx = fmax(mx, static_cast<double>(xr[j]));
  double sum = 0.0;
  for (int64_t j = 0; j < cols; ++j) sum = __dadd_rn(sum, exp(static_cast<double>(xr[j]) - mx));
  for (int64_t j = 0; j < cols; ++j)
    o[i * cols + j] = __double2float_rn(__ddiv_rn(exp(static_cast<double>(xr[j]) - mx), sum));
}

// SAGE mean fix-up on a summed aggregate: float(r * (1/max(1,cnt))) in double
// (graphops.cpp:304-314).
__global__ void k_scale_rows(float* __restrict__ x, int64_t rows, int64_t cols,
                             const int64_t* __restrict__ cnt) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * cols) return;
  const int64_t c = cnt[t / cols];
  const double inv = __ddiv_rn(1.0, static_cast<double>(c > 1 ? c : 1));
  x[t] = __double2float_rn(__dmul_rn(static_cast<double>(x[t]), inv));
}

// gamma*(x-mean)/max(sigma,1e-12) + beta in double (graphops.cpp:337-355).
__global__ void k_bn(const float* __restrict__ x, int64_t rows, int64_t cols,
                     const float* __restrict__ g, const float* __restrict__ b,
                     const float* __restrict__ m, const float* __restrict__ sg,
                     float* __restrict__ o) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * cols) return;
  const int64_t j = t % cols;
  const double sigma = fmax(static_cast<double>(sg[j]), 1e-12);
  const double num = __dmul_rn(static_cast<double>(g[j]),
                               __dsub_rn(static_cast<double>(x[t]), static_cast<double>(m[j])));
  o[t] = __double2float_rn(__dadd_rn(__ddiv_rn(num, sigma), static_cast<double>(b[j])));
}

// BatchNorm [ReLU] [binarize] fused: floats out, or warp per (row, word)
// with lanes over columns and one ballot per packed word.
__global__ void k_bn_act_f(const float* __restrict__ x, int64_t n, int64_t cols, const FEpi e, float* __restrict__ o) {
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    o[t] = fepi_apply(e, x[t], t % cols);
}
__global__ void k_bn_act_b(const float* __restrict__ x, int64_t rows, int64_t cols, const FEpi e) {
  const int64_t words = (cols + 31) / 32;
  const int lane = threadIdx.x & 31;
  for (int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < rows * words;
       w += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t i = w / words, k = 32 * (w % words) + lane;
    fepi_store_lane(e, nullptr, i, cols, k, k < cols ? x[i * cols + k] : 0.0f);
    if (lane == 0 && w % words == words - 1)
      for (int64_t p = words; p < e.bspw; ++p) e.bits[i * e.bspw + p] = 0u;  // 64-bit word padding
  }
}

// x * row[i] * col[j] in double, left to right (kernels.cpp:560-571).
__global__ void k_scl(const float* __restrict__ x, int64_t rows, int64_t cols,
                      const float* __restrict__ r, const float* __restrict__ c,
                      float* __restrict__ o) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * cols) return;
  const int64_t i = t / cols, j = t % cols;
  o[t] = __double2float_rn(__dmul_rn(__dmul_rn(static_cast<double>(r[i]), static_cast<double>(x[t])),
                                     static_cast<double>(c[j])));
}

// MM.FFF: double accumulation in k order (kernels.cpp:193-212).
__global__ void k_dense_mm(const float* __restrict__ a, const float* __restrict__ w, int64_t rows,
                           int64_t k, int64_t cols, float* __restrict__ o) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * cols) return;
  const int64_t i = t / cols, j = t % cols;
  double acc = 0.0;
  for (int64_t kk = 0; kk < k; ++kk)
    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(a[i * k + kk]), static_cast<double>(w[kk * cols + j])));
  o[t] = __double2float_rn(acc);
}

// CONCAT.BBB: bit-contiguous repack, one thread per output word (:648-667).
__global__ void k_concat_bits(const uint32_t* __restrict__ a, int64_t ca,
                              const uint32_t* __restrict__ b, int64_t cb, int64_t rows,
                              int64_t sa, int64_t sb, int64_t so, uint32_t* __restrict__ o) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * so) return;
  const int64_t i = t / so, w = t % so;
  uint32_t v = 0;
  for (int q = 0; q < 32; ++q) {
    const int64_t j = 32 * w + q;
    uint32_t bit = 0;
    if (j < ca) bit = bit_of(a, sa, i, j);
    else if (j < ca + cb) bit = bit_of(b, sb, i, j - ca);
    v |= bit << (31 - q);
  }
  o[t] = v;
}

__global__ void k_concat_f(const float* __restrict__ a, int64_t ca, const float* __restrict__ b,
                           int64_t cb, int64_t rows, float* __restrict__ o) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t c = ca + cb;
  if (t >= rows * c) return;
  const int64_t i = t / c, j = t % c;
  o[t] = j < ca ? a[i * ca + j] : b[i * cb + (j - ca)];
}

}  // namespace

void add_bbb(const uint32_t* a, const uint32_t* b, int64_t words, uint32_t* out, cudaStream_t s) {
  if (words == 0) return;
  k_or<<<grid1(words), 256, 0, s>>>(a, b, words, out);
  BG_LAUNCH_CHECK();
}

void add_bbf(const uint32_t* a, const uint32_t* b, int64_t rows, int64_t cols, int wb, float* out,
             cudaStream_t s, bool fuse_relu) {
  if (rows * cols == 0) return;
  const int64_t threads = rows * ((cols + 31) / 32);
  if (fuse_relu)
    k_add_bbf<true><<<grid1(threads), 256, 0, s>>>(a, b, rows, cols, spw(cols, wb), out);
  else
    k_add_bbf<false><<<grid1(threads), 256, 0, s>>>(a, b, rows, cols, spw(cols, wb), out);
  BG_LAUNCH_CHECK();
}

void add_fff(const float* a, const float* b, int64_t n, float* out, cudaStream_t s, bool fuse_relu) {
  if (n == 0) return;
  const bool v4 = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                    reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  const int64_t threads = cdiv(n, 4);
  if (v4) {
    if (fuse_relu) k_add_fff<true><<<grid1(threads), 256, 0, s>>>(a, b, n, out);
    else k_add_fff<false><<<grid1(threads), 256, 0, s>>>(a, b, n, out);
  } else {
    if (fuse_relu) k_add_fff1<true><<<grid1(n), 256, 0, s>>>(a, b, n, out);
    else k_add_fff1<false><<<grid1(n), 256, 0, s>>>(a, b, n, out);
  }
  BG_LAUNCH_CHECK();
}

void relu(float* x, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) k_relu<<<grid1(cdiv(n, 4)), 256, 0, s>>>(x, n);
  else k_relu1<<<grid1(n), 256, 0, s>>>(x, n);
  BG_LAUNCH_CHECK();
}

void softmax_rows(const float* x, int64_t rows, int64_t cols, float* out, cudaStream_t s) {
  if (rows == 0) return;
  // narrow rows (Flickr's 7 classes: 10 vs 14 us): lane per row; wider rows
  // keep the element-parallel staged kernel (Reddit's 41: 58 vs 128 us --
  // 41 exps and divisions per lane at 139 registers)
  if (cols >= 1 && cols <= 16 && x != out && std::getenv("BG_SOFTMAX_STAGED") == nullptr) {
    auto go = [&](auto kern) {
      const int64_t blocks = std::min<int64_t>(cdiv(rows, 4 * kSlRows), static_cast<int64_t>(sm_count()) * 16);
      kern<<<static_cast<unsigned>(blocks), 128, 0, s>>>(x, rows, static_cast<int>(cols), out);
    };
    if (cols <= 8) go(k_softmax_lane<8>);
    else go(k_softmax_lane<16>);
    BG_LAUNCH_CHECK();
    return;
  }
  if (cols >= 2 && cols <= kSmMaxCols && x != out && reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(out) % 16 == 0) {
    // t / cols == umulhi(t, ceil(2^32 / cols)) for t < kSmRows cols (error kSmRows cols^2 < 2^32)
    const uint32_t cmagic = static_cast<uint32_t>(((uint64_t{1} << 32) + cols - 1) / cols);
    const int64_t blocks = std::min<int64_t>(cdiv(rows, kSmWarps * kSmRows), static_cast<int64_t>(sm_count()) * 32);
    k_softmax_staged<<<static_cast<unsigned>(blocks), kSmWarps * 32, 0, s>>>(x, rows, static_cast<int>(cols),
                                                                            cmagic, out);
  } else {
    k_softmax<<<grid1(rows, 128), 128, 0, s>>>(x, rows, cols, out);
  }
  BG_LAUNCH_CHECK();
}

void scale_rows_double(float* x, int64_t rows, int64_t cols, const int64_t* cnt, cudaStream_t s) {
  if (rows * cols == 0) return;
  k_scale_rows<<<grid1(rows * cols), 256, 0, s>>>(x, rows, cols, cnt);
  BG_LAUNCH_CHECK();
}

void batchnorm(const float* x, int64_t rows, int64_t cols, const float* g, const float* b,
               const float* m, const float* sg, float* out, cudaStream_t s) {
  if (rows * cols == 0) return;
  k_bn<<<grid1(rows * cols), 256, 0, s>>>(x, rows, cols, g, b, m, sg, out);
  BG_LAUNCH_CHECK();
}

void bn_act(const float* x, int64_t rows, int64_t cols, const FEpi& e, float* out_f, cudaStream_t s) {
  if (rows * cols == 0) return;
  if (e.bits) k_bn_act_b<<<grid1(rows * ((cols + 31) / 32) * 32), 256, 0, s>>>(x, rows, cols, e);
  else k_bn_act_f<<<grid1(rows * cols), 256, 0, s>>>(x, rows * cols, cols, e, out_f);
  BG_LAUNCH_CHECK();
}

void scl(const float* x, int64_t rows, int64_t cols, const float* r, const float* c, float* out,
         cudaStream_t s) {
  if (rows * cols == 0) return;
  k_scl<<<grid1(rows * cols), 256, 0, s>>>(x, rows, cols, r, c, out);
  BG_LAUNCH_CHECK();
}

void dense_mm(const float* a, const float* w, int64_t rows, int64_t k, int64_t cols, float* out,
              cudaStream_t s) {
  if (rows * cols == 0) return;
  k_dense_mm<<<grid1(rows * cols), 256, 0, s>>>(a, w, rows, k, cols, out);
  BG_LAUNCH_CHECK();
}

void concat_bits(const uint32_t* a, int64_t ca, const uint32_t* b, int64_t cb, int64_t rows,
                 int wb, uint32_t* out, cudaStream_t s) {
  const int64_t so = spw(ca + cb, wb);
  if (rows * so == 0) return;
  k_concat_bits<<<grid1(rows * so), 256, 0, s>>>(a, ca, b, cb, rows, spw(ca, wb), spw(cb, wb), so,
                                                 out);
  BG_LAUNCH_CHECK();
}

void concat_f(const float* a, int64_t ca, const float* b, int64_t cb, int64_t rows, float* out,
              cudaStream_t s) {
  if (rows * (ca + cb) == 0) return;
  k_concat_f<<<grid1(rows * (ca + cb)), 256, 0, s>>>(a, ca, b, cb, rows, out);
  BG_LAUNCH_CHECK();
}

}  // namespace bg
