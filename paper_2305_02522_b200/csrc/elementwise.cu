// Small glue kernels of the layer chain: ADD variants, ReLU, softmax, SAGE
// mean fix-up, BatchNorm, SCL, dense MM.FFF and CONCAT.
// ref: kernels.cpp:193-212, :560-668; graphops.cpp:89-97, :304-314, :337-386.
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
__global__ void k_add_bbf(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                          int64_t rows, int64_t cols, int64_t spw, float* __restrict__ o) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * cols) return;
  const int64_t i = t / cols, j = t % cols;
  o[t] = static_cast<float>(2 * static_cast<int>(bit_of(a, spw, i, j) + bit_of(b, spw, i, j)) - 2);
}

// ADD.FFF: float(double(a) + b) (:603-607).
__global__ void k_add_fff(const float* __restrict__ a, const float* __restrict__ b, int64_t n,
                          float* __restrict__ o) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) o[t] = __double2float_rn(__dadd_rn(static_cast<double>(a[t]), static_cast<double>(b[t])));
}

__global__ void k_relu(float* __restrict__ x, int64_t n) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) x[t] = x[t] > 0.0f ? x[t] : 0.0f;
}

// Row softmax in double, sequential column order (graphops.cpp:372-386).
// A warp stages 32 rows (contiguous) through shared memory with coalesced
// loads/stores.  The order-sensitive parts -- the row max and the sequential
// double sum -- run lane per row; exp(x - max) (cached as double, the value
// the reference recomputes identically) and the division run element-parallel.
constexpr int kSmWarps = 2;
constexpr int kSmMaxCols = 48;

__global__ void __launch_bounds__(kSmWarps * 32)
    k_softmax_staged(const float* __restrict__ x, int64_t rows, int cols, float* __restrict__ o) {
  __shared__ float buf[kSmWarps][32 * (kSmMaxCols + 1)];
  __shared__ double ex[kSmWarps][32 * kSmMaxCols];
  __shared__ double rmx[kSmWarps][32], rsum[kSmWarps][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ld = cols | 1;
  float* b = buf[warp];
  double* e = ex[warp];
  for (int64_t r0 = (static_cast<int64_t>(blockIdx.x) * kSmWarps + warp) * 32; r0 < rows;
       r0 += static_cast<int64_t>(gridDim.x) * kSmWarps * 32) {
    const int nr = static_cast<int>(rows - r0 < 32 ? rows - r0 : 32);
    const int n = nr * cols;
    const float* src = x + r0 * cols;
    for (int t = lane, r = 0, c = lane; t < n; t += 32) {  // (r, c) = divmod(t, cols)
      while (c >= cols) c -= cols, ++r;
      b[r * ld + c] = src[t];
      c += 32;
    }
    __syncwarp();
    if (lane < nr) {
      const float* xr = b + lane * ld;
      double mx = -INFINITY;
      for (int j = 0; j < cols; ++j) mx = fmax(mx, static_cast<double>(xr[j]));
      rmx[warp][lane] = mx;
    }
    __syncwarp();
    for (int t = lane, r = 0, c = lane; t < n; t += 32) {
      while (c >= cols) c -= cols, ++r;
      e[r * cols + c] = exp_nonpos(static_cast<double>(b[r * ld + c]) - rmx[warp][r]);
      c += 32;
    }
    __syncwarp();
    if (lane < nr) {
      const double* er = e + lane * cols;
      double sum = 0.0;
      for (int j = 0; j < cols; ++j) sum = __dadd_rn(sum, er[j]);
      rsum[warp][lane] = __drcp_rn(sum);
    }
    __syncwarp();
    float* dst = o + r0 * cols;
    for (int t = lane, r = 0, c = lane; t < n; t += 32) {
      while (c >= cols) c -= cols, ++r;
      dst[t] = __double2float_rn(__dmul_rn(e[r * cols + c], rsum[warp][r]));
      c += 32;
    }
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
             cudaStream_t s) {
  if (rows * cols == 0) return;
  k_add_bbf<<<grid1(rows * cols), 256, 0, s>>>(a, b, rows, cols, spw(cols, wb), out);
  BG_LAUNCH_CHECK();
}

void add_fff(const float* a, const float* b, int64_t n, float* out, cudaStream_t s) {
  if (n == 0) return;
  k_add_fff<<<grid1(n), 256, 0, s>>>(a, b, n, out);
  BG_LAUNCH_CHECK();
}

void relu(float* x, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  k_relu<<<grid1(n), 256, 0, s>>>(x, n);
  BG_LAUNCH_CHECK();
}

void softmax_rows(const float* x, int64_t rows, int64_t cols, float* out, cudaStream_t s) {
  if (rows == 0) return;
  if (cols >= 1 && cols <= kSmMaxCols && x != out) {
    const int64_t blocks = std::min<int64_t>(cdiv(rows, kSmWarps * 32), static_cast<int64_t>(sm_count()) * 32);
    k_softmax_staged<<<static_cast<unsigned>(blocks), kSmWarps * 32, 0, s>>>(x, rows, static_cast<int>(cols), out);
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
