// Bit packing primitives: binarize (warp ballot), L1 reconstruction scales,
// unpack and bit transpose.  ref: bitdense.cpp.
#include "ops.cuh"

namespace bg {
namespace {

constexpr int kWordsPerWarp = 8;

// One warp packs kWordsPerWarp consecutive words of one row: every lane loads
// its column of each 32-column group (coalesced 128 B per load, all loads in
// flight before the ballots), the ballot of (x >= 0) is the word with lane l
// at bit l, and __brev puts column 32w at the MSB (ref: bitdense.cpp:71-88;
// NaN compares false -> 0, -0.0 >= 0 -> 1, exactly like the reference).
__global__ void k_binarize(const float* __restrict__ x, int64_t rows, int64_t cols, int64_t spw,
                           int64_t groups, uint32_t* __restrict__ out) {
  const int64_t unit = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (unit >= rows * groups) return;
  const int lane = threadIdx.x & 31;
  const int64_t row = unit / groups;
  const int64_t w0 = (unit % groups) * kWordsPerWarp;
  const float* xr = x + row * cols;
  float v[kWordsPerWarp];
#pragma unroll
  for (int m = 0; m < kWordsPerWarp; ++m) {
    const int64_t j = 32 * (w0 + m) + lane;
    v[m] = j < cols ? __ldg(xr + j) : -1.0f;
  }
  uint32_t mine = 0;
#pragma unroll
  for (int m = 0; m < kWordsPerWarp; ++m) {
    const uint32_t word = __brev(__ballot_sync(0xFFFFFFFFu, v[m] >= 0.0f));
    if (lane == m) mine = word;
  }
  if (lane < kWordsPerWarp && w0 + lane < spw) out[row * spw + w0 + lane] = mine;
}

// Row scales for rows of a multiple of 4 floats: as k_l1_rows, but each
// stage is 32 rows x 128 columns loaded with float4s (one 512-byte row per
// warp instruction), then lane r sums row r in column order from shared
// memory (stride 129: conflict-free).
constexpr int kL1Warps = 2;
__global__ void __launch_bounds__(32 * kL1Warps)
    k_l1_rows4(const float* __restrict__ x, int64_t rows, int64_t cols, float* __restrict__ out) {
  __shared__ float tile[kL1Warps][32][129];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = (static_cast<int64_t>(blockIdx.x) * kL1Warps + warp) * 32;
  if (row0 >= rows) return;
  double acc = 0.0;
  for (int64_t c0 = 0; c0 < cols; c0 += 128) {
    const int64_t j = c0 + 4 * lane;
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {
      const int64_t i = row0 + r;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < rows && j < cols) v = __ldg(reinterpret_cast<const float4*>(x + i * cols + j));
      float* t = &tile[warp][r][4 * lane];
      t[0] = v.x, t[1] = v.y, t[2] = v.z, t[3] = v.w;
    }
    __syncwarp();
    const int64_t cmax = cols - c0 < 128 ? cols - c0 : 128;
    for (int t = 0; t < cmax; ++t) acc += fabs(static_cast<double>(tile[warp][lane][t]));
    __syncwarp();
  }
  const int64_t i = row0 + lane;
  if (i < rows) {
    const double mean = cols > 0 ? acc / static_cast<double>(cols) : 0.0;
    out[i] = static_cast<float>(mean > 1e-12 ? mean : 1e-12);
  }
}

// Row scales: each warp owns 32 rows; a 32x32 tile is staged through shared
// memory with coalesced loads, then lane r sums row r's entries in column
// order (the reference's sequential double accumulation, bitdense.cpp:95-102).
__global__ void k_l1_rows(const float* __restrict__ x, int64_t rows, int64_t cols,
                          float* __restrict__ out) {
  __shared__ float tile[8][32][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = (static_cast<int64_t>(blockIdx.x) * 8 + warp) * 32;
  if (row0 >= rows) return;
  double acc = 0.0;
  for (int64_t c0 = 0; c0 < cols; c0 += 32) {
    for (int r = 0; r < 32; ++r) {
      const int64_t i = row0 + r, j = c0 + lane;
      tile[warp][r][lane] = (i < rows && j < cols) ? __ldg(x + i * cols + j) : 0.0f;
    }
    __syncwarp();
    const int64_t cmax = cols - c0 < 32 ? cols - c0 : 32;
    for (int t = 0; t < cmax; ++t) acc += fabs(static_cast<double>(tile[warp][lane][t]));
    __syncwarp();
  }
  const int64_t i = row0 + lane;
  if (i < rows) {
    const double mean = cols > 0 ? acc / static_cast<double>(cols) : 0.0;
    out[i] = static_cast<float>(mean > 1e-12 ? mean : 1e-12);
  }
}

// Column scales: one thread per column walks the rows in order (coalesced
// across the warp).
__global__ void k_l1_cols(const float* __restrict__ x, int64_t rows, int64_t cols,
                          float* __restrict__ out) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  double acc = 0.0;
  for (int64_t t = 0; t < rows; ++t) acc += fabs(static_cast<double>(__ldg(x + t * cols + j)));
  const double mean = rows > 0 ? acc / static_cast<double>(rows) : 0.0;
  out[j] = static_cast<float>(mean > 1e-12 ? mean : 1e-12);
}

__global__ void k_unpack(const uint32_t* __restrict__ bits, int64_t rows, int64_t cols,
                         int64_t spw, float lo, float* __restrict__ out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * cols) return;
  const int64_t i = t / cols, j = t % cols;
  out[t] = ((bits[i * spw + j / 32] >> (31 - (j & 31))) & 1u) ? 1.0f : lo;
}

// out (cols x rows bits): thread per output word gathers 32 input rows.
__global__ void k_transpose(const uint32_t* __restrict__ in, int64_t rows, int64_t cols,
                            int64_t spw_in, int64_t spw_out, uint32_t* __restrict__ out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= cols * spw_out) return;
  const int64_t j = t / spw_out, wi = t % spw_out;
  uint32_t v = 0;
  const uint32_t sh = 31 - static_cast<uint32_t>(j & 31);
  for (int b = 0; b < 32; ++b) {
    const int64_t i = 32 * wi + b;
    if (i < rows) v |= ((__ldg(in + i * spw_in + j / 32) >> sh) & 1u) << (31 - b);
  }
  out[t] = v;
}

}  // namespace

void binarize(const float* x, int64_t rows, int64_t cols, int wb, uint32_t* out, cudaStream_t s) {
  const int64_t w = spw(cols, wb);
  if (rows == 0 || w == 0) return;
  const int64_t groups = cdiv(w, kWordsPerWarp);
  const int64_t warps = rows * groups;
  k_binarize<<<static_cast<unsigned>(cdiv(warps, 8)), 256, 0, s>>>(x, rows, cols, w, groups, out);
  BG_LAUNCH_CHECK();
}

void l1_scales(const float* x, int64_t rows, int64_t cols, int axis, float* out, cudaStream_t s) {
  if (axis == BG_AXIS_ROW) {
    if (rows == 0) return;
    if (cols % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0)
      k_l1_rows4<<<static_cast<unsigned>(cdiv(rows, 32 * kL1Warps)), 32 * kL1Warps, 0, s>>>(x, rows, cols, out);
    else
      k_l1_rows<<<static_cast<unsigned>(cdiv(rows, 256)), 256, 0, s>>>(x, rows, cols, out);
  } else {
    if (cols == 0) return;
    k_l1_cols<<<static_cast<unsigned>(cdiv(cols, 128)), 128, 0, s>>>(x, rows, cols, out);
  }
  BG_LAUNCH_CHECK();
}

void unpack(const uint32_t* bits, int64_t rows, int64_t cols, int wb, int semantics, float* out,
            cudaStream_t s) {
  if (rows * cols == 0) return;
  const float lo = semantics == BG_PLUS_MINUS ? -1.0f : 0.0f;
  k_unpack<<<static_cast<unsigned>(cdiv(rows * cols, 256)), 256, 0, s>>>(bits, rows, cols,
                                                                          spw(cols, wb), lo, out);
  BG_LAUNCH_CHECK();
}

void transpose_bits(const uint32_t* in, int64_t rows, int64_t cols, int wb, uint32_t* out,
                    cudaStream_t s) {
  const int64_t so = spw(rows, wb);
  if (cols * so == 0) return;
  k_transpose<<<static_cast<unsigned>(cdiv(cols * so, 256)), 256, 0, s>>>(in, rows, cols,
                                                                          spw(cols, wb), so, out);
  BG_LAUNCH_CHECK();
}

}  // namespace bg
