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

#include "ops.cuh"

namespace bg {
namespace {

constexpr int kWarps = 8;
constexpr int kMaxOutPerLane = 8;  // output columns per lane per pass (256 per pass)

template <bool AF, bool OUTB, int M>
__global__ void __launch_bounds__(kWarps * 32)
    k_bmm(const uint32_t* __restrict__ a_bits, const float* __restrict__ a_f,
          const float* __restrict__ alpha, const uint32_t* __restrict__ wt,
          const float* __restrict__ beta, int64_t rows, int64_t k, int64_t n, int64_t kspw,
          int64_t ld, int64_t c0, int64_t nc, int64_t ospw, uint32_t* __restrict__ out_bits,
          float* __restrict__ out_f) {
  extern __shared__ uint32_t smem[];
  uint32_t* sw = smem;                       // nc x ld transposed weight words
  uint32_t* srow = smem + nc * ld;           // kWarps x kspw packed activation rows
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t t = threadIdx.x; t < nc * kspw; t += blockDim.x) {
    const int64_t j = t / kspw, w = t % kspw;
    sw[j * ld + w] = __ldg(wt + (c0 + j) * kspw + w);
  }
  __syncthreads();
  uint32_t* arow = srow + warp * kspw;
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * kWarps + warp; row < rows;
       row += static_cast<int64_t>(gridDim.x) * kWarps) {
    if (AF) {
      const float* xr = a_f + row * k;
      for (int64_t w0 = 0; w0 < kspw; w0 += 8) {
        float v[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const int64_t j = 32 * (w0 + m) + lane;
          v[m] = j < k ? __ldg(xr + j) : -1.0f;
        }
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const uint32_t word = __brev(__ballot_sync(0xFFFFFFFFu, v[m] >= 0.0f));
          if (lane == m && w0 + m < kspw) arow[w0 + m] = word;
        }
      }
    } else {
      for (int64_t w = lane; w < kspw; w += 32) arow[w] = __ldg(a_bits + row * kspw + w);
    }
    __syncwarp();
    int diff[M];
#pragma unroll
    for (int m = 0; m < M; ++m) diff[m] = 0;
    const uint32_t* swl = sw + lane * ld;
    for (int64_t w = 0; w < kspw; ++w) {
      const uint32_t aw = arow[w];
#pragma unroll
      for (int m = 0; m < M; ++m) diff[m] += __popc(aw ^ swl[32 * m * ld + w]);
    }
    __syncwarp();
    if (OUTB) {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int64_t j = 32 * m + lane;
        const bool bit = j < nc && (k - 2 * static_cast<int64_t>(diff[m])) >= 0;
        const uint32_t word = __brev(__ballot_sync(0xFFFFFFFFu, bit));
        if (lane == 0) out_bits[row * ospw + c0 / 32 + m] = word;
      }
      // zero the storage-padding words of 64-bit rows after the last pass
      if (lane == 0 && c0 + nc == n)
        for (int64_t w = (n + 31) / 32; w < ospw; ++w) out_bits[row * ospw + w] = 0;
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

template <bool AF, bool OUTB>
void launch(const BmmArgs& a, cudaStream_t s) {
  auto pick = [](int64_t nc) {
    return nc <= 32 ? k_bmm<AF, OUTB, 1> : nc <= 64 ? k_bmm<AF, OUTB, 2>
         : nc <= 128 ? k_bmm<AF, OUTB, 4> : k_bmm<AF, OUTB, 8>;
  };
  const int64_t kspw = spw(a.k, a.wb);
  const int64_t ld = kspw | 1;
  const int64_t ospw = spw(a.n, a.wb);
  const int64_t pass = 32 * kMaxOutPerLane;
  int64_t blocks = std::min<int64_t>(cdiv(a.rows, kWarps), static_cast<int64_t>(sm_count()) * 8);
  blocks = std::max<int64_t>(blocks, 1);
  for (int64_t c0 = 0; c0 < a.n; c0 += pass) {
    const int64_t nc = std::min(pass, a.n - c0);
    const size_t smem = static_cast<size_t>(cdiv(nc, 32) * 32 * ld + kWarps * kspw) * 4;
    auto kern = pick(nc);
    if (smem > 48 * 1024) BG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      static_cast<int>(smem)));
    if (smem > 200 * 1024) fail("bmm: inner dimension too large for one pass");
    kern<<<static_cast<unsigned>(blocks), kWarps * 32, smem, s>>>(
        a.a_bits, a.a_f, a.alpha, a.wt, a.beta, a.rows, a.k, a.n, kspw, ld, c0, nc, ospw,
        a.out_bits, a.out_f);
    BG_LAUNCH_CHECK();
  }
}

}  // namespace

void bmm(const BmmArgs& a, cudaStream_t s) {
  if (a.rows == 0 || a.n == 0) return;
  const bool af = a.a_f != nullptr, ob = a.out_bits != nullptr;
  if (af && ob) launch<true, true>(a, s);
  else if (af) launch<true, false>(a, s);
  else if (ob) launch<false, true>(a, s);
  else launch<false, false>(a, s);
}

}  // namespace bg
