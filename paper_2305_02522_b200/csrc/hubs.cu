// Hub rows of BSpMM.BBB / BBF (power-law degree profiles).
//
// The BB aggregation kernels (window.cu k_win_bb, sliver.cu k_sl_bb /
// k_bv_bb) give one warp -- or one lane -- a node row: a row of 10^5
// neighbours then runs ~10^5 / 256 dependent gather rounds in one warp while
// the rest of the GPU idles, and the windowed kernel's 16-bit step counts and
// 12-bit counters cannot hold it at all.  Rows of degree >= kHubDeg are
// therefore taken out of those kernels (they see the row as empty) and
// counted here, split over the SMs:
//   k_hub_count  warp per chunk of kHubChunk tiles of a hub's tile row: lane
//                per tile, every set bit of the hub's nibble gathers the
//                neighbour's feature words into bit-sliced counters, a
//                butterfly reduces the 32 lanes (slot_reduce) and lane b adds
//                the count of bit b to the hub's int32 counter (atomicAdd);
//   k_hub_final  block per hub: out = 2*count - deg (BBF) or the bit
//                count >= ceil(deg/2) (BBB, kernels.cpp:440-454), and the
//                counters back to zero for the next call.
// Counting is order-free (integer), so the split changes nothing in the
// results: bit-identical to the reference's per-row walk (kernels.cpp:254-455).
#include <algorithm>
#include <climits>
#include <vector>

#include "ops.cuh"
#include "tilewalk.cuh"

namespace bg {
namespace {

constexpr int kHubChunk = 32 * 16;  // tiles per warp: 16 per lane
constexpr int kHubNP = 7;           // <= 16 tiles x 4 bits = 64 per lane
constexpr int kHubNQ = kHubNP + 5;  // after the 32-lane reduction

__device__ __forceinline__ void add1(uint32_t (&P)[kHubNP], uint32_t v) {
#pragma unroll
  for (int q = 0; q < kHubNP; ++q) {
    const uint32_t c = P[q] & v;
    P[q] ^= v;
    v = c;
  }
}

// Chunk record: x,y = first tile (u64), z = tiles, w = hub index << 2 | row in tile row.
// blockIdx.y: group of G feature words.
template <int G>
__global__ void __launch_bounds__(256)
    k_hub_count(const uint4* __restrict__ chunks, int64_t nchunks, const int32_t* __restrict__ hub_rows,
                int64_t r0, int64_t r1, const uint32_t* __restrict__ ci, const uint16_t* __restrict__ tiles,
                const uint32_t* __restrict__ x, int64_t xspw, int32_t* __restrict__ cnt) {
  const int64_t c = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (c >= nchunks) return;
  const int lane = threadIdx.x & 31;
  const uint4 ch = chunks[c];
  const int64_t h = ch.w >> 2;
  const int r = static_cast<int>(ch.w & 3u);
  const int64_t row = hub_rows[h];
  if (row < r0 || row >= r1) return;  // warp-uniform
  const uint64_t t0 = (static_cast<uint64_t>(ch.y) << 32) | ch.x;
  const int64_t w0 = static_cast<int64_t>(blockIdx.y) * G;
  uint32_t P[G][kHubNP];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int q = 0; q < kHubNP; ++q) P[g][q] = 0u;
  for (uint32_t k = lane; k < ch.z; k += 32) {
    const uint32_t nib = (static_cast<uint32_t>(ld_nc_u16(tiles + t0 + k)) >> (12 - 4 * r)) & 0xFu;
    if (!nib) continue;
    const int64_t j0 = 4 * static_cast<int64_t>(ld_nc_u32(ci + t0 + k));
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (!((nib >> (3 - b)) & 1u)) continue;
      const uint32_t* xr = x + (j0 + b) * xspw + w0;
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (w0 + g < xspw) add1(P[g], __ldg(xr + g));
    }
  }
  int32_t* hc = cnt + h * xspw * 32;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (w0 + g >= xspw) break;  // block-uniform
    uint32_t Q[kHubNQ];
    slot_reduce<1, kHubNP, kHubNQ>(P[g], Q);
    const uint32_t v = plane_count<kHubNQ>(Q, lane);
    if (v) atomicAdd(hc + (w0 + g) * 32 + lane, static_cast<int32_t>(v));
  }
}

// Block per hub, thread per (word, bit).
__global__ void k_hub_final(const int32_t* __restrict__ hub_rows, int64_t nhubs, int64_t r0, int64_t r1,
                            const int32_t* __restrict__ degree, int64_t xspw, int64_t f, int32_t* __restrict__ cnt,
                            uint32_t* __restrict__ out_bits, float* __restrict__ out_f, const FEpi ep) {
  const int64_t h = blockIdx.x;
  if (h >= nhubs) return;
  const int64_t i = hub_rows[h];
  if (i < r0 || i >= r1) return;
  const int64_t deg = degree[i];
  int32_t* hc = cnt + h * xspw * 32;
  const int lane = threadIdx.x & 31;
  for (int64_t w = threadIdx.x >> 5; w < xspw; w += blockDim.x >> 5) {
    const int64_t k = 32 * w + lane;
    const int64_t c = hc[k];
    hc[k] = 0;
    if (out_bits) {
      const uint32_t word = __brev(__ballot_sync(0xFFFFFFFFu, k < f && 2 * c - deg >= 0));
      if (lane == 0) out_bits[i * xspw + w] = word;
    } else {
      fepi_store_lane(ep, out_f, i, f, k, static_cast<float>(2 * c - deg));
    }
  }
}

}  // namespace

void frdc_hubs(bg_frdc& m, cudaStream_t s) {
  auto& H = m.hub;
  if (H.n >= 0) return;
  H.n = 0;
  H.nchunks = 0;
  H.max_light_deg = m.max_deg;
  if (m.max_deg < kHubDeg || m.rows == 0) return;
  // one-time host pass over the degrees and the hub tile rows' extents
  std::vector<int32_t> deg(static_cast<size_t>(m.rows));
  std::vector<uint64_t> rp(static_cast<size_t>(m.tile_rows) + 1);
  BG_CUDA(cudaMemcpyAsync(deg.data(), m.deg(), deg.size() * 4, cudaMemcpyDeviceToHost, s));
  BG_CUDA(cudaMemcpyAsync(rp.data(), m.rp(), rp.size() * 8, cudaMemcpyDeviceToHost, s));
  BG_CUDA(cudaStreamSynchronize(s));
  std::vector<int32_t> rows;
  std::vector<uint4> chunks;
  int64_t light = 0;
  for (int64_t i = 0; i < m.rows; ++i) {
    if (deg[i] < kHubDeg) {
      light = std::max<int64_t>(light, deg[i]);
      continue;
    }
    const uint32_t h = static_cast<uint32_t>(rows.size());
    rows.push_back(static_cast<int32_t>(i));
    const uint64_t a = rp[i / 4], b = rp[i / 4 + 1];
    for (uint64_t t = a; t < b; t += kHubChunk)
      chunks.push_back(make_uint4(static_cast<uint32_t>(t), static_cast<uint32_t>(t >> 32),
                                  static_cast<uint32_t>(std::min<uint64_t>(kHubChunk, b - t)),
                                  h << 2 | static_cast<uint32_t>(i & 3)));
  }
  H.max_light_deg = light;
  H.n = static_cast<int64_t>(rows.size());
  H.nchunks = static_cast<int64_t>(chunks.size());
  H.rows.alloc(std::max<size_t>(rows.size() * 4, 4));
  H.chunks.alloc(std::max<size_t>(chunks.size() * 16, 16));
  BG_CUDA(cudaMemcpyAsync(H.rows.p, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, s));
  BG_CUDA(cudaMemcpyAsync(H.chunks.p, chunks.data(), chunks.size() * 16, cudaMemcpyHostToDevice, s));
  BG_CUDA(cudaStreamSynchronize(s));
  ++m.gen;
}

int64_t light_max_deg(bg_frdc& m, cudaStream_t s) {
  frdc_hubs(m, s);
  return m.hub.max_light_deg;
}

void hub_bb(bg_frdc& A, const uint32_t* x, int64_t f, int64_t xspw, uint32_t* out_bits, float* out_f,
            cudaStream_t s, int64_t r0, int64_t r1) {
  frdc_hubs(A, s);
  auto& H = A.hub;
  if (H.n == 0 || xspw == 0) return;
  if (H.cnt_words < xspw) {  // counters (zero between calls): grown eagerly, never while capturing
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    BG_CUDA(cudaStreamIsCapturing(s, &cap));
    if (cap != cudaStreamCaptureStatusNone) fail("hub_bb: counters not sized before capture");
    H.cnt.alloc(static_cast<size_t>(H.n * xspw * 32) * 4);
    BG_CUDA(cudaMemsetAsync(H.cnt.p, 0, H.cnt.bytes, s));
    H.cnt_words = xspw;
    ++A.gen;
  }
  auto* cnt = H.cnt.as<int32_t>();
  const unsigned blocks = static_cast<unsigned>(cdiv(H.nchunks * 32, 256));
  const auto* ch = H.chunks.as<uint4>();
  const auto* hr = H.rows.as<int32_t>();
  if (xspw <= 1) {
    k_hub_count<1><<<dim3(blocks, 1), 256, 0, s>>>(ch, H.nchunks, hr, r0, r1, A.ci(), A.ti(), x, xspw, cnt);
  } else if (xspw <= 2) {
    k_hub_count<2><<<dim3(blocks, 1), 256, 0, s>>>(ch, H.nchunks, hr, r0, r1, A.ci(), A.ti(), x, xspw, cnt);
  } else {
    k_hub_count<4><<<dim3(blocks, static_cast<unsigned>(cdiv(xspw, 4))), 256, 0, s>>>(ch, H.nchunks, hr, r0, r1,
                                                                                     A.ci(), A.ti(), x, xspw, cnt);
  }
  BG_LAUNCH_CHECK();
  k_hub_final<<<static_cast<unsigned>(H.n), 128, 0, s>>>(hr, H.n, r0, r1, A.deg(), xspw, f, cnt, out_bits, out_f, current_fepi());
  BG_LAUNCH_CHECK();
}

}  // namespace bg
