// Device construction of the FRDC bit-tile adjacency and the graph bundle.
// ref: bitsparse.cpp:40-112 (FrdcMatrix, frdc_from_edges),
//      graphops.cpp:18-33, :135-170 (row_popcounts, normalize, prepare_graph).
//
// Build-once path: 64-bit tile keys -> CUB radix sort -> head flags + scan ->
// OR-reduce payload bits per tile -> per-tile-row histogram + scan.  The three
// arrays come out byte-identical to the reference's std::sort + run-length
// loop because both produce the keys in ascending order and OR the same bits.
#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "ops.cuh"

namespace bg {
namespace {

__global__ void k_keys(const int64_t* __restrict__ src, const int64_t* __restrict__ dst, int64_t e,
                       int64_t n, uint64_t tcols, bool loops, bool drop_self, uint64_t sentinel,
                       uint64_t* __restrict__ keys, unsigned long long* __restrict__ dropped,
                       unsigned long long* __restrict__ bad) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < e) {
    const int64_t s = src[t], d = dst[t];
    if (s < 0 || s >= n || d < 0 || d >= n) {
      atomicMin(bad, static_cast<unsigned long long>(t));
      keys[t] = sentinel;
      return;
    }
    if (drop_self && s == d) {
      atomicAdd(dropped, 1ull);
      keys[t] = sentinel;
      return;
    }
    const uint64_t key = static_cast<uint64_t>(s >> 2) * tcols + static_cast<uint64_t>(d >> 2);
    keys[t] = (key << 4) | static_cast<uint64_t>(4 * (s & 3) + (d & 3));
  } else if (loops && t < e + n) {
    const int64_t i = t - e;
    const uint64_t key = static_cast<uint64_t>(i >> 2) * tcols + static_cast<uint64_t>(i >> 2);
    keys[t] = (key << 4) | static_cast<uint64_t>(5 * (i & 3));
  }
}

__global__ void k_heads(const uint64_t* __restrict__ k, int64_t valid, uint32_t* __restrict__ flag) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= valid) return;
  flag[t] = (t == 0 || (k[t] >> 4) != (k[t - 1] >> 4)) ? 1u : 0u;
}

__global__ void k_scatter(const uint64_t* __restrict__ k, const uint32_t* __restrict__ idx1,
                          int64_t valid, uint64_t tcols, uint32_t* __restrict__ tiles32,
                          uint32_t* __restrict__ col_ind, unsigned long long* __restrict__ row_cnt) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= valid) return;
  const uint64_t key = k[t] >> 4;
  const uint32_t i = idx1[t] - 1;  // inclusive scan of head flags
  atomicOr(tiles32 + i, 1u << (15 - static_cast<uint32_t>(k[t] & 15)));
  if (t == 0 || (k[t - 1] >> 4) != key) {
    col_ind[i] = static_cast<uint32_t>(key % tcols);
    atomicAdd(row_cnt + key / tcols, 1ull);
  }
}

__global__ void k_narrow(const uint32_t* __restrict__ a, int64_t n, uint16_t* __restrict__ b) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) b[t] = static_cast<uint16_t>(a[t]);
}

// Warp per tile row: per-node-row set-bit counts (ref: graphops.cpp:18-33).
__global__ void k_degree(const uint64_t* __restrict__ rp, const uint16_t* __restrict__ tiles,
                         int64_t trows, int64_t rows, int32_t* __restrict__ deg,
                         unsigned long long* __restrict__ nbits, int* __restrict__ maxdeg) {
  const int64_t tr = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (tr >= trows) return;
  const int lane = threadIdx.x & 31;
  int c[4] = {0, 0, 0, 0};
  for (uint64_t k = rp[tr] + lane; k < rp[tr + 1]; k += 32) {
    const uint32_t t = tiles[k];
#pragma unroll
    for (int r = 0; r < 4; ++r) c[r] += __popc((t >> (12 - 4 * r)) & 0xFu);
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
    for (int o = 16; o; o >>= 1) c[r] += __shfl_xor_sync(0xFFFFFFFFu, c[r], o);
  if (lane == 0) {
    int tot = 0, mx = 0;
    for (int r = 0; r < 4; ++r) {
      const int64_t row = 4 * tr + r;
      if (row < rows) {
        deg[row] = c[r];
        tot += c[r];
        mx = c[r] > mx ? c[r] : mx;
      }
    }
    atomicAdd(nbits, static_cast<unsigned long long>(tot));
    atomicMax(maxdeg, mx);
  }
}

// Warp per tile row: lane p sums, per node row, the bits of tiles p, p+32, ...;
// groups of G lanes are then summed and the maximum kept (G = 4 and 8).
__global__ void k_slot_max(const uint64_t* __restrict__ rp, const uint16_t* __restrict__ tiles,
                           int64_t trows, int* __restrict__ out) {
  const int64_t tr = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (tr >= trows) return;
  const int lane = threadIdx.x & 31;
  int c[4] = {0, 0, 0, 0};
  for (uint64_t k = rp[tr] + lane; k < rp[tr + 1]; k += 32) {
    const uint32_t t = tiles[k];
#pragma unroll
    for (int r = 0; r < 4; ++r) c[r] += __popc((t >> (12 - 4 * r)) & 0xFu);
  }
  int m4 = 0, m8 = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    int v = c[r];
    v += __shfl_xor_sync(0xFFFFFFFFu, v, 1);
    v += __shfl_xor_sync(0xFFFFFFFFu, v, 2);
    m4 = v > m4 ? v : m4;
    v += __shfl_xor_sync(0xFFFFFFFFu, v, 4);
    m8 = v > m8 ? v : m8;
  }
  if (lane == 0 || lane == 4 || lane == 8 || lane == 12 || lane == 16 || lane == 20 ||
      lane == 24 || lane == 28) {
    atomicMax(out, m4);
    atomicMax(out + 1, m8);
  }
}

// Warp per tile row: nonzero nibbles per node row, padded to a multiple of
// kSliverPad entries (the aggregation kernels then need no bounds checks).
__global__ void k_sliver_count(const uint64_t* __restrict__ rp, const uint16_t* __restrict__ tiles,
                               int64_t trows, int64_t rows, const int32_t* __restrict__ deg,
                               unsigned long long* __restrict__ cnt, int* __restrict__ maxima) {
  const int64_t tr = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (tr >= trows) return;
  const int lane = threadIdx.x & 31;
  int c[4] = {0, 0, 0, 0};
  for (uint64_t k = rp[tr] + lane; k < rp[tr + 1]; k += 32) {
    const uint32_t t = tiles[k];
#pragma unroll
    for (int r = 0; r < 4; ++r) c[r] += ((t >> (12 - 4 * r)) & 0xFu) != 0;
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    for (int o = 16; o; o >>= 1) c[r] += __shfl_xor_sync(0xFFFFFFFFu, c[r], o);
    if (lane == 0 && 4 * tr + r < rows) {
      const int padded = (c[r] + kSliverPad - 1) / kSliverPad * kSliverPad;
      cnt[4 * tr + r] = static_cast<unsigned long long>(padded);
      if (deg[4 * tr + r] < kHubDeg) {  // hub rows: hubs.cu
        atomicMax(maxima, padded);
        atomicMax(maxima + 1, deg[4 * tr + r] - c[r]);
      }
    }
  }
}

// Sliver entry of one nonzero nibble of tile column `col`: the node column of
// its first set bit (bit 3-c of the nibble is local column c) and a 3-bit
// mask of the following columns present (bit k-1 <-> first + k).
__device__ __forceinline__ uint32_t sliver_entry(uint32_t col, uint32_t nib) {
  const uint32_t c0 = __clz(nib) - 28;  // lowest local column present
  uint32_t extra = 0;
#pragma unroll
  for (int k = 1; k < 4; ++k)
    if (c0 + k < 4 && ((nib >> (3 - c0 - k)) & 1u)) extra |= 1u << (k - 1);
  return ((4 * col + c0) << 3) | extra;
}

// Warp per tile row: ballot-compact each row's nonzero nibbles in tile order,
// then the row's padding entries.
__global__ void k_sliver_fill(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                              const uint16_t* __restrict__ tiles, int64_t trows, int64_t rows,
                              const unsigned long long* __restrict__ srp,
                              uint32_t* __restrict__ out) {
  const int64_t tr = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (tr >= trows) return;
  const int lane = threadIdx.x & 31;
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  unsigned long long pos[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) pos[r] = 4 * tr + r < rows ? srp[4 * tr + r] : 0;
  for (uint64_t base = rp[tr]; base < rp[tr + 1]; base += 32) {
    const uint64_t k = base + lane;
    uint32_t t = 0, col = 0;
    if (k < rp[tr + 1]) {
      t = tiles[k];
      col = ci[k];
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t nib = (t >> (12 - 4 * r)) & 0xFu;
      const uint32_t mask = __ballot_sync(0xFFFFFFFFu, nib != 0);
      if (nib) out[pos[r] + __popc(mask & lt)] = sliver_entry(col, nib);
      pos[r] += __popc(mask);
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if (4 * tr + r < rows)
      for (unsigned long long k = pos[r] + lane; k < srp[4 * tr + r + 1]; k += 32) out[k] = kSliverSentinel;
}

__global__ void k_graph_scales(const int32_t* __restrict__ deg_loops,
                               const int32_t* __restrict__ deg_raw, int64_t n,
                               float* __restrict__ norm, float* __restrict__ mean,
                               float* __restrict__ ones, int64_t* __restrict__ cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // ref: graphops.cpp:141 -- float(1 / sqrt(double(deg))) ; :164 float divide
  norm[i] = static_cast<float>(1.0 / sqrt(static_cast<double>(deg_loops[i])));
  const int64_t c = deg_raw[i];
  cnt[i] = c;
  mean[i] = 1.0f / static_cast<float>(c > 1 ? c : 1);
  ones[i] = 1.0f;
}

unsigned grid1(int64_t n, int bs = 256) { return static_cast<unsigned>(cdiv(n, bs)); }

}  // namespace

void frdc_finalize(bg_frdc& m, cudaStream_t s) {
  m.nslivers = -1;  // derived views are rebuilt on next use
  ++m.gen;
  m.hub.n = -1;
  m.hub.cnt_words = 0;
  m.win.T = 0;
  m.nbits_view = -1;
  m.degree.alloc(static_cast<size_t>(std::max<int64_t>(m.rows, 1)) * 4);
  BG_CUDA(cudaMemsetAsync(m.degree.p, 0, m.degree.bytes, s));
  DevBuf stats(16);
  BG_CUDA(cudaMemsetAsync(stats.p, 0, 16, s));
  auto* nbits = stats.as<unsigned long long>();
  auto* maxdeg = reinterpret_cast<int*>(stats.as<char>() + 8);
  if (m.tile_rows > 0)
    k_degree<<<grid1(m.tile_rows * 32), 256, 0, s>>>(m.rp(), m.ti(), m.tile_rows, m.rows,
                                                     m.degree.as<int32_t>(), nbits, maxdeg);
  BG_LAUNCH_CHECK();
  DevBuf slots(8);
  BG_CUDA(cudaMemsetAsync(slots.p, 0, 8, s));
  if (m.tile_rows > 0)
    k_slot_max<<<grid1(m.tile_rows * 32), 256, 0, s>>>(m.rp(), m.ti(), m.tile_rows, slots.as<int>());
  BG_LAUNCH_CHECK();
  unsigned long long h[2] = {0, 0};
  int hs[2] = {0, 0};
  BG_CUDA(cudaMemcpyAsync(h, stats.p, 16, cudaMemcpyDeviceToHost, s));
  BG_CUDA(cudaMemcpyAsync(hs, slots.p, 8, cudaMemcpyDeviceToHost, s));
  BG_CUDA(cudaStreamSynchronize(s));
  m.nnz_bits = static_cast<int64_t>(h[0]);
  m.max_deg = static_cast<int64_t>(static_cast<int>(h[1] & 0xFFFFFFFFull));
  m.max_slot[0] = hs[0];
  m.max_slot[1] = hs[1];
}

void frdc_slivers(bg_frdc& m, cudaStream_t s) {
  if (m.nslivers >= 0) return;
  if (4 * m.tile_cols >= (int64_t{1} << 29)) fail("FRDC: too many node columns for the sliver view");
  const size_t n1 = static_cast<size_t>(m.rows) + 1;
  DevBuf cnt(n1 * 8), maxima(8);
  m.sliver_ptr.alloc(n1 * 8);
  BG_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes, s));
  BG_CUDA(cudaMemsetAsync(maxima.p, 0, 8, s));
  BG_CUDA(cudaMemsetAsync(m.sliver_ptr.p, 0, m.sliver_ptr.bytes, s));
  if (m.tile_rows > 0)
    k_sliver_count<<<grid1(m.tile_rows * 32), 256, 0, s>>>(m.rp(), m.ti(), m.tile_rows, m.rows,
                                                           m.deg(), cnt.as<unsigned long long>(),
                                                           maxima.as<int>());
  BG_LAUNCH_CHECK();
  int hm[2] = {0, 0};
  BG_CUDA(cudaMemcpyAsync(hm, maxima.p, 8, cudaMemcpyDeviceToHost, s));
  size_t tmp_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, cnt.as<unsigned long long>(),
                                m.sliver_ptr.as<unsigned long long>() + 1, static_cast<int>(m.rows), s);
  DevBuf tmp(std::max<size_t>(tmp_bytes, 1));
  if (m.rows > 0)
    cub::DeviceScan::InclusiveSum(tmp.p, tmp_bytes, cnt.as<unsigned long long>(),
                                  m.sliver_ptr.as<unsigned long long>() + 1, static_cast<int>(m.rows), s);
  BG_LAUNCH_CHECK();
  unsigned long long total = 0;
  BG_CUDA(cudaMemcpyAsync(&total, m.sliver_ptr.as<unsigned long long>() + m.rows, 8,
                          cudaMemcpyDeviceToHost, s));
  BG_CUDA(cudaStreamSynchronize(s));
  m.slivers.alloc(std::max<size_t>(static_cast<size_t>(total) * 4, 4));
  if (m.tile_rows > 0)
    k_sliver_fill<<<grid1(m.tile_rows * 32), 256, 0, s>>>(
        m.rp(), m.ci(), m.ti(), m.tile_rows, m.rows, m.sliver_ptr.as<unsigned long long>(),
        m.slivers.as<uint32_t>());
  BG_LAUNCH_CHECK();
  BG_CUDA(cudaStreamSynchronize(s));
  m.nslivers = static_cast<int64_t>(total);
  ++m.gen;
  m.max_sl_row = hm[0];
  m.max_extra_bits = hm[1];
}

std::unique_ptr<bg_frdc> frdc_build(const int64_t* src, const int64_t* dst, int64_t e, int64_t n,
                                    bool add_self_loops, bool drop_self_edges, cudaStream_t s) {
  if (n < 0) fail("frdc_from_edges: negative node count");
  if (e < 0) fail("frdc_from_edges: negative edge count");
  const int64_t tcols = (n + 3) / 4;
  if (tcols > 0xFFFFFFFEll) fail("frdc_from_edges: graph too large");
  auto m = std::make_unique<bg_frdc>();
  m->rows = m->cols = n;
  m->tile_rows = m->tile_cols = tcols;
  const int64_t total = e + (add_self_loops ? n : 0);
  if (total >= (int64_t{1} << 32)) fail("frdc_from_edges: more than 2^32 entries");
  m->row_ptr.alloc(static_cast<size_t>(tcols + 1) * 8);
  BG_CUDA(cudaMemsetAsync(m->row_ptr.p, 0, m->row_ptr.bytes, s));
  if (total == 0) {
    frdc_finalize(*m, s);
    return m;
  }
  const uint64_t sentinel = (static_cast<uint64_t>(tcols) * static_cast<uint64_t>(tcols)) << 4;
  int end_bit = 1;
  while (end_bit < 64 && (sentinel >> end_bit)) ++end_bit;

  DevBuf keys(static_cast<size_t>(total) * 8), keys2(static_cast<size_t>(total) * 8);
  DevBuf counters(16);
  BG_CUDA(cudaMemsetAsync(counters.p, 0, 8, s));
  BG_CUDA(cudaMemsetAsync(counters.as<char>() + 8, 0xFF, 8, s));
  auto* dropped = counters.as<unsigned long long>();
  auto* bad = dropped + 1;
  k_keys<<<grid1(total), 256, 0, s>>>(src, dst, e, n, static_cast<uint64_t>(tcols), add_self_loops,
                                      drop_self_edges, sentinel, keys.as<uint64_t>(), dropped, bad);
  BG_LAUNCH_CHECK();
  unsigned long long hc[2];
  BG_CUDA(cudaMemcpyAsync(hc, counters.p, 16, cudaMemcpyDeviceToHost, s));
  BG_CUDA(cudaStreamSynchronize(s));
  if (hc[1] != ~0ull) {
    int64_t es = 0, ed = 0;
    BG_CUDA(cudaMemcpy(&es, src + hc[1], 8, cudaMemcpyDeviceToHost));
    BG_CUDA(cudaMemcpy(&ed, dst + hc[1], 8, cudaMemcpyDeviceToHost));
    fail("frdc_from_edges: edge " + std::to_string(hc[1]) + " = (" + std::to_string(es) + ", " +
         std::to_string(ed) + ") out of range for " + std::to_string(n) + " nodes");
  }
  const int64_t valid = total - static_cast<int64_t>(hc[0]);
  if (valid == 0) {
    frdc_finalize(*m, s);
    return m;
  }

  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                 static_cast<int>(total), 0, end_bit, s);
  size_t scan_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, static_cast<uint32_t*>(nullptr),
                                static_cast<uint32_t*>(nullptr), static_cast<int>(total), s);
  size_t rscan_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, rscan_bytes, static_cast<unsigned long long*>(nullptr),
                                static_cast<unsigned long long*>(nullptr),
                                static_cast<int>(std::max<int64_t>(tcols, 1)), s);
  DevBuf tmp(std::max(tmp_bytes, std::max(scan_bytes, rscan_bytes)));
  cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                 static_cast<int>(total), 0, end_bit, s);
  BG_LAUNCH_CHECK();
  const uint64_t* sk = keys2.as<uint64_t>();
  keys = DevBuf();  // release

  DevBuf flag(static_cast<size_t>(valid) * 4), idx(static_cast<size_t>(valid) * 4);
  k_heads<<<grid1(valid), 256, 0, s>>>(sk, valid, flag.as<uint32_t>());
  BG_LAUNCH_CHECK();
  cub::DeviceScan::InclusiveSum(tmp.p, scan_bytes, flag.as<uint32_t>(), idx.as<uint32_t>(),
                                static_cast<int>(valid), s);
  BG_LAUNCH_CHECK();
  uint32_t nnz32 = 0;
  BG_CUDA(cudaMemcpyAsync(&nnz32, idx.as<uint32_t>() + valid - 1, 4, cudaMemcpyDeviceToHost, s));
  BG_CUDA(cudaStreamSynchronize(s));
  m->nnz = nnz32;
  flag = DevBuf();

  DevBuf tiles32(static_cast<size_t>(m->nnz) * 4);
  DevBuf rowcnt(static_cast<size_t>(tcols) * 8);
  m->col_ind.alloc(static_cast<size_t>(m->nnz) * 4);
  m->tiles.alloc(static_cast<size_t>(m->nnz) * 2);
  BG_CUDA(cudaMemsetAsync(tiles32.p, 0, tiles32.bytes, s));
  BG_CUDA(cudaMemsetAsync(rowcnt.p, 0, rowcnt.bytes, s));
  k_scatter<<<grid1(valid), 256, 0, s>>>(sk, idx.as<uint32_t>(), valid,
                                         static_cast<uint64_t>(tcols), tiles32.as<uint32_t>(),
                                         m->col_ind.as<uint32_t>(),
                                         rowcnt.as<unsigned long long>());
  BG_LAUNCH_CHECK();
  k_narrow<<<grid1(m->nnz), 256, 0, s>>>(tiles32.as<uint32_t>(), m->nnz, m->tiles.as<uint16_t>());
  BG_LAUNCH_CHECK();
  cub::DeviceScan::InclusiveSum(tmp.p, rscan_bytes, rowcnt.as<unsigned long long>(),
                                m->row_ptr.as<unsigned long long>() + 1, static_cast<int>(tcols),
                                s);
  BG_LAUNCH_CHECK();
  frdc_finalize(*m, s);  // synchronizes; temporaries are safe to free after
  return m;
}

namespace {
uint16_t allowed_tile_mask(int rmax, int cmax) {
  uint16_t msk = 0;
  for (int r = 0; r < rmax; ++r)
    for (int c = 0; c < cmax; ++c) msk |= static_cast<uint16_t>(1u << (15 - (4 * r + c)));
  return msk;
}
}  // namespace

// ref: FrdcMatrix constructor validation (bitsparse.cpp:40-70).
std::unique_ptr<bg_frdc> frdc_from_host(int64_t rows, int64_t cols, const uint64_t* rp,
                                        const uint32_t* ci, const uint16_t* ti, int64_t nnz,
                                        cudaStream_t s) {
  if (rows < 0 || cols < 0) fail("FRDC: negative dimension");
  const int64_t trows = (rows + 3) / 4, tcols = (cols + 3) / 4;
  if (tcols > 0xFFFFFFFEll) fail("FRDC: too many tile columns");
  if (!rp) fail("FRDC: row_ptr length mismatch");
  if (rp[0] != 0 || rp[trows] != static_cast<uint64_t>(nnz))
    fail("FRDC: offsets do not match payload");
  const int rrem = static_cast<int>(rows & 3), crem = static_cast<int>(cols & 3);
  for (int64_t r = 0; r < trows; ++r) {
    if (rp[r] > rp[r + 1]) fail("FRDC: row_ptr not monotone");
    const int rmax = (rrem && r == trows - 1) ? rrem : 4;
    for (uint64_t k = rp[r]; k < rp[r + 1]; ++k) {
      if (k > rp[r] && ci[k - 1] >= ci[k]) fail("FRDC: tile columns not strictly increasing");
      if (ci[k] >= static_cast<uint64_t>(tcols)) fail("FRDC: tile column out of range");
      if (ti[k] == 0) fail("FRDC: stored all-zero tile");
      const int cmax = (crem && ci[k] == static_cast<uint64_t>(tcols) - 1) ? crem : 4;
      if (ti[k] & ~allowed_tile_mask(rmax, cmax))
        fail("FRDC: boundary tile has bits outside the node range");
    }
  }
  auto m = std::make_unique<bg_frdc>();
  m->rows = rows;
  m->cols = cols;
  m->tile_rows = trows;
  m->tile_cols = tcols;
  m->nnz = nnz;
  m->row_ptr.alloc(static_cast<size_t>(trows + 1) * 8);
  m->col_ind.alloc(static_cast<size_t>(nnz) * 4);
  m->tiles.alloc(static_cast<size_t>(nnz) * 2);
  BG_CUDA(cudaMemcpyAsync(m->row_ptr.p, rp, m->row_ptr.bytes, cudaMemcpyHostToDevice, s));
  if (nnz) {
    BG_CUDA(cudaMemcpyAsync(m->col_ind.p, ci, m->col_ind.bytes, cudaMemcpyHostToDevice, s));
    BG_CUDA(cudaMemcpyAsync(m->tiles.p, ti, m->tiles.bytes, cudaMemcpyHostToDevice, s));
  }
  frdc_finalize(*m, s);
  return m;
}

namespace {
__global__ void k_rebase(const uint64_t* __restrict__ rp, int64_t n, uint64_t base, uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = rp[i] - base;
}
}  // namespace

// Node rows [row0, row1) of A as a standalone FRDC (rows row1-row0, the same
// columns): row0 is a multiple of 4, row1 too unless it is A.rows, so the
// slice is whole tile rows -- row_ptr rebased, col_ind / tiles copied.
std::unique_ptr<bg_frdc> frdc_slice(const bg_frdc& A, int64_t row0, int64_t row1, cudaStream_t s) {
  if (row0 < 0 || row1 < row0 || row1 > A.rows || row0 % 4 || (row1 % 4 && row1 != A.rows))
    fail("FRDC slice: rows must be whole tile rows inside the matrix");
  const int64_t t0 = row0 / 4, t1 = cdiv(row1, 4);
  uint64_t ends[2] = {0, 0};
  BG_CUDA(cudaMemcpyAsync(&ends[0], A.rp() + t0, 8, cudaMemcpyDeviceToHost, s));
  BG_CUDA(cudaMemcpyAsync(&ends[1], A.rp() + t1, 8, cudaMemcpyDeviceToHost, s));
  BG_CUDA(cudaStreamSynchronize(s));
  auto m = std::make_unique<bg_frdc>();
  m->rows = row1 - row0;
  m->cols = A.cols;
  m->tile_rows = t1 - t0;
  m->tile_cols = A.tile_cols;
  m->nnz = static_cast<int64_t>(ends[1] - ends[0]);
  m->row_ptr.alloc(static_cast<size_t>(m->tile_rows + 1) * 8);
  m->col_ind.alloc(static_cast<size_t>(std::max<int64_t>(m->nnz, 1)) * 4);
  m->tiles.alloc(static_cast<size_t>(std::max<int64_t>(m->nnz, 1)) * 2);
  k_rebase<<<grid1(m->tile_rows + 1), 256, 0, s>>>(A.rp() + t0, m->tile_rows + 1, ends[0], m->row_ptr.as<uint64_t>());
  BG_LAUNCH_CHECK();
  if (m->nnz) {
    BG_CUDA(cudaMemcpyAsync(m->col_ind.p, A.ci() + ends[0], static_cast<size_t>(m->nnz) * 4,
                            cudaMemcpyDeviceToDevice, s));
    BG_CUDA(cudaMemcpyAsync(m->tiles.p, A.ti() + ends[0], static_cast<size_t>(m->nnz) * 2,
                            cudaMemcpyDeviceToDevice, s));
  }
  frdc_finalize(*m, s);
  return m;
}

// A rank's share of a prepared graph (SURVEY §8e "each GPU holds its FRDC
// slice"): both adjacency structures cut to node rows [row0, row1); the
// per-node scale vectors stay whole (O(n): the column scales of an
// aggregation index every node).
std::unique_ptr<bg_graph> graph_shard(const bg_graph& g, int64_t row0, int64_t row1, cudaStream_t s) {
  if (g.row0 != 0 || g.structure->rows != g.n) fail("graph shard: the source must be a whole graph");
  auto o = std::make_unique<bg_graph>();
  o->n = g.n;
  o->row0 = row0;
  o->structure = frdc_slice(*g.structure, row0, row1, s);
  o->raw = frdc_slice(*g.raw, row0, row1, s);
  auto copy = [&](DevBuf& d, const DevBuf& src) {
    d.alloc(src.bytes);
    if (src.bytes) BG_CUDA(cudaMemcpyAsync(d.p, src.p, src.bytes, cudaMemcpyDeviceToDevice, s));
  };
  copy(o->norm, g.norm);
  copy(o->mean_row, g.mean_row);
  copy(o->ones, g.ones);
  copy(o->neighbor_count, g.neighbor_count);
  BG_CUDA(cudaStreamSynchronize(s));
  return o;
}

std::unique_ptr<bg_graph> prepare_graph(const int64_t* src, const int64_t* dst, int64_t e,
                                        int64_t n, cudaStream_t s) {
  auto g = std::make_unique<bg_graph>();
  g->n = n;
  g->structure = frdc_build(src, dst, e, n, /*add_self_loops=*/true, /*drop_self=*/false, s);
  g->raw = frdc_build(src, dst, e, n, /*add_self_loops=*/false, /*drop_self=*/true, s);
  const size_t nn = static_cast<size_t>(std::max<int64_t>(n, 1));
  g->norm.alloc(nn * 4);
  g->mean_row.alloc(nn * 4);
  g->ones.alloc(nn * 4);
  g->neighbor_count.alloc(nn * 8);
  if (n > 0)
    k_graph_scales<<<grid1(n), 256, 0, s>>>(g->structure->deg(), g->raw->deg(), n,
                                            g->norm.as<float>(), g->mean_row.as<float>(),
                                            g->ones.as<float>(), g->neighbor_count.as<int64_t>());
  BG_LAUNCH_CHECK();
  BG_CUDA(cudaStreamSynchronize(s));
  return g;
}

}  // namespace bg
