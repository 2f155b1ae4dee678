// Tile sets, dense expansion and statistics of a device FRDC matrix
// (ref: TileSet / gather_tileset / tileset_count / frdc_to_dense / frdc_stats,
// bitsparse.hpp:62-90, bitsparse.cpp:114-169).
//
// A tile set is the gather unit of the paper's Algorithm 1 (lines 1-5):
// ts = word_bits/4 consecutive tiles of one tile row, their four nibble rows
// concatenated into four words (slot s at bits [wb-1-4s, wb-4-4s]), with the
// tile column per slot (0xFFFFFFFF past the end of the row).  On the device
// every tile set of the matrix is assembled at once, one thread per set,
// after an exclusive scan of the per-tile-row set counts; the single-set
// entry point is the same kernel over one set.  The expansion to a dense
// ZeroOne bit matrix ORs each tile's four nibbles into the row words.
#include <cub/device/device_scan.cuh>

#include "ops.cuh"

namespace bg {
namespace {

__global__ void k_set_counts(const uint64_t* __restrict__ rp, int64_t tile_rows, int ts,
                             uint64_t* __restrict__ cnt) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r <= tile_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    cnt[r] = r < tile_rows ? (rp[r + 1] - rp[r] + ts - 1) / ts : 0;  // ref: bitsparse.cpp:129-134
}

// One thread per tile set.  set_ptr[r] = first set of tile row r.
__global__ void k_gather_sets(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                              const uint16_t* __restrict__ ti, int64_t tile_rows,
                              const uint64_t* __restrict__ set_ptr, int wb, int64_t r_only,
                              int64_t set_only, bg_tileset* __restrict__ out) {
  const uint64_t total = r_only >= 0 ? 1 : set_ptr[tile_rows];
  const int ts = wb / 4;
  for (uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    int64_t r, s;
    if (r_only >= 0) {
      r = r_only;
      s = set_only;
    } else {  // the tile row owning set g: last r with set_ptr[r] <= g
      int64_t lo = 0, hi = tile_rows - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (set_ptr[mid] <= g) lo = mid;
        else hi = mid - 1;
      }
      r = lo;
      s = static_cast<int64_t>(g - set_ptr[r]);
    }
    bg_tileset t;
    t.ts = ts;
    t.reserved = 0;
    uint64_t rows[4] = {0, 0, 0, 0};
    const uint64_t begin = rp[r] + static_cast<uint64_t>(s) * ts, end = rp[r + 1];
    for (int k = 0; k < 16; ++k) {  // ref: bitsparse.cpp:146-158
      const uint64_t e = begin + static_cast<uint64_t>(k);
      const bool live = k < ts && e < end;
      t.cols[k] = live ? ci[e] : BG_TILESET_PAD_COL;
      if (live) {
        const uint32_t tile = ti[e];
        const int shift = wb - 4 - 4 * k;
#pragma unroll
        for (int n = 0; n < 4; ++n) rows[n] |= static_cast<uint64_t>((tile >> (12 - 4 * n)) & 0xFu) << shift;
      }
    }
#pragma unroll
    for (int n = 0; n < 4; ++n) t.rows[n] = rows[n];
    out[r_only >= 0 ? 0 : g] = t;
  }
}

// One thread per stored tile: its four nibbles ORed into the owning row words
// (ZeroOne bits, MSB first; 64-bit words are big-endian u32 pairs, so the
// u32 addressing is the same for both widths).
__global__ void k_frdc_to_dense(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                                const uint16_t* __restrict__ ti, int64_t tile_rows, int64_t rows,
                                int64_t words_per_row, uint32_t* __restrict__ out) {
  const int64_t nnz = static_cast<int64_t>(rp[tile_rows]);
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t lo = 0, hi = tile_rows - 1;  // tile row of tile k
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (rp[mid] <= static_cast<uint64_t>(k)) lo = mid;
      else hi = mid - 1;
    }
    const uint32_t t = ti[k];
    const int64_t c0 = 4 * static_cast<int64_t>(ci[k]);
    const int64_t word = c0 >> 5;
    const int sh = 28 - static_cast<int>(c0 & 31);  // a tile's 4 columns never straddle a word
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      const int64_t i = 4 * lo + n;
      const uint32_t nib = (t >> (12 - 4 * n)) & 0xFu;
      if (nib && i < rows) atomicOr(out + i * words_per_row + word, nib << sh);
    }
  }
}

void check_tileset_wb(int wb, const char* who) {
  if (wb != 32 && wb != 64) fail(std::string(who) + ": word_bits must be 32 or 64");
}

int grid_for(int64_t n) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 16LL * sm_count())));
}

}  // namespace
}  // namespace bg

using namespace bg;

extern "C" {

int bg_tileset_count(const bg_frdc* m, int64_t tile_row, int word_bits, int64_t* count) {
  return guard([&] {
    if (!m || !count) fail("tileset_count: null argument");
    check_tileset_wb(word_bits, "tileset_count");
    if (tile_row < 0 || tile_row >= m->tile_rows) fail("tileset_count: tile_row out of range");
    uint64_t rp[2];
    BG_CUDA(cudaMemcpy(rp, m->rp() + tile_row, sizeof rp, cudaMemcpyDeviceToHost));
    const int ts = word_bits / 4;
    *count = static_cast<int64_t>((rp[1] - rp[0] + ts - 1) / ts);
  });
}

int bg_gather_tileset(const bg_frdc* m, int64_t tile_row, int64_t set_index, int word_bits, bg_tileset* out) {
  int64_t sets = 0;
  return guard([&] {
    if (!m || !out) fail("gather_tileset: null argument");
    // ref: bitsparse.cpp:137-143 (checks and messages in this order)
    check_tileset_wb(word_bits, "gather_tileset");
    if (tile_row < 0 || tile_row >= m->tile_rows) fail("gather_tileset: tile_row out of range");
    uint64_t rp[2];
    BG_CUDA(cudaMemcpy(rp, m->rp() + tile_row, sizeof rp, cudaMemcpyDeviceToHost));
    sets = static_cast<int64_t>((rp[1] - rp[0] + word_bits / 4 - 1) / (word_bits / 4));
    if (set_index < 0 || set_index >= sets) fail("gather_tileset: set_index out of range");
    DevBuf d(sizeof(bg_tileset));
    k_gather_sets<<<1, 32>>>(m->rp(), m->ci(), m->ti(), m->tile_rows, nullptr, word_bits, tile_row,
                             set_index, d.as<bg_tileset>());
    BG_LAUNCH_CHECK();
    BG_CUDA(cudaMemcpy(out, d.p, sizeof(bg_tileset), cudaMemcpyDeviceToHost));
  });
}

int bg_tileset_ptr(const bg_frdc* m, int word_bits, uint64_t* set_ptr, int64_t* total, bg_stream stream) {
  return guard([&] {
    if (!m || !set_ptr) fail("tileset_ptr: null argument");
    check_tileset_wb(word_bits, "tileset_ptr");
    cudaStream_t s = S(stream);
    const int64_t n = m->tile_rows + 1;
    DevBuf cnt(static_cast<size_t>(n) * 8);
    k_set_counts<<<grid_for(n), 256, 0, s>>>(m->rp(), m->tile_rows, word_bits / 4, cnt.as<uint64_t>());
    BG_LAUNCH_CHECK();
    size_t tmp = 0;
    BG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.as<uint64_t>(), set_ptr, n, s));
    DevBuf t(std::max<size_t>(tmp, 1));
    BG_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, cnt.as<uint64_t>(), set_ptr, n, s));
    uint64_t tot = 0;
    BG_CUDA(cudaMemcpyAsync(&tot, set_ptr + m->tile_rows, 8, cudaMemcpyDeviceToHost, s));
    BG_CUDA(cudaStreamSynchronize(s));
    if (total) *total = static_cast<int64_t>(tot);
  });
}

int bg_gather_tilesets(const bg_frdc* m, int word_bits, const uint64_t* set_ptr, int64_t total,
                       bg_tileset* sets, bg_stream stream) {
  return guard([&] {
    if (!m || !set_ptr) fail("gather_tilesets: null argument");
    check_tileset_wb(word_bits, "gather_tilesets");
    if (total <= 0 || m->tile_rows == 0) return;
    if (!sets) fail("gather_tilesets: null output");
    k_gather_sets<<<grid_for(total), 256, 0, S(stream)>>>(m->rp(), m->ci(), m->ti(), m->tile_rows, set_ptr,
                                                          word_bits, -1, 0, sets);
    BG_LAUNCH_CHECK();
  });
}

int bg_frdc_to_dense(const bg_frdc* m, int word_bits, uint32_t* out, bg_stream stream) {
  return guard([&] {
    if (!m) fail("frdc_to_dense: null matrix");
    if (word_bits != 32 && word_bits != 64) fail("BitDenseMatrix: word_bits must be 32 or 64");
    const int64_t wpr = spw(m->cols, word_bits);
    const size_t bytes = static_cast<size_t>(m->rows * wpr) * 4;
    if (!bytes) return;
    if (!out) fail("frdc_to_dense: null output");
    cudaStream_t s = S(stream);
    BG_CUDA(cudaMemsetAsync(out, 0, bytes, s));
    if (m->nnz && m->tile_rows)
      k_frdc_to_dense<<<grid_for(m->nnz), 256, 0, s>>>(m->rp(), m->ci(), m->ti(), m->tile_rows, m->rows, wpr,
                                                       out);
    BG_LAUNCH_CHECK();
  });
}

int bg_frdc_stats_get(const bg_frdc* m, bg_frdc_stats* out) {
  return guard([&] {
    if (!m || !out) fail("frdc_stats: null argument");
    // ref: bitsparse.cpp:162-169 (nnz_bits is counted once at build)
    out->nnz_tiles = static_cast<uint64_t>(m->nnz);
    out->nnz_bits = static_cast<uint64_t>(m->nnz_bits);
    out->bytes = static_cast<uint64_t>(m->tile_rows + 1) * 8 + static_cast<uint64_t>(m->nnz) * 6;
    out->fill_ratio = m->nnz ? static_cast<double>(m->nnz_bits) / (16.0 * static_cast<double>(m->nnz)) : 0.0;
  });
}

}  // extern "C"
