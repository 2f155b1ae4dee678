// Internal launchers shared by the C ABI entry points and the model engine.
#pragma once

#include <memory>

#include "common.cuh"

// Device-resident FRDC matrix (ref: FrdcMatrix, bitsparse.hpp:26-60) plus the
// per-node-row degree the aggregation kernels use for thresholds.
constexpr int kSliverPad = 8;
constexpr uint32_t kSliverSentinel = 0xFFFFFFF8u;  // node column 2^29-1, no extra bits
constexpr int kBitPad = 64;

// Node rows at least this long are hub rows of the BB aggregations (hubs.cu).
constexpr int kHubDeg = 2048;

namespace bg {
// Fused epilogue of an F-output aggregation (north-star item 4): when the
// aggregation's F result feeds BatchNorm [ReLU] [Binarize] (graphops.cpp:
// 337-355, :89-97; binarize bitdense.cpp:83), the kernels apply BatchNorm
// (and ReLU) to each value as they produce it and either store the floats or
// -- with a following Binarize -- the packed sign bits only, so the
// activation never round-trips through HBM unpacked.  Set by the executor
// around the call (FEpiScope); zero = plain store.
struct FEpi {
  const float* g = nullptr;  // BatchNorm gamma, beta, mean, sigma (g null: none)
  const float* b = nullptr;
  const float* m = nullptr;
  const float* s = nullptr;
  int relu = 0;
  uint32_t* bits = nullptr;  // binarize-pack output: MSB-first u32 words, bspw per row
  int64_t bspw = 0;
};
const FEpi& current_fepi();
struct FEpiScope {
  explicit FEpiScope(const FEpi& e);
  ~FEpiScope();
  FEpiScope(const FEpiScope&) = delete;
  FEpiScope& operator=(const FEpiScope&) = delete;
};

// BatchNorm in double with the reference's operation order, then ReLU.
__device__ __forceinline__ float fepi_apply(const FEpi& e, float v, int64_t k) {
  if (e.g) {
    const double sigma = fmax(static_cast<double>(e.s[k]), 1e-12);
    const double num = __dmul_rn(static_cast<double>(e.g[k]), __dsub_rn(static_cast<double>(v), static_cast<double>(e.m[k])));
    v = __double2float_rn(__dadd_rn(__ddiv_rn(num, sigma), static_cast<double>(e.b[k])));
  }
  if (e.relu) v = v > 0.0f ? v : 0.0f;
  return v;
}

// One thread owns output word wd (columns 32*wd .. 32*wd+31) of row i:
// val(bb) is the plain value of column 32*wd+bb.  Stores the epilogue's
// floats or, with e.bits, the packed word (columns >= f stay zero).
template <class V>
__device__ __forceinline__ void fepi_store_word(const FEpi& e, float* out_f, int64_t i, int64_t f, int64_t wd, V&& val) {
  if (e.bits) {
    uint32_t w = 0;
    for (int bb = 0; bb < 32; ++bb) {
      const int64_t k = 32 * wd + bb;
      if (k >= f) break;
      if (fepi_apply(e, val(bb), k) >= 0.0f) w |= 0x80000000u >> bb;
    }
    e.bits[i * e.bspw + wd] = w;
  } else {
    for (int bb = 0; bb < 32; ++bb) {
      const int64_t k = 32 * wd + bb;
      if (k >= f) break;
      out_f[i * f + k] = fepi_apply(e, val(bb), k);
    }
  }
}

// Lanes of a warp own columns fbase+lane (fbase a multiple of 32, the call
// warp-uniform): store value v of column k through the epilogue.
__device__ __forceinline__ void fepi_store_lane(const FEpi& e, float* out_f, int64_t i, int64_t f, int64_t k, float v) {
  const float y = k < f ? fepi_apply(e, v, k) : 0.0f;
  if (e.bits) {
    const uint32_t word = __brev(__ballot_sync(0xFFFFFFFFu, k < f && y >= 0.0f));
    if ((threadIdx.x & 31) == 0) e.bits[i * e.bspw + (k >> 5)] = word;
  } else if (k < f) {
    out_f[i * f + k] = y;
  }
}
}  // namespace bg

struct bg_frdc {
  int64_t rows = 0, cols = 0, tile_rows = 0, tile_cols = 0, nnz = 0, nnz_bits = 0;
  int64_t max_deg = 0;
  // Most bits of one node row that land in the tiles of G consecutive lanes
  // (tile k of a tile row goes to lane k % 32) -- sizes the bit-sliced
  // counters of the aggregation kernels.  Index: 0 -> G=4, 1 -> G=8.
  int64_t max_slot[2] = {0, 0};
  // Bumped whenever the arrays change (finalize) or a derived view below is
  // (re)built: a CUDA graph captured over the views' pointers is valid only
  // while gen is unchanged.
  uint64_t gen = 0;
  bg::DevBuf row_ptr;  // u64[tile_rows + 1]
  bg::DevBuf col_ind;  // u32[nnz]
  bg::DevBuf tiles;    // u16[nnz]
  bg::DevBuf degree;   // i32[rows]
  // Node-major view of the same bit tiles, built once on first use
  // (frdc_slivers): for node row i, one u32 per nonzero 1x4 nibble of its
  // tiles, ascending tile column (the reference's walk order,
  // kernels.cpp:218-234): (node column of the nibble's first bit) << 3 | mask
  // of the following columns present (bit k-1 <-> first + k).  Each row is
  // padded to a multiple of kSliverPad entries with kSliverSentinel.
  bg::DevBuf sliver_ptr;  // u64[rows + 1]
  bg::DevBuf slivers;     // u32[nslivers]
  int64_t nslivers = -1;  // -1: not built
  // most entries (padded) / most (bits - slivers) in one node row of degree
  // < kHubDeg (the hub rows are counted by hub_bb)
  int64_t max_sl_row = 0;
  int64_t max_extra_bits = 0;
  // Bit-entry view (frdc_bitview), built once on first use: for node row i,
  // the node column of every adjacency bit in ascending order (the
  // reference's walk order), padded to a multiple of kBitPad entries with the
  // column count (the index of the zero record the consumers append).
  bg::DevBuf bit_ptr;   // u64[rows + 1]
  bg::DevBuf bit_cols;  // u32
  int64_t nbits_view = -1;  // -1: not built
  // Column-windowed view (window.cu), built once on first use: node rows in
  // blocks of T (one CTA, one row per thread), node columns in half-windows of
  // Wn (one shared-memory ring slot).  Each warp of each block owns one stream
  // of ELL groups (4 u16 entries per lane per 256-byte group) covering all nw
  // steps in order: stream base seg[b*(T/32)+v], step lengths steplen[.. *nw + k].
  struct Windows {
    int T = 0, Wn = 0, nw = 0, nb = 0, rw = 0;  // T: rows per block; rw: rows per warp stream
    bg::DevBuf seg;      // u32[nb*(T/32) + 1] stream bases, in ELL groups
    bg::DevBuf steplen;  // u16[nb*(T/32)*nw] groups per step
    bg::DevBuf ell;      // u16 entries (ring record index)
  } win;
  // Hub rows (hubs.cu), found once on first use: node rows of degree >=
  // kHubDeg.  The BB aggregation kernels see them as empty rows and hub_bb
  // counts them split over the SMs.
  struct Hubs {
    int64_t n = -1;  // -1: not built
    int64_t nchunks = 0;
    int64_t max_light_deg = 0;  // largest degree of the other rows
    bg::DevBuf rows;            // i32[n]
    bg::DevBuf chunks;          // uint4[nchunks]: first tile, tiles, hub << 2 | row in tile row
    bg::DevBuf cnt;             // i32[n * cnt_words * 32], zero between calls
    int64_t cnt_words = 0;
  } hub;
  const uint64_t* srp() const { return sliver_ptr.as<uint64_t>(); }
  const uint32_t* sl() const { return slivers.as<uint32_t>(); }
  const uint64_t* rp() const { return row_ptr.as<uint64_t>(); }
  const uint32_t* ci() const { return col_ind.as<uint32_t>(); }
  const uint16_t* ti() const { return tiles.as<uint16_t>(); }
  const int32_t* deg() const { return degree.as<int32_t>(); }
};

struct bg_graph {
  int64_t n = 0;     // node count of the whole graph
  int64_t row0 = 0;  // a shard: the FRDC rows are node rows [row0, row0 + structure->rows)
  std::unique_ptr<bg_frdc> structure, raw;
  bg::DevBuf norm, mean_row, ones, neighbor_count;
};

namespace bg {

// ---- bitdense.cu ---------------------------------------------------------
void binarize(const float* x, int64_t rows, int64_t cols, int wb, uint32_t* out, cudaStream_t s);
// mean |x| per row (axis 0) or column (axis 1), double in index order.
void l1_scales(const float* x, int64_t rows, int64_t cols, int axis, float* out, cudaStream_t s);
void unpack(const uint32_t* bits, int64_t rows, int64_t cols, int wb, int semantics, float* out,
            cudaStream_t s);
void transpose_bits(const uint32_t* in, int64_t rows, int64_t cols, int wb, uint32_t* out,
                    cudaStream_t s);

// ---- frdc.cu -------------------------------------------------------------
// drop_self_edges: skip (s, s) input edges (the loop-free structure of
// prepare_graph, graphops.cpp:149-154).
std::unique_ptr<bg_frdc> frdc_build(const int64_t* src, const int64_t* dst, int64_t e, int64_t n,
                                    bool add_self_loops, bool drop_self_edges, cudaStream_t s);
std::unique_ptr<bg_frdc> frdc_from_host(int64_t rows, int64_t cols, const uint64_t* rp,
                                        const uint32_t* ci, const uint16_t* ti, int64_t nnz,
                                        cudaStream_t s);
void frdc_finalize(bg_frdc& m, cudaStream_t s);  // degree, nnz_bits, max_deg
// ---- container.cu: FRDC container I/O (bitsparse.cpp:171-222) -----------
size_t frdc_container_bytes(const bg_frdc& m);
void frdc_serialize(const bg_frdc& m, int word_bits, void* buf);
std::unique_ptr<bg_frdc> frdc_deserialize(const void* buf, size_t len, int* word_bits, cudaStream_t s);
void frdc_write_file(const bg_frdc& m, int word_bits, const char* path);
std::unique_ptr<bg_frdc> frdc_read_file(const char* path, int* word_bits, cudaStream_t s);
void frdc_slivers(bg_frdc& m, cudaStream_t s);   // build the node-major sliver view once
void frdc_bitview(bg_frdc& m, cudaStream_t s);   // build the bit-entry view once (from slivers)
std::unique_ptr<bg_graph> prepare_graph(const int64_t* src, const int64_t* dst, int64_t e,
                                        int64_t n, cudaStream_t s);
std::unique_ptr<bg_frdc> frdc_slice(const bg_frdc& A, int64_t row0, int64_t row1, cudaStream_t s);
std::unique_ptr<bg_graph> graph_shard(const bg_graph& g, int64_t row0, int64_t row1, cudaStream_t s);

// ---- bmm.cu --------------------------------------------------------------
// Binary product against transposed weight bits wt (n x spw(k)).
//   a_bits != nullptr: packed +-1 rows (rows x spw(k)); else a_f fp32 rows x k,
//   binarized on the fly (fused FBB/FBF prologue).
// out_bits: B output (dot >= 0, no scale), else out_f = float((alpha*dot)*beta).
struct BmmArgs {
  const uint32_t* a_bits = nullptr;
  const float* a_f = nullptr;
  const float* alpha = nullptr;  // per-row scale or null (1.0)
  const uint32_t* wt = nullptr;
  const float* beta = nullptr;  // per-column scale or null (1.0)
  int64_t rows = 0, k = 0, n = 0;
  int wb = 32;
  uint32_t* out_bits = nullptr;
  float* out_f = nullptr;
  // Paired F->B product (two weight matrices on one fp32 input, the input
  // read once): wt holds W1's n columns, zero rows up to n1pad = 32*ceil(n/32),
  // then W2's n2 columns; the second result goes to out_bits2.
  uint32_t* out_bits2 = nullptr;
  int64_t n2 = 0;
};
void bmm(const BmmArgs& a, cudaStream_t s);
// Both products of a paired BmmArgs; false (nothing launched) when no kernel
// takes the pair, so the caller runs the two products separately.
bool bmm_pair(const BmmArgs& a, cudaStream_t s);
// fbb_tc.cu: F->B products (and pairs) on tcgen05.mma.kind::i8; false when not eligible
bool fbb_tc(const BmmArgs& a, cudaStream_t s);
// fbb_bulk.cu: F-input products (B or F output, <= 128 columns, pairs) with
// every row requested at kernel start by bulk copies; false when not eligible
bool fbb_bulk(const BmmArgs& a, cudaStream_t s);
// fbb_tmem.cu: F->B products with the A operand in tensor memory (wide K)
bool fbb_tmem(const BmmArgs& a, cudaStream_t s, bool pair = false);

// ---- bspmm.cu ------------------------------------------------------------
// Integer path (BBB / BBF): out(i,k) = 2*#{j in N(i): x_jk = 1} - deg_i.
// [row0, row1): node rows to produce (tile-row aligned start); -1 = all.
void bspmm_bb(const bg_frdc& A, const uint32_t* x, int64_t f, int wb, uint32_t* out_bits,
              float* out_f, cudaStream_t s, int64_t row0 = 0, int64_t row1 = -1);
// Real-valued walk: F activations (x_f) or B activations with factorized
// adjacency (x_bits + col_scale).  Ascending-j double accumulation.
struct SpmmFArgs {
  const float* x_f = nullptr;
  const uint32_t* x_bits = nullptr;
  int xwb = 32;
  const float* row_scale = nullptr;
  const float* col_scale = nullptr;
  int64_t f = 0;
  uint32_t* out_bits = nullptr;
  int owb = 32;
  float* out_f = nullptr;
};
void bspmm_f(const bg_frdc& A, const SpmmFArgs& a, cudaStream_t s, int64_t row0 = 0,
             int64_t row1 = -1);

// ---- gcn_fused.cu: MM.BBF + BSpMM.FBF (+ softmax) without materializing Y ----
// rec_buf holds n + 1 64-byte records (the last one zero, for padding entries).
bool gcn1_fused_supported(const bg_frdc& A, int64_t K, int wb, int64_t C);
void gcn1_records(const uint32_t* h, int64_t n, int64_t K, int wb, const uint32_t* wt,
                  const float* beta, int64_t C, uint32_t* rec_buf, cudaStream_t s);
void gcn1_aggregate(const bg_frdc& A, const uint32_t* rec_buf, int64_t K, int wb,
                    const uint32_t* wt, const float* beta, int64_t C, float* logits, float* probs,
                    cudaStream_t s, int64_t row0 = 0, int64_t row1 = -1);

// ---- sliver.cu: the same aggregations over the node-major sliver view -----
// (builds the view on first use, so the first call synchronizes once)
void sliver_bb(bg_frdc& A, const uint32_t* x, int64_t f, int wb, uint32_t* out_bits, float* out_f,
               cudaStream_t s, int64_t r0 = 0, int64_t r1 = -1);
void sliver_f(bg_frdc& A, const SpmmFArgs& a, cudaStream_t s, int64_t r0 = 0, int64_t r1 = -1);
void sliver_gcn1_records(const uint32_t* h, int64_t n, int64_t K, int wb, const uint32_t* wt,
                         const float* beta, int64_t C, uint32_t* rec, cudaStream_t s);
void sliver_gcn1_aggregate(bg_frdc& A, const uint32_t* rec, int64_t K, int wb, const uint32_t* wt,
                           const float* beta, int64_t C, float* logits, float* probs,
                           cudaStream_t s, int64_t r0 = 0, int64_t r1 = -1);
// Aggregation layout (bg_set_aggregation; BG_AGG_* of bitgnn_b200.h).  All
// layouts produce identical results.  aggregation_generation() changes on
// every set, so captured CUDA graphs are re-recorded.
int aggregation_mode();
int window_nodes_setting();  // 0 = default window size
uint64_t aggregation_generation();
void set_aggregation(int mode, int window_nodes);
inline bool use_slivers() { return aggregation_mode() != BG_AGG_TILES; }

// ---- window.cu: BSpMM.BBB/BBF with the packed operand staged in shared
// memory one column window at a time (bulk async copies), for graphs dense
// enough that streaming the operand costs less than per-edge L2 gathers.
// Returns false (nothing launched) when the shape is not eligible or the mode
// is SLIVERS/TILES; mode WINDOW skips the cost model (tests).
bool window_bb(bg_frdc& A, const uint32_t* x, int64_t f, int wb, uint32_t* out_bits,
               float* out_f, cudaStream_t s, int64_t r0, int64_t r1);
// sliver.cu: BBB/BBF for short rows (lane group per row over the bit-entry
// view); false when not eligible (mode != AUTO, > 8 words, average degree >= 64).
// hubs.cu: the hub rows of [r0, r1) (BSpMM.BBB / BBF), after the main kernel
void frdc_hubs(bg_frdc& m, cudaStream_t s);
int64_t light_max_deg(bg_frdc& m, cudaStream_t s);  // largest degree below kHubDeg
void hub_bb(bg_frdc& A, const uint32_t* x, int64_t f, int64_t xspw, uint32_t* out_bits, float* out_f,
            cudaStream_t s, int64_t r0, int64_t r1);
bool rowgroup_bb(bg_frdc& A, const uint32_t* x, int64_t f, int64_t xspw, uint32_t* out_bits, float* out_f,
                 cudaStream_t s, int64_t r0, int64_t r1);

// ---- packed.cu: two-valued F activations kept as bits ----------------------
void and_words(const uint32_t* a, const uint32_t* b, int64_t n, uint32_t* out, cudaStream_t s);
void expand_packed(const uint32_t* bits, int64_t rows, int64_t cols, int wb, float pval, float* out, cudaStream_t s);
// every row of an F->B product on an all-ones input (the binarized packed tensor)
void packed_const_rows(const uint32_t* wt, int64_t k, int64_t n, int wb, int64_t rows, uint32_t* out,
                       cudaStream_t s);
bool packed_fbf_supported(int64_t n);
// MM.FBF on rows [r0, r1) of a packed input (+ the row softmax into probs)
// (table: packed_fbf_table_bytes of workspace)
size_t packed_fbf_table_bytes(int64_t k, int64_t n);
void packed_fbf(const uint32_t* bits, int64_t r0, int64_t r1, int64_t k, int xwb, float pval, const uint32_t* wt,
                int wb, const float* beta, int64_t n, float* logits, float* probs, float* table, cudaStream_t s);

// ---- elementwise.cu ------------------------------------------------------
void add_bbb(const uint32_t* a, const uint32_t* b, int64_t words, uint32_t* out, cudaStream_t s);
void add_bbf(const uint32_t* a, const uint32_t* b, int64_t rows, int64_t cols, int wb, float* out,
             cudaStream_t s, bool fuse_relu = false);
void add_fff(const float* a, const float* b, int64_t n, float* out, cudaStream_t s, bool fuse_relu = false);
void relu(float* x, int64_t n, cudaStream_t s);
void softmax_rows(const float* x, int64_t rows, int64_t cols, float* out, cudaStream_t s);
void scale_rows_double(float* x, int64_t rows, int64_t cols, const int64_t* cnt, cudaStream_t s);
// BatchNorm [+ ReLU] [+ binarize-pack] in one pass over x (the epilogue of
// an F producer that does not take FEpi itself): out_bits (bspw words per
// row) instead of out_f when non-null.
void bn_act(const float* x, int64_t rows, int64_t cols, const FEpi& e, float* out_f, cudaStream_t s);
void batchnorm(const float* x, int64_t rows, int64_t cols, const float* g, const float* b,
               const float* m, const float* sg, float* out, cudaStream_t s);
void scl(const float* x, int64_t rows, int64_t cols, const float* r, const float* c, float* out,
         cudaStream_t s);
void dense_mm(const float* a, const float* w, int64_t rows, int64_t k, int64_t cols, float* out,
              cudaStream_t s);
void concat_bits(const uint32_t* a, int64_t ca, const uint32_t* b, int64_t cb, int64_t rows,
                 int wb, uint32_t* out, cudaStream_t s);
void concat_f(const float* a, int64_t ca, const float* b, int64_t cb, int64_t rows, float* out,
              cudaStream_t s);

}  // namespace bg
