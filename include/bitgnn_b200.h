/*
 * bitgnn_b200.h -- C ABI of the B200-native binary-GNN inference path.
 *
 * This is the drop-in boundary for the reference's operator API in
 * /root/reference/proj/include/bitgnn (abbreviated "ref:").  Each entry point
 * names the reference interface it replaces.  Plain pointers and sizes only:
 * device buffers are CUDA device pointers, streams are cudaStream_t passed as
 * void*.  Every call returns a status code; bg_last_error() holds the message
 * (thread-local), worded like the reference's exception text so the C++ shim
 * (include/bitgnn_b200/bitgnn.hpp) can rethrow the reference's exception types:
 *
 *   BG_INVALID_ARGUMENT -> std::invalid_argument   (contract violations)
 *   BG_RUNTIME_ERROR    -> std::runtime_error      (layer failures, I/O)
 *   BG_LOGIC_ERROR      -> std::logic_error
 *   BG_CUDA_ERROR       -> std::runtime_error      (device failure)
 *
 * Layouts are the reference's (ref: bitdense.hpp:55-60, bitsparse.hpp:22-25):
 * row-major; packed rows of ceil(cols/word_bits)*(word_bits/32) u32 words,
 * column j at bit 31 - j%32 of word j/32 (MSB first), padding bits zero;
 * FRDC = CSR over 4x4 bit tiles (u64 row_ptr, u32 col_ind, u16 tiles with
 * bit (r,c) at 15-(4r+c)).  All kernels are sm_100a CUDA; there is no CPU
 * fallback: a call on a machine without a B200 fails with BG_CUDA_ERROR.
 */
#ifndef BITGNN_B200_H
#define BITGNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BG_OK 0
#define BG_INVALID_ARGUMENT 1
#define BG_RUNTIME_ERROR 2
#define BG_LOGIC_ERROR 3
#define BG_CUDA_ERROR 4

typedef void* bg_stream; /* cudaStream_t; NULL = legacy default stream */

const char* bg_last_error(void);
int bg_version(void);

/* ---- aggregation layout (process-wide tuning, like the OpenMP thread count
 * of the reference; every layout gives identical results) ------------------
 * AUTO picks per call: column windows staged in shared memory for dense
 * graphs (BBB/BBF, 4-word rows), node-major slivers otherwise.  window_nodes
 * = 0 keeps the default window size (tests use small windows).  Initial
 * values come from env BG_AGGREGATION=auto|slivers|tiles|window and
 * BG_WINDOW_NODES. */
enum { BG_AGG_AUTO = 0, BG_AGG_SLIVERS = 1, BG_AGG_TILES = 2, BG_AGG_WINDOW = 3 };
int bg_set_aggregation(int mode, int window_nodes);
int bg_get_aggregation(int* mode, int* window_nodes);
/* Whole-forward persistent kernel for small graphs (one cooperative launch
 * for a binary GCN chain, results identical to the layer-by-layer forward).
 * Off by default (measured slower on B200 than the captured layer-by-layer
 * forward); enable = 1 turns it on process-wide (as does env
 * BG_PERSISTENT=1).  Traced and timed forwards always run layer by layer. */
int bg_set_persistent(int enable);

/* ---- device memory (so C/C++ hosts need no CUDA headers) ---------------- */
enum { BG_COPY_H2D = 0, BG_COPY_D2H = 1, BG_COPY_D2D = 2 };
int bg_device_count(int* count);
int bg_device_alloc(size_t bytes, void** out); /* cudaMalloc; 0 bytes -> NULL */
int bg_device_free(void* p);
/* Copy on `stream`, then wait for the stream (synchronous for the caller). */
int bg_memcpy(void* dst, const void* src, size_t bytes, int kind, bg_stream stream);
int bg_memset(void* dst, int value, size_t bytes, bg_stream stream);
int bg_stream_synchronize(bg_stream stream);

/* ---- enums (ref: kernels.hpp:15-33, bitdense.hpp:15-16, graphops.hpp:44-55) */
enum { BG_F = 0, BG_B = 1 };                                  /* Precision */
enum { BG_BMM = 0, BG_BSPMM = 1, BG_ADD = 2, BG_CONCAT = 3 }; /* KernelOp */
enum { BG_AXIS_ROW = 0, BG_AXIS_COL = 1 };                    /* Axis */
enum { BG_ZERO_ONE = 0, BG_PLUS_MINUS = 1 };                  /* BitSemantics */
enum { /* TrinaryStrategy; accepted and semantically inert (ref: test_kernels.cpp:276-303) */
       BG_STRATEGY_DEFAULT = -1,
       BG_IF_ELSE = 0,
       BG_AND_ANDNOT = 1,
       BG_TWO_AND_MINUS_POPC = 2 };
enum { /* LayerKind */
       BG_LAYER_GCN = 0,
       BG_LAYER_SAGE = 1,
       BG_LAYER_GRAPHCONV = 2,
       BG_LAYER_FC = 3,
       BG_LAYER_AGGREGATE = 4,
       BG_LAYER_RELU = 5,
       BG_LAYER_BATCHNORM = 6,
       BG_LAYER_SOFTMAX = 7,
       BG_LAYER_BINARIZE = 8,
       BG_LAYER_SCALE = 9 };

/* ref: KernelVariant (kernels.hpp:23-33) */
typedef struct bg_variant {
  int32_t op, in1, in2, out;
} bg_variant;

int bg_variant_parse(const char* text, bg_variant* out);      /* ref: KernelVariant::parse */
int bg_variant_valid(bg_variant v);                           /* ref: KernelVariant::valid, 1/0 */
int bg_variant_name(bg_variant v, char* buf, size_t buf_len); /* ref: KernelVariant::name */

/* A matrix operand in device memory: ref MatOperand = variant<DenseMatrix,
 * BitOperand> (kernels.hpp:37-42).  F: data = float[rows*cols].  B: data =
 * uint32[rows*bg_storage_words_per_row(cols, word_bits)], optional scale
 * (float[rows] for Axis::Row, float[cols] for Axis::Col), NULL when absent. */
typedef struct bg_mat {
  int32_t precision;
  int32_t word_bits;
  int32_t semantics;
  int32_t scale_axis;
  int64_t rows, cols;
  void* data;
  float* scale;
} bg_mat;

/* ref: BitDenseMatrix::storage_words_per_row (bitdense.hpp:72-73) */
int64_t bg_storage_words_per_row(int64_t cols, int word_bits);

/* ---- bitdense (ref: bitdense.hpp:110-141) ------------------------------- */
/* ref: binarize (bitdense.cpp:71-88): bit = (x >= 0) */
int bg_binarize(const float* x, int64_t rows, int64_t cols, int word_bits, uint32_t* out,
                bg_stream stream);
/* ref: binarize_with_scale (bitdense.cpp:90-104): mean |x| in double, floor 1e-12 */
int bg_binarize_with_scale(const float* x, int64_t rows, int64_t cols, int axis, int word_bits,
                           uint32_t* out_bits, float* out_scale, bg_stream stream);
/* ref: unpack (bitdense.cpp:106-114) */
int bg_unpack(const uint32_t* bits, int64_t rows, int64_t cols, int word_bits, int semantics,
              float* out, bg_stream stream);
/* ref: transpose (bitdense.cpp:189-210): out is cols x rows bits */
int bg_transpose(const uint32_t* in, int64_t rows, int64_t cols, int word_bits, uint32_t* out,
                 bg_stream stream);

/* ---- bitsparse (ref: bitsparse.hpp:26-81) -------------------------------- */
typedef struct bg_frdc bg_frdc; /* device-resident FrdcMatrix, immutable after build */

typedef struct bg_frdc_info {
  int64_t node_rows, node_cols, tile_rows, tile_cols, nnz_tiles, nnz_bits, max_row_degree;
  const uint64_t* row_ptr; /* device, tile_rows + 1 */
  const uint32_t* col_ind; /* device, nnz_tiles */
  const uint16_t* tiles;   /* device, nnz_tiles */
  const int32_t* degree;   /* device, node_rows: set bits per node row */
} bg_frdc_info;

/* ref: frdc_from_edges (bitsparse.cpp:72-112), built on the device.  src/dst
 * are DEVICE int64 arrays of n_edges directed (src, dst) pairs. */
int bg_frdc_from_edges(const int64_t* src, const int64_t* dst, int64_t n_edges, int64_t n_nodes,
                       int add_self_loops, bg_frdc** out, bg_stream stream);
/* ref: FrdcMatrix constructor (bitsparse.cpp:40-70) with its validation; HOST arrays. */
int bg_frdc_from_host(int64_t node_rows, int64_t node_cols, const uint64_t* row_ptr,
                      const uint32_t* col_ind, const uint16_t* tiles, int64_t nnz_tiles,
                      bg_frdc** out, bg_stream stream);
int bg_frdc_info_get(const bg_frdc* m, bg_frdc_info* info);
/* Copy the three FRDC arrays to HOST buffers (row_ptr: tile_rows+1, others nnz). */
int bg_frdc_download(const bg_frdc* m, uint64_t* row_ptr, uint32_t* col_ind, uint16_t* tiles);
/* Tile sets: the gather unit of Algorithm 1 (ref: TileSet, bitsparse.hpp:62-71):
 * ts = word_bits/4 consecutive tiles of a tile row, nibble row n of slot s at
 * bits [word_bits-1-4s, word_bits-4-4s] of rows[n]; cols[s] = tile column,
 * BG_TILESET_PAD_COL past the end of the row (and for slots >= ts). */
#define BG_TILESET_PAD_COL 0xFFFFFFFFu
typedef struct bg_tileset {
  int32_t ts;
  int32_t reserved;
  uint64_t rows[4];
  uint32_t cols[16];
} bg_tileset;
/* ref: tileset_count (bitsparse.cpp:129-134) */
int bg_tileset_count(const bg_frdc* m, int64_t tile_row, int word_bits, int64_t* count);
/* ref: gather_tileset (bitsparse.cpp:136-160), one set into a HOST struct;
 * the reference's checks and messages (word_bits, tile_row, set_index). */
int bg_gather_tileset(const bg_frdc* m, int64_t tile_row, int64_t set_index, int word_bits,
                      bg_tileset* out);
/* Every tile set of the matrix on the device (Algorithm 1 lines 1-5 for all
 * tile rows at once).  set_ptr: DEVICE u64[tile_rows + 1], the exclusive scan
 * of tileset_count (set_ptr[r] = first set of tile row r); *total = sets.
 * sets: DEVICE bg_tileset[total], set set_ptr[r] + s = gather_tileset(m, r, s). */
int bg_tileset_ptr(const bg_frdc* m, int word_bits, uint64_t* set_ptr, int64_t* total, bg_stream stream);
int bg_gather_tilesets(const bg_frdc* m, int word_bits, const uint64_t* set_ptr, int64_t total,
                       bg_tileset* sets, bg_stream stream);
/* ref: frdc_to_dense (bitsparse.cpp:114-127): ZeroOne bits, DEVICE
 * node_rows x bg_storage_words_per_row(node_cols, word_bits) u32. */
int bg_frdc_to_dense(const bg_frdc* m, int word_bits, uint32_t* out, bg_stream stream);
/* ref: FrdcStats / frdc_stats (bitsparse.hpp:83-90, bitsparse.cpp:162-169) */
typedef struct bg_frdc_stats {
  uint64_t nnz_tiles, nnz_bits, bytes;
  double fill_ratio; /* nnz_bits / (16 nnz_tiles), 0 when empty */
} bg_frdc_stats;
int bg_frdc_stats_get(const bg_frdc* m, bg_frdc_stats* out);
/* FRDC container (ref: write_frdc / read_frdc, bitsparse.cpp:171-222; layout
 * bitsparse.hpp:92-96): little-endian bytes identical to the reference writer.
 * Format and I/O faults are BG_RUNTIME_ERROR with the reference's messages
 * ("FRDC: bad magic", "FRDC: truncated file", ...); a payload that fails the
 * FrdcMatrix checks is BG_INVALID_ARGUMENT.  Reads stage through pinned host
 * memory straight to the device. */
int bg_frdc_serialized_size(const bg_frdc* m, size_t* bytes);
int bg_frdc_serialize(const bg_frdc* m, int word_bits, void* buf, size_t buf_len);
int bg_frdc_deserialize(const void* buf, size_t len, bg_frdc** out, int* word_bits, bg_stream stream);
int bg_frdc_write_file(const bg_frdc* m, int word_bits, const char* path);
int bg_frdc_read_file(const char* path, bg_frdc** out, int* word_bits, bg_stream stream);

/* ---- graph file readers (ref: graphio.hpp:11-24, graphio.cpp:72-176) -------
 * Host edge lists: "src dst [weight]" lines ('#'/'%' comments), MatrixMarket
 * coordinate (pattern/real/integer, general/symmetric; 1-based, mirrored when
 * symmetric or undirected), and load_graph's sniffing of a file (FRDC
 * container -> its edges, "%%MatrixMarket" -> MM, else an edge list).
 * forced_nodes = -1 infers the node count.  Errors: BG_RUNTIME_ERROR with the
 * reference's "name:line: message" text.  The result is a host-side handle:
 * read its arrays with bg_edges_info (valid until bg_edges_destroy), then
 * build the device graph with bg_frdc_from_edges / bg_prepare_graph. */
typedef struct bg_edges bg_edges;
int bg_read_edge_list(const char* text, size_t len, const char* name, int64_t forced_nodes, int undirected,
                      bg_edges** out);
int bg_read_matrix_market(const char* text, size_t len, const char* name, int undirected, bg_edges** out);
int bg_load_graph(const char* path, int64_t forced_nodes, int undirected, bg_edges** out);
int bg_edges_info(const bg_edges* e, int64_t* node_count, int64_t* n_edges, const int64_t** src,
                  const int64_t** dst, const double** weights, int64_t* n_weights);
void bg_edges_destroy(bg_edges* e);
/* Fault hook (ref: runreport.cpp:55-63): flip bit 0 of stored tile k % nnz. */
int bg_frdc_corrupt_tile(bg_frdc* m, int64_t k);
void bg_frdc_destroy(bg_frdc* m);

/* ---- graph bundle (ref: GraphBundle, prepare_graph, graphops.hpp:17-40) --- */
typedef struct bg_graph bg_graph;
typedef struct bg_graph_info {
  int64_t n;
  const bg_frdc* structure;      /* A + I */
  const bg_frdc* raw;            /* A, explicit self edges stripped */
  const float* norm;             /* device: float(1/sqrt(double deg(A+I))) */
  const float* mean_row;         /* device: 1.0f / float(max(1, neighbor_count)) */
  const float* ones;             /* device: 1.0f */
  const int64_t* neighbor_count; /* device */
} bg_graph_info;

/* ref: prepare_graph (graphops.cpp:146-170); src/dst DEVICE int64 arrays. */
int bg_prepare_graph(const int64_t* src, const int64_t* dst, int64_t n_edges, int64_t n_nodes,
                     bg_graph** out, bg_stream stream);
int bg_graph_info_get(const bg_graph* g, bg_graph_info* info);
/* Engine-side fault hook for verify (ref: runreport.cpp:55-63): corrupts A+I. */
int bg_graph_corrupt_tile(bg_graph* g, int64_t k);
void bg_graph_destroy(bg_graph* g);

/* ---- kernel families (ref: kernels.hpp:63-97) -------------------------- */
/* Output descriptors: fill precision/shape/word_bits of the result the op
 * would produce (data/scale left NULL) so callers can allocate it. */
int bg_bmm_out_desc(bg_variant v, const bg_mat* a, const bg_mat* w, int word_bits, bg_mat* out);
int bg_bspmm_out_desc(bg_variant v, const bg_frdc* adj, const bg_mat* x, int word_bits,
                      bg_mat* out);

/* ref: bmm (kernels.cpp:140-191).  out is caller-allocated per bg_bmm_out_desc. */
int bg_bmm(bg_variant v, const bg_mat* a, const bg_mat* w, int word_bits, bg_mat* out,
           bg_stream stream);
/* ref: bspmm (kernels.cpp:413-556).  row_scale/col_scale (device, len
 * node_rows/node_cols) factorize the adjacency; both NULL for in2 = B. */
int bg_bspmm(bg_variant v, const bg_frdc* adj, const float* row_scale, const float* col_scale,
             const bg_mat* x, int strategy, int word_bits, bg_mat* out, bg_stream stream);
/* ref: add (kernels.cpp:593-625) */
int bg_add(bg_variant v, const bg_mat* a, const bg_mat* b, bg_mat* out, bg_stream stream);
/* ref: concat (kernels.cpp:627-668) */
int bg_concat(bg_variant v, const bg_mat* a, const bg_mat* b, bg_mat* out, bg_stream stream);
/* ref: scl (kernels.cpp:560-571) */
int bg_scl(const float* x, int64_t rows, int64_t cols, const float* row, const float* col,
           float* out, bg_stream stream);
/* ref: dense_mm (kernels.cpp:193-212), double accumulation in k order */
int bg_dense_mm(const float* a, const float* w, int64_t rows, int64_t k, int64_t cols, float* out,
                bg_stream stream);
/* ref: relu_inplace (graphops.cpp:89-97); binary operands are left untouched */
int bg_relu_inplace(bg_mat* x, bg_stream stream);
/* ref: softmax_rows (graphops.cpp:372-386) */
int bg_softmax_rows(const float* x, int64_t rows, int64_t cols, float* out, bg_stream stream);
/* ref: batchnorm_infer (graphops.cpp:337-355); parameters are device arrays of len cols */
int bg_batchnorm_infer(const float* x, int64_t rows, int64_t cols, const float* gamma,
                       const float* beta, const float* mean, const float* sigma, float* out,
                       bg_stream stream);
/* ref: fused_mm_spmm (kernels.cpp:670-677): adj * (x * w), requires mm.out == spmm.in1 */
int bg_fused_mm_spmm(bg_variant mm, bg_variant spmm, const bg_mat* x, const bg_mat* w,
                     const bg_frdc* adj, const float* row_scale, const float* col_scale,
                     int strategy, bg_mat* out, bg_stream stream);

/* ---- models (ref: LayerSpec / ModelSpec / run_model, graphops.hpp:57-133) --- */
typedef struct bg_layer_desc {
  int32_t kind; /* BG_LAYER_* */
  int32_t n_plan;
  bg_variant plan[4];
  const float* w1; /* HOST fp32, row-major */
  int64_t w1_rows, w1_cols;
  const float* w2;
  int64_t w2_rows, w2_cols;
  int32_t relu;
  const float *bn_gamma, *bn_beta, *bn_mean, *bn_sigma; /* HOST, optional (BatchNorm) */
  int64_t bn_len;
  const float* scale_row; /* HOST, optional (Scale) */
  int64_t scale_row_len;
  const float* scale_col;
  int64_t scale_col_len;
} bg_layer_desc;

typedef struct bg_model bg_model;
typedef struct bg_trace bg_trace; /* BIN-point trace, below */

/* Single layers (ref: gcn_layer / sage_layer / graphconv_layer,
 * graphops.hpp:94-105, graphops.cpp:270-335): x is a DEVICE operand, l the
 * layer's plan and HOST weights (l->kind is ignored: the function names the
 * kind), g the graph (A+I for gcn, loop-free A with mean / ones scales for
 * sage / graph conv).  BIN points are appended to `trace` (may be NULL) with
 * labels prefix + "mm.bin_in" ... as the reference's LayerHooks record them.
 * out is caller-allocated per bg_layer_out_desc.  Synchronous.  Errors are the
 * reference's (std::invalid_argument "gcn_conv: expected {mm, spmm} plan and
 * weights", kernel contract messages), not wrapped in "layer i". */
int bg_layer_out_desc(int kind, const bg_layer_desc* l, const bg_mat* x, int word_bits, bg_mat* out);
int bg_gcn_layer(const bg_mat* x, const bg_layer_desc* l, const bg_graph* g, int strategy,
                 bg_trace* trace, const char* prefix, int word_bits, bg_mat* out, bg_stream stream);
int bg_sage_layer(const bg_mat* x, const bg_layer_desc* l, const bg_graph* g, int strategy,
                  bg_trace* trace, const char* prefix, int word_bits, bg_mat* out, bg_stream stream);
int bg_graphconv_layer(const bg_mat* x, const bg_layer_desc* l, const bg_graph* g, int strategy,
                       bg_trace* trace, const char* prefix, int word_bits, bg_mat* out, bg_stream stream);

/* ref: validate_model (graphops.cpp:245-268).  Returns the number of
 * problems; the messages, '\n'-separated and worded like the reference's,
 * go to buf. */
int bg_validate_model(int has_graph, int input_precision, const bg_layer_desc* layers,
                      int n_layers, char* buf, size_t buf_len);

/* Builds a device-resident model; weights are uploaded and binarized once
 * with their column scales, as run_mm_slot does per call (graphops.cpp:47-77).
 * Invalid models fail with BG_INVALID_ARGUMENT and the run_model message. */
int bg_model_create(const bg_graph* graph, int input_precision, int strategy, int word_bits,
                    const bg_layer_desc* layers, int n_layers, bg_model** out, bg_stream stream);
void bg_model_destroy(bg_model* m);
/* Shape of the model output for an input with `rows` rows. */
int bg_model_output_cols(const bg_model* m, int64_t* cols);
/* Capture each forward as one CUDA graph after the first run (default on). */
int bg_model_set_graph_capture(bg_model* m, int enable);

/* ref: run_model (graphops.cpp:390-484).  x0 in device memory; out and
 * logits (softmax input; may be NULL) are device float[rows*out_cols]. */
int bg_model_forward(bg_model* m, const bg_mat* x0, float* out, float* logits, bg_stream stream);

/* End-to-end call with HOST buffers: H2D of x (pipelined with the first
 * layer), forward, D2H of out/logits (logits may be NULL).  Synchronous. */
int bg_model_forward_host(bg_model* m, const float* x_host, int64_t rows, int64_t cols,
                          float* out_host, float* logits_host, bg_stream stream);

/* BIN-point trace (ref: RunTrace, graphops.hpp:114-122) */
int bg_trace_create(bg_trace** out);
void bg_trace_destroy(bg_trace* t);
int bg_model_forward_traced(bg_model* m, const bg_mat* x0, float* out, float* logits,
                            bg_trace* trace, bg_stream stream);
int bg_trace_size(const bg_trace* t);
/* bits: device pointer owned by the trace, rows x storage_words_per_row(cols) */
int bg_trace_point(const bg_trace* t, int i, const char** label, int64_t* rows, int64_t* cols,
                   int* word_bits, const uint32_t** bits);

/* ---- verification (ref: verify_model / VerifyReport, runreport.hpp:13-31,
 * runreport.cpp:51-135) -----------------------------------------------------
 * The engine's BIN points and logits against a reference run supplied by the
 * caller (the dense oracle, the reference engine, a recorded trace), compared
 * on the device: bit mismatches over the valid columns with the first one
 * (label, row, col) in trace order, max |e - o| / max(1, |o|), and argmax
 * agreement with the reference's exact-tie rule; pass = no mismatch, full
 * agreement, max_rel <= tolerance.  compare_bits = 0 is the reference's
 * full-precision mode (no BIN points compared).  A trace of another length or
 * a misaligned point is BG_LOGIC_ERROR with the reference's message. */
typedef struct bg_verify_report {
  double max_rel_logit_error;
  int64_t bin_points, bin_values, bin_mismatches;
  char first_mismatch_label[64];
  int64_t first_mismatch_row, first_mismatch_col; /* -1 when no mismatch */
  double argmax_agreement;
  double tolerance;
  int32_t pass;
} bg_verify_report;
typedef struct bg_ref_point { /* one reference BIN point, HOST packed bits */
  const char* label;
  int64_t rows, cols;
  int32_t word_bits;
  const uint32_t* bits; /* rows x bg_storage_words_per_row(cols, word_bits) */
} bg_ref_point;
/* A recorded engine trace + DEVICE logits (rows x cols) vs the reference
 * (ref_logits: HOST double rows x cols). */
int bg_verify_trace(const bg_trace* engine, const float* engine_logits, int64_t rows, int64_t cols,
                    const bg_ref_point* ref, int n_ref, const double* ref_logits, int compare_bits,
                    double tolerance, bg_verify_report* out, bg_stream stream);
/* Traced forward of `m` on x0 (device), then bg_verify_trace against the
 * reference (ref_logits HOST double ref_rows x ref_cols). */
int bg_model_verify(bg_model* m, const bg_mat* x0, const bg_ref_point* ref, int n_ref, const double* ref_logits,
                    int64_t ref_rows, int64_t ref_cols, int compare_bits, double tolerance,
                    bg_verify_report* out, bg_stream stream);

/* Per-kernel timing (ref: KernelTiming + record_ns hooks, graphops.cpp:53-84),
 * measured with CUDA events on `stream`. */
typedef struct bg_kernel_timing {
  char label[64];
  double ms;
} bg_kernel_timing;
int bg_model_forward_timed(bg_model* m, const bg_mat* x0, float* out, float* logits,
                           bg_kernel_timing* timings, int cap, int* n, bg_stream stream);

/* ---- row-sharded multi-GPU forward (one process per GPU) ---------------- */
/* New capability (the reference is single-process): node rows
 * are split into contiguous tile-row ranges with about equal FRDC tiles; each
 * rank computes its rows of every layer and the operand of every neighbour
 * aggregation is all-gathered over NVLink with NCCL. */

/* HOST: bounds[0..world] (multiples of 4, bounds[world] = n) from an FRDC
 * row_ptr (tile_rows + 1 entries). */
int bg_partition_bounds(const uint64_t* row_ptr, int64_t tile_rows, int64_t n, int world_size,
                        int64_t* bounds);
/* Row range [row_begin, row_end) of rank `rank` for the graph's A+I structure. */
int bg_partition_rows(const bg_graph* g, int world_size, int rank, int64_t* row_begin,
                      int64_t* row_end);

typedef struct bg_comm bg_comm; /* NCCL communicator, one rank per GPU */
/* Rank 0 creates the id and ships its bytes to every rank (e.g. through
 * torch.distributed); every rank then calls bg_comm_create on its device. */
int bg_comm_unique_id(uint8_t* id, size_t id_len);
int bg_comm_create(int world_size, int rank, const uint8_t* id, size_t id_len, bg_comm** out);
void bg_comm_destroy(bg_comm* c);
/* An exchange through the caller's transport instead of NCCL (tests, hosts
 * without NVLink peers): before each neighbour aggregation the engine
 * synchronizes `stream` and calls fn(ctx, buf, row_bytes, bounds, world, rank,
 * stream) on the host.  buf is a DEVICE buffer of bounds[world] rows of
 * row_bytes, rows [bounds[rank], bounds[rank+1]) produced by this rank; fn
 * must fill every other rank's rows and return 0 (nonzero fails the forward
 * with BG_RUNTIME_ERROR).  A forward using it is never graph-captured. */
typedef int (*bg_allgather_fn)(void* ctx, void* buf, int64_t row_bytes, const int64_t* bounds, int world_size,
                               int rank, bg_stream stream);
int bg_comm_create_external(int world_size, int rank, bg_allgather_fn fn, void* ctx, bg_comm** out);

/* A rank's share of a prepared graph: both adjacency structures cut to node
 * rows [row_begin, row_end) (whole tile rows: multiples of 4, or the node
 * count), the per-node scale vectors kept whole.  The source graph may be
 * destroyed afterwards, so a rank holds FRDC/world of the adjacency.  A model
 * on a shard runs bg_model_forward_sharded for that rank's range only. */
int bg_graph_shard(const bg_graph* g, int64_t row_begin, int64_t row_end, bg_graph** out, bg_stream stream);

/* Sharded ref: run_model.  With a communicator, x/out/logits hold this
 * rank's rows [bounds[rank], bounds[rank+1]) only.  With comm == NULL every
 * rank's range is computed in this process on this device ("virtual ranks",
 * x/out/logits full size) -- the same per-range kernels, no exchange.  With
 * an NCCL communicator on a non-default stream the forward is captured as
 * one CUDA graph from its second call with the same binding. */
int bg_model_forward_sharded(bg_model* m, bg_comm* comm, const bg_mat* x, const int64_t* bounds,
                             int world_size, int rank, float* out, float* logits,
                             bg_stream stream);
/* The same forward with per-op CUDA-event times (labels as bg_model_forward_timed,
 * plus "layerI.allgather" for each exchange); synchronizes the stream. */
int bg_model_forward_sharded_timed(bg_model* m, bg_comm* comm, const bg_mat* x, const int64_t* bounds,
                                   int world_size, int rank, float* out, bg_kernel_timing* timings, int cap,
                                   int* n, bg_stream stream);

/* ---- deterministic synthetic inputs (ref: rng.hpp:16-80) --------------- */
typedef struct bg_rng bg_rng;
int bg_rng_create(uint64_t seed, bg_rng** out);
void bg_rng_destroy(bg_rng* r);
/* float(uniform*2-1) draws, row-major, into a HOST buffer (ref: random_dense) */
int bg_rng_dense(bg_rng* r, int64_t rows, int64_t cols, float* out_host);
/* ref: random_edges; HOST outputs of capacity m; *count = edges written */
int bg_rng_edges(bg_rng* r, int64_t nodes, int64_t m, int allow_self, int64_t* src_host,
                 int64_t* dst_host, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* BITGNN_B200_H */
