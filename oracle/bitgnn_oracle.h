/*
 * bitgnn_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the BitGNN CPU reference (/root/reference/proj) for
 * the binary-GNN inference hot path.  It exists so the CUDA product can be
 * checked against the reference algorithm on the GPU box, where
 * /root/reference is absent.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it; the product never does.
 *
 * Parity of this restatement is pinned two ways:
 *   - the reference's own known-answer tests (proj/tests/test_*.cpp) restated in
 *     tests/test_oracle_golden.py;
 *   - fixtures produced by the real reference compiled from
 *     /root/reference/proj/src (oracle/_ref, tests/golden/make_golden.py).
 *
 * Every function cites the reference file:line it follows.  Layout
 * conventions are the reference's: row-major, MSB-first u32 bit words, a
 * 64-bit logical word is a big-endian pair of u32 (bitdense.hpp:55-60).
 */
#ifndef BITGNN_ORACLE_H
#define BITGNN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OG_F = 0, OG_B = 1 };
enum { OG_BMM = 0, OG_BSPMM = 1, OG_ADD = 2, OG_CONCAT = 3 };
enum { OG_ROW = 0, OG_COL = 1 };

/* ---- rng.hpp:16-80 ------------------------------------------------------ */
typedef struct og_rng {
  uint64_t mt[312];
  int idx;
} og_rng;

void og_rng_seed(og_rng* r, uint64_t seed);
uint64_t og_rng_next(og_rng* r);
double og_rng_uniform(og_rng* r);
int64_t og_rng_index(og_rng* r, int64_t n);
void og_random_dense(og_rng* r, int64_t rows, int64_t cols, float* out);
/* Returns the number of edges written (<= m). */
int64_t og_random_edges(og_rng* r, int64_t nodes, int64_t m, int allow_self, int64_t* src,
                        int64_t* dst);

/* ---- bitdense.cpp ------------------------------------------------------- */
int64_t og_spw(int64_t cols, int word_bits);
void og_binarize(const float* x, int64_t rows, int64_t cols, int word_bits, uint32_t* out);
void og_l1_scales(const float* x, int64_t rows, int64_t cols, int axis, float* out);
void og_transpose_bits(const uint32_t* in, int64_t rows, int64_t cols, int word_bits,
                       uint32_t* out);

/* ---- bitsparse.cpp ------------------------------------------------------ */
typedef struct og_frdc {
  int64_t rows, cols, nnz;
  uint64_t* row_ptr; /* tile_rows + 1 */
  uint32_t* col_ind; /* nnz */
  uint16_t* tiles;   /* nnz */
} og_frdc;

/* 0 on success; -1 when an endpoint is out of range (*bad = edge index). */
int og_frdc_from_edges(int64_t n, const int64_t* src, const int64_t* dst, int64_t e,
                       int self_loops, og_frdc* out, int64_t* bad);
void og_frdc_free(og_frdc* m);
void og_row_popcounts(const og_frdc* m, int64_t* deg);
int64_t og_frdc_nnz_bits(const og_frdc* m);

/* Tile sets (ref: TileSet, bitsparse.hpp:62-71): same layout as bg_tileset. */
typedef struct og_tileset {
  int32_t ts, reserved;
  uint64_t rows[4];
  uint32_t cols[16];
} og_tileset;
/* ref: tileset_count (bitsparse.cpp:129-134) */
int64_t og_tileset_count(const og_frdc* m, int64_t tile_row, int word_bits);
/* ref: gather_tileset (bitsparse.cpp:136-160); 0, or nonzero with og_error() */
int og_gather_tileset(const og_frdc* m, int64_t tile_row, int64_t set_index, int word_bits,
                      og_tileset* out);
/* ref: frdc_to_dense (bitsparse.cpp:114-127): ZeroOne rows x og_spw(cols) words */
void og_frdc_to_dense(const og_frdc* m, int word_bits, uint32_t* out);

/* ---- kernels.cpp -------------------------------------------------------- */
typedef struct og_variant {
  int op, in1, in2, out;
} og_variant;

/* A matrix operand: full precision (f) or packed +-1 bits (bits) with an
 * optional reconstruction scale (NULL when absent). */
typedef struct og_mat {
  int prec;
  int64_t rows, cols;
  int word_bits;
  float* f;
  uint32_t* bits;
  float* scale;
} og_mat;

/* Output operands are allocated by the oracle; release with og_mat_free. */
void og_mat_free(og_mat* m);

/* 0 on success, nonzero on a contract violation (message in og_error()). */
int og_bmm(og_variant v, const og_mat* a, const og_mat* w, int word_bits, og_mat* out);
int og_bspmm(og_variant v, const og_frdc* adj, const float* row_scale, const float* col_scale,
             const og_mat* x, int word_bits, og_mat* out);
int og_add(og_variant v, const og_mat* a, const og_mat* b, og_mat* out);
void og_relu(og_mat* x);
void og_softmax_rows(const float* x, int64_t rows, int64_t cols, float* out);
const char* og_error(void);

/* ---- graphops.cpp ------------------------------------------------------- */
typedef struct og_graph {
  int64_t n;
  og_frdc structure; /* A + I */
  og_frdc raw;       /* A, explicit self edges stripped */
  float* norm;       /* (deg of A+I)^-1/2 */
  float* mean_row;   /* 1 / max(1, neighbour count) */
  float* ones;
  int64_t* neighbor_count;
} og_graph;

int og_prepare_graph(int64_t n, const int64_t* src, const int64_t* dst, int64_t e, og_graph* g);
void og_graph_free(og_graph* g);

enum { OG_GCN = 0, OG_SAGE = 1, OG_GRAPHCONV = 2, OG_FC = 3, OG_SOFTMAX = 7 };

typedef struct og_layer {
  int kind;
  int nplan;
  og_variant plan[4];
  const float* w1;
  int64_t w1_rows, w1_cols;
  const float* w2;
  int64_t w2_rows, w2_cols;
  int relu;
} og_layer;

/* Trace sink: called for every binarization point, in reference order. */
typedef void (*og_trace_fn)(void* ctx, const char* label, const uint32_t* bits, int64_t rows,
                            int64_t cols, int word_bits);

/* Runs the layer chain (graphops.cpp:390-484).  logits receives the softmax
 * input (or the model output when there is no softmax); out receives the
 * final output.  Shapes: out/logits rows x out_cols (returned in *out_cols). */
int og_run_model(const og_layer* layers, int nlayers, int word_bits, const og_graph* g,
                 const float* x0, int64_t rows, int64_t cols, float** out, float** logits,
                 int64_t* out_cols, og_trace_fn trace, void* ctx);
void og_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
