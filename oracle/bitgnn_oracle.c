/*
 * bitgnn_oracle.c -- TEST INFRASTRUCTURE ONLY (see bitgnn_oracle.h).
 *
 * Scalar, single-threaded restatement of the reference hot path.  Reference
 * citations are into /root/reference/proj (abbreviated "ref:").  Compiled with
 * -ffp-contract=off so double arithmetic follows the reference's evaluation
 * order operation by operation.
 */
#include "bitgnn_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];

const char* og_error(void) { return g_err; }

static int fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return 1;
}

void og_free(void* p) { free(p); }

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz ? sz : 1);
  if (!p) {
    fprintf(stderr, "oracle: out of memory (%zu x %zu)\n", n, sz);
    abort();
  }
  return p;
}

/* ======================================================================== */
/* rng.hpp:16-80 -- std::mt19937_64 (pinned by the C++ standard) and the     */
/* reference's distribution-free mappings.                                   */
/* ======================================================================== */

#define MT_N 312
#define MT_M 156

void og_rng_seed(og_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
}

static void mt_twist(og_rng* r) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
    uint64_t xa = x >> 1;
    if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->idx = 0;
}

uint64_t og_rng_next(og_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* ref: rng.hpp:24 */
double og_rng_uniform(og_rng* r) { return (double)(og_rng_next(r) >> 11) * 0x1.0p-53; }

/* ref: rng.hpp:30-38 (rejection sampling, no distribution classes) */
int64_t og_rng_index(og_rng* r, int64_t n) {
  uint64_t un = (uint64_t)n;
  uint64_t limit = UINT64_MAX - UINT64_MAX % un;
  uint64_t v;
  do {
    v = og_rng_next(r);
  } while (v >= limit);
  return (int64_t)(v % un);
}

/* ref: rng.hpp:46-53 -- float(uniform*2-1), row-major draw order */
void og_random_dense(og_rng* r, int64_t rows, int64_t cols, float* out) {
  for (int64_t i = 0; i < rows * cols; ++i) out[i] = (float)(og_rng_uniform(r) * 2.0 - 1.0);
}

/* ref: rng.hpp:66-80 -- self draws nudged to d+1, dropped if still self */
int64_t og_random_edges(og_rng* r, int64_t nodes, int64_t m, int allow_self, int64_t* src,
                        int64_t* dst) {
  int64_t k = 0;
  for (int64_t t = 0; t < m; ++t) {
    int64_t s = og_rng_index(r, nodes);
    int64_t d = og_rng_index(r, nodes);
    if (!allow_self && s == d) {
      d = (d + 1) % nodes;
      if (s == d) continue;
    }
    src[k] = s;
    dst[k] = d;
    ++k;
  }
  return k;
}

/* ======================================================================== */
/* bitdense.cpp                                                              */
/* ======================================================================== */

/* ref: bitdense.hpp:72-73 -- ceil(cols/wb) words of wb bits, in u32 units */
int64_t og_spw(int64_t cols, int word_bits) {
  return (cols + word_bits - 1) / word_bits * (word_bits / 32);
}

/* ref: bitdense.cpp:71-88 -- bit = (x >= 0), column j at bit 31 - j%32 */
void og_binarize(const float* x, int64_t rows, int64_t cols, int word_bits, uint32_t* out) {
  const int64_t spw = og_spw(cols, word_bits);
  for (int64_t i = 0; i < rows; ++i) {
    const float* src = x + i * cols;
    for (int64_t w = 0; w < spw; ++w) {
      uint32_t v = 0;
      int64_t j0 = 32 * w;
      int64_t bmax = cols - j0 < 32 ? cols - j0 : 32;
      for (int64_t b = 0; b < bmax; ++b)
        if (src[j0 + b] >= 0) v |= 1u << (31 - b);
      out[i * spw + w] = v;
    }
  }
}

/* ref: bitdense.cpp:90-104 -- mean |x| accumulated in double in index order,
 * floored at 1e-12, stored as float */
void og_l1_scales(const float* x, int64_t rows, int64_t cols, int axis, float* out) {
  const int64_t len = axis == OG_ROW ? rows : cols;
  const int64_t span = axis == OG_ROW ? cols : rows;
  for (int64_t k = 0; k < len; ++k) {
    double acc = 0;
    for (int64_t t = 0; t < span; ++t)
      acc += fabs((double)(axis == OG_ROW ? x[k * cols + t] : x[t * cols + k]));
    double mean = span > 0 ? acc / (double)span : 0.0;
    out[k] = (float)(mean > 1e-12 ? mean : 1e-12);
  }
}

/* ref: bitdense.cpp:178-210 -- result is the bit transpose (a straight
 * bit-by-bit definition; the reference's 32x32 block walk computes the same
 * matrix, pinned by test_bitdense.cpp:172-199). */
void og_transpose_bits(const uint32_t* in, int64_t rows, int64_t cols, int word_bits,
                       uint32_t* out) {
  const int64_t spw_in = og_spw(cols, word_bits);
  const int64_t spw_out = og_spw(rows, word_bits);
  memset(out, 0, (size_t)(cols * spw_out) * 4);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j)
      if ((in[i * spw_in + j / 32] >> (31 - (j & 31))) & 1u)
        out[j * spw_out + i / 32] |= 1u << (31 - (i & 31));
}

/* ======================================================================== */
/* bitsparse.cpp                                                             */
/* ======================================================================== */

/* LSD radix sort of u64 keys over the low `bits` bits; equivalent to the
 * reference's std::sort (bitsparse.cpp:94) for the resulting order. */
static void radix_sort_u64(uint64_t* a, int64_t n, int bits) {
  if (n < 2) return;
  uint64_t* buf = (uint64_t*)xcalloc((size_t)n, 8);
  uint64_t *src = a, *dst = buf;
  const int D = 11;
  for (int shift = 0; shift < bits; shift += D) {
    int64_t cnt[1 << 11];
    memset(cnt, 0, sizeof cnt);
    for (int64_t i = 0; i < n; ++i) cnt[(src[i] >> shift) & ((1 << D) - 1)]++;
    int64_t sum = 0;
    for (int d = 0; d < (1 << D); ++d) {
      int64_t c = cnt[d];
      cnt[d] = sum;
      sum += c;
    }
    for (int64_t i = 0; i < n; ++i) dst[cnt[(src[i] >> shift) & ((1 << D) - 1)]++] = src[i];
    uint64_t* t = src;
    src = dst;
    dst = t;
  }
  if (src != a) memcpy(a, src, (size_t)n * 8);
  free(buf);
}

/* ref: bitsparse.cpp:72-112 -- key = (tile_row*tile_cols + tile_col) << 4 |
 * local bit, sorted, runs OR-ed into the u16 payload at bit 15 - local,
 * row_ptr max-scanned. */
int og_frdc_from_edges(int64_t n, const int64_t* src, const int64_t* dst, int64_t e,
                       int self_loops, og_frdc* out, int64_t* bad) {
  const int64_t tcols = (n + 3) / 4;
  const int64_t trows = tcols;
  int64_t total = e + (self_loops ? n : 0);
  uint64_t* keys = (uint64_t*)xcalloc((size_t)total, 8);
  int64_t k = 0;
  for (int64_t t = 0; t < e; ++t) {
    int64_t s = src[t], d = dst[t];
    if (s < 0 || s >= n || d < 0 || d >= n) {
      if (bad) *bad = t;
      free(keys);
      return -1;
    }
    uint64_t key = (uint64_t)(s / 4) * (uint64_t)tcols + (uint64_t)(d / 4);
    keys[k++] = (key << 4) | (uint64_t)(4 * (s & 3) + (d & 3));
  }
  if (self_loops)
    for (int64_t i = 0; i < n; ++i) {
      uint64_t key = (uint64_t)(i / 4) * (uint64_t)tcols + (uint64_t)(i / 4);
      keys[k++] = (key << 4) | (uint64_t)(4 * (i & 3) + (i & 3));
    }
  uint64_t maxkey = trows > 0 ? (((uint64_t)trows * (uint64_t)tcols) << 4) : 1;
  int bits = 1;
  while (bits < 64 && (maxkey >> bits)) ++bits;
  radix_sort_u64(keys, total, bits);

  out->rows = n;
  out->cols = n;
  out->row_ptr = (uint64_t*)xcalloc((size_t)trows + 1, 8);
  out->col_ind = (uint32_t*)xcalloc((size_t)total, 4);
  out->tiles = (uint16_t*)xcalloc((size_t)total, 2);
  int64_t nt = 0;
  int64_t p = 0;
  while (p < total) {
    uint64_t key = keys[p] >> 4;
    uint16_t payload = 0;
    for (; p < total && (keys[p] >> 4) == key; ++p)
      payload |= (uint16_t)(1u << (15 - (keys[p] & 15)));
    out->col_ind[nt] = (uint32_t)(key % (uint64_t)tcols);
    out->tiles[nt] = payload;
    ++nt;
    out->row_ptr[key / (uint64_t)tcols + 1] = (uint64_t)nt;
  }
  for (int64_t r = 1; r <= trows; ++r)
    if (out->row_ptr[r] < out->row_ptr[r - 1]) out->row_ptr[r] = out->row_ptr[r - 1];
  out->nnz = nt;
  free(keys);
  return 0;
}

void og_frdc_free(og_frdc* m) {
  free(m->row_ptr);
  free(m->col_ind);
  free(m->tiles);
  memset(m, 0, sizeof *m);
}

/* ref: tileset_count, bitsparse.cpp:129-134 */
int64_t og_tileset_count(const og_frdc* m, int64_t tile_row, int word_bits) {
  const int64_t ts = word_bits / 4;
  const int64_t nt = (int64_t)(m->row_ptr[tile_row + 1] - m->row_ptr[tile_row]);
  return (nt + ts - 1) / ts;
}

/* ref: gather_tileset, bitsparse.cpp:136-160 (checks and messages in order) */
int og_gather_tileset(const og_frdc* m, int64_t tile_row, int64_t set_index, int word_bits,
                      og_tileset* out) {
  if (word_bits != 32 && word_bits != 64) return fail("gather_tileset: word_bits must be 32 or 64");
  if (tile_row < 0 || tile_row >= (m->rows + 3) / 4) return fail("gather_tileset: tile_row out of range");
  memset(out, 0, sizeof *out);
  out->ts = word_bits / 4;
  if (set_index < 0 || set_index >= og_tileset_count(m, tile_row, word_bits))
    return fail("gather_tileset: set_index out of range");
  for (int s = 0; s < 16; ++s) out->cols[s] = 0xFFFFFFFFu;
  const uint64_t begin = m->row_ptr[tile_row] + (uint64_t)set_index * (uint64_t)out->ts;
  const uint64_t end = m->row_ptr[tile_row + 1];
  for (int s = 0; s < out->ts; ++s) {
    const uint64_t k = begin + (uint64_t)s;
    if (k >= end) break;
    out->cols[s] = m->col_ind[k];
    const uint16_t t = m->tiles[k];
    const int shift = word_bits - 4 - 4 * s;
    for (int n = 0; n < 4; ++n) out->rows[n] |= (uint64_t)((t >> (12 - 4 * n)) & 0xF) << shift;
  }
  return 0;
}

/* ref: frdc_to_dense, bitsparse.cpp:114-127 (MSB-first bits, u32 storage) */
void og_frdc_to_dense(const og_frdc* m, int word_bits, uint32_t* out) {
  const int64_t w = og_spw(m->cols, word_bits), trows = (m->rows + 3) / 4;
  memset(out, 0, (size_t)(m->rows * w) * 4);
  for (int64_t r = 0; r < trows; ++r)
    for (uint64_t k = m->row_ptr[r]; k < m->row_ptr[r + 1]; ++k)
      for (int rl = 0; rl < 4; ++rl)
        for (int cl = 0; cl < 4; ++cl)
          if ((m->tiles[k] >> (15 - (4 * rl + cl))) & 1) {
            const int64_t i = 4 * r + rl, j = 4 * (int64_t)m->col_ind[k] + cl;
            out[i * w + j / 32] |= 1u << (31 - (j & 31));
          }
}

/* ref: graphops.cpp:18-33 */
void og_row_popcounts(const og_frdc* a, int64_t* deg) {
  const int64_t trows = (a->rows + 3) / 4;
  memset(deg, 0, (size_t)a->rows * 8);
  for (int64_t tr = 0; tr < trows; ++tr)
    for (uint64_t k = a->row_ptr[tr]; k < a->row_ptr[tr + 1]; ++k) {
      uint16_t t = a->tiles[k];
      for (int r = 0; r < 4; ++r) {
        int64_t row = tr * 4 + r;
        if (row >= a->rows) break;
        deg[row] += __builtin_popcount((t >> (12 - 4 * r)) & 0xF);
      }
    }
}

int64_t og_frdc_nnz_bits(const og_frdc* a) {
  int64_t s = 0;
  for (int64_t k = 0; k < a->nnz; ++k) s += __builtin_popcount(a->tiles[k]);
  return s;
}

/* ======================================================================== */
/* kernels.cpp                                                               */
/* ======================================================================== */

void og_mat_free(og_mat* m) {
  free(m->f);
  free(m->bits);
  free(m->scale);
  memset(m, 0, sizeof *m);
}

static int bit_at(const uint32_t* bits, int64_t spw, int64_t i, int64_t j) {
  return (int)((bits[i * spw + j / 32] >> (31 - (j & 31))) & 1u);
}

/* ref: kernels.cpp:30-41 -- n - 2*popc(a ^ b) over whole storage rows */
static int32_t pm1_dot(const uint32_t* a, const uint32_t* b, int64_t spw, int64_t n) {
  int64_t diff = 0;
  for (int64_t k = 0; k < spw; ++k) diff += __builtin_popcount(a[k] ^ b[k]);
  return (int32_t)(n - 2 * diff);
}

/* One resolved bmm side: bits + optional scale (kernels.cpp:52-77). */
typedef struct side {
  const uint32_t* bits;
  const float* scale;
  int64_t rows, cols;
  int wb;
  uint32_t* own_bits;
  float* own_scale;
} side;

static int resolve_side(int tag, const og_mat* m, int axis, const char* which, side* s, int wb) {
  memset(s, 0, sizeof *s);
  if (tag == OG_F) {
    if (m->prec != OG_F) return fail("bmm: %s is tagged F but operand is binary", which);
    s->own_bits = (uint32_t*)xcalloc((size_t)(m->rows * og_spw(m->cols, wb)), 4);
    og_binarize(m->f, m->rows, m->cols, wb, s->own_bits);
    s->own_scale = (float*)xcalloc((size_t)(axis == OG_ROW ? m->rows : m->cols), 4);
    og_l1_scales(m->f, m->rows, m->cols, axis, s->own_scale);
    s->bits = s->own_bits;
    s->scale = s->own_scale;
    s->wb = wb;
  } else {
    if (m->prec != OG_B) return fail("bmm: %s is tagged B but operand is full-precision", which);
    s->bits = m->bits;
    s->scale = m->scale;
    s->wb = m->word_bits;
  }
  s->rows = m->rows;
  s->cols = m->cols;
  return 0;
}

/* ref: kernels.cpp:140-191 */
int og_bmm(og_variant v, const og_mat* a, const og_mat* w, int word_bits, og_mat* out) {
  memset(out, 0, sizeof *out);
  if (v.op != OG_BMM) return fail("bmm: not a BMM variant");
  if (v.in1 == OG_F && v.in2 == OG_F && v.out == OG_F) return fail("bmm: FFF is not supported");
  if (v.in1 == OG_B && a->prec == OG_B) word_bits = a->word_bits;
  if (v.in2 == OG_B && w->prec == OG_B) word_bits = w->word_bits;
  side sa, sw;
  if (resolve_side(v.in1, a, OG_ROW, "in1", &sa, word_bits)) return 1;
  if (resolve_side(v.in2, w, OG_COL, "in2", &sw, word_bits)) {
    free(sa.own_bits);
    free(sa.own_scale);
    return 1;
  }
  int rc = 0;
  if (sa.cols != sw.rows) {
    rc = fail("bmm: inner dimensions disagree");
    goto done;
  }
  if (sa.wb != sw.wb) {
    rc = fail("bmm: operand word widths disagree");
    goto done;
  }
  {
    const int64_t rows = sa.rows, cols = sw.cols, k = sa.cols;
    const int64_t spw = og_spw(k, sa.wb);
    uint32_t* wt = (uint32_t*)xcalloc((size_t)(cols * spw), 4);
    og_transpose_bits(sw.bits, sw.rows, sw.cols, sw.wb, wt);
    out->rows = rows;
    out->cols = cols;
    out->word_bits = sa.wb;
    if (v.out == OG_B) {
      /* SCL elimination (kernels.cpp:159-161): no scale on B outputs */
      const int64_t ospw = og_spw(cols, sa.wb);
      out->prec = OG_B;
      out->bits = (uint32_t*)xcalloc((size_t)(rows * ospw), 4);
      for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j)
          if (pm1_dot(sa.bits + i * spw, wt + j * spw, spw, k) >= 0)
            out->bits[i * ospw + j / 32] |= 1u << (31 - (j & 31));
    } else {
      out->prec = OG_F;
      out->f = (float*)xcalloc((size_t)(rows * cols), 4);
      for (int64_t i = 0; i < rows; ++i) {
        const double alpha = sa.scale ? (double)sa.scale[i] : 1.0;
        for (int64_t j = 0; j < cols; ++j) {
          const double beta = sw.scale ? (double)sw.scale[j] : 1.0;
          out->f[i * cols + j] =
              (float)(alpha * (double)pm1_dot(sa.bits + i * spw, wt + j * spw, spw, k) * beta);
        }
      }
    }
    free(wt);
  }
done:
  free(sa.own_bits);
  free(sa.own_scale);
  free(sw.own_bits);
  free(sw.own_scale);
  return rc;
}

/* Ascending-column neighbour walk of one node row (kernels.cpp:218-234:
 * tile sets in order, slots ascending, local columns ascending). */
typedef void (*visit_fn)(void* ctx, int64_t j);
static void walk_row(const og_frdc* a, int64_t i, visit_fn f, void* ctx) {
  const int64_t tr = i / 4;
  const int n = (int)(i & 3);
  for (uint64_t k = a->row_ptr[tr]; k < a->row_ptr[tr + 1]; ++k) {
    unsigned nib = (a->tiles[k] >> (12 - 4 * n)) & 0xF;
    for (int c = 0; c < 4; ++c)
      if (nib & (8u >> c)) f(ctx, 4 * (int64_t)a->col_ind[k] + c);
  }
}

typedef struct acc_ctx {
  const og_mat* x;
  const float* col_scale; /* NULL: weight 1 */
  double* d;
  int64_t deg, pos_count_unused;
  int64_t* cnt; /* BB path: +1 counts */
} acc_ctx;

static void visit_bb(void* c, int64_t j) {
  acc_ctx* a = (acc_ctx*)c;
  const int64_t spw = og_spw(a->x->cols, a->x->word_bits);
  for (int64_t k = 0; k < a->x->cols; ++k) a->cnt[k] += bit_at(a->x->bits, spw, j, k);
  a->deg++;
}

static void visit_bf(void* c, int64_t j) {
  acc_ctx* a = (acc_ctx*)c;
  const int64_t spw = og_spw(a->x->cols, a->x->word_bits);
  const double wj = (double)a->col_scale[j];
  for (int64_t k = 0; k < a->x->cols; ++k) a->d[k] += bit_at(a->x->bits, spw, j, k) ? wj : -wj;
}

static void visit_f(void* c, int64_t j) {
  acc_ctx* a = (acc_ctx*)c;
  const double wj = a->col_scale ? (double)a->col_scale[j] : 1.0;
  const float* xr = a->x->f + j * a->x->cols;
  for (int64_t k = 0; k < a->x->cols; ++k) a->d[k] += wj * (double)xr[k];
}

/* ref: kernels.cpp:413-556 */
int og_bspmm(og_variant v, const og_frdc* adj, const float* row_scale, const float* col_scale,
             const og_mat* x, int word_bits, og_mat* out) {
  memset(out, 0, sizeof *out);
  if (v.op != OG_BSPMM) return fail("bspmm: not a BSpMM variant");
  if (v.in2 == OG_F && (!row_scale || !col_scale))
    return fail("bspmm: needs a factorized adjacency (row and col scales)");
  if (v.in2 == OG_B && (row_scale || col_scale))
    return fail("bspmm: takes the raw structure, not a factorized adjacency");
  if (v.in1 == OG_B && x->prec != OG_B) return fail("bspmm: in1 tag B requires a binary operand");
  if (v.in1 == OG_F && x->prec != OG_F)
    return fail("bspmm: in1 tag F requires a full-precision operand");
  if (v.in1 == OG_B && x->scale) return fail("bspmm: unexpected scale on the activation operand");
  if (x->rows != adj->cols) return fail("bspmm: activation row count != adjacency node_cols");
  const int64_t rows = adj->rows, f = x->cols;
  const int owb = v.in1 == OG_B ? x->word_bits : word_bits;
  const int64_t ospw = og_spw(f, owb);
  out->rows = rows;
  out->cols = f;
  out->word_bits = owb;
  if (v.out == OG_B) {
    out->prec = OG_B;
    out->bits = (uint32_t*)xcalloc((size_t)(rows * ospw), 4);
  } else {
    out->prec = OG_F;
    out->f = (float*)xcalloc((size_t)(rows * f), 4);
  }
  double* d = (double*)xcalloc((size_t)f, 8);
  int64_t* cnt = (int64_t*)xcalloc((size_t)f, 8);
  for (int64_t i = 0; i < rows; ++i) {
    acc_ctx c = {x, col_scale, d, 0, 0, cnt};
    memset(d, 0, (size_t)f * 8);
    memset(cnt, 0, (size_t)f * 8);
    if (v.in1 == OG_B && v.in2 == OG_B) {
      /* integer path (kernels.cpp:254-333, emit :440-464): 2*cnt - deg */
      walk_row(adj, i, visit_bb, &c);
      for (int64_t k = 0; k < f; ++k) {
        int64_t s = 2 * cnt[k] - c.deg;
        if (v.out == OG_B) {
          if (s >= 0) out->bits[i * ospw + k / 32] |= 1u << (31 - (k & 31));
        } else {
          out->f[i * f + k] = (float)s;
        }
      }
      continue;
    }
    double si = 1.0;
    if (v.in1 == OG_B) {
      /* binary activations, factorized adjacency (kernels.cpp:467-510) */
      walk_row(adj, i, visit_bf, &c);
      si = (double)row_scale[i];
    } else {
      /* full-precision activations (kernels.cpp:512-555) */
      if (v.in2 == OG_B) c.col_scale = NULL;
      walk_row(adj, i, visit_f, &c);
      si = v.in2 == OG_F ? (double)row_scale[i] : 1.0;
    }
    for (int64_t k = 0; k < f; ++k) {
      if (v.out == OG_B) {
        if (si * d[k] >= 0) out->bits[i * ospw + k / 32] |= 1u << (31 - (k & 31));
      } else {
        out->f[i * f + k] = (float)(si * d[k]);
      }
    }
  }
  free(d);
  free(cnt);
  return 0;
}

/* ref: kernels.cpp:593-625 */
int og_add(og_variant v, const og_mat* a, const og_mat* b, og_mat* out) {
  memset(out, 0, sizeof *out);
  if (v.op != OG_ADD) return fail("add: not an ADD variant");
  if (a->rows != b->rows || a->cols != b->cols) return fail("add: operand shapes disagree");
  const int64_t rows = a->rows, cols = a->cols;
  out->rows = rows;
  out->cols = cols;
  if (v.in1 == OG_F) {
    out->prec = OG_F;
    out->f = (float*)xcalloc((size_t)(rows * cols), 4);
    for (int64_t t = 0; t < rows * cols; ++t) out->f[t] = (float)((double)a->f[t] + (double)b->f[t]);
    return 0;
  }
  if (a->word_bits != b->word_bits) return fail("add: operand word widths disagree");
  const int64_t spw = og_spw(cols, a->word_bits);
  if (v.out == OG_B) {
    out->prec = OG_B;
    out->word_bits = a->word_bits;
    out->bits = (uint32_t*)xcalloc((size_t)(rows * spw), 4);
    for (int64_t t = 0; t < rows * spw; ++t) out->bits[t] = a->bits[t] | b->bits[t];
    return 0;
  }
  out->prec = OG_F;
  out->f = (float*)xcalloc((size_t)(rows * cols), 4);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j)
      out->f[i * cols + j] =
          (float)(2 * (bit_at(a->bits, spw, i, j) + bit_at(b->bits, spw, i, j)) - 2);
  return 0;
}

/* ref: graphops.cpp:89-97 -- F only */
void og_relu(og_mat* x) {
  if (x->prec != OG_F) return;
  for (int64_t t = 0; t < x->rows * x->cols; ++t) x->f[t] = x->f[t] > 0 ? x->f[t] : 0.0f;
}

/* ref: graphops.cpp:372-386 */
void og_softmax_rows(const float* x, int64_t rows, int64_t cols, float* out) {
  for (int64_t i = 0; i < rows; ++i) {
    const float* xr = x + i * cols;
    double mx = -INFINITY;
    for (int64_t j = 0; j < cols; ++j) mx = (double)xr[j] > mx ? (double)xr[j] : mx;
    double sum = 0.0;
    for (int64_t j = 0; j < cols; ++j) sum += exp((double)xr[j] - mx);
    for (int64_t j = 0; j < cols; ++j) out[i * cols + j] = (float)(exp((double)xr[j] - mx) / sum);
  }
}

/* ======================================================================== */
/* graphops.cpp                                                              */
/* ======================================================================== */

/* ref: graphops.cpp:135-170 */
int og_prepare_graph(int64_t n, const int64_t* src, const int64_t* dst, int64_t e, og_graph* g) {
  memset(g, 0, sizeof *g);
  int64_t bad = -1;
  g->n = n;
  if (og_frdc_from_edges(n, src, dst, e, 1, &g->structure, &bad))
    return fail("frdc_from_edges: edge %lld out of range", (long long)bad);
  int64_t* deg = (int64_t*)xcalloc((size_t)n, 8);
  og_row_popcounts(&g->structure, deg);
  g->norm = (float*)xcalloc((size_t)n, 4);
  for (int64_t i = 0; i < n; ++i) g->norm[i] = (float)(1.0 / sqrt((double)deg[i]));
  int64_t* ls = (int64_t*)xcalloc((size_t)e, 8);
  int64_t* ld = (int64_t*)xcalloc((size_t)e, 8);
  int64_t m = 0;
  for (int64_t t = 0; t < e; ++t)
    if (src[t] != dst[t]) {
      ls[m] = src[t];
      ld[m] = dst[t];
      ++m;
    }
  og_frdc_from_edges(n, ls, ld, m, 0, &g->raw, &bad);
  free(ls);
  free(ld);
  g->neighbor_count = deg;
  og_row_popcounts(&g->raw, g->neighbor_count);
  g->mean_row = (float*)xcalloc((size_t)n, 4);
  g->ones = (float*)xcalloc((size_t)n, 4);
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = g->neighbor_count[i] > 1 ? g->neighbor_count[i] : 1;
    g->mean_row[i] = 1.0f / (float)c;
    g->ones[i] = 1.0f;
  }
  return 0;
}

void og_graph_free(og_graph* g) {
  og_frdc_free(&g->structure);
  og_frdc_free(&g->raw);
  free(g->norm);
  free(g->mean_row);
  free(g->ones);
  free(g->neighbor_count);
  memset(g, 0, sizeof *g);
}

static void emit_bits(og_trace_fn tr, void* ctx, const char* prefix, const char* suffix,
                      const uint32_t* bits, int64_t rows, int64_t cols, int wb) {
  if (!tr) return;
  char label[128];
  snprintf(label, sizeof label, "%s%s", prefix, suffix);
  tr(ctx, label, bits, rows, cols, wb);
}

/* ref: graphops.cpp:47-77 (run_mm_slot) */
static int mm_slot(og_variant mm, og_mat* x, const float* w, int64_t wr, int64_t wc,
                   const char* label, int wb, og_trace_fn tr, void* ctx, og_mat* out) {
  if (tr) {
    if (mm.in1 == OG_F && x->prec == OG_F) {
      uint32_t* b = (uint32_t*)xcalloc((size_t)(x->rows * og_spw(x->cols, wb)), 4);
      og_binarize(x->f, x->rows, x->cols, wb, b);
      emit_bits(tr, ctx, label, ".bin_in", b, x->rows, x->cols, wb);
      free(b);
    }
    uint32_t* b = (uint32_t*)xcalloc((size_t)(wr * og_spw(wc, wb)), 4);
    og_binarize(w, wr, wc, wb, b);
    emit_bits(tr, ctx, label, ".bin_w", b, wr, wc, wb);
    free(b);
  }
  og_mat wop;
  memset(&wop, 0, sizeof wop);
  wop.rows = wr;
  wop.cols = wc;
  if (mm.in2 == OG_B) {
    wop.prec = OG_B;
    wop.word_bits = wb;
    wop.bits = (uint32_t*)xcalloc((size_t)(wr * og_spw(wc, wb)), 4);
    og_binarize(w, wr, wc, wb, wop.bits);
    wop.scale = (float*)xcalloc((size_t)wc, 4);
    og_l1_scales(w, wr, wc, OG_COL, wop.scale);
  } else {
    wop.prec = OG_F;
    wop.f = (float*)w;
  }
  int rc = og_bmm(mm, x, &wop, wb, out);
  if (wop.prec == OG_B) og_mat_free(&wop);
  if (rc) return rc;
  if (mm.out == OG_B) emit_bits(tr, ctx, label, ".out", out->bits, out->rows, out->cols, out->word_bits);
  return 0;
}

static int spmm_slot(og_variant sp, const og_frdc* a, const float* rs, const float* cs,
                     og_mat* x, const char* label, int wb, og_trace_fn tr, void* ctx,
                     og_mat* out) {
  int rc = og_bspmm(sp, a, rs, cs, x, wb, out);
  if (rc) return rc;
  if (sp.out == OG_B) emit_bits(tr, ctx, label, ".out", out->bits, out->rows, out->cols, out->word_bits);
  return 0;
}

/* ref: graphops.cpp:390-484 (with gcn_layer :270-285, neighborhood_layer
 * :289-321, FC :434-438, softmax :451-460) */
int og_run_model(const og_layer* layers, int nlayers, int wb, const og_graph* g,
                 const float* x0, int64_t rows, int64_t cols, float** out, float** logits,
                 int64_t* out_cols, og_trace_fn tr, void* ctx) {
  og_mat cur;
  memset(&cur, 0, sizeof cur);
  cur.prec = OG_F;
  cur.rows = rows;
  cur.cols = cols;
  cur.f = (float*)xcalloc((size_t)(rows * cols), 4);
  memcpy(cur.f, x0, (size_t)(rows * cols) * 4);
  *logits = NULL;
  char prefix[64], label[96];
  for (int li = 0; li < nlayers; ++li) {
    const og_layer* l = &layers[li];
    snprintf(prefix, sizeof prefix, "layer%d.", li);
    og_mat nxt;
    memset(&nxt, 0, sizeof nxt);
    int rc = 0;
    if (l->kind == OG_GCN) {
      og_mat h;
      snprintf(label, sizeof label, "%smm", prefix);
      rc = mm_slot(l->plan[0], &cur, l->w1, l->w1_rows, l->w1_cols, label, wb, tr, ctx, &h);
      if (rc) goto err;
      snprintf(label, sizeof label, "%sspmm", prefix);
      const int fac = l->plan[1].in2 == OG_F;
      rc = spmm_slot(l->plan[1], &g->structure, fac ? g->norm : NULL, fac ? g->norm : NULL, &h,
                     label, wb, tr, ctx, &nxt);
      og_mat_free(&h);
      if (rc) goto err;
      if (l->relu) og_relu(&nxt);
    } else if (l->kind == OG_SAGE || l->kind == OG_GRAPHCONV) {
      const int mean = l->kind == OG_SAGE;
      og_mat hs, hn, agg;
      snprintf(label, sizeof label, "%smm_self", prefix);
      rc = mm_slot(l->plan[0], &cur, l->w1, l->w1_rows, l->w1_cols, label, wb, tr, ctx, &hs);
      if (rc) goto err;
      snprintf(label, sizeof label, "%smm_neigh", prefix);
      rc = mm_slot(l->plan[1], &cur, l->w2, l->w2_rows, l->w2_cols, label, wb, tr, ctx, &hn);
      if (rc) goto err;
      const og_variant sp = l->plan[2];
      const int fac = sp.in2 == OG_F;
      snprintf(label, sizeof label, "%sspmm", prefix);
      rc = spmm_slot(sp, &g->raw, fac ? (mean ? g->mean_row : g->ones) : NULL,
                     fac ? g->ones : NULL, &hn, label, wb, tr, ctx, &agg);
      og_mat_free(&hn);
      if (rc) goto err;
      if (mean && sp.in2 == OG_B && sp.out == OG_F) {
        /* ref: graphops.cpp:304-314 -- double multiply by 1/max(1,cnt) */
        for (int64_t i = 0; i < agg.rows; ++i) {
          int64_t c = g->neighbor_count[i] > 1 ? g->neighbor_count[i] : 1;
          double inv = 1.0 / (double)c;
          for (int64_t j = 0; j < agg.cols; ++j)
            agg.f[i * agg.cols + j] = (float)((double)agg.f[i * agg.cols + j] * inv);
        }
      }
      rc = og_add(l->plan[3], &hs, &agg, &nxt);
      og_mat_free(&hs);
      og_mat_free(&agg);
      if (rc) goto err;
      if (l->plan[3].out == OG_B)
        emit_bits(tr, ctx, prefix, "add.out", nxt.bits, nxt.rows, nxt.cols, nxt.word_bits);
      if (l->relu) og_relu(&nxt);
    } else if (l->kind == OG_FC) {
      snprintf(label, sizeof label, "%smm", prefix);
      rc = mm_slot(l->plan[0], &cur, l->w1, l->w1_rows, l->w1_cols, label, wb, tr, ctx, &nxt);
      if (rc) goto err;
      if (l->relu) og_relu(&nxt);
    } else if (l->kind == OG_SOFTMAX) {
      *logits = (float*)xcalloc((size_t)(cur.rows * cur.cols), 4);
      memcpy(*logits, cur.f, (size_t)(cur.rows * cur.cols) * 4);
      nxt.prec = OG_F;
      nxt.rows = cur.rows;
      nxt.cols = cur.cols;
      nxt.f = (float*)xcalloc((size_t)(cur.rows * cur.cols), 4);
      og_softmax_rows(cur.f, cur.rows, cur.cols, nxt.f);
    } else {
      rc = fail("layer %d: unsupported kind %d", li, l->kind);
      goto err;
    }
    og_mat_free(&cur);
    cur = nxt;
    continue;
  err:
    og_mat_free(&cur);
    return rc;
  }
  if (cur.prec != OG_F) {
    og_mat_free(&cur);
    return fail("model output must be full precision");
  }
  if (!*logits) {
    *logits = (float*)xcalloc((size_t)(cur.rows * cur.cols), 4);
    memcpy(*logits, cur.f, (size_t)(cur.rows * cur.cols) * 4);
  }
  *out = cur.f;
  *out_cols = cur.cols;
  cur.f = NULL;
  og_mat_free(&cur);
  return 0;
}
