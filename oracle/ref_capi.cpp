// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library, compiled
// straight from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libbitgnn_ref.so.  It lets the Python tests and bench.py's
// reference arm drive the real reference (bitgnn::prepare_graph,
// bitgnn::build_model, bitgnn::run_model, bitgnn::bench_model) without
// linking it into the product.  No reference source is copied here; only the
// reference's public headers are included.
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "bitgnn/bitsparse.hpp"
#include "bitgnn/graphio.hpp"
#include "bitgnn/graphops.hpp"
#include "bitgnn/kernelbench.hpp"
#include "bitgnn/kernels.hpp"
#include "bitgnn/modelconfig.hpp"
#include "bitgnn/oracle.hpp"
#include "bitgnn/rng.hpp"
#include "bitgnn/runreport.hpp"
#include "bitgnn/tune.hpp"

using namespace bitgnn;

namespace {

thread_local std::string g_err;

struct RefGraph {
  std::shared_ptr<const GraphBundle> g;
  EdgeList edges;
};

struct RefModel {
  BuiltModel bm;
};

int guard(const std::exception& e) {
  g_err = e.what();
  return 1;
}

}  // namespace

extern "C" {

typedef void (*ref_trace_fn)(void* ctx, const char* label, const uint32_t* bits, int64_t rows,
                             int64_t cols, int word_bits);

const char* ref_error(void) { return g_err.c_str(); }

int ref_max_threads(void) { return omp_get_max_threads(); }
void ref_set_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
}

// rng.hpp:66-80 through the reference's own Rng.
int64_t ref_random_edges(uint64_t seed, int64_t nodes, int64_t m, int allow_self, int64_t* src,
                         int64_t* dst) {
  Rng rng(seed);
  EdgeList e = random_edges(rng, nodes, m, allow_self != 0);
  for (size_t k = 0; k < e.edges.size(); ++k) {
    src[k] = e.edges[k].first;
    dst[k] = e.edges[k].second;
  }
  return static_cast<int64_t>(e.edges.size());
}

void ref_random_dense(uint64_t seed, int64_t rows, int64_t cols, float* out) {
  Rng rng(seed);
  DenseMatrix m = random_dense(rng, rows, cols);
  std::memcpy(out, m.row(0), static_cast<size_t>(rows * cols) * sizeof(float));
}

// graphops.cpp:146-170 (prepare_graph) on the given edges.
void* ref_graph_create(int64_t n, const int64_t* src, const int64_t* dst, int64_t e) {
  try {
    auto h = std::make_unique<RefGraph>();
    h->edges.node_count = n;
    h->edges.edges.reserve(static_cast<size_t>(e));
    for (int64_t k = 0; k < e; ++k) h->edges.edges.emplace_back(src[k], dst[k]);
    h->g = prepare_graph(h->edges);
    return h.release();
  } catch (const std::exception& ex) {
    guard(ex);
    return nullptr;
  }
}

// GraphBundle assembled from FRDC arrays (A+I and loop-free A) through the
// reference's own validating FrdcMatrix constructor, with the scales derived
// exactly as prepare_graph does (graphops.cpp:135-170).  Used by the bounded
// CPU-baseline sample to skip the reference's single-threaded 44 s sort; the
// arrays are the ones the parity tests prove byte-identical.
void* ref_graph_from_frdc(int64_t n, const uint64_t* rp, const uint32_t* ci, const uint16_t* ti,
                          int64_t nnz, const uint64_t* rp2, const uint32_t* ci2,
                          const uint16_t* ti2, int64_t nnz2) {
  try {
    const size_t tr = static_cast<size_t>((n + 3) / 4) + 1;
    auto mk = [&](const uint64_t* r, const uint32_t* c, const uint16_t* t, int64_t z) {
      return FrdcMatrix(n, n, std::vector<uint64_t>(r, r + tr), std::vector<uint32_t>(c, c + z),
                        std::vector<uint16_t>(t, t + z));
    };
    auto deg_of = [&](const FrdcMatrix& a) {
      std::vector<int64_t> d(static_cast<size_t>(n), 0);
      for (int64_t t = 0; t + 1 < static_cast<int64_t>(a.row_ptr().size()); ++t)
        for (uint64_t k = a.row_ptr()[t]; k < a.row_ptr()[t + 1]; ++k)
          for (int r = 0; r < 4 && 4 * t + r < n; ++r)
            d[static_cast<size_t>(4 * t + r)] += __builtin_popcount((a.tiles()[k] >> (12 - 4 * r)) & 0xF);
      return d;
    };
    auto g = std::make_shared<GraphBundle>();
    g->structure = mk(rp, ci, ti, nnz);
    g->raw = mk(rp2, ci2, ti2, nnz2);
    std::vector<int64_t> dl = deg_of(g->structure);
    std::vector<Real> s(dl.size());
    for (size_t i = 0; i < dl.size(); ++i) s[i] = static_cast<Real>(1.0 / std::sqrt(static_cast<double>(dl[i])));
    g->norm_row = ScaleVector(Axis::Row, s);
    g->norm_col = ScaleVector(Axis::Col, std::move(s));
    g->neighbor_count = deg_of(g->raw);
    std::vector<Real> mean(dl.size()), ones(dl.size(), Real(1));
    for (size_t i = 0; i < mean.size(); ++i)
      mean[i] = Real(1) / static_cast<Real>(std::max<int64_t>(1, g->neighbor_count[i]));
    g->mean_row = ScaleVector(Axis::Row, std::move(mean));
    g->ones_row = ScaleVector(Axis::Row, ones);
    g->ones_col = ScaleVector(Axis::Col, std::move(ones));
    auto h = std::make_unique<RefGraph>();
    h->edges.node_count = n;
    h->g = g;
    return h.release();
  } catch (const std::exception& ex) {
    guard(ex);
    return nullptr;
  }
}

void ref_graph_free(void* h) { delete static_cast<RefGraph*>(h); }

// which: 0 = A+I (structure), 1 = loop-free A (raw).
int ref_graph_frdc(void* h, int which, int64_t* nnz, const uint64_t** row_ptr,
                   const uint32_t** col_ind, const uint16_t** tiles) {
  auto* g = static_cast<RefGraph*>(h);
  const FrdcMatrix& m = which == 0 ? g->g->structure : g->g->raw;
  *nnz = m.nnz_tiles();
  *row_ptr = m.row_ptr().data();
  *col_ind = m.col_ind().data();
  *tiles = m.tiles().data();
  return 0;
}

int ref_graph_scales(void* h, const float** norm, const float** mean_row,
                     const int64_t** neighbor_count) {
  auto* g = static_cast<RefGraph*>(h);
  *norm = g->g->norm_row.values().data();
  *mean_row = g->g->mean_row.values().data();
  *neighbor_count = g->g->neighbor_count.data();
  return 0;
}

// modelconfig.cpp:99-173 (build_model).  plan: '|'-separated chains, empty
// for the default plan of `model`.
void* ref_model_build(void* graph, const char* model, int64_t features, int64_t hidden,
                      int64_t classes, uint64_t seed, int word_bits, const char* plan,
                      int64_t nodes) {
  try {
    ModelConfig cfg;
    cfg.model = model;
    cfg.features = features;
    cfg.hidden = hidden;
    cfg.classes = classes;
    cfg.seed = seed;
    cfg.word_bits = word_bits;
    if (plan && *plan) {
      std::string p(plan);
      size_t s = 0;
      while (s <= p.size()) {
        size_t e = p.find('|', s);
        if (e == std::string::npos) e = p.size();
        if (e > s) cfg.plan.push_back(p.substr(s, e - s));
        s = e + 1;
      }
    }
    auto h = std::make_unique<RefModel>();
    std::shared_ptr<const GraphBundle> g =
        graph ? static_cast<RefGraph*>(graph)->g : std::shared_ptr<const GraphBundle>();
    h->bm = build_model(cfg, g, nodes);
    return h.release();
  } catch (const std::exception& ex) {
    guard(ex);
    return nullptr;
  }
}

void ref_model_free(void* h) { delete static_cast<RefModel*>(h); }

const float* ref_model_features(void* h, int64_t* rows, int64_t* cols) {
  auto* m = static_cast<RefModel*>(h);
  *rows = m->bm.features.rows();
  *cols = m->bm.features.cols();
  return m->bm.features.row(0);
}

int ref_model_layers(void* h) { return static_cast<int>(static_cast<RefModel*>(h)->bm.spec.layers.size()); }

// which: 1 = w1, 2 = w2.  Returns NULL when the layer has no such weight.
const float* ref_model_weight(void* h, int layer, int which, int64_t* rows, int64_t* cols) {
  auto* m = static_cast<RefModel*>(h);
  const LayerSpec& l = m->bm.spec.layers[static_cast<size_t>(layer)];
  const auto& w = which == 1 ? l.w1 : l.w2;
  if (!w) return nullptr;
  *rows = w->rows();
  *cols = w->cols();
  return w->row(0);
}

// graphops.cpp:390-484 with a RunTrace; logits = softmax input.
int ref_model_run(void* h, const float* x, int64_t rows, int64_t cols, float* logits,
                  float* out, ref_trace_fn trace, void* ctx) {
  try {
    auto* m = static_cast<RefModel*>(h);
    const DenseMatrix* x0 = &m->bm.features;
    DenseMatrix own;
    if (x) {
      own = DenseMatrix(rows, cols);
      std::memcpy(own.row(0), x, static_cast<size_t>(rows * cols) * sizeof(float));
      x0 = &own;
    }
    RunTrace tr;
    DenseMatrix o = run_model(m->bm.spec, MatOperand(*x0), &tr);
    if (trace)
      for (const auto& p : tr.points) {
        std::vector<uint32_t> words(static_cast<size_t>(p.bits.rows() * p.bits.storage_words_per_row()));
        for (int64_t i = 0; i < p.bits.rows(); ++i) {
          auto r = p.bits.row_span(i);
          std::memcpy(words.data() + i * p.bits.storage_words_per_row(), r.data(), r.size() * 4);
        }
        trace(ctx, p.label.c_str(), words.data(), p.bits.rows(), p.bits.cols(), p.bits.word_bits());
      }
    if (logits)
      std::memcpy(logits, tr.logits.row(0),
                  static_cast<size_t>(tr.logits.rows() * tr.logits.cols()) * sizeof(float));
    if (out) std::memcpy(out, o.row(0), static_cast<size_t>(o.rows() * o.cols()) * sizeof(float));
    return 0;
  } catch (const std::exception& ex) {
    return guard(ex);
  }
}

// Wall-clock forward timing through the reference's own run_model (the body
// of bench_model, runreport.cpp:241-277), one call per invocation so the
// caller controls warm-up/steps.  Returns milliseconds, or -1 on error.
double ref_model_time_forward(void* h) {
  try {
    auto* m = static_cast<RefModel*>(h);
    auto t0 = std::chrono::steady_clock::now();
    DenseMatrix o = run_model(m->bm.spec, MatOperand(m->bm.features));
    auto t1 = std::chrono::steady_clock::now();
    volatile float sink = o.rows() ? o.at(0, 0) : 0.0f;
    (void)sink;
    return std::chrono::duration<double, std::milli>(t1 - t0).count();
  } catch (const std::exception& ex) {
    guard(ex);
    return -1.0;
  }
}

// Per-kernel breakdown of one forward (graphops.cpp:53-55 record_ns hooks).
int ref_model_kernel_times(void* h, int cap, char* labels, int label_len, double* ms) {
  try {
    auto* m = static_cast<RefModel*>(h);
    std::vector<KernelTiming> t;
    run_model(m->bm.spec, MatOperand(m->bm.features), nullptr, &t);
    int n = 0;
    for (const auto& k : t) {
      if (n >= cap) break;
      std::strncpy(labels + n * label_len, k.label.c_str(), static_cast<size_t>(label_len - 1));
      labels[n * label_len + label_len - 1] = 0;
      ms[n] = static_cast<double>(k.ns) / 1e6;
      ++n;
    }
    return n;
  } catch (const std::exception& ex) {
    guard(ex);
    return -1;
  }
}

// The reference's own single-thread kernel benchmark (kernelbench.cpp:110-186):
// BSpMM.BBB over a random graph vs a naive CSR SpMM.  edges = adjacency bits
// the tiled kernel walked (kernelbench.cpp:143/179), parsed from its result name.
int ref_bench_bspmm_bbb(int64_t nodes, double density, int64_t cols, uint64_t seed, int word_bits,
                        double* engine_ms, double* baseline_ms, int64_t* edges, int* match) {
  try {
    KernelBenchResult r = bench_bspmm_bbb(nodes, density, cols, seed, word_bits);
    *engine_ms = r.engine_ms;
    *baseline_ms = r.baseline_ms;
    *match = r.values_match ? 1 : 0;
    const std::string key = " nodes, ";
    size_t p = r.name.find(key);
    *edges = p == std::string::npos ? -1 : std::strtoll(r.name.c_str() + p + key.size(), nullptr, 10);
    return 0;
  } catch (const std::exception& ex) {
    return guard(ex);
  }
}

// The reference's own tile-set gather and dense expansion over FRDC arrays
// (bitsparse.cpp:114-160), through its validating FrdcMatrix constructor.
namespace {
FrdcMatrix frdc_of(int64_t rows, int64_t cols, const uint64_t* rp, const uint32_t* ci,
                   const uint16_t* ti, int64_t nnz) {
  const size_t tr = static_cast<size_t>((rows + 3) / 4) + 1;
  return FrdcMatrix(rows, cols, std::vector<uint64_t>(rp, rp + tr), std::vector<uint32_t>(ci, ci + nnz),
                    std::vector<uint16_t>(ti, ti + nnz));
}
}  // namespace

int ref_gather_tileset(int64_t rows, int64_t cols, const uint64_t* rp, const uint32_t* ci,
                       const uint16_t* ti, int64_t nnz, int64_t tile_row, int64_t set_index,
                       int word_bits, int32_t* ts, uint64_t* out_rows, uint32_t* out_cols) {
  try {
    TileSet t = gather_tileset(frdc_of(rows, cols, rp, ci, ti, nnz), tile_row, set_index, word_bits);
    *ts = t.ts;
    for (int i = 0; i < 4; ++i) out_rows[i] = t.rows[static_cast<size_t>(i)];
    for (int i = 0; i < 16; ++i) out_cols[i] = t.cols[static_cast<size_t>(i)];
    return 0;
  } catch (const std::exception& ex) {
    return guard(ex);
  }
}

int ref_frdc_to_dense(int64_t rows, int64_t cols, const uint64_t* rp, const uint32_t* ci,
                      const uint16_t* ti, int64_t nnz, int word_bits, uint32_t* out) {
  try {
    BitDenseMatrix d = frdc_to_dense(frdc_of(rows, cols, rp, ci, ti, nnz), word_bits);
    const int64_t w = d.storage_words_per_row();
    for (int64_t i = 0; i < d.rows(); ++i) std::memcpy(out + i * w, d.row_span(i).data(), static_cast<size_t>(w) * 4);
    return 0;
  } catch (const std::exception& ex) {
    return guard(ex);
  }
}

// Kernel-level access for fixtures: binarize (bitdense.cpp:71-88).
void ref_binarize(const float* x, int64_t rows, int64_t cols, int word_bits, uint32_t* out) {
  DenseMatrix m(rows, cols);
  std::memcpy(m.row(0), x, static_cast<size_t>(rows * cols) * sizeof(float));
  BitDenseMatrix b = binarize(m, word_bits);
  for (int64_t i = 0; i < rows; ++i) {
    auto r = b.row_span(i);
    std::memcpy(out + i * b.storage_words_per_row(), r.data(), r.size() * 4);
  }
}

// The reference's plan enumeration (tune.cpp:119-125) for a model skeleton
// (skeleton_of, tune.cpp:84-96): writes the plans as lines of '|'-joined layer
// chains into buf; returns the number of plans or -1 (error / buffer short).
int64_t ref_enumerate_plans(const char* model, int layers, char* buf, int64_t cap) {
  try {
    std::vector<LayerKind> kinds;
    const std::string m(model);
    if (m == "gcn") {
      kinds.assign(layers, LayerKind::GcnConv);
    } else if (m == "sage") {
      kinds.assign(layers, LayerKind::SageConv);
    } else {
      kinds.assign(layers - 1, LayerKind::GraphConv);
      kinds.push_back(LayerKind::FullyConnected);
    }
    const auto plans = enumerate_plans(kinds, Precision::F);
    std::string out;
    for (const auto& p : plans) {
      for (size_t i = 0; i < p.size(); ++i) out += (i ? "|" : "") + p[i];
      out += "\n";
    }
    if (static_cast<int64_t>(out.size()) + 1 > cap) return -1;
    std::memcpy(buf, out.c_str(), out.size() + 1);
    return static_cast<int64_t>(plans.size());
  } catch (const std::exception& e) {
    guard(e);
    return -1;
  }
}

// An arbitrary layer list through the reference's run_model (graphops.cpp:
// 390-484): layer kinds in LayerKind order (graphops.hpp:42-53), plan as a
// '+'-joined chain (parse_plan_chain), optional weights / BatchNorm / Scale
// parameters, graph optional.  Output and logits are malloc'd (free with
// ref_free); the trace callback sees every BIN point.
typedef struct {
  int kind;
  const char* plan;
  const float* w1;
  int64_t w1_rows, w1_cols;
  const float* w2;
  int64_t w2_rows, w2_cols;
  int relu;
  const float *bn_gamma, *bn_beta, *bn_mean, *bn_sigma;
  int64_t bn_len;
  const float* scale_row;
  int64_t scale_row_len;
  const float* scale_col;
  int64_t scale_col_len;
} ref_layer;

int ref_spec_run(void* graph, const ref_layer* layers, int n, int word_bits, const float* x, int64_t rows,
                 int64_t cols, float** out, float** logits, int64_t* out_cols, ref_trace_fn trace, void* ctx) {
  try {
    ModelSpec spec;
    spec.word_bits = word_bits;
    if (graph) spec.graph = static_cast<RefGraph*>(graph)->g;
    auto dense = [](const float* p, int64_t r, int64_t c) {
      auto d = std::make_shared<DenseMatrix>(r, c);
      if (r * c) std::memcpy(d->row(0), p, static_cast<size_t>(r * c) * sizeof(float));
      return d;
    };
    auto vec = [](const float* p, int64_t len) { return std::vector<Real>(p, p + len); };
    for (int i = 0; i < n; ++i) {
      const ref_layer& d = layers[i];
      LayerSpec l;
      l.kind = static_cast<LayerKind>(d.kind);
      if (d.plan && *d.plan) l.plan = parse_plan_chain(d.plan);
      if (d.w1) l.w1 = dense(d.w1, d.w1_rows, d.w1_cols);
      if (d.w2) l.w2 = dense(d.w2, d.w2_rows, d.w2_cols);
      l.relu = d.relu != 0;
      if (d.bn_gamma)
        l.bn = BatchNormParams{vec(d.bn_gamma, d.bn_len), vec(d.bn_beta, d.bn_len), vec(d.bn_mean, d.bn_len),
                               vec(d.bn_sigma, d.bn_len)};
      if (d.scale_row) l.scale_row = ScaleVector(Axis::Row, vec(d.scale_row, d.scale_row_len));
      if (d.scale_col) l.scale_col = ScaleVector(Axis::Col, vec(d.scale_col, d.scale_col_len));
      spec.layers.push_back(std::move(l));
    }
    DenseMatrix x0(rows, cols);
    if (rows * cols) std::memcpy(x0.row(0), x, static_cast<size_t>(rows * cols) * sizeof(float));
    RunTrace tr;
    DenseMatrix o = run_model(spec, MatOperand(x0), &tr);
    if (trace)
      for (const auto& p : tr.points) {
        std::vector<uint32_t> words(static_cast<size_t>(p.bits.rows() * p.bits.storage_words_per_row()));
        for (int64_t r = 0; r < p.bits.rows(); ++r) {
          auto sp = p.bits.row_span(r);
          std::memcpy(words.data() + r * p.bits.storage_words_per_row(), sp.data(), sp.size() * 4);
        }
        trace(ctx, p.label.c_str(), words.data(), p.bits.rows(), p.bits.cols(), p.bits.word_bits());
      }
    *out_cols = o.cols();
    const size_t nb = static_cast<size_t>(o.rows() * o.cols()) * sizeof(float);
    *out = static_cast<float*>(std::malloc(std::max<size_t>(nb, 4)));
    *logits = static_cast<float*>(std::malloc(std::max<size_t>(nb, 4)));
    if (nb) std::memcpy(*out, o.row(0), nb);
    const bool has_logits = tr.logits.rows() * tr.logits.cols() == o.rows() * o.cols() && nb;
    if (has_logits) std::memcpy(*logits, tr.logits.row(0), nb);
    else if (nb) std::memcpy(*logits, o.row(0), nb);
    return 0;
  } catch (const std::exception& ex) {
    return guard(ex);
  }
}

// One layer through the reference's own gcn_layer / sage_layer /
// graphconv_layer (graphops.cpp:270-335), with LayerHooks recording every BIN
// point.  x: F (float rows x cols) or B (packed PlusMinus bits, x_wb).  The
// result is malloc'd (free with ref_free): floats for F, packed words for B.
int ref_layer_run(void* graph, const ref_layer* d, int word_bits, int x_prec, const void* x, int64_t rows,
                  int64_t cols, int x_wb, const char* prefix, int* out_prec, void** out, int64_t* out_rows,
                  int64_t* out_cols, int* out_wb, ref_trace_fn trace, void* ctx) {
  try {
    LayerSpec l;
    l.kind = static_cast<LayerKind>(d->kind);
    if (d->plan && *d->plan) l.plan = parse_plan_chain(d->plan);
    auto dense = [](const float* p, int64_t r, int64_t c) {
      auto m = std::make_shared<DenseMatrix>(r, c);
      if (r * c) std::memcpy(m->row(0), p, static_cast<size_t>(r * c) * sizeof(float));
      return m;
    };
    if (d->w1) l.w1 = dense(d->w1, d->w1_rows, d->w1_cols);
    if (d->w2) l.w2 = dense(d->w2, d->w2_rows, d->w2_cols);
    l.relu = d->relu != 0;
    MatOperand xo;
    if (x_prec == 0) {
      DenseMatrix m(rows, cols);
      if (rows * cols) std::memcpy(m.row(0), x, static_cast<size_t>(rows * cols) * sizeof(float));
      xo = std::move(m);
    } else {
      BitDenseMatrix b(rows, cols, BitSemantics::PlusMinus, x_wb);
      const int64_t w = b.storage_words_per_row();
      for (int64_t r = 0; r < rows; ++r)
        std::memcpy(b.row_span(r).data(), static_cast<const uint32_t*>(x) + r * w, static_cast<size_t>(w) * 4);
      xo = BitOperand{std::move(b), std::nullopt};
    }
    LayerHooks hooks;
    hooks.record_bits = [&](const std::string& label, const BitDenseMatrix& b) {
      if (!trace) return;
      const int64_t w = b.storage_words_per_row();
      std::vector<uint32_t> words(static_cast<size_t>(b.rows() * w));
      for (int64_t r = 0; r < b.rows(); ++r) std::memcpy(words.data() + r * w, b.row_span(r).data(), static_cast<size_t>(w) * 4);
      trace(ctx, label.c_str(), words.data(), b.rows(), b.cols(), b.word_bits());
    };
    const GraphBundle& g = *static_cast<RefGraph*>(graph)->g;
    const std::string pre = prefix ? prefix : "";
    MatOperand r = d->kind == static_cast<int>(LayerKind::GcnConv)
                       ? gcn_layer(xo, l, g, std::nullopt, &hooks, pre, word_bits)
                   : d->kind == static_cast<int>(LayerKind::SageConv)
                       ? sage_layer(xo, l, g, std::nullopt, &hooks, pre, word_bits)
                       : graphconv_layer(xo, l, g, std::nullopt, &hooks, pre, word_bits);
    if (std::holds_alternative<DenseMatrix>(r)) {
      const DenseMatrix& o = std::get<DenseMatrix>(r);
      *out_prec = 0;
      *out_rows = o.rows();
      *out_cols = o.cols();
      *out_wb = 32;
      const size_t nb = static_cast<size_t>(o.rows() * o.cols()) * 4;
      *out = std::malloc(std::max<size_t>(nb, 4));
      if (nb) std::memcpy(*out, o.row(0), nb);
    } else {
      const BitDenseMatrix& b = std::get<BitOperand>(r).bits;
      const int64_t w = b.storage_words_per_row();
      *out_prec = 1;
      *out_rows = b.rows();
      *out_cols = b.cols();
      *out_wb = b.word_bits();
      *out = std::malloc(std::max<size_t>(static_cast<size_t>(b.rows() * w) * 4, 4));
      for (int64_t i = 0; i < b.rows(); ++i)
        std::memcpy(static_cast<uint32_t*>(*out) + i * w, b.row_span(i).data(), static_cast<size_t>(w) * 4);
    }
    return 0;
  } catch (const std::exception& ex) {
    return guard(ex);
  }
}

// The reference's dense oracle (oracle.cpp:194-317) on a built model and the
// graph's edges: BIN points as packed bits (sign > 0 -> 1, the comparison of
// runreport.cpp:92-93) through the trace callback, logits in double
// (malloc'd, free with ref_free).  full_precision selects Mode::FullPrecision.
int ref_oracle_run(void* graph, void* model, int full_precision, int word_bits, ref_trace_fn trace, void* ctx,
                   double** logits, int64_t* rows, int64_t* cols) {
  try {
    auto* g = static_cast<RefGraph*>(graph);
    auto* m = static_cast<RefModel*>(model);
    oracle::Config cfg;
    cfg.mode = full_precision ? oracle::Config::Mode::FullPrecision : oracle::Config::Mode::SimulatedBinarization;
    oracle::GraphDense gd = oracle::graph_from_edges(g->edges);
    oracle::Trace tr;
    oracle::run_model(m->bm.spec, oracle::Mat::from(m->bm.features), gd, cfg, &tr);
    if (trace)
      for (const auto& p : tr.points) {
        BitDenseMatrix b(p.signs.rows, p.signs.cols, BitSemantics::PlusMinus, word_bits);
        for (int64_t i = 0; i < p.signs.rows; ++i)
          for (int64_t j = 0; j < p.signs.cols; ++j) b.set_bit(i, j, p.signs.at(i, j) > 0);
        const int64_t w = b.storage_words_per_row();
        std::vector<uint32_t> words(static_cast<size_t>(b.rows() * w));
        for (int64_t r = 0; r < b.rows(); ++r) std::memcpy(words.data() + r * w, b.row_span(r).data(), static_cast<size_t>(w) * 4);
        trace(ctx, p.label.c_str(), words.data(), b.rows(), b.cols(), word_bits);
      }
    *rows = tr.logits.rows;
    *cols = tr.logits.cols;
    *logits = static_cast<double*>(std::malloc(std::max<size_t>(tr.logits.v.size() * 8, 8)));
    if (!tr.logits.v.empty()) std::memcpy(*logits, tr.logits.v.data(), tr.logits.v.size() * 8);
    return 0;
  } catch (const std::exception& ex) {
    return guard(ex);
  }
}

// The reference's own verify_model (runreport.cpp:51-135), report fields out.
int ref_verify_model(void* graph, void* model, int full_precision, double tolerance, int64_t corrupt_tile,
                     double* max_rel, int64_t* counts /* points, values, mismatches, row, col */, char* label,
                     int label_len, double* agreement, int* pass) {
  try {
    auto* g = static_cast<RefGraph*>(graph);
    auto* m = static_cast<RefModel*>(model);
    oracle::Config cfg;
    cfg.mode = full_precision ? oracle::Config::Mode::FullPrecision : oracle::Config::Mode::SimulatedBinarization;
    cfg.tolerance = tolerance;
    VerifyReport r = verify_model(m->bm.spec, m->bm.features, g->edges, cfg, corrupt_tile);
    *max_rel = r.max_rel_logit_error;
    counts[0] = r.bin_points;
    counts[1] = r.bin_values;
    counts[2] = r.bin_mismatches;
    counts[3] = r.first_mismatch_row;
    counts[4] = r.first_mismatch_col;
    std::strncpy(label, r.first_mismatch_label.c_str(), static_cast<size_t>(label_len - 1));
    label[label_len - 1] = 0;
    *agreement = r.argmax_agreement;
    *pass = r.pass ? 1 : 0;
    return 0;
  } catch (const std::exception& ex) {
    return guard(ex);
  }
}

void ref_free(void* p) { std::free(p); }

// graphio.cpp readers.  kind 0: read_edge_list(text), 1: read_matrix_market
// (text), 2: load_graph(path = text).  Arrays are malloc'd (ref_free).
int ref_read_graph(int kind, const char* text, size_t len, const char* name, int64_t forced, int undirected,
                   int64_t* node_count, int64_t* n_edges, int64_t** src, int64_t** dst, int64_t* n_weights,
                   double** weights) {
  try {
    EdgeList e;
    if (kind == 2) {
      e = load_graph(std::string(text, len), forced, undirected != 0);
    } else {
      std::istringstream in(std::string(text, len));
      e = kind == 0 ? read_edge_list(in, name, forced, undirected != 0)
                    : read_matrix_market(in, name, undirected != 0);
    }
    *node_count = e.node_count;
    *n_edges = static_cast<int64_t>(e.edges.size());
    *src = static_cast<int64_t*>(std::malloc(std::max<size_t>(e.edges.size(), 1) * 8));
    *dst = static_cast<int64_t*>(std::malloc(std::max<size_t>(e.edges.size(), 1) * 8));
    for (size_t k = 0; k < e.edges.size(); ++k) (*src)[k] = e.edges[k].first, (*dst)[k] = e.edges[k].second;
    *n_weights = static_cast<int64_t>(e.weights.size());
    *weights = static_cast<double*>(std::malloc(std::max<size_t>(e.weights.size(), 1) * 8));
    for (size_t k = 0; k < e.weights.size(); ++k) (*weights)[k] = e.weights[k];
    return 0;
  } catch (const std::exception& ex) {
    return guard(ex);
  }
}

}  // extern "C"
