// extern "C" entry points (include/bitgnn_b200.h).  Every function converts
// exceptions into status codes; the message stays in bg_last_error().
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <random>
#include <sstream>

#include "engine.cuh"
#include "model.cuh"

namespace bg {

namespace {
thread_local std::string g_last_error;
thread_local Pool g_op_pool;  // temporaries of op-level calls (synchronous)
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

int sm_count() {
  static int n = [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
    return v;
  }();
  return n;
}

namespace {

void need(const void* p, const char* what) {
  if (!p) fail(std::string("null ") + what);
}

void copy_out(const Op& r, bg_mat* out, cudaStream_t s) {
  need(out, "output operand");
  if (out->precision != r.prec || out->rows != r.rows || out->cols != r.cols ||
      (r.prec == BG_B && out->word_bits != r.wb))
    fail("output operand shape/precision does not match the result");
  if (r.bytes()) need(out->data, "output data");  // an empty result needs no buffer
  const void* src = r.prec == BG_F ? static_cast<const void*>(r.f) : static_cast<const void*>(r.bits);
  if (r.bytes()) BG_CUDA(cudaMemcpyAsync(out->data, src, r.bytes(), cudaMemcpyDeviceToDevice, s));
  out->semantics = BG_PLUS_MINUS;
  out->scale = nullptr;
}

void sync(cudaStream_t s) { BG_CUDA(cudaStreamSynchronize(s)); }



}  // namespace
}  // namespace bg

namespace bg {

// Changes whenever either adjacency of the graph rebuilds a view (or is
// corrupted by the fault hook): captured forwards are then re-recorded.
uint64_t graph_generation(const bg_graph* g) {
  if (!g) return 0;
  return (g->structure ? g->structure->gen : 0) * 0x9E3779B97F4A7C15ull + (g->raw ? g->raw->gen : 0);
}

void run_captured(bg_model& m, bg_model::CaptureSlot& slot, bg_model::Key k, cudaStream_t st,
                  const std::function<void()>& run) {
  k.agg_gen = aggregation_generation() * 2 + (persistent_forced() ? 1 : 0);  // settings the graph was recorded with
  // Any other entry point sharing the pool (traced, timed, host, the other
  // slot) may have grown a slot since the capture: pool_gen then differs and
  // the graph, which holds the old pointers, is re-recorded.
  k.pool_gen = m.pool.gen;
  k.graph_gen = graph_generation(m.graph);
  if (slot.exec && k == slot.key) {
    BG_CUDA(cudaGraphLaunch(slot.exec, st));
    return;
  }
  if (!(k == slot.key)) {
    // First run with this binding: eager, which also sizes the pool.
    slot.reset();
    run();
    slot.key = k;
    slot.key.pool_gen = m.pool.gen;
    slot.key.graph_gen = graph_generation(m.graph);
    return;
  }
  // Second run with the same binding: capture and replay from now on.
  cudaGraph_t graph = nullptr;
  BG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  try {
    run();
  } catch (...) {
    cudaStreamEndCapture(st, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  BG_CUDA(cudaStreamEndCapture(st, &graph));
  BG_CUDA(cudaGraphInstantiate(&slot.exec, graph, 0));
  cudaGraphDestroy(graph);
  BG_CUDA(cudaGraphLaunch(slot.exec, st));
}

}  // namespace bg

using namespace bg;

extern "C" {

const char* bg_last_error(void) { return bg::g_last_error.c_str(); }
int bg_version(void) { return 100; }

int bg_set_aggregation(int mode, int window_nodes) {
  return guard([&] { set_aggregation(mode, window_nodes); });
}

int bg_set_persistent(int enable) {
  return guard([&] { set_persistent_forced(enable != 0); });
}

int bg_get_aggregation(int* mode, int* window_nodes) {
  return guard([&] {
    if (mode) *mode = aggregation_mode();
    if (window_nodes) *window_nodes = window_nodes_setting();
  });
}

int bg_device_count(int* count) {
  return guard([&] {
    need(count, "output");
    BG_CUDA(cudaGetDeviceCount(count));
  });
}
int bg_device_alloc(size_t bytes, void** out) {
  return guard([&] {
    need(out, "output");
    *out = nullptr;
    if (bytes) BG_CUDA(cudaMalloc(out, bytes));
  });
}
int bg_device_free(void* p) {
  return guard([&] {
    if (p) BG_CUDA(cudaFree(p));
  });
}
int bg_memcpy(void* dst, const void* src, size_t bytes, int kind, bg_stream s) {
  return guard([&] {
    if (!bytes) return;
    need(dst, "destination");
    need(src, "source");
    const cudaMemcpyKind k = kind == BG_COPY_H2D   ? cudaMemcpyHostToDevice
                             : kind == BG_COPY_D2H ? cudaMemcpyDeviceToHost
                             : kind == BG_COPY_D2D ? cudaMemcpyDeviceToDevice
                                                   : (fail("bg_memcpy: unknown copy kind"), cudaMemcpyDefault);
    BG_CUDA(cudaMemcpyAsync(dst, src, bytes, k, S(s)));
    sync(S(s));
  });
}
int bg_memset(void* dst, int value, size_t bytes, bg_stream s) {
  return guard([&] {
    if (!bytes) return;
    need(dst, "destination");
    BG_CUDA(cudaMemsetAsync(dst, value, bytes, S(s)));
  });
}
int bg_stream_synchronize(bg_stream s) {
  return guard([&] { sync(S(s)); });
}

int64_t bg_storage_words_per_row(int64_t cols, int word_bits) { return spw(cols, word_bits); }

int bg_variant_parse(const char* text, bg_variant* out) {
  return guard([&] {
    need(text, "text");
    need(out, "output");
    *out = variant_parse(text);
  });
}
int bg_variant_valid(bg_variant v) { return variant_valid(v) ? 1 : 0; }
int bg_variant_name(bg_variant v, char* buf, size_t len) {
  return guard([&] {
    const std::string n = variant_name(v);
    if (!buf || len <= n.size()) fail("buffer too small");
    std::memcpy(buf, n.c_str(), n.size() + 1);
  });
}

// ---- bitdense ---------------------------------------------------------------
static void check_wb(int wb) {
  if (wb != 32 && wb != 64) fail("BitDenseMatrix: word_bits must be 32 or 64");
}

int bg_binarize(const float* x, int64_t rows, int64_t cols, int wb, uint32_t* out, bg_stream s) {
  return guard([&] {
    check_wb(wb);
    if (rows < 0 || cols < 0) fail("BitDenseMatrix: negative dimension");
    binarize(x, rows, cols, wb, out, S(s));
  });
}

int bg_binarize_with_scale(const float* x, int64_t rows, int64_t cols, int axis, int wb,
                           uint32_t* out_bits, float* out_scale, bg_stream s) {
  return guard([&] {
    check_wb(wb);
    if (rows < 0 || cols < 0) fail("BitDenseMatrix: negative dimension");
    binarize(x, rows, cols, wb, out_bits, S(s));
    l1_scales(x, rows, cols, axis, out_scale, S(s));
  });
}

int bg_unpack(const uint32_t* bits, int64_t rows, int64_t cols, int wb, int semantics, float* out,
              bg_stream s) {
  return guard([&] {
    check_wb(wb);
    unpack(bits, rows, cols, wb, semantics, out, S(s));
  });
}

int bg_transpose(const uint32_t* in, int64_t rows, int64_t cols, int wb, uint32_t* out,
                 bg_stream s) {
  return guard([&] {
    check_wb(wb);
    transpose_bits(in, rows, cols, wb, out, S(s));
  });
}

// ---- FRDC / graph --------------------------------------------------------------
int bg_frdc_from_edges(const int64_t* src, const int64_t* dst, int64_t e, int64_t n, int loops,
                       bg_frdc** out, bg_stream s) {
  return guard([&] {
    need(out, "output");
    *out = frdc_build(src, dst, e, n, loops != 0, false, S(s)).release();
  });
}

int bg_frdc_from_host(int64_t rows, int64_t cols, const uint64_t* rp, const uint32_t* ci,
                      const uint16_t* ti, int64_t nnz, bg_frdc** out, bg_stream s) {
  return guard([&] {
    need(out, "output");
    *out = frdc_from_host(rows, cols, rp, ci, ti, nnz, S(s)).release();
  });
}

int bg_frdc_info_get(const bg_frdc* m, bg_frdc_info* info) {
  return guard([&] {
    need(m, "frdc");
    need(info, "info");
    info->node_rows = m->rows;
    info->node_cols = m->cols;
    info->tile_rows = m->tile_rows;
    info->tile_cols = m->tile_cols;
    info->nnz_tiles = m->nnz;
    info->nnz_bits = m->nnz_bits;
    info->max_row_degree = m->max_deg;
    info->row_ptr = m->rp();
    info->col_ind = m->ci();
    info->tiles = m->ti();
    info->degree = m->deg();
  });
}

int bg_frdc_download(const bg_frdc* m, uint64_t* rp, uint32_t* ci, uint16_t* ti) {
  return guard([&] {
    need(m, "frdc");
    if (rp) BG_CUDA(cudaMemcpy(rp, m->row_ptr.p, static_cast<size_t>(m->tile_rows + 1) * 8, cudaMemcpyDeviceToHost));
    if (ci && m->nnz) BG_CUDA(cudaMemcpy(ci, m->col_ind.p, static_cast<size_t>(m->nnz) * 4, cudaMemcpyDeviceToHost));
    if (ti && m->nnz) BG_CUDA(cudaMemcpy(ti, m->tiles.p, static_cast<size_t>(m->nnz) * 2, cudaMemcpyDeviceToHost));
  });
}

int bg_frdc_serialized_size(const bg_frdc* m, size_t* bytes) {
  return guard([&] {
    need(m, "frdc");
    need(bytes, "output");
    *bytes = frdc_container_bytes(*m);
  });
}

int bg_frdc_serialize(const bg_frdc* m, int word_bits, void* buf, size_t buf_len) {
  return guard([&] {
    need(m, "frdc");
    need(buf, "buffer");
    if (buf_len < frdc_container_bytes(*m)) fail("write_frdc: buffer too small");
    frdc_serialize(*m, word_bits, buf);
  });
}

int bg_frdc_deserialize(const void* buf, size_t len, bg_frdc** out, int* word_bits, bg_stream s) {
  return guard([&] {
    need(out, "output");
    if (!buf && len) fail("null buffer");
    *out = frdc_deserialize(buf, len, word_bits, S(s)).release();
  });
}

int bg_frdc_write_file(const bg_frdc* m, int word_bits, const char* path) {
  return guard([&] {
    need(m, "frdc");
    frdc_write_file(*m, word_bits, path);
  });
}

int bg_frdc_read_file(const char* path, bg_frdc** out, int* word_bits, bg_stream s) {
  return guard([&] {
    need(out, "output");
    *out = frdc_read_file(path, word_bits, S(s)).release();
  });
}

int bg_frdc_corrupt_tile(bg_frdc* m, int64_t k) {
  return guard([&] {
    need(m, "frdc");
    if (m->nnz == 0) return;
    const int64_t i = ((k % m->nnz) + m->nnz) % m->nnz;
    uint16_t t = 0;
    BG_CUDA(cudaMemcpy(&t, m->tiles.as<uint16_t>() + i, 2, cudaMemcpyDeviceToHost));
    t = static_cast<uint16_t>(t ^ 1u);
    BG_CUDA(cudaMemcpy(m->tiles.as<uint16_t>() + i, &t, 2, cudaMemcpyHostToDevice));
    frdc_finalize(*m, nullptr);
  });
}

void bg_frdc_destroy(bg_frdc* m) { delete m; }

int bg_prepare_graph(const int64_t* src, const int64_t* dst, int64_t e, int64_t n, bg_graph** out,
                     bg_stream s) {
  return guard([&] {
    need(out, "output");
    *out = prepare_graph(src, dst, e, n, S(s)).release();
  });
}

int bg_graph_info_get(const bg_graph* g, bg_graph_info* info) {
  return guard([&] {
    need(g, "graph");
    need(info, "info");
    info->n = g->n;
    info->structure = g->structure.get();
    info->raw = g->raw.get();
    info->norm = g->norm.as<float>();
    info->mean_row = g->mean_row.as<float>();
    info->ones = g->ones.as<float>();
    info->neighbor_count = g->neighbor_count.as<int64_t>();
  });
}

int bg_graph_corrupt_tile(bg_graph* g, int64_t k) {
  need(g, "graph");
  return bg_frdc_corrupt_tile(g->structure.get(), k);
}

void bg_graph_destroy(bg_graph* g) { delete g; }

// ---- ops ---------------------------------------------------------------------
int bg_bmm_out_desc(bg_variant v, const bg_mat* a, const bg_mat* w, int wb, bg_mat* out) {
  return guard([&] {
    need(out, "output");
    Op o = bmm_out_desc(v, op_from_mat(a), op_from_mat(w), wb);
    std::memset(out, 0, sizeof *out);
    op_to_mat(o, out);
  });
}

int bg_bspmm_out_desc(bg_variant v, const bg_frdc* adj, const bg_mat* x, int wb, bg_mat* out) {
  return guard([&] {
    need(out, "output");
    Op o = bspmm_out_desc(v, adj, op_from_mat(x), wb);
    std::memset(out, 0, sizeof *out);
    op_to_mat(o, out);
  });
}

int bg_bmm(bg_variant v, const bg_mat* a, const bg_mat* w, int wb, bg_mat* out, bg_stream s) {
  return guard([&] {
    g_op_pool.reset();
    const Op wo = op_from_mat(w);
    Op r = run_bmm(v, op_from_mat(a), &wo, nullptr, wb, g_op_pool, S(s));
    copy_out(r, out, S(s));
    sync(S(s));
  });
}

int bg_bspmm(bg_variant v, const bg_frdc* adj, const float* rs, const float* cs, const bg_mat* x,
             int strategy, int wb, bg_mat* out, bg_stream s) {
  (void)strategy;  // all TrinaryStrategy rewritings produce identical results
  return guard([&] {
    g_op_pool.reset();
    Op r = run_bspmm(v, adj, rs, cs, op_from_mat(x), wb, g_op_pool, S(s));
    copy_out(r, out, S(s));
    sync(S(s));
  });
}

int bg_add(bg_variant v, const bg_mat* a, const bg_mat* b, bg_mat* out, bg_stream s) {
  return guard([&] {
    g_op_pool.reset();
    Op r = run_add(v, op_from_mat(a), op_from_mat(b), g_op_pool, S(s));
    copy_out(r, out, S(s));
    sync(S(s));
  });
}

int bg_concat(bg_variant v, const bg_mat* a, const bg_mat* b, bg_mat* out, bg_stream s) {
  return guard([&] {
    g_op_pool.reset();
    Op r = run_concat(v, op_from_mat(a), op_from_mat(b), g_op_pool, S(s));
    copy_out(r, out, S(s));
    sync(S(s));
  });
}

int bg_scl(const float* x, int64_t rows, int64_t cols, const float* r, const float* c, float* out,
           bg_stream s) {
  return guard([&] { scl(x, rows, cols, r, c, out, S(s)); });
}

int bg_dense_mm(const float* a, const float* w, int64_t rows, int64_t k, int64_t cols, float* out,
                bg_stream s) {
  return guard([&] { dense_mm(a, w, rows, k, cols, out, S(s)); });
}

int bg_relu_inplace(bg_mat* x, bg_stream s) {
  return guard([&] {
    Op o = op_from_mat(x);
    if (o.prec == BG_F) relu(o.f, o.rows * o.cols, S(s));
  });
}

int bg_softmax_rows(const float* x, int64_t rows, int64_t cols, float* out, bg_stream s) {
  return guard([&] { softmax_rows(x, rows, cols, out, S(s)); });
}

int bg_batchnorm_infer(const float* x, int64_t rows, int64_t cols, const float* g, const float* b,
                       const float* m, const float* sg, float* out, bg_stream s) {
  return guard([&] { batchnorm(x, rows, cols, g, b, m, sg, out, S(s)); });
}

int bg_fused_mm_spmm(bg_variant mm, bg_variant sp, const bg_mat* x, const bg_mat* w,
                     const bg_frdc* adj, const float* rs, const float* cs, int strategy,
                     bg_mat* out, bg_stream s) {
  (void)strategy;
  return guard([&] {
    if (mm.out != sp.in1)
      fail("fused_mm_spmm: precision chain mismatch (" + variant_name(mm) + " -> " +
           variant_name(sp) + ")");
    g_op_pool.reset();
    const Op wo = op_from_mat(w);
    Op h = run_bmm(mm, op_from_mat(x), &wo, nullptr, 32, g_op_pool, S(s));
    Op r = run_bspmm(sp, adj, rs, cs, h, 32, g_op_pool, S(s));
    copy_out(r, out, S(s));
    sync(S(s));
  });
}

// ---- single layers (ref: gcn_layer / sage_layer / graphconv_layer) -----------
namespace {

// The reference's own slot checks (graphops.cpp:273, :292-294), then one layer
// through the model executor on a throw-away one-layer model: weights
// binarized with their column scales as run_mm_slot does per call
// (graphops.cpp:47-77), BIN points appended to `trace` under `prefix`.
void layer_call(int kind, const bg_mat* x, const bg_layer_desc* l, const bg_graph* g, int strategy,
                bg_trace* trace, const char* prefix, int wb, bg_mat* out, bg_stream stream) {
  need(x, "input operand");
  need(l, "layer");
  need(g, "graph");
  check_wb(wb);
  if (kind == BG_LAYER_GCN) {
    if (l->n_plan != 2 || !l->w1) fail("gcn_conv: expected {mm, spmm} plan and weights");
  } else if (l->n_plan != 4 || !l->w1 || !l->w2) {
    fail("expected {mm_self, mm_neigh, spmm, add} plan and two weight matrices");
  }
  cudaStream_t s = S(stream);
  const Op x0 = op_from_mat(x);
  bg_model m;
  m.graph = g;
  m.input_prec = x0.prec;
  m.strategy = strategy;
  m.wb = wb;
  m.capture = false;
  LayerInfo info = layer_info(*l);
  info.kind = kind;
  m.infos.push_back(info);
  m.layers.resize(1);
  ModelLayer& ml = m.layers[0];
  ml.info = info;
  ml.relu = l->relu != 0;
  ml.w1.upload(l->w1, l->w1_rows, l->w1_cols, wb, s);
  if (kind != BG_LAYER_GCN) ml.w2.upload(l->w2, l->w2_rows, l->w2_cols, wb, s);
  LayerCall call;
  call.prefix = prefix ? prefix : "";
  forward_impl(m, x0, nullptr, nullptr, trace, nullptr, s, nullptr, &call);
  copy_out(call.result, out, s);
  sync(s);
}

}  // namespace

int bg_layer_out_desc(int kind, const bg_layer_desc* l, const bg_mat* x, int word_bits, bg_mat* out) {
  return guard([&] {
    need(l, "layer");
    need(x, "input operand");
    need(out, "output");
    check_wb(word_bits);
    const int slot = kind == BG_LAYER_GCN ? 1 : 3;
    if (kind != BG_LAYER_GCN && kind != BG_LAYER_SAGE && kind != BG_LAYER_GRAPHCONV)
      fail("layer_out_desc: kind must be gcn_conv, sage_conv or graph_conv");
    // the layer functions' own slot checks (graphops.cpp:273, :292-294)
    if (kind == BG_LAYER_GCN && (l->n_plan != 2 || !l->w1)) fail("gcn_conv: expected {mm, spmm} plan and weights");
    if (kind != BG_LAYER_GCN && (l->n_plan != 4 || !l->w1 || !l->w2))
      fail("expected {mm_self, mm_neigh, spmm, add} plan and two weight matrices");
    std::memset(out, 0, sizeof *out);
    out->precision = l->plan[slot].out;
    out->rows = x->rows;
    out->cols = l->w1_cols;
    out->word_bits = out->precision == BG_B ? word_bits : 32;
    out->semantics = BG_PLUS_MINUS;
  });
}

int bg_gcn_layer(const bg_mat* x, const bg_layer_desc* l, const bg_graph* g, int strategy, bg_trace* trace,
                 const char* prefix, int word_bits, bg_mat* out, bg_stream s) {
  return guard([&] { layer_call(BG_LAYER_GCN, x, l, g, strategy, trace, prefix, word_bits, out, s); });
}

int bg_sage_layer(const bg_mat* x, const bg_layer_desc* l, const bg_graph* g, int strategy, bg_trace* trace,
                  const char* prefix, int word_bits, bg_mat* out, bg_stream s) {
  return guard([&] { layer_call(BG_LAYER_SAGE, x, l, g, strategy, trace, prefix, word_bits, out, s); });
}

int bg_graphconv_layer(const bg_mat* x, const bg_layer_desc* l, const bg_graph* g, int strategy,
                       bg_trace* trace, const char* prefix, int word_bits, bg_mat* out, bg_stream s) {
  return guard([&] { layer_call(BG_LAYER_GRAPHCONV, x, l, g, strategy, trace, prefix, word_bits, out, s); });
}

// ---- models -----------------------------------------------------------------
int bg_validate_model(int has_graph, int input_precision, const bg_layer_desc* layers, int n,
                      char* buf, size_t len) {
  std::vector<LayerInfo> infos;
  for (int i = 0; i < n; ++i) infos.push_back(layer_info(layers[i]));
  const auto errs = validate_model(has_graph != 0, input_precision, infos);
  std::string joined;
  for (size_t i = 0; i < errs.size(); ++i) joined += (i ? "\n" : "") + errs[i];
  if (buf && len) {
    const size_t k = std::min(len - 1, joined.size());
    std::memcpy(buf, joined.data(), k);
    buf[k] = 0;
  }
  return static_cast<int>(errs.size());
}

int bg_model_create(const bg_graph* graph, int input_precision, int strategy, int wb,
                    const bg_layer_desc* layers, int n, bg_model** out, bg_stream s) {
  return guard([&] {
    need(out, "output");
    check_wb(wb);
    auto m = std::make_unique<bg_model>();
    m->graph = graph;
    m->input_prec = input_precision;
    m->strategy = strategy;
    m->wb = wb;
    for (int i = 0; i < n; ++i) m->infos.push_back(layer_info(layers[i]));
    {
      const auto errs = validate_model(graph != nullptr, input_precision, m->infos);
      if (!errs.empty()) {
        std::ostringstream os;
        os << "invalid model:";
        for (const auto& e : errs) os << "\n  " << e;
        fail(os.str());
      }
    }
    m->layers.resize(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      const bg_layer_desc& d = layers[i];
      ModelLayer& l = m->layers[static_cast<size_t>(i)];
      l.info = m->infos[static_cast<size_t>(i)];
      l.relu = d.relu != 0;
      if (d.w1) l.w1.upload(d.w1, d.w1_rows, d.w1_cols, wb, S(s));
      if (d.w2) l.w2.upload(d.w2, d.w2_rows, d.w2_cols, wb, S(s));
      auto up = [&](DevBuf& b, const float* h, int64_t len) {
        b.alloc(static_cast<size_t>(std::max<int64_t>(len, 1)) * 4);
        if (len) BG_CUDA(cudaMemcpyAsync(b.p, h, static_cast<size_t>(len) * 4, cudaMemcpyHostToDevice, S(s)));
      };
      if (l.info.has_bn) {
        l.bn_len = d.bn_len;
        up(l.bn_g, d.bn_gamma, d.bn_len);
        up(l.bn_b, d.bn_beta, d.bn_len);
        up(l.bn_m, d.bn_mean, d.bn_len);
        up(l.bn_s, d.bn_sigma, d.bn_len);
      }
      if (l.info.has_scale) {
        l.sr_len = d.scale_row_len;
        l.sc_len = d.scale_col_len;
        up(l.sr, d.scale_row, d.scale_row_len);
        up(l.sc, d.scale_col, d.scale_col_len);
      }
    }
    BG_CUDA(cudaStreamSynchronize(S(s)));
    *out = m.release();
  });
}

void bg_model_destroy(bg_model* m) { delete m; }

int bg_model_output_cols(const bg_model* m, int64_t* cols) {
  return guard([&] {
    need(m, "model");
    need(cols, "cols");
    int64_t c = -1;
    for (const auto& l : m->layers)
      if (l.info.has_w1) c = l.w1.cols;
    if (c < 0) c = m->last_out_cols;
    if (c < 0) fail("output width depends on the input (no weighted layer)");
    *cols = c;
  });
}

int bg_model_set_graph_capture(bg_model* m, int enable) {
  return guard([&] {
    need(m, "model");
    m->capture = enable != 0;
    if (!m->capture) {
      m->fwd.reset();
      m->sharded.reset();
    }
  });
}

int bg_model_forward(bg_model* m, const bg_mat* x0, float* out, float* logits, bg_stream s) {
  return guard([&] {
    need(m, "model");
    const Op x = op_from_mat(x0);
    cudaStream_t st = S(s);
    auto run = [&] { forward_impl(*m, x, out, logits, nullptr, nullptr, st); };
    if (!m->capture || st == nullptr) {
      run();
      return;
    }
    bg_model::Key k;
    k.x = x.prec == BG_F ? static_cast<const void*>(x.f) : static_cast<const void*>(x.bits);
    k.rows = x.rows;
    k.cols = x.cols;
    k.prec = x.prec;
    k.wb = x.wb;
    k.out = out;
    k.logits = logits;
    k.s = st;
    run_captured(*m, m->fwd, k, st, run);
  });
}

// Host buffers in and out (the reference-facing call).  The fp32 input
// streams in row chunks on an internal copy stream while layer 0's MM runs
// on the chunks that have landed; the last layer produces its output per row
// chunk and each chunk is copied out as soon as it is ready.  Results and
// their order are those of bg_model_forward.
int bg_model_forward_host(bg_model* m, const float* xh, int64_t rows, int64_t cols, float* outh,
                          float* logh, bg_stream s) {
  int64_t oc = 0;
  int rc = bg_model_output_cols(m, &oc);
  if (rc) return rc;
  return guard([&] {
    need(xh, "input");
    need(outh, "output");
    cudaStream_t st = S(s);
    const size_t xb = static_cast<size_t>(rows * cols) * 4, ob = static_cast<size_t>(rows * oc) * 4;
    if (m->hx.bytes < xb) m->hx.alloc(xb);
    if (m->hout.bytes < ob) m->hout.alloc(ob);
    if (logh && m->hlog.bytes < ob) m->hlog.alloc(ob);
    const int nc = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8, rows / 4096)));
    if (!m->copy_stream) BG_CUDA(cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking));
    while (m->chunk_events.size() < static_cast<size_t>(2 * nc + 1)) {
      cudaEvent_t e;
      BG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      m->chunk_events.push_back(e);
    }
    cudaStream_t cs = m->copy_stream;
    cudaEvent_t* in_ev = m->chunk_events.data();
    cudaEvent_t* out_ev = in_ev + nc;
    cudaEvent_t done_ev = in_ev[2 * nc];
    std::vector<int64_t> bounds(nc + 1);
    for (int c = 0; c <= nc; ++c) bounds[c] = rows * c / nc / 16 * 16;
    bounds[nc] = rows;
    // BG_HOST_TRACE=1: print the timeline of this call (stderr) -- last input
    // byte landed, forward done, last output byte back -- for the e2e analysis
    static const bool trace_tl = std::getenv("BG_HOST_TRACE") != nullptr;
    cudaEvent_t tl[4] = {};
    if (trace_tl)
      for (auto& e : tl) BG_CUDA(cudaEventCreate(&e));
    // the copy stream starts after everything already queued on the caller's stream
    BG_CUDA(cudaEventRecord(done_ev, st));
    BG_CUDA(cudaStreamWaitEvent(cs, done_ev, 0));
    if (trace_tl) BG_CUDA(cudaEventRecord(tl[0], cs));
    auto* hx = m->hx.as<float>();
    for (int c = 0; c < nc; ++c) {
      const size_t off = static_cast<size_t>(bounds[c] * cols), n = static_cast<size_t>((bounds[c + 1] - bounds[c]) * cols);
      if (n) BG_CUDA(cudaMemcpyAsync(hx + off, xh + off, n * 4, cudaMemcpyHostToDevice, cs));
      BG_CUDA(cudaEventRecord(in_ev[c], cs));
    }
    if (trace_tl) BG_CUDA(cudaEventRecord(tl[1], cs));
    StreamChunks sc;
    sc.in = RowChunks{nc, bounds.data(), in_ev};
    sc.out = RowChunks{nc, bounds.data(), out_ev};
    const Op x0 = [&] {
      Op o;
      o.prec = BG_F;
      o.rows = rows;
      o.cols = cols;
      o.f = hx;
      return o;
    }();
    if (x0.prec != m->input_prec) fail("model input tag does not match the provided operand");
    forward_impl(*m, x0, m->hout.as<float>(), logh ? m->hlog.as<float>() : nullptr, nullptr, nullptr, st, &sc);
    if (trace_tl) BG_CUDA(cudaEventRecord(tl[2], st));
    auto* ho = m->hout.as<float>();
    if (sc.out_done) {
      for (int c = 0; c < nc; ++c) {
        const size_t off = static_cast<size_t>(bounds[c] * oc), n = static_cast<size_t>((bounds[c + 1] - bounds[c]) * oc);
        BG_CUDA(cudaStreamWaitEvent(cs, out_ev[c], 0));
        if (n) BG_CUDA(cudaMemcpyAsync(outh + off, ho + off, n * 4, cudaMemcpyDeviceToHost, cs));
      }
    }
    BG_CUDA(cudaEventRecord(done_ev, st));
    BG_CUDA(cudaStreamWaitEvent(cs, done_ev, 0));
    if (!sc.out_done) BG_CUDA(cudaMemcpyAsync(outh, ho, ob, cudaMemcpyDeviceToHost, cs));
    if (logh) BG_CUDA(cudaMemcpyAsync(logh, m->hlog.p, ob, cudaMemcpyDeviceToHost, cs));
    if (trace_tl) BG_CUDA(cudaEventRecord(tl[3], cs));
    BG_CUDA(cudaStreamSynchronize(cs));
    BG_CUDA(cudaStreamSynchronize(st));
    if (trace_tl) {
      float a = 0, b = 0, c = 0;
      BG_CUDA(cudaEventElapsedTime(&a, tl[0], tl[1]));
      BG_CUDA(cudaEventElapsedTime(&b, tl[0], tl[2]));
      BG_CUDA(cudaEventElapsedTime(&c, tl[0], tl[3]));
      std::fprintf(stderr, "host_tl: inputs landed %.3f ms, forward done %.3f ms, outputs back %.3f ms (%d chunks)\n",
                   a, b, c, nc);
      for (auto& e : tl) cudaEventDestroy(e);
    }
  });
}

int bg_trace_create(bg_trace** out) {
  return guard([&] {
    need(out, "output");
    *out = new bg_trace();
  });
}
void bg_trace_destroy(bg_trace* t) { delete t; }

int bg_model_forward_traced(bg_model* m, const bg_mat* x0, float* out, float* logits, bg_trace* t,
                            bg_stream s) {
  return guard([&] {
    need(m, "model");
    need(t, "trace");
    t->pts.clear();
    forward_impl(*m, op_from_mat(x0), out, logits, t, nullptr, S(s));
    BG_CUDA(cudaStreamSynchronize(S(s)));
  });
}

int bg_trace_size(const bg_trace* t) { return t ? static_cast<int>(t->pts.size()) : 0; }

int bg_trace_point(const bg_trace* t, int i, const char** label, int64_t* rows, int64_t* cols,
                   int* wb, const uint32_t** bits) {
  return guard([&] {
    need(t, "trace");
    if (i < 0 || i >= static_cast<int>(t->pts.size())) fail("trace point index out of range");
    const TracePoint& p = t->pts[static_cast<size_t>(i)];
    if (label) *label = p.label.c_str();
    if (rows) *rows = p.rows;
    if (cols) *cols = p.cols;
    if (wb) *wb = p.wb;
    if (bits) *bits = p.bits.as<uint32_t>();
  });
}

int bg_model_forward_timed(bg_model* m, const bg_mat* x0, float* out, float* logits,
                           bg_kernel_timing* timings, int cap, int* n, bg_stream s) {
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
  int rc = guard([&] {
    need(m, "model");
    forward_impl(*m, op_from_mat(x0), out, logits, nullptr, &ev, S(s));
    BG_CUDA(cudaStreamSynchronize(S(s)));
    int k = 0;
    for (const auto& e : ev) {
      if (k >= cap) break;
      float ms = 0.0f;
      BG_CUDA(cudaEventElapsedTime(&ms, e.second.first, e.second.second));
      std::memset(timings[k].label, 0, sizeof timings[k].label);
      std::strncpy(timings[k].label, e.first.c_str(), sizeof timings[k].label - 1);
      timings[k].ms = ms;
      ++k;
    }
    if (n) *n = k;
  });
  for (auto& e : ev) {
    cudaEventDestroy(e.second.first);
    cudaEventDestroy(e.second.second);
  }
  return rc;
}

// ---- multi-GPU row partition ------------------------------------------------
int bg_partition_rows(const bg_graph* g, int world, int rank, int64_t* r0, int64_t* r1) {
  int rc = guard([&] {
    need(g, "graph");
    if (world < 1 || rank < 0 || rank >= world) fail("partition: bad rank/world size");
  });
  if (rc) return rc;
  std::vector<uint64_t> rp;
  std::vector<int64_t> bounds(static_cast<size_t>(world) + 1);
  rc = guard([&] {
    const bg_frdc& A = *g->structure;
    rp.resize(static_cast<size_t>(A.tile_rows + 1));
    BG_CUDA(cudaMemcpy(rp.data(), A.row_ptr.p, rp.size() * 8, cudaMemcpyDeviceToHost));
  });
  if (rc) return rc;
  rc = bg_partition_bounds(rp.data(), g->structure->tile_rows, g->n, world, bounds.data());
  if (rc) return rc;
  *r0 = bounds[static_cast<size_t>(rank)];
  *r1 = bounds[static_cast<size_t>(rank) + 1];
  return BG_OK;
}

// ---- synthetic inputs (ref: rng.hpp:16-80) ------------------------------------
}  // extern "C"

struct bg_rng {
  std::mt19937_64 g;
  explicit bg_rng(uint64_t seed) : g(seed) {}
  double uniform() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
  int64_t index(int64_t n) {
    const uint64_t un = static_cast<uint64_t>(n);
    const uint64_t limit = UINT64_MAX - UINT64_MAX % un;
    uint64_t v;
    do v = g();
    while (v >= limit);
    return static_cast<int64_t>(v % un);
  }
};

extern "C" {

int bg_rng_create(uint64_t seed, bg_rng** out) {
  return guard([&] {
    need(out, "output");
    *out = new bg_rng(seed);
  });
}
void bg_rng_destroy(bg_rng* r) { delete r; }

int bg_rng_dense(bg_rng* r, int64_t rows, int64_t cols, float* out) {
  return guard([&] {
    need(r, "rng");
    for (int64_t i = 0; i < rows * cols; ++i) out[i] = static_cast<float>(r->uniform() * 2.0 - 1.0);
  });
}

int bg_rng_edges(bg_rng* r, int64_t nodes, int64_t m, int allow_self, int64_t* src, int64_t* dst,
                 int64_t* count) {
  return guard([&] {
    need(r, "rng");
    if (nodes <= 0) fail("random_edges: nodes must be positive");
    int64_t k = 0;
    for (int64_t t = 0; t < m; ++t) {
      const int64_t a = r->index(nodes);
      int64_t b = r->index(nodes);
      if (!allow_self && a == b) {
        b = (b + 1) % nodes;
        if (a == b) continue;
      }
      src[k] = a;
      dst[k] = b;
      ++k;
    }
    if (count) *count = k;
  });
}

}  // extern "C"
