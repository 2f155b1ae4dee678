// C++ host API test (include/bitgnn_b200/bitgnn.hpp), written the way the
// reference's own doctest suites exercise bitgnn:: (proj/tests/test_kernels.cpp,
// test_graphops.cpp): same calls, same exception types and messages.
//   test_shim --cpu : host-side logic, no device needed (variant algebra,
//                     validate_model, exception mapping, loud failure without GPU)
//   test_shim --gpu : every op through the C++ API on the B200, compared with
//                     the C oracle (oracle/bitgnn_oracle.h -- test infrastructure)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "bitgnn_b200/bitgnn.hpp"
extern "C" {
#include "bitgnn_oracle.h"
}

namespace b = bitgnn_b200;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    if (cond) ++g_pass;                                                          \
    else {                                                                       \
      ++g_fail;                                                                  \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
    }                                                                            \
  } while (0)

template <class E>
static bool throws(const std::function<void()>& f, const char* prefix = nullptr) {
  try {
    f();
  } catch (const E& e) {
    if (prefix && std::strncmp(e.what(), prefix, std::strlen(prefix)) != 0) {
      std::fprintf(stderr, "  message was: %s\n", e.what());
      return false;
    }
    return true;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "  wrong exception: %s\n", e.what());
    return false;
  }
  return false;
}

static b::DenseMatrix random_dense(og_rng* r, int64_t rows, int64_t cols) {
  b::DenseMatrix m(rows, cols);
  og_random_dense(r, rows, cols, m.data());
  return m;
}

// ---------------------------------------------------------------- CPU part --
static void test_cpu() {
  // ref: test_kernels.cpp:79-112 -- variant tables and names
  int counts[4] = {0, 0, 0, 0};
  for (int op = 0; op < 4; ++op)
    for (int a = 0; a < 2; ++a)
      for (int c = 0; c < 2; ++c)
        for (int o = 0; o < 2; ++o)
          counts[op] += b::KernelVariant{static_cast<b::KernelOp>(op), static_cast<b::Precision>(a),
                                         static_cast<b::Precision>(c), static_cast<b::Precision>(o)}
                            .valid();
  CHECK(counts[0] == 7 && counts[1] == 8 && counts[2] == 3 && counts[3] == 3);
  CHECK(b::KernelVariant::parse("MM.FBB").name() == "BMM.FBB");
  CHECK(b::KernelVariant::parse("bspmm.bbf").name() == "BSpMM.BBF");
  CHECK((b::KernelVariant::parse("BSpMM.FBF") ==
         b::KernelVariant{b::KernelOp::BSpMM, b::Precision::F, b::Precision::B, b::Precision::F}));
  CHECK(!b::KernelVariant::parse("BMM.FFF").valid());
  CHECK(throws<std::invalid_argument>([] { b::KernelVariant::parse("BMM.XYZ"); }));
  CHECK(throws<std::invalid_argument>([] { b::ScaleVector(b::Axis::Row, {1.0f, 0.0f}); }));

  // ref: validate_model messages (graphops.cpp:245-268)
  auto W = std::make_shared<const b::DenseMatrix>(4, 4, 1.0f);
  b::ModelSpec m;
  m.layers.push_back({b::LayerKind::GcnConv, {b::KernelVariant::parse("MM.FBB"), b::KernelVariant::parse("BSpMM.BBB")}, W});
  m.layers.push_back({b::LayerKind::GcnConv, {b::KernelVariant::parse("MM.BBF"), b::KernelVariant::parse("BSpMM.FBF")}, W});
  m.layers.push_back({b::LayerKind::Softmax, {}});
  auto errs = b::validate_model(m);
  CHECK(errs.size() == 1 && errs[0] == "model uses graph layers but carries no graph");
  m.layers[1].plan[1] = b::KernelVariant::parse("BSpMM.BBB");  // chain ends at B
  errs = b::validate_model(m);
  CHECK(errs.size() >= 2);

  // SCL elimination (graphops.cpp:357-368)
  b::ModelSpec sm;
  b::LayerSpec scale;
  scale.kind = b::LayerKind::Scale;
  b::LayerSpec binz;
  binz.kind = b::LayerKind::Binarize;
  sm.layers = {m.layers[0], scale, binz, scale, m.layers[2]};
  const b::ModelSpec r = b::rewrite_eliminate_scl(sm);
  CHECK(r.layers.size() == 4 && r.layers[1].kind == b::LayerKind::Binarize && r.layers[2].kind == b::LayerKind::Scale);

  // graph readers (graphio.cpp:72-176): host parsing, no device needed
  std::istringstream el("# a comment\n1 2 0.5\n0 5\n");
  const b::EdgeList e = b::read_edge_list(el, "two.txt", -1, true);
  CHECK(e.node_count == 6 && e.edges.size() == 4 && e.edges[2].first == 2 && e.edges[2].second == 1 &&
        e.weights.size() == 1 && e.weights[0] == 0.5);
  std::istringstream bad("0 1\nfoo bar\n");
  CHECK(throws<std::runtime_error>([&] { b::read_edge_list(bad, "broken.txt"); }, "broken.txt:2: expected \"src dst\""));
  std::istringstream mm("%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 0.5\n3 3 1.0\n");
  const b::EdgeList me = b::read_matrix_market(mm, "mm.mtx");
  CHECK(me.node_count == 3 && me.edges.size() == 3);
  CHECK(throws<std::runtime_error>([&] { b::load_graph("/nonexistent/x.txt"); }, "/nonexistent/x.txt: cannot open"));
}

// Without a device every op fails loudly (no CPU fallback).
static void test_no_device() {
  CHECK(throws<std::runtime_error>([] { b::binarize(b::DenseMatrix(2, 3, 1.0f)); }));
}

// ---------------------------------------------------------------- GPU part --
static og_mat og_dense(const b::DenseMatrix& m) {
  og_mat o{};
  o.prec = OG_F;
  o.rows = m.rows();
  o.cols = m.cols();
  o.word_bits = 32;
  o.f = const_cast<float*>(m.data());
  return o;
}
static og_mat og_bits(const b::BitOperand& x) {
  og_mat o{};
  o.prec = OG_B;
  o.rows = x.bits.rows();
  o.cols = x.bits.cols();
  o.word_bits = x.bits.word_bits();
  o.bits = const_cast<uint32_t*>(x.bits.data());
  o.scale = x.scale ? const_cast<float*>(x.scale->values().data()) : nullptr;
  return o;
}
static bool same(const b::MatOperand& got, const og_mat& want) {
  if (b::operand_rows(got) != want.rows || b::operand_cols(got) != want.cols) return false;
  if (const auto* f = std::get_if<b::DenseMatrix>(&got)) {
    if (want.prec != OG_F) return false;
    return std::memcmp(f->data(), want.f, f->payload_bytes()) == 0;
  }
  const auto& x = std::get<b::BitOperand>(got);
  if (want.prec != OG_B || x.bits.word_bits() != want.word_bits) return false;
  return std::memcmp(x.bits.data(), want.bits, x.bits.payload_bytes()) == 0;
}
static og_variant ogv(const char* s) {
  const auto v = b::KernelVariant::parse(s).c();
  return og_variant{v.op, v.in1, v.in2, v.out};
}

static void test_gpu() {
  og_rng r;
  og_rng_seed(&r, 4242);
  // binarize (ref: bitdense.cpp:71-88), both word widths
  for (int wb : {32, 64}) {
    b::DenseMatrix X = random_dense(&r, 37, 100);
    b::BitDenseMatrix bits = b::binarize(X, wb);
    std::vector<uint32_t> want(static_cast<size_t>(37 * og_spw(100, wb)));
    og_binarize(X.data(), 37, 100, wb, want.data());
    CHECK(std::memcmp(bits.data(), want.data(), want.size() * 4) == 0);
    auto [b2, sc] = b::binarize_with_scale(X, b::Axis::Col, wb);
    std::vector<float> wsc(100);
    og_l1_scales(X.data(), 37, 100, OG_COL, wsc.data());
    CHECK(b2 == bits && std::memcmp(sc.values().data(), wsc.data(), 400) == 0);
    CHECK(b::transpose(b::transpose(bits)) == bits);
  }

  // FRDC from edges, byte-identical (ref: bitsparse.cpp:72-112)
  const int64_t n = 300, e = 3000;
  std::vector<int64_t> s(e), d(e);
  const int64_t ne = og_random_edges(&r, n, e, 0, s.data(), d.data());
  b::EdgeList el;
  el.node_count = n;
  for (int64_t k = 0; k < ne; ++k) el.edges.emplace_back(s[static_cast<size_t>(k)], d[static_cast<size_t>(k)]);
  b::FrdcMatrix A = b::frdc_from_edges(el, true);
  og_frdc oA{};
  int64_t bad = 0;
  CHECK(og_frdc_from_edges(n, s.data(), d.data(), ne, 1, &oA, &bad) == 0);
  CHECK(A.nnz_tiles() == oA.nnz && std::memcmp(A.row_ptr().data(), oA.row_ptr, A.row_ptr().size() * 8) == 0 &&
        std::memcmp(A.col_ind().data(), oA.col_ind, oA.nnz * 4) == 0 &&
        std::memcmp(A.tiles().data(), oA.tiles, oA.nnz * 2) == 0);

  // bmm (ref: kernels.cpp:140-191): weights carry their column scales
  b::DenseMatrix X = random_dense(&r, n, 70), W = random_dense(&r, 70, 40);
  auto [wbits, wsc] = b::binarize_with_scale(W, b::Axis::Col);
  b::BitOperand Wop{wbits, wsc};
  for (const char* v : {"BMM.FBB", "BMM.FBF"}) {
    auto got = b::bmm(b::KernelVariant::parse(v), X, Wop);
    og_mat oa = og_dense(X), ow = og_bits(Wop), out{};
    CHECK(og_bmm(ogv(v), &oa, &ow, 32, &out) == 0);
    CHECK(same(got, out));
    og_mat_free(&out);
  }
  b::BitOperand H{std::get<b::BitOperand>(b::bmm(b::KernelVariant::parse("BMM.FBB"), X, Wop)).bits, std::nullopt};
  for (const char* v : {"BMM.BBB", "BMM.BBF"}) {
    b::DenseMatrix W2 = random_dense(&r, 40, 9);
    auto [w2b, w2s] = b::binarize_with_scale(W2, b::Axis::Col);
    b::BitOperand W2op{w2b, w2s};
    auto got = b::bmm(b::KernelVariant::parse(v), H, W2op);
    og_mat oa = og_bits(H), ow = og_bits(W2op), out{};
    CHECK(og_bmm(ogv(v), &oa, &ow, 32, &out) == 0);
    CHECK(same(got, out));
    og_mat_free(&out);
  }

  // bspmm (ref: kernels.cpp:254-555): integer and real-valued paths
  b::AdjacencyOperand adj{&A, nullptr, nullptr};
  for (const char* v : {"BSpMM.BBB", "BSpMM.BBF"}) {
    auto got = b::bspmm(b::KernelVariant::parse(v), adj, H);
    og_mat ox = og_bits(H), out{};
    CHECK(og_bspmm(ogv(v), &oA, nullptr, nullptr, &ox, 32, &out) == 0);
    CHECK(same(got, out));
    og_mat_free(&out);
  }
  {
    auto got = b::bspmm(b::KernelVariant::parse("BSpMM.FBF"), adj, X);
    og_mat ox = og_dense(X), out{};
    CHECK(og_bspmm(ogv("BSpMM.FBF"), &oA, nullptr, nullptr, &ox, 32, &out) == 0);
    CHECK(same(got, out));
    og_mat_free(&out);
  }
  // contract violations keep the reference's exception type
  CHECK(throws<std::invalid_argument>([&] { b::bspmm(b::KernelVariant::parse("BSpMM.BBB"), adj, X); }));
  CHECK(throws<std::invalid_argument>([&] { b::bmm(b::KernelVariant::parse("BMM.FBB"), H, Wop); }));

  // run_model: Cora-like GCN, traced, against og_run_model (graphops.cpp:390-484)
  auto g = b::prepare_graph(el);
  og_graph og{};
  CHECK(og_prepare_graph(n, s.data(), d.data(), ne, &og) == 0);
  CHECK(g->structure() == A);
  b::DenseMatrix W1 = random_dense(&r, 70, 16), W2 = random_dense(&r, 16, 5);
  b::ModelSpec m;
  m.graph = g;
  m.layers.push_back({b::LayerKind::GcnConv, {b::KernelVariant::parse("MM.FBB"), b::KernelVariant::parse("BSpMM.BBB")},
                      std::make_shared<const b::DenseMatrix>(W1)});
  m.layers.push_back({b::LayerKind::GcnConv, {b::KernelVariant::parse("MM.BBF"), b::KernelVariant::parse("BSpMM.FBF")},
                      std::make_shared<const b::DenseMatrix>(W2)});
  m.layers.push_back({b::LayerKind::Softmax, {}});
  CHECK(b::validate_model(m).empty());
  CHECK(std::string(b::layer_kind_name(b::LayerKind::GcnConv)) == "gcn_conv");
  b::RunTrace trace;
  std::vector<b::KernelTiming> timings;
  b::DenseMatrix out = b::run_model(m, X, &trace, &timings);

  og_layer ol[3] = {};
  ol[0].kind = 0; ol[0].nplan = 2; ol[0].plan[0] = ogv("MM.FBB"); ol[0].plan[1] = ogv("BSpMM.BBB");
  ol[0].w1 = W1.data(); ol[0].w1_rows = 70; ol[0].w1_cols = 16; ol[0].relu = 1;
  ol[1].kind = 0; ol[1].nplan = 2; ol[1].plan[0] = ogv("MM.BBF"); ol[1].plan[1] = ogv("BSpMM.FBF");
  ol[1].w1 = W2.data(); ol[1].w1_rows = 16; ol[1].w1_cols = 5;
  ol[2].kind = 7;
  float *oo = nullptr, *olg = nullptr;
  int64_t oc = 0;
  CHECK(og_run_model(ol, 3, 32, &og, X.data(), n, 70, &oo, &olg, &oc, nullptr, nullptr) == 0);
  CHECK(oc == 5 && std::memcmp(out.data(), oo, out.payload_bytes()) == 0);
  CHECK(std::memcmp(trace.logits.data(), olg, trace.logits.payload_bytes()) == 0);
  CHECK(!trace.points.empty() && trace.points.front().bits.rows() == n);
  CHECK(!timings.empty());
  og_free(oo);
  og_free(olg);

  // resident model: repeated (graph-captured) forwards are identical
  b::Model model(m);
  b::DenseMatrix lg1, lg2;
  b::DenseMatrix o1 = model.forward(X, &lg1), o2 = model.forward(X, &lg2);
  CHECK(o1 == out && o2 == out && lg1 == trace.logits && lg2 == lg1);

  // single layers (ref: gcn_layer, graphops.cpp:270-285): the two layer calls
  // compose to the model's logits; the hooks see the model's BIN points
  {
    std::vector<std::string> labels;
    b::LayerHooks hooks;
    hooks.record_bits = [&](const std::string& l, const b::BitDenseMatrix&) { labels.push_back(l); };
    b::MatOperand h1 = b::gcn_layer(X, m.layers[0], *m.graph, std::nullopt, &hooks, "layer0.");
    b::MatOperand h2 = b::gcn_layer(h1, m.layers[1], *m.graph, std::nullopt, &hooks, "layer1.");
    CHECK(std::get<b::DenseMatrix>(h2) == trace.logits);
    CHECK(labels.size() == trace.points.size());
    for (size_t i = 0; i < labels.size() && i < trace.points.size(); ++i) CHECK(labels[i] == trace.points[i].label);
    b::LayerSpec bad = m.layers[0];
    bad.plan.pop_back();
    CHECK(throws<std::invalid_argument>([&] { b::gcn_layer(X, bad, *m.graph); },
                                        "gcn_conv: expected {mm, spmm} plan and weights"));
  }

  // tile sets (ref: test_bitsparse.cpp:131-161)
  {
    b::EdgeList row;
    row.node_count = 40;
    for (int c = 0; c < 10; ++c) row.edges.emplace_back(0, 4 * c);
    b::FrdcMatrix T = b::frdc_from_edges(row, false);
    CHECK(b::tileset_count(T, 0, 32) == 2 && b::tileset_count(T, 0, 64) == 1);
    b::TileSet s0 = b::gather_tileset(T, 0, 0, 32), s1 = b::gather_tileset(T, 0, 1, 32);
    CHECK(s0.ts == 8 && s0.rows[0] == 0x88888888u && s1.rows[0] == 0x88000000u && s1.cols[2] == b::TileSet::kPadCol);
    CHECK(b::gather_tileset(T, 0, 0, 64).rows[0] == 0x8888888888000000ull);
    CHECK(throws<std::invalid_argument>([&] { b::gather_tileset(T, 0, 2, 32); },
                                        "gather_tileset: set_index out of range"));
    b::BitDenseMatrix D = b::frdc_to_dense(T);
    CHECK(D.bit(0, 0) && D.bit(0, 36) && !D.bit(0, 1) && !D.bit(1, 0));
    b::FrdcStats st = b::frdc_stats(T);
    CHECK(st.nnz_tiles == 10 && st.nnz_bits == 10 && st.fill_ratio == 10.0 / 160.0);
  }

  // layer failures: std::runtime_error("layer i (kind): ...") (graphops.cpp:476-479)
  b::DenseMatrix Xbad = random_dense(&r, n, 69);
  CHECK(throws<std::runtime_error>([&] { b::run_model(m, Xbad); }, "layer 0 (gcn_conv): "));
  og_graph_free(&og);
  og_frdc_free(&oA);
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "--cpu";
  test_cpu();
  int ndev = 0;
  const bool have_gpu = bg_device_count(&ndev) == BG_OK && ndev > 0;
  if (mode == "--gpu") {
    if (!have_gpu) {
      std::fprintf(stderr, "no CUDA device\n");
      return 2;
    }
    test_gpu();
  } else if (!have_gpu) {
    test_no_device();
  }
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
