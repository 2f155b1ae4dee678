// Device-resident model and the layer-chain executor (ref: graphops.cpp:172-484).
//
// run_model's semantics are kept operation for operation (validation
// messages, trace labels and order, timing labels, exception wrapping); the
// difference is where the work happens: weights are uploaded and binarized
// once, every operator is a CUDA kernel on the caller's stream, and a forward
// with a fixed input binding is captured into one CUDA graph and replayed.
#include <algorithm>
#include <sstream>

#include "engine.cuh"
#include "model.cuh"

namespace bg {

// ---- validation (ref: graphops.cpp:103-268) ---------------------------------
namespace {

bool is_dense_fff(bg_variant v) {
  return v.op == BG_BMM && v.in1 == BG_F && v.in2 == BG_F && v.out == BG_F;
}

void check_slot(std::vector<std::string>* errors, const std::string& where, bg_variant v, int want) {
  if (v.op != want) {
    static const char* names[] = {"MM", "SpMM", "ADD", "CONCAT"};
    if (errors)
      errors->push_back(where + ": expected a " + names[want] + " variant, got " + variant_name(v));
    return;
  }
  if (!variant_valid(v) && !is_dense_fff(v))
    if (errors) errors->push_back(where + ": unsupported variant " + variant_name(v));
}

}  // namespace

int layer_output_precision(const LayerInfo& l, int in, std::vector<std::string>* errors) {
  auto err = [&](const std::string& m) {
    if (errors) errors->push_back(std::string(layer_kind_name(l.kind)) + ": " + m);
  };
  auto need_plan = [&](size_t n) {
    if (l.plan.size() != n) {
      err("expected " + std::to_string(n) + " plan slots, got " + std::to_string(l.plan.size()));
      return false;
    }
    return true;
  };
  const auto& p = l.plan;
  switch (l.kind) {
    case BG_LAYER_GCN: {
      if (!need_plan(2)) return in;
      check_slot(errors, "gcn_conv mm", p[0], BG_BMM);
      check_slot(errors, "gcn_conv spmm", p[1], BG_BSPMM);
      if (!l.has_w1) err("missing weights");
      if (p[0].in1 != in) err("mm input tag does not match incoming value");
      if (p[0].out != p[1].in1) err("mm output tag does not feed the spmm input");
      return p[1].out;
    }
    case BG_LAYER_SAGE:
    case BG_LAYER_GRAPHCONV: {
      if (!need_plan(4)) return in;
      check_slot(errors, "mm_self", p[0], BG_BMM);
      check_slot(errors, "mm_neigh", p[1], BG_BMM);
      check_slot(errors, "spmm", p[2], BG_BSPMM);
      check_slot(errors, "add", p[3], BG_ADD);
      if (!l.has_w1 || !l.has_w2) err("missing weights");
      if (p[0].in1 != in || p[1].in1 != in) err("mm input tags do not match incoming value");
      if (p[1].out != p[2].in1) err("mm_neigh output tag does not feed the spmm input");
      if (p[3].in1 != p[0].out) err("add input 1 tag does not match mm_self output");
      if (p[3].in2 != p[2].out) err("add input 2 tag does not match spmm output");
      return p[3].out;
    }
    case BG_LAYER_FC: {
      if (!need_plan(1)) return in;
      check_slot(errors, "fc mm", p[0], BG_BMM);
      if (!l.has_w1) err("missing weights");
      if (p[0].in1 != in) err("mm input tag does not match incoming value");
      return p[0].out;
    }
    case BG_LAYER_AGGREGATE: {
      if (!need_plan(1)) return in;
      check_slot(errors, "aggregate spmm", p[0], BG_BSPMM);
      if (p[0].in1 != in) err("spmm input tag does not match incoming value");
      return p[0].out;
    }
    case BG_LAYER_RELU:
      need_plan(0);
      return in;
    case BG_LAYER_BATCHNORM:
      need_plan(0);
      if (in != BG_F) err("expects a full-precision input");
      if (!l.has_bn) err("missing parameters");
      return BG_F;
    case BG_LAYER_SOFTMAX:
      need_plan(0);
      if (in != BG_F) err("expects a full-precision input");
      return BG_F;
    case BG_LAYER_BINARIZE:
      need_plan(0);
      if (in != BG_F) err("expects a full-precision input");
      return BG_B;
    case BG_LAYER_SCALE:
      need_plan(0);
      if (in != BG_F) err("expects a full-precision input");
      if (!l.has_scale) err("missing factors");
      return BG_F;
  }
  return in;
}

std::vector<std::string> validate_model(bool has_graph, int input_prec,
                                        const std::vector<LayerInfo>& layers) {
  std::vector<std::string> errors;
  if (!has_graph) {
    bool needs_graph = false;
    for (const auto& l : layers)
      if (l.kind == BG_LAYER_GCN || l.kind == BG_LAYER_SAGE || l.kind == BG_LAYER_GRAPHCONV ||
          l.kind == BG_LAYER_AGGREGATE)
        needs_graph = true;
    if (needs_graph) errors.push_back("model uses graph layers but carries no graph");
  }
  if (layers.empty()) errors.push_back("model has no layers");
  int cur = input_prec;
  for (size_t i = 0; i < layers.size(); ++i) {
    std::vector<std::string> local;
    cur = layer_output_precision(layers[i], cur, &local);
    for (auto& e : local) errors.push_back("layer " + std::to_string(i) + " " + e);
  }
  if (!layers.empty() && cur != BG_F)
    errors.push_back("model output must be full precision, got a binary tail");
  return errors;
}

LayerInfo layer_info(const bg_layer_desc& d) {
  LayerInfo l;
  l.kind = d.kind;
  for (int k = 0; k < d.n_plan && k < 4; ++k) l.plan.push_back(d.plan[k]);
  if (d.n_plan > 4) l.plan.resize(static_cast<size_t>(d.n_plan), bg_variant{});
  l.has_w1 = d.w1 != nullptr;
  l.has_w2 = d.w2 != nullptr;
  l.has_bn = d.bn_gamma && d.bn_beta && d.bn_mean && d.bn_sigma;
  l.has_scale = d.scale_row && d.scale_col;
  return l;
}

// ---- weights ------------------------------------------------------------------
void WeightDev::upload(const float* host, int64_t r, int64_t c, int wb_, cudaStream_t s) {
  rows = r;
  cols = c;
  wb = wb_;
  f.alloc(static_cast<size_t>(std::max<int64_t>(r * c, 1)) * 4);
  bits.alloc(static_cast<size_t>(std::max<int64_t>(r * spw(c, wb), 1)) * 4);
  scale.alloc(static_cast<size_t>(std::max<int64_t>(c, 1)) * 4);
  wt.alloc(static_cast<size_t>(std::max<int64_t>(c * spw(r, wb), 1)) * 4);
  if (r * c) BG_CUDA(cudaMemcpyAsync(f.p, host, static_cast<size_t>(r * c) * 4, cudaMemcpyHostToDevice, s));
  binarize(f.as<float>(), r, c, wb, bits.as<uint32_t>(), s);
  l1_scales(f.as<float>(), r, c, BG_AXIS_COL, scale.as<float>(), s);
  transpose_bits(bits.as<uint32_t>(), r, c, wb, wt.as<uint32_t>(), s);
}

WeightCache WeightDev::cache() const {
  WeightCache c;
  c.wbits = bits.as<uint32_t>();
  c.wt = wt.as<uint32_t>();
  c.scale = scale.as<float>();
  c.f = f.as<float>();
  c.rows = rows;
  c.cols = cols;
  c.wb = wb;
  return c;
}

// ---- executor -------------------------------------------------------------------
namespace {

struct Hooks {
  bg_trace* trace = nullptr;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>>* timing = nullptr;
  cudaStream_t s = nullptr;

  void bits(const std::string& label, const uint32_t* b, int64_t rows, int64_t cols, int wb) {
    if (!trace) return;
    TracePoint p;
    p.label = label;
    p.rows = rows;
    p.cols = cols;
    p.wb = wb;
    const size_t bytes = static_cast<size_t>(rows * spw(cols, wb)) * 4;
    p.bits.alloc(std::max<size_t>(bytes, 4));
    if (bytes) BG_CUDA(cudaMemcpyAsync(p.bits.p, b, bytes, cudaMemcpyDeviceToDevice, s));
    trace->pts.push_back(std::move(p));
  }
  void begin(const std::string& label) {
    if (!timing) return;
    cudaEvent_t a, b;
    BG_CUDA(cudaEventCreate(&a));
    BG_CUDA(cudaEventCreate(&b));
    BG_CUDA(cudaEventRecord(a, s));
    timing->push_back({label, {a, b}});
  }
  void end() {
    if (!timing) return;
    BG_CUDA(cudaEventRecord(timing->back().second.second, s));
  }
};

}  // namespace

// W1 | zero rows to a 32-column boundary | W2 as one transposed weight array
// (the paired product's layout, ops.cuh BmmArgs), built on first use.
const uint32_t* paired_weights(ModelLayer& l, int wb, cudaStream_t s) {
  const WeightDev &w1 = l.w1, &w2 = l.w2;
  const int64_t kspw = spw(w1.rows, wb), n = w1.cols, n1pad = 32 * cdiv(n, 32);
  if (!l.wt_pair.p) {
    const size_t bytes = static_cast<size_t>((n1pad + n) * kspw) * 4;
    l.wt_pair.alloc(bytes);
    BG_CUDA(cudaMemsetAsync(l.wt_pair.p, 0, bytes, s));
    BG_CUDA(cudaMemcpyAsync(l.wt_pair.p, w1.wt.p, static_cast<size_t>(n * kspw) * 4, cudaMemcpyDeviceToDevice, s));
    BG_CUDA(cudaMemcpyAsync(l.wt_pair.as<uint32_t>() + n1pad * kspw, w2.wt.p, static_cast<size_t>(n * kspw) * 4,
                            cudaMemcpyDeviceToDevice, s));
  }
  return l.wt_pair.as<uint32_t>();
}

namespace {

struct Exec {
  bg_model& m;
  Hooks& h;
  cudaStream_t s;
  const float* x0f = nullptr;           // the model input (fp32), when streamed in
  const RowChunks* in_chunks = nullptr;  // its row chunks (host entry point)

  // ref: run_mm_slot (graphops.cpp:47-77)
  // every chunk of a streamed input has landed (before any op that is not a
  // chunk-aware MM reads it)
  void wait_all_in() {
    if (!in_chunks) return;
    for (int c = 0; c < in_chunks->n; ++c) BG_CUDA(cudaStreamWaitEvent(s, in_chunks->ready[c], 0));
  }

  Op mm_slot(bg_variant mm, const Op& x, const WeightDev& w, const std::string& label) {
    if (mm.op != BG_BMM) fail(label + ": plan slot expects an MM variant");
    if (x.packed()) {
      if (is_dense_fff(mm) || (mm.out == BG_F && !packed_fbf_supported(w.cols)) || w.wb != m.wb ||
          spw(w.cols, m.wb) > 64)
        return mm_slot(mm, materialize(x, m.pool, s), w, label);
      return mm_packed(mm, x, w, label, nullptr);
    }
    if (in_chunks && x.f == x0f && (is_dense_fff(mm) || h.trace)) wait_all_in();
    if (is_dense_fff(mm)) {
      if (x.prec != BG_F) fail(label + ": MM.FFF expects a full-precision input");
      if (x.cols != w.rows) fail("dense_mm: inner dimensions disagree");
      Op o;
      o.prec = BG_F;
      o.rows = x.rows;
      o.cols = w.cols;
      o.f = static_cast<float*>(m.pool.get(o.bytes()));
      h.begin(label + "[MM.FFF]");
      dense_mm(x.f, w.f.as<float>(), x.rows, x.cols, w.cols, o.f, s);
      h.end();
      return o;
    }
    if (h.trace) {
      if (mm.in1 == BG_F && x.prec == BG_F) {
        auto* b = static_cast<uint32_t*>(m.pool.get(static_cast<size_t>(x.rows * spw(x.cols, m.wb)) * 4));
        binarize(x.f, x.rows, x.cols, m.wb, b, s);
        h.bits(label + ".bin_in", b, x.rows, x.cols, m.wb);
      }
      h.bits(label + ".bin_w", w.bits.as<uint32_t>(), w.rows, w.cols, w.wb);
    }
    const WeightCache wc = w.cache();
    h.begin(label + "[" + variant_name(mm) + "]");
    const RowChunks* streamed = (in_chunks && x.prec == BG_F && x.f == x0f) ? in_chunks : nullptr;
    Op r = run_bmm(mm, x, nullptr, &wc, m.wb, m.pool, s, streamed);
    h.end();
    if (mm.out == BG_B) h.bits(label + ".out", r.bits, r.rows, r.cols, r.wb);
    return r;
  }

  // An F-input product on a packed two-valued input (packed.cu): the
  // binarized input is all ones, so B outputs are one constant row and
  // MM.FBF needs one popcount per row; probs: the following softmax fused.
  Op mm_packed(bg_variant mm, const Op& x, const WeightDev& w, const std::string& label, float* probs,
               const RowChunks* out_chunks = nullptr, bool keep_logits = true) {
    if (mm.in1 != BG_F) fail("bmm: in1 is tagged F but operand is binary");
    if (!variant_valid(mm)) fail("bmm: " + variant_name(mm) + " is not a supported variant");
    if (x.cols != w.rows) fail("bmm: inner dimensions disagree");
    if (h.trace) {
      const Op xf = materialize(x, m.pool, s);
      auto* b = static_cast<uint32_t*>(m.pool.get(static_cast<size_t>(x.rows * spw(x.cols, m.wb)) * 4));
      binarize(xf.f, x.rows, x.cols, m.wb, b, s);
      h.bits(label + ".bin_in", b, x.rows, x.cols, m.wb);
      h.bits(label + ".bin_w", w.bits.as<uint32_t>(), w.rows, w.cols, w.wb);
    }
    Op r;
    r.rows = x.rows;
    r.cols = w.cols;
    r.wb = m.wb;
    h.begin(label + "[" + variant_name(mm) + "]");
    if (mm.out == BG_B) {
      r.prec = BG_B;
      r.bits = static_cast<uint32_t*>(m.pool.get(r.bytes()));
      packed_const_rows(w.wt.as<uint32_t>(), w.rows, w.cols, m.wb, x.rows, r.bits, s);
    } else {
      r.prec = BG_F;
      r.f = static_cast<float*>(m.pool.get(r.bytes()));
      auto* tab = static_cast<float*>(m.pool.get(packed_fbf_table_bytes(x.cols, w.cols)));
      if (out_chunks) {
        for (int c = 0; c < out_chunks->n; ++c) {
          packed_fbf(x.bits, out_chunks->bounds[c], out_chunks->bounds[c + 1], x.cols, x.wb, x.pval,
                     w.wt.as<uint32_t>(), m.wb, w.scale.as<float>(), w.cols, keep_logits ? r.f : nullptr, probs, tab, s);
          BG_CUDA(cudaEventRecord(out_chunks->ready[c], s));
        }
      } else {
        packed_fbf(x.bits, 0, x.rows, x.cols, x.wb, x.pval, w.wt.as<uint32_t>(), m.wb, w.scale.as<float>(),
                   w.cols, keep_logits ? r.f : nullptr, probs, tab, s);
      }
    }
    h.end();
    if (mm.out == BG_B) h.bits(label + ".out", r.bits, r.rows, r.cols, r.wb);
    return r;
  }

  // The two MMs of a SAGE / GraphConv layer when both are F -> B on the same
  // fp32 input (MM.FBB / MM.FFB): one paired product reads the input once
  // (bmm_pair).  Untraced forwards only (the traced one keeps the per-slot
  // BIN points); false when the shapes do not pair.
  bool mm_pair(ModelLayer& l, const Op& x, const std::string& prefix, Op& hs, Op& hn) {
    const bg_variant p0 = l.info.plan[0], p1 = l.info.plan[1];
    auto fb = [](bg_variant v) { return v.op == BG_BMM && v.in1 == BG_F && v.out == BG_B; };
    if (h.trace || !fb(p0) || !fb(p1) || x.prec != BG_F || x.scale || x.packed()) return false;
    const WeightDev &w1 = l.w1, &w2 = l.w2;
    if (w1.rows != w2.rows || w1.cols != w2.cols || w1.wb != m.wb || w2.wb != m.wb || x.cols != w1.rows)
      return false;
    const int64_t n = w1.cols;
    const uint32_t* wtp = paired_weights(l, m.wb, s);
    Op a, b;
    a.prec = b.prec = BG_B;
    a.rows = b.rows = x.rows;
    a.cols = b.cols = n;
    a.wb = b.wb = m.wb;
    a.bits = static_cast<uint32_t*>(m.pool.get(a.bytes()));
    b.bits = static_cast<uint32_t*>(m.pool.get(b.bytes()));
    BmmArgs k;
    k.k = x.cols;
    k.n = n;
    k.n2 = n;
    k.wb = m.wb;
    k.wt = wtp;
    const int64_t ospw = spw(n, m.wb);
    h.begin(prefix + "mm_pair[" + variant_name(p0) + "]");
    const bool streamed = in_chunks && x.f == x0f;
    const int nc = streamed ? in_chunks->n : 1;
    bool ok = true;
    for (int c = 0; c < nc && ok; ++c) {
      const int64_t r0 = streamed ? in_chunks->bounds[c] : 0, r1 = streamed ? in_chunks->bounds[c + 1] : x.rows;
      if (streamed) BG_CUDA(cudaStreamWaitEvent(s, in_chunks->ready[c], 0));
      k.rows = r1 - r0;
      k.a_f = x.f + r0 * x.cols;
      k.out_bits = a.bits + r0 * ospw;
      k.out_bits2 = b.bits + r0 * ospw;
      const bool paired = bmm_pair(k, s);
      if (!paired && c == 0) {
        ok = false;
      } else if (!paired) {  // a later chunk the pair kernels do not take: one product at a time
        BmmArgs one = k;
        one.out_bits2 = nullptr;
        one.n2 = 0;
        one.wt = w1.wt.as<uint32_t>();
        bmm(one, s);
        one.wt = w2.wt.as<uint32_t>();
        one.out_bits = k.out_bits2;
        bmm(one, s);
      }
    }
    h.end();
    if (!ok) {
      if (h.timing) {  // drop the empty span
        cudaEventDestroy(h.timing->back().second.first);
        cudaEventDestroy(h.timing->back().second.second);
        h.timing->pop_back();
      }
      return false;
    }
    hs = a;
    hn = b;
    return true;
  }

  Op spmm_slot(bg_variant sp, const bg_frdc* adj, const float* rs, const float* cs, const Op& x,
               const std::string& label) {
    h.begin(label + "[" + variant_name(sp) + "]");
    Op r = run_bspmm(sp, adj, rs, cs, x, m.wb, m.pool, s);
    h.end();
    if (sp.out == BG_B) h.bits(label + ".out", r.bits, r.rows, r.cols, r.wb);
    return r;
  }

  Op own_f(const Op& x) {  // fresh copy for in-place ops on caller memory
    Op o = x;
    o.f = static_cast<float*>(m.pool.get(x.bytes()));
    BG_CUDA(cudaMemcpyAsync(o.f, x.f, x.bytes(), cudaMemcpyDeviceToDevice, s));
    return o;
  }

  // Fused epilogue (ops.cuh FEpi): layers bn, bn+1, .. that are BatchNorm
  // [ReLU] [Binarize] fold into the stores of the F result before them.
  // Returns how many layers it covers (0: none).
  size_t plan_epi(size_t bn, int64_t cols, FEpi& e, size_t& bin_layer) {
    static const bool on = [] {
      const char* v = std::getenv("BG_FUSE_EPI");
      return !(v && std::atoi(v) == 0);
    }();
    const size_t nl = m.layers.size();
    if (!on || bn >= nl || m.layers[bn].info.kind != BG_LAYER_BATCHNORM) return 0;
    const size_t i = bn - 1;  // the producer's layer (wraps for bn == 0; only i + k is used)
    const ModelLayer& bnl = m.layers[bn];
    if (bnl.bn_len != cols) return 0;  // the unfused path reports the mismatch
    e = FEpi{};
    e.g = bnl.bn_g.as<float>();
    e.b = bnl.bn_b.as<float>();
    e.m = bnl.bn_m.as<float>();
    e.s = bnl.bn_s.as<float>();
    size_t n = 1;
    if (i + n + 1 < nl && m.layers[i + n + 1].info.kind == BG_LAYER_RELU) {
      e.relu = 1;
      ++n;
    }
    if (i + n + 1 < nl && m.layers[i + n + 1].info.kind == BG_LAYER_BINARIZE) {
      bin_layer = i + n + 1;
      ++n;
    }
    return n;
  }

  // The packed output of a fused binarize (zeroed when 64-bit words pad a column).
  Op bits_out(int64_t rows, int64_t cols, FEpi& e) {
    Op o;
    o.prec = BG_B;
    o.rows = rows;
    o.cols = cols;
    o.wb = m.wb;
    o.bits = static_cast<uint32_t*>(m.pool.get(o.bytes()));
    e.bits = o.bits;
    e.bspw = spw(cols, m.wb);
    if (e.bspw * 32 - cols >= 32) BG_CUDA(cudaMemsetAsync(o.bits, 0, o.bytes(), s));
    return o;
  }

  // An F aggregation with its BatchNorm [ReLU] [Binarize] epilogue; advances i
  // past the fused layers.
  bool spmm_epi(size_t& i, bg_variant sp, const bg_frdc* adj, const float* rs, const float* cs, const Op& x,
                const std::string& label, Op& cur) {
    if (sp.out != BG_F) return false;
    FEpi e;
    size_t bin_layer = 0;
    const size_t n = plan_epi(i + 1, x.cols, e, bin_layer);
    if (n == 0) return false;
    Op bits;
    if (bin_layer) bits = bits_out(adj->rows, x.cols, e);
    {
      FEpiScope scope(e);
      cur = spmm_slot(sp, adj, rs, cs, x, label);
    }
    if (bin_layer) {
      cur = bits;
      h.bits("layer" + std::to_string(bin_layer) + ".bin.out", cur.bits, cur.rows, cur.cols, cur.wb);
    }
    i += n;
    return true;
  }

  void relu_inplace(Op& x, const Op& x0) {
    if (x.prec != BG_F || x.packed()) return;  // ref: graphops.cpp:89-97; packed values are >= 0
    if (x.f == x0.f) x = own_f(x);
    relu(x.f, x.rows * x.cols, s);
  }
};

}  // namespace

void forward_impl(bg_model& m, const Op& x0, float* out, float* logits, bg_trace* trace,
                  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>>* timing,
                  cudaStream_t s, StreamChunks* chunks, LayerCall* single) {
  if (!single) {
    std::vector<std::string> errors = validate_model(m.graph != nullptr, m.input_prec, m.infos);
    if (!errors.empty()) {
      std::ostringstream os;
      os << "invalid model:";
      for (const auto& e : errors) os << "\n  " << e;
      fail(os.str());
    }
    if (x0.prec != m.input_prec) fail("model input tag does not match the provided operand");
  }
  m.pool.reset();
  if (!trace && !timing && !chunks && !single && persistent_forward(m, x0, out, logits, s)) {
    m.last_out_cols = m.layers[m.layers.size() - 2].w1.cols;
    return;
  }
  Hooks h;
  h.trace = trace;
  h.timing = timing;
  h.s = s;
  Exec ex{m, h, s};
  if (chunks && chunks->in.n > 0 && x0.prec == BG_F) {
    ex.x0f = x0.f;
    ex.in_chunks = &chunks->in;
  }
  if (ex.in_chunks && !m.layers.empty()) {
    const int k0 = m.layers[0].info.kind;  // only MM slots stream; anything else reads all of x0
    if (k0 != BG_LAYER_GCN && k0 != BG_LAYER_SAGE && k0 != BG_LAYER_GRAPHCONV && k0 != BG_LAYER_FC) ex.wait_all_in();
  }
  // final output produced per row chunk (so its copy-out overlaps the rest)
  auto chunked_out = [&](size_t layer_after) {
    return chunks && chunks->out.n > 0 && layer_after == m.layers.size();
  };
  Op cur = x0;
  bool logits_set = false;
  float* fused_probs = nullptr;   // softmax already produced by a fused epilogue
  const float* fused_logits = nullptr;
  const size_t nl = m.layers.size();
  for (size_t i = 0; i < nl; ++i) {
    ModelLayer& l = m.layers[i];
    const std::string prefix = single ? single->prefix : "layer" + std::to_string(i) + ".";
    try {
      switch (l.info.kind) {
        case BG_LAYER_GCN: {  // ref: gcn_layer, graphops.cpp:270-285
          const bg_variant mm = l.info.plan[0], sp = l.info.plan[1];
          const bool bbf_fbf = mm.op == BG_BMM && mm.in1 == BG_B && mm.in2 == BG_B &&
                               mm.out == BG_F && sp.op == BG_BSPMM && sp.in1 == BG_F &&
                               sp.in2 == BG_B && sp.out == BG_F;
          if (bbf_fbf && !l.relu && cur.prec == BG_B && cur.sem == BG_PLUS_MINUS && !cur.scale &&
              cur.wb == m.wb && cur.cols == l.w1.rows && cur.rows == m.graph->structure->cols &&
              gcn1_fused_supported(*m.graph->structure, cur.cols, cur.wb, l.w1.cols)) {
            // Fused MM.BBF + BSpMM.FBF (+ the following Softmax): bit-identical
            // logits without materializing the N x C intermediate (gcn_fused.cu).
            if (h.trace) h.bits(prefix + "mm.bin_w", l.w1.bits.as<uint32_t>(), l.w1.rows, l.w1.cols, l.w1.wb);
            const bg_frdc& A = *m.graph->structure;
            auto* recs = static_cast<uint32_t*>(m.pool.get(static_cast<size_t>(A.cols + 1) * 64));  // + zero record
            h.begin(prefix + "mm[" + variant_name(mm) + "]");
            gcn1_records(cur.bits, A.cols, cur.cols, cur.wb, l.w1.wt.as<uint32_t>(),
                         l.w1.scale.as<float>(), l.w1.cols, recs, s);
            h.end();
            Op o;
            o.prec = BG_F;
            o.rows = A.rows;
            o.cols = l.w1.cols;
            o.f = static_cast<float*>(m.pool.get(o.bytes()));
            float* probs = nullptr;
            if (i + 1 < nl && m.layers[i + 1].info.kind == BG_LAYER_SOFTMAX) {
              probs = (i + 2 == nl && out) ? out : static_cast<float*>(m.pool.get(o.bytes()));
              fused_probs = probs;
              fused_logits = o.f;
            }
            // the logits are only written when something reads them (a fused
            // softmax that is the model's output, no caller logits, no trace)
            const bool keep_lg = !probs || logits || h.trace || h.timing || single || i + 2 != nl;
            h.begin(prefix + "spmm[" + variant_name(sp) + "]");
            if (probs == out && out && chunked_out(i + 2)) {
              for (int c = 0; c < chunks->out.n; ++c) {
                const int64_t r0 = chunks->out.bounds[c], r1 = chunks->out.bounds[c + 1];
                if (r1 > r0)
                  gcn1_aggregate(A, recs, cur.cols, cur.wb, l.w1.wt.as<uint32_t>(), l.w1.scale.as<float>(),
                                 l.w1.cols, keep_lg ? o.f : nullptr, probs, s, r0, r1);
                BG_CUDA(cudaEventRecord(chunks->out.ready[c], s));
              }
              chunks->out_done = true;
            } else {
              gcn1_aggregate(A, recs, cur.cols, cur.wb, l.w1.wt.as<uint32_t>(), l.w1.scale.as<float>(),
                             l.w1.cols, keep_lg ? o.f : nullptr, probs, s);
            }
            h.end();
            cur = o;
            break;
          }
          Op hh = ex.mm_slot(l.info.plan[0], cur, l.w1, prefix + "mm");
          const bool fac = sp.in2 == BG_F;
          const float* sc = fac ? m.graph->norm.as<float>() : nullptr;
          if (!single && !l.relu && ex.spmm_epi(i, sp, m.graph->structure.get(), sc, sc, hh, prefix + "spmm", cur))
            break;
          cur = ex.spmm_slot(sp, m.graph->structure.get(), sc, sc, hh, prefix + "spmm");
          if (l.relu) ex.relu_inplace(cur, x0);
          break;
        }
        case BG_LAYER_SAGE:
        case BG_LAYER_GRAPHCONV: {  // ref: neighborhood_layer, graphops.cpp:289-321
          const bool mean = l.info.kind == BG_LAYER_SAGE;
          Op hs, hn;
          if (!ex.mm_pair(l, cur, prefix, hs, hn)) {
            hs = ex.mm_slot(l.info.plan[0], cur, l.w1, prefix + "mm_self");
            hn = ex.mm_slot(l.info.plan[1], cur, l.w2, prefix + "mm_neigh");
          }
          const bg_variant sp = l.info.plan[2];
          const bool fac = sp.in2 == BG_F;
          const float* rs = fac ? (mean ? m.graph->mean_row.as<float>() : m.graph->ones.as<float>()) : nullptr;
          const float* cs = fac ? m.graph->ones.as<float>() : nullptr;
          Op agg = ex.spmm_slot(sp, m.graph->raw.get(), rs, cs, hn, prefix + "spmm");
          if (mean && sp.in2 == BG_B && sp.out == BG_F)
            scale_rows_double(agg.f, agg.rows, agg.cols, m.graph->neighbor_count.as<int64_t>(), s);
          // the layer's ReLU rides in the ADD kernel when the sum is F (on a B
          // sum it is a no-op, graphops.cpp:89-97)
          const bg_variant av = l.info.plan[3];
          if (av.op == BG_ADD && av.in1 == BG_B && av.out == BG_F && l.relu && hs.prec == BG_B && agg.prec == BG_B) {
            // ReLU(ADD.BBF) = 2 (a AND b): kept packed (packed.cu), 1/32 of the fp32 bytes
            cur = run_add_relu_packed(av, hs, agg, m.pool, s);
            break;
          }
          cur = run_add(av, hs, agg, m.pool, s, l.relu && av.out == BG_F);
          if (l.info.plan[3].out == BG_B) h.bits(prefix + "add.out", cur.bits, cur.rows, cur.cols, cur.wb);
          break;
        }
        case BG_LAYER_FC: {
          const bg_variant mm = l.info.plan[0];
          if (cur.packed() && mm.op == BG_BMM && mm.in1 == BG_F && mm.in2 == BG_B && mm.out == BG_F && !l.relu &&
              i + 1 < nl && m.layers[i + 1].info.kind == BG_LAYER_SOFTMAX && packed_fbf_supported(l.w1.cols) &&
              cur.cols == l.w1.rows && l.w1.wb == m.wb) {
            // MM.FBF on the packed input with the following softmax in the
            // same pass: logits and probabilities from one popcount per row
            float* probs = (i + 2 == nl && out) ? out : static_cast<float*>(m.pool.get(
                static_cast<size_t>(cur.rows * l.w1.cols) * 4));
            const bool chunked = probs == out && out && chunked_out(i + 2);
            // the logits are only written when something reads them
            const bool keep = logits || h.trace || h.timing || single || i + 2 != nl;
            Op o = ex.mm_packed(mm, cur, l.w1, prefix + "mm", probs, chunked ? &chunks->out : nullptr, keep);
            if (chunked) chunks->out_done = true;
            fused_probs = probs;
            fused_logits = o.f;
            cur = o;
            break;
          }
          cur = ex.mm_slot(l.info.plan[0], cur, l.w1, prefix + "mm");
          if (l.relu) ex.relu_inplace(cur, x0);
          break;
        }
        case BG_LAYER_AGGREGATE: {
          cur = materialize(cur, m.pool, s);
          const bg_variant sp = l.info.plan[0];
          const bool fac = sp.in2 == BG_F;
          const float* sc = fac ? m.graph->norm.as<float>() : nullptr;
          if (!single && ex.spmm_epi(i, sp, m.graph->structure.get(), sc, sc, cur, prefix + "spmm", cur)) break;
          cur = ex.spmm_slot(sp, m.graph->structure.get(), sc, sc, cur, prefix + "spmm");
          break;
        }
        case BG_LAYER_RELU:
          ex.relu_inplace(cur, x0);
          break;
        case BG_LAYER_BATCHNORM: {
          if (cur.prec != BG_F) fail("bad variant access");
          cur = materialize(cur, m.pool, s);
          if (l.bn_len != cur.cols)
            fail("batchnorm: parameter lengths do not match " + std::to_string(cur.cols) + " columns");
          FEpi e;
          size_t bin_layer = 0;
          // BatchNorm [ReLU] [Binarize] of an F producer without its own
          // epilogue: one pass (plan_epi looks from the layer before)
          const size_t n = single ? 0 : ex.plan_epi(i, cur.cols, e, bin_layer);
          if (n > 0) {
            Op o = cur;
            if (bin_layer) {
              o = ex.bits_out(cur.rows, cur.cols, e);
            } else {
              o.f = static_cast<float*>(m.pool.get(cur.bytes()));
            }
            bn_act(cur.f, cur.rows, cur.cols, e, o.f, s);
            if (bin_layer) h.bits("layer" + std::to_string(bin_layer) + ".bin.out", o.bits, o.rows, o.cols, o.wb);
            cur = o;
            i += n - 1;
            break;
          }
          Op o = cur;
          o.f = static_cast<float*>(m.pool.get(cur.bytes()));
          batchnorm(cur.f, cur.rows, cur.cols, l.bn_g.as<float>(), l.bn_b.as<float>(),
                    l.bn_m.as<float>(), l.bn_s.as<float>(), o.f, s);
          cur = o;
          break;
        }
        case BG_LAYER_SOFTMAX: {
          if (cur.prec != BG_F) fail("bad variant access");
          cur = materialize(cur, m.pool, s);
          if (logits) {
            BG_CUDA(cudaMemcpyAsync(logits, cur.f, cur.bytes(), cudaMemcpyDeviceToDevice, s));
            logits_set = true;
          }
          Op o = cur;
          if (fused_probs && cur.f == fused_logits) {
            o.f = fused_probs;  // computed in the fused aggregation epilogue
            h.begin(prefix + "softmax");
            h.end();
          } else {
            o.f = (i + 1 == nl && out) ? out : static_cast<float*>(m.pool.get(cur.bytes()));
            h.begin(prefix + "softmax");
            if (o.f == out && chunked_out(i + 1)) {
              for (int c = 0; c < chunks->out.n; ++c) {
                const int64_t r0 = chunks->out.bounds[c], r1 = chunks->out.bounds[c + 1];
                if (r1 > r0) softmax_rows(cur.f + r0 * cur.cols, r1 - r0, cur.cols, o.f + r0 * cur.cols, s);
                BG_CUDA(cudaEventRecord(chunks->out.ready[c], s));
              }
              chunks->out_done = true;
            } else {
              softmax_rows(cur.f, cur.rows, cur.cols, o.f, s);
            }
            h.end();
          }
          cur = o;
          break;
        }
        case BG_LAYER_BINARIZE: {
          if (cur.prec != BG_F) fail("bad variant access");
          cur = materialize(cur, m.pool, s);
          Op o;
          o.prec = BG_B;
          o.rows = cur.rows;
          o.cols = cur.cols;
          o.wb = m.wb;
          o.bits = static_cast<uint32_t*>(m.pool.get(o.bytes()));
          binarize(cur.f, cur.rows, cur.cols, m.wb, o.bits, s);
          h.bits(prefix + "bin.out", o.bits, o.rows, o.cols, o.wb);
          cur = o;
          break;
        }
        case BG_LAYER_SCALE: {
          if (cur.prec != BG_F) fail("bad variant access");
          cur = materialize(cur, m.pool, s);
          if (l.sr_len != cur.rows || l.sc_len != cur.cols) fail("scl: scale length mismatch");
          Op o = cur;
          o.f = static_cast<float*>(m.pool.get(cur.bytes()));
          scl(cur.f, cur.rows, cur.cols, l.sr.as<float>(), l.sc.as<float>(), o.f, s);
          cur = o;
          break;
        }
        default:
          fail("unknown layer kind");
      }
    } catch (const cuda_error&) {
      throw;
    } catch (const std::exception& e) {
      if (single) throw;  // a layer function reports its own errors unwrapped
      throw std::runtime_error("layer " + std::to_string(i) + " (" + layer_kind_name(l.info.kind) +
                               "): " + e.what());
    }
  }
  cur = materialize(cur, m.pool, s);  // a packed two-valued result leaves as fp32
  if (single) {
    single->result = cur;
    return;
  }
  if (cur.prec != BG_F) fail("model output must be full precision");
  if (out && cur.f != out)
    BG_CUDA(cudaMemcpyAsync(out, cur.f, cur.bytes(), cudaMemcpyDeviceToDevice, s));
  if (logits && !logits_set)
    BG_CUDA(cudaMemcpyAsync(logits, cur.f, cur.bytes(), cudaMemcpyDeviceToDevice, s));
  m.last_out_cols = cur.cols;
}

}  // namespace bg
