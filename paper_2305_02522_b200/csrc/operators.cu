// Operator dispatch with the reference's argument checks and messages
// (ref: kernels.cpp:95-191, :413-465, :573-668).
#include <cctype>

#include "engine.cuh"

namespace bg {

void* Pool::get(size_t bytes) {
  bytes = bytes ? (bytes + 255) / 256 * 256 : 256;
  if (next < bufs.size()) {
    if (bufs[next].bytes < bytes) {
      bufs[next].alloc(bytes);
      ++gen;
    }
    return bufs[next++].p;
  }
  bufs.emplace_back(bytes);
  ++gen;
  return bufs[next++].p;
}

Op op_from_mat(const bg_mat* m) {
  if (!m) fail("null operand");
  Op o;
  o.prec = m->precision;
  o.rows = m->rows;
  o.cols = m->cols;
  o.wb = m->word_bits ? m->word_bits : 32;
  o.sem = m->semantics;
  if (o.prec == BG_F) o.f = static_cast<float*>(m->data);
  else o.bits = static_cast<uint32_t*>(m->data);
  o.scale = m->scale;
  o.scale_axis = m->scale_axis;
  if (o.prec != BG_F && o.prec != BG_B) fail("operand precision must be F or B");
  if (o.prec == BG_B && o.wb != 32 && o.wb != 64)
    fail("BitDenseMatrix: word_bits must be 32 or 64");
  if (o.rows < 0 || o.cols < 0) fail("operand: negative dimension");
  return o;
}

void op_to_mat(const Op& o, bg_mat* m) {
  m->precision = o.prec;
  m->rows = o.rows;
  m->cols = o.cols;
  m->word_bits = o.wb;
  m->semantics = o.sem;
  m->scale_axis = o.scale_axis;
  m->data = o.prec == BG_F ? static_cast<void*>(o.f) : static_cast<void*>(o.bits);
  m->scale = const_cast<float*>(o.scale);
}

std::string variant_name(bg_variant v) {
  static const char* ops[] = {"BMM", "BSpMM", "ADD", "CONCAT"};
  auto c = [](int p) { return p == BG_F ? 'F' : 'B'; };
  std::string s = (v.op >= 0 && v.op < 4) ? ops[v.op] : "?";
  return s + "." + c(v.in1) + c(v.in2) + c(v.out);
}

// ref: KernelVariant::valid (kernels.cpp:81-91)
bool variant_valid(bg_variant v) {
  const bool all_f = v.in1 == BG_F && v.in2 == BG_F && v.out == BG_F;
  switch (v.op) {
    case BG_BMM: return !all_f;
    case BG_BSPMM: return true;
    case BG_ADD:
    case BG_CONCAT: return all_f || (v.in1 == BG_B && v.in2 == BG_B);
  }
  return false;
}

// ref: KernelVariant::parse (kernels.cpp:99-121)
bg_variant variant_parse(const std::string& text) {
  const size_t dot = text.find('.');
  if (dot == std::string::npos || text.size() - dot - 1 != 3)
    fail("KernelVariant: cannot parse '" + text + "'");
  std::string op = text.substr(0, dot);
  for (char& ch : op) ch = static_cast<char>(std::toupper(static_cast<unsigned char>(ch)));
  bg_variant v{};
  if (op == "BMM" || op == "MM") v.op = BG_BMM;
  else if (op == "BSPMM") v.op = BG_BSPMM;
  else if (op == "ADD") v.op = BG_ADD;
  else if (op == "CONCAT") v.op = BG_CONCAT;
  else fail("KernelVariant: unknown op '" + text + "'");
  int32_t* slots[3] = {&v.in1, &v.in2, &v.out};
  for (int i = 0; i < 3; ++i) {
    const char ch = text[dot + 1 + static_cast<size_t>(i)];
    if (ch == 'F' || ch == 'f') *slots[i] = BG_F;
    else if (ch == 'B' || ch == 'b') *slots[i] = BG_B;
    else fail("KernelVariant: bad precision letter in '" + text + "'");
  }
  return v;
}

const char* layer_kind_name(int k) {
  switch (k) {
    case BG_LAYER_GCN: return "gcn_conv";
    case BG_LAYER_SAGE: return "sage_conv";
    case BG_LAYER_GRAPHCONV: return "graph_conv";
    case BG_LAYER_FC: return "fc";
    case BG_LAYER_AGGREGATE: return "aggregate";
    case BG_LAYER_RELU: return "relu";
    case BG_LAYER_BATCHNORM: return "batchnorm";
    case BG_LAYER_SOFTMAX: return "softmax";
    case BG_LAYER_BINARIZE: return "binarize";
    case BG_LAYER_SCALE: return "scale";
  }
  return "?";
}

namespace {

// Resolution of one BMM side (ref: resolve_bmm_side, kernels.cpp:52-77).
void check_bmm_side(int tag, const Op& m, int axis, const char* which) {
  const std::string w = which;
  if (tag == BG_F) {
    if (m.prec != BG_F) fail("bmm: " + w + " is tagged F but operand is binary");
  } else {
    if (m.prec != BG_B) fail("bmm: " + w + " is tagged B but operand is full-precision");
    if (m.sem != BG_PLUS_MINUS) fail("bmm: " + w + " must carry PlusMinus bits");
    if (m.scale && m.scale_axis != axis) fail("bmm: " + w + " scale has the wrong axis");
  }
}

}  // namespace

Op bmm_out_desc(bg_variant v, const Op& a, const Op& w, int word_bits) {
  if (v.op != BG_BMM) fail("bmm: variant " + variant_name(v) + " is not a BMM variant");
  if (!variant_valid(v)) fail("bmm: " + variant_name(v) + " is not a supported variant");
  if (v.in1 == BG_B && a.prec == BG_B) word_bits = a.wb;
  if (v.in2 == BG_B && w.prec == BG_B) word_bits = w.wb;
  if (word_bits != 32 && word_bits != 64) fail("BitDenseMatrix: word_bits must be 32 or 64");
  check_bmm_side(v.in1, a, BG_AXIS_ROW, "in1");
  check_bmm_side(v.in2, w, BG_AXIS_COL, "in2");
  const int awb = v.in1 == BG_F ? word_bits : a.wb;
  const int wwb = v.in2 == BG_F ? word_bits : w.wb;
  if (a.cols != w.rows) fail("bmm: inner dimensions disagree");
  if (awb != wwb) fail("bmm: operand word widths disagree");
  Op o;
  o.prec = v.out;
  o.rows = a.rows;
  o.cols = w.cols;
  o.wb = awb;
  return o;
}

Op run_bmm(bg_variant v, const Op& a, const Op* w, const WeightCache* wc, int word_bits,
           Pool& pool, cudaStream_t s, const RowChunks* in_chunks) {
  // Only FBB-type products stream row chunks; every other variant reads the
  // whole activation (row scales included), so it waits for all chunks first.
  const bool stream_rows = in_chunks && in_chunks->n > 0 && v.in1 == BG_F && v.out == BG_B;
  if (in_chunks && !stream_rows)
    for (int c = 0; c < in_chunks->n; ++c) BG_CUDA(cudaStreamWaitEvent(s, in_chunks->ready[c], 0));
  Op wdesc;
  Op wtmp;
  if (wc && v.in2 == BG_F) {
    // A cached layout is only valid at the width it was packed with; an
    // activation that pins another width re-binarizes the fp32 weights the
    // way bmm does for F-tagged weights (kernels.cpp:144-149).
    int pinned = word_bits;
    if (v.in1 == BG_B && a.prec == BG_B) pinned = a.wb;
    if (pinned != wc->wb) {
      wtmp.prec = BG_F;
      wtmp.rows = wc->rows;
      wtmp.cols = wc->cols;
      wtmp.f = const_cast<float*>(wc->f);
      w = &wtmp;
      wc = nullptr;
    }
  }
  if (wc) {
    // Model path: weights were binarized once with their column scales
    // (run_mm_slot, graphops.cpp:64-70); both in2 tags resolve to these.
    wdesc.prec = v.in2;
    wdesc.rows = wc->rows;
    wdesc.cols = wc->cols;
    wdesc.wb = wc->wb;
    wdesc.scale = wc->scale;
    wdesc.scale_axis = BG_AXIS_COL;
    if (v.in2 == BG_F) wdesc.f = const_cast<float*>(wc->f);
  } else {
    wdesc = *w;
  }
  Op out = bmm_out_desc(v, a, wdesc, word_bits);
  const int wb = out.wb;

  // Weight side: transposed +-1 bits and column scales.
  const uint32_t* wt = nullptr;
  const float* beta = nullptr;
  if (wc) {
    wt = wc->wt;
    beta = wc->scale;
  } else if (v.in2 == BG_F) {
    auto* wbits = static_cast<uint32_t*>(pool.get(static_cast<size_t>(w->rows * spw(w->cols, wb)) * 4));
    auto* sc = static_cast<float*>(pool.get(static_cast<size_t>(w->cols) * 4));
    binarize(w->f, w->rows, w->cols, wb, wbits, s);
    l1_scales(w->f, w->rows, w->cols, BG_AXIS_COL, sc, s);
    auto* t = static_cast<uint32_t*>(pool.get(static_cast<size_t>(w->cols * spw(w->rows, wb)) * 4));
    transpose_bits(wbits, w->rows, w->cols, wb, t, s);
    wt = t;
    beta = sc;
  } else {
    auto* t = static_cast<uint32_t*>(pool.get(static_cast<size_t>(w->cols * spw(w->rows, wb)) * 4));
    transpose_bits(w->bits, w->rows, w->cols, wb, t, s);
    wt = t;
    beta = w->scale;
  }

  BmmArgs k;
  k.rows = a.rows;
  k.k = a.cols;
  k.n = out.cols;
  k.wb = wb;
  k.wt = wt;
  if (v.in1 == BG_F) {
    k.a_f = a.f;
    if (v.out == BG_F) {
      auto* al = static_cast<float*>(pool.get(static_cast<size_t>(a.rows) * 4));
      l1_scales(a.f, a.rows, a.cols, BG_AXIS_ROW, al, s);
      k.alpha = al;
    }
  } else {
    k.a_bits = a.bits;
    k.alpha = a.scale;
  }
  if (v.out == BG_B) {
    out.bits = static_cast<uint32_t*>(pool.get(out.bytes()));
    k.out_bits = out.bits;
  } else {
    out.f = static_cast<float*>(pool.get(out.bytes()));
    k.out_f = out.f;
    k.beta = beta;
  }
  if (stream_rows) {
    // streamed input: each chunk of rows as soon as its copy has landed
    const int64_t ospw = spw(out.cols, wb);
    for (int c = 0; c < in_chunks->n; ++c) {
      const int64_t r0 = in_chunks->bounds[c], r1 = in_chunks->bounds[c + 1];
      BG_CUDA(cudaStreamWaitEvent(s, in_chunks->ready[c], 0));
      if (r1 <= r0) continue;
      BmmArgs kc = k;
      kc.rows = r1 - r0;
      kc.a_f = a.f + r0 * a.cols;
      kc.out_bits = out.bits + r0 * ospw;
      bmm(kc, s);
    }
    return out;
  }
  bmm(k, s);
  return out;
}

Op bspmm_out_desc(bg_variant v, const bg_frdc* adj, const Op& x, int word_bits) {
  if (v.op != BG_BSPMM) fail("bspmm: variant " + variant_name(v) + " is not a BSpMM variant");
  if (!adj) fail("bspmm: missing adjacency structure");
  if (v.in1 == BG_B) {
    if (x.prec != BG_B) fail("bspmm: in1 tag B requires a binary operand");
    if (x.sem != BG_PLUS_MINUS) fail("bspmm: binary activations must be PlusMinus");
    if (x.scale) fail("bspmm: unexpected scale on the activation operand");
  } else if (x.prec != BG_F) {
    fail("bspmm: in1 tag F requires a full-precision operand");
  }
  if (x.rows != adj->cols) fail("bspmm: activation row count != adjacency node_cols");
  Op o;
  o.prec = v.out;
  o.rows = adj->rows;
  o.cols = x.cols;
  o.wb = v.in1 == BG_B ? x.wb : word_bits;
  if (o.prec == BG_B && o.wb != 32 && o.wb != 64) fail("BitDenseMatrix: word_bits must be 32 or 64");
  return o;
}

Op run_bspmm(bg_variant v, const bg_frdc* adj, const float* rs, const float* cs, const Op& x,
             int word_bits, Pool& pool, cudaStream_t s) {
  if (v.op != BG_BSPMM) fail("bspmm: variant " + variant_name(v) + " is not a BSpMM variant");
  if (!adj) fail("bspmm: missing adjacency structure");
  if (v.in2 == BG_F) {
    if (!rs || !cs)
      fail("bspmm: " + variant_name(v) + " needs a factorized adjacency (row and col scales)");
  } else if (rs || cs) {
    fail("bspmm: " + variant_name(v) + " takes the raw structure, not a factorized adjacency");
  }
  Op out = bspmm_out_desc(v, adj, x, word_bits);
  if (out.prec == BG_B) out.bits = static_cast<uint32_t*>(pool.get(out.bytes()));
  else out.f = static_cast<float*>(pool.get(out.bytes()));
  if (v.in1 == BG_B && v.in2 == BG_B) {
    bspmm_bb(*adj, x.bits, x.cols, x.wb, out.bits, out.f, s);
  } else {
    SpmmFArgs a;
    a.f = x.cols;
    if (v.in1 == BG_B) {
      a.x_bits = x.bits;
      a.xwb = x.wb;
    } else {
      a.x_f = x.f;
    }
    a.row_scale = v.in2 == BG_F ? rs : nullptr;
    a.col_scale = v.in2 == BG_F ? cs : nullptr;
    a.out_bits = out.bits;
    a.owb = out.wb;
    a.out_f = out.f;
    bspmm_f(*adj, a, s);
  }
  return out;
}

namespace {

void binary_pair(bg_variant v, const Op& a, const Op& b, const char* what) {
  const std::string w = what;
  if (a.prec != BG_B || b.prec != BG_B) fail(w + ": " + variant_name(v) + " requires binary operands");
  if (a.scale || b.scale) fail(w + ": unexpected scale on binary operand");
  if (a.sem != BG_PLUS_MINUS || b.sem != BG_PLUS_MINUS) fail(w + ": binary operands must be PlusMinus");
  if (a.wb != b.wb) fail(w + ": operand word widths disagree");
}

}  // namespace

Op run_add(bg_variant v, const Op& a, const Op& b, Pool& pool, cudaStream_t s, bool fuse_relu) {
  if (v.op != BG_ADD) fail("add: variant " + variant_name(v) + " is not an ADD variant");
  if (!variant_valid(v)) fail("add: " + variant_name(v) + " is not a supported variant");
  if (a.rows != b.rows || a.cols != b.cols) fail("add: operand shapes disagree");
  Op out;
  out.rows = a.rows;
  out.cols = a.cols;
  if (v.in1 == BG_F) {
    if (a.prec != BG_F || b.prec != BG_F) fail("add: FFF requires full-precision operands");
    out.prec = BG_F;
    out.f = static_cast<float*>(pool.get(out.bytes()));
    add_fff(a.f, b.f, a.rows * a.cols, out.f, s, fuse_relu);
    return out;
  }
  binary_pair(v, a, b, "add");
  out.wb = a.wb;
  if (v.out == BG_B) {
    out.prec = BG_B;
    out.bits = static_cast<uint32_t*>(pool.get(out.bytes()));
    add_bbb(a.bits, b.bits, a.rows * spw(a.cols, a.wb), out.bits, s);
  } else {
    out.prec = BG_F;
    out.f = static_cast<float*>(pool.get(out.bytes()));
    add_bbf(a.bits, b.bits, a.rows, a.cols, a.wb, out.f, s, fuse_relu);
  }
  return out;
}

Op run_add_relu_packed(bg_variant v, const Op& a, const Op& b, Pool& pool, cudaStream_t s) {
  if (v.op != BG_ADD) fail("add: variant " + variant_name(v) + " is not an ADD variant");
  if (!variant_valid(v)) fail("add: " + variant_name(v) + " is not a supported variant");
  if (a.rows != b.rows || a.cols != b.cols) fail("add: operand shapes disagree");
  if (v.in1 != BG_B || v.out != BG_F) fail("add: packed ReLU sum needs ADD.BBF");
  binary_pair(v, a, b, "add");
  Op out;
  out.prec = BG_F;
  out.rows = a.rows;
  out.cols = a.cols;
  out.wb = a.wb;
  out.pval = 2.0f;  // ReLU(2 (a + b) - 2) = 2 (a AND b)  (kernels.cpp:619-624)
  out.bits = static_cast<uint32_t*>(pool.get(out.bytes()));
  and_words(a.bits, b.bits, a.rows * spw(a.cols, a.wb), out.bits, s);
  return out;
}

Op materialize(const Op& x, Pool& pool, cudaStream_t s) {
  if (!x.packed()) return x;
  Op o;
  o.prec = BG_F;
  o.rows = x.rows;
  o.cols = x.cols;
  o.f = static_cast<float*>(pool.get(static_cast<size_t>(x.rows * x.cols) * 4));
  expand_packed(x.bits, x.rows, x.cols, x.wb, x.pval, o.f, s);
  return o;
}

Op run_concat(bg_variant v, const Op& a, const Op& b, Pool& pool, cudaStream_t s) {
  if (v.op != BG_CONCAT) fail("concat: variant " + variant_name(v) + " is not a CONCAT variant");
  if (!variant_valid(v)) fail("concat: " + variant_name(v) + " is not a supported variant");
  if (a.rows != b.rows) fail("concat: operand row counts disagree");
  Op out;
  out.rows = a.rows;
  out.cols = a.cols + b.cols;
  if (v.in1 == BG_F || v.out == BG_F) {
    if (v.in1 == BG_F && (a.prec != BG_F || b.prec != BG_F))
      fail("concat: FFF requires full-precision operands");
    const float *fa = a.f, *fb = b.f;
    if (v.in1 == BG_B) {
      binary_pair(v, a, b, "concat");
      auto* ua = static_cast<float*>(pool.get(static_cast<size_t>(a.rows * a.cols) * 4));
      auto* ub = static_cast<float*>(pool.get(static_cast<size_t>(b.rows * b.cols) * 4));
      unpack(a.bits, a.rows, a.cols, a.wb, a.sem, ua, s);
      unpack(b.bits, b.rows, b.cols, b.wb, b.sem, ub, s);
      fa = ua;
      fb = ub;
    }
    out.prec = BG_F;
    out.f = static_cast<float*>(pool.get(out.bytes()));
    concat_f(fa, a.cols, fb, b.cols, a.rows, out.f, s);
    return out;
  }
  binary_pair(v, a, b, "concat");
  out.prec = BG_B;
  out.wb = a.wb;
  out.bits = static_cast<uint32_t*>(pool.get(out.bytes()));
  concat_bits(a.bits, a.cols, b.bits, b.cols, a.rows, a.wb, out.bits, s);
  return out;
}

// The active fused epilogue (ops.cuh FEpi): per host thread, scoped by the
// executor around one aggregation.
namespace {
thread_local FEpi g_fepi;
}  // namespace
const FEpi& current_fepi() { return g_fepi; }
FEpiScope::FEpiScope(const FEpi& e) { g_fepi = e; }
FEpiScope::~FEpiScope() { g_fepi = FEpi{}; }

}  // namespace bg
