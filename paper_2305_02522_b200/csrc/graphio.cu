// Graph file readers (ref: graphio.hpp / graphio.cpp:72-176): whitespace
// "src dst [weight]" edge lists, MatrixMarket coordinate files, and the FRDC
// container decoded back to its edges, with load_graph's format sniffing.
//
// Host code: text parsing is byte work with no parallel structure worth a
// kernel, so the lines are scanned with a hand-rolled tokenizer (the
// reference uses one istringstream per line).  The accepted grammar, the
// edge order and every error message follow the reference: errors are
// runtime_error "name:line: message" (BG_RUNTIME_ERROR).  The FRDC branch
// reads the container straight to the device (container.cu) and decodes its
// tiles on the host in the reference's order.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

#include "ops.cuh"

struct bg_edges {
  int64_t node_count = 0;
  std::vector<int64_t> src, dst;
  std::vector<double> weights;  // may be shorter than the edge list (ref: EdgeList::weights)
};

namespace bg {
namespace {

[[noreturn]] void fail_at(const std::string& name, int64_t line, const std::string& msg) {
  throw std::runtime_error(name + ":" + std::to_string(line) + ": " + msg);
}

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

bool blank_or_comment(const char* b, const char* e) {
  while (b < e && (*b == ' ' || *b == '\t' || *b == '\r')) ++b;
  return b == e || *b == '#' || *b == '%';
}

// One line's tokens, with istream >> semantics for the types read here.
struct Cursor {
  const char* p;
  const char* e;
  void skip() {
    while (p < e && is_space(*p)) ++p;
  }
  // istream >> int64_t: optional sign, at least one digit, no overflow.
  bool int64(int64_t& v) {
    skip();
    const char* q = p;
    bool neg = false;
    if (q < e && (*q == '+' || *q == '-')) neg = *q++ == '-';
    if (q == e || *q < '0' || *q > '9') return false;
    uint64_t acc = 0;
    const uint64_t lim = neg ? uint64_t{1} << 63 : (uint64_t{1} << 63) - 1;
    for (; q < e && *q >= '0' && *q <= '9'; ++q) {
      const uint64_t d = static_cast<uint64_t>(*q - '0');
      if (acc > (lim - d) / 10) return false;
      acc = acc * 10 + d;
    }
    v = neg ? static_cast<int64_t>(0 - acc) : static_cast<int64_t>(acc);
    p = q;
    return true;
  }
  // istream >> double (libstdc++ num_get): the longest [sign] digits [.
  // digits] [e [sign] digits] prefix is consumed, then converted.  Returns 1
  // on success, 0 on failure with characters consumed, -1 on failure with
  // nothing consumed.  *eof: the extraction ran into the end of the line.
  int real(double& v, bool* eof) {
    skip();
    const char* q = p;
    if (q < e && (*q == '+' || *q == '-')) ++q;
    bool digits = false;
    while (q < e && *q >= '0' && *q <= '9') ++q, digits = true;
    if (q < e && *q == '.') {
      ++q;
      while (q < e && *q >= '0' && *q <= '9') ++q, digits = true;
    }
    if (digits && q < e && (*q == 'e' || *q == 'E')) {
      ++q;
      if (q < e && (*q == '+' || *q == '-')) ++q;
      while (q < e && *q >= '0' && *q <= '9') ++q;
    }
    *eof = q == e;
    if (q == p) return -1;
    const std::string tok(p, q);
    p = q;
    char* end = nullptr;
    errno = 0;
    const double d = std::strtod(tok.c_str(), &end);
    if (!digits || end != tok.c_str() + tok.size() || errno == ERANGE) return 0;
    v = d;
    return 1;
  }
  std::string word() {
    skip();
    const char* q = p;
    while (q < e && !is_space(*q)) ++q;
    std::string w(p, q);
    p = q;
    return w;
  }
};

// std::getline over a buffer: calls f(begin, end, line_number) per line.
template <class F>
void each_line(const char* text, size_t len, F&& f) {
  const char* p = text;
  const char* end = text + len;
  int64_t lineno = 0;
  while (p < end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    const char* le = nl ? nl : end;
    if (!f(p, le, ++lineno)) return;
    p = nl ? nl + 1 : end;
  }
}

void finish(bg_edges& e, const std::string& name, int64_t forced_nodes, bool undirected) {
  int64_t max_idx = -1;
  for (size_t k = 0; k < e.src.size(); ++k) max_idx = std::max({max_idx, e.src[k], e.dst[k]});
  if (forced_nodes >= 0) {
    if (max_idx >= forced_nodes)
      throw std::runtime_error(name + ": node index " + std::to_string(max_idx) + " does not fit the requested " +
                               std::to_string(forced_nodes) + " nodes");
    e.node_count = forced_nodes;
  } else {
    e.node_count = max_idx + 1;
  }
  if (undirected) {
    const size_t n = e.src.size();
    e.src.reserve(2 * n);
    e.dst.reserve(2 * n);
    for (size_t k = 0; k < n; ++k)
      if (e.src[k] != e.dst[k]) {
        e.src.push_back(e.dst[k]);
        e.dst.push_back(e.src[k]);
      }
  }
}

// ref: read_edge_list (graphio.cpp:72-99)
std::unique_ptr<bg_edges> edge_list(const char* text, size_t len, const std::string& name, int64_t forced,
                                    bool undirected) {
  auto e = std::make_unique<bg_edges>();
  each_line(text, len, [&](const char* b, const char* le, int64_t lineno) {
    if (blank_or_comment(b, le)) return true;
    Cursor c{b, le};
    int64_t s, d;
    if (!c.int64(s) || !c.int64(d)) fail_at(name, lineno, "expected \"src dst\", got \"" + std::string(b, le) + "\"");
    double w = 0;
    bool eof = false;
    const int r = c.real(w, &eof);
    if (r == 1) {  // optional weight column, kept but irrelevant to the 0/1 structure
      e->weights.resize(e->src.size(), 1.0);
      e->weights.push_back(w);
    } else if (!eof) {
      fail_at(name, lineno, "trailing token \"" + c.word() + "\"");
    }
    if (s < 0 || d < 0) fail_at(name, lineno, "negative node index");
    e->src.push_back(s);
    e->dst.push_back(d);
    return true;
  });
  finish(*e, name, forced, undirected);
  return e;
}

// ref: read_matrix_market (graphio.cpp:101-155)
std::unique_ptr<bg_edges> matrix_market(const char* text, size_t len, const std::string& name, bool undirected) {
  if (len == 0) fail_at(name, 1, "empty file");
  auto e = std::make_unique<bg_edges>();
  int64_t rows = 0, cols = 0, nnz = 0, seen = 0, last = 0;
  bool has_value = false, mirror = false;
  int stage = 0;  // 0 header, 1 size line, 2 entries
  each_line(text, len, [&](const char* b, const char* le, int64_t lineno) {
    last = lineno;
    if (stage == 0) {
      Cursor c{b, le};
      const std::string banner = c.word(), object = c.word(), format = c.word(), field = c.word(),
                        symmetry = c.word();
      if (banner != "%%MatrixMarket" || object != "matrix" || format != "coordinate")
        fail_at(name, 1, "expected a MatrixMarket coordinate header");
      if (field != "pattern" && field != "real" && field != "integer")
        fail_at(name, 1, "unsupported field \"" + field + "\"");
      if (symmetry != "general" && symmetry != "symmetric")
        fail_at(name, 1, "unsupported symmetry \"" + symmetry + "\"");
      has_value = field != "pattern";
      mirror = symmetry == "symmetric" || undirected;
      stage = 1;
      return true;
    }
    if (blank_or_comment(b, le)) return true;
    Cursor c{b, le};
    if (stage == 1) {
      if (!c.int64(rows) || !c.int64(cols) || !c.int64(nnz)) fail_at(name, lineno, "expected \"rows cols nnz\"");
      if (rows <= 0 || cols <= 0) fail_at(name, lineno, "missing size line");
      if (rows != cols)
        fail_at(name, lineno, "adjacency must be square, got " + std::to_string(rows) + "x" + std::to_string(cols));
      e->node_count = rows;
      if (nnz > 0) {
        e->src.reserve(static_cast<size_t>(std::min<int64_t>(nnz, int64_t{1} << 28)) * (mirror ? 2 : 1));
        e->dst.reserve(e->src.capacity());
      }
      stage = 2;
      return true;
    }
    int64_t i, j;
    if (!c.int64(i) || !c.int64(j)) fail_at(name, lineno, "expected \"row col\", got \"" + std::string(b, le) + "\"");
    double v;
    bool eof;
    if (has_value && c.real(v, &eof) != 1) fail_at(name, lineno, "missing value");
    if (i < 1 || i > rows || j < 1 || j > cols) fail_at(name, lineno, "index out of range");
    e->src.push_back(i - 1);
    e->dst.push_back(j - 1);
    if (mirror && i != j) {
      e->src.push_back(j - 1);
      e->dst.push_back(i - 1);
    }
    ++seen;
    return true;
  });
  if (stage < 2) fail_at(name, std::max<int64_t>(last, 1), "missing size line");
  if (seen != nnz)
    throw std::runtime_error(name + ": header promised " + std::to_string(nnz) + " entries, file holds " +
                             std::to_string(seen));
  return e;
}

// ref: read_frdc_edges (graphio.cpp:46-70): tiles in storage order, the set
// bits of a tile from bit 0 up (row-major position 15 down to 0).
std::unique_ptr<bg_edges> frdc_edges(const std::string& path, const std::string& bytes, int64_t forced,
                                     bool undirected) {
  int wb = 0;
  auto m = frdc_deserialize(bytes.data(), bytes.size(), &wb, nullptr);  // the bytes load_graph read
  const int64_t tr = (m->rows + 3) / 4;
  std::vector<uint64_t> rp(static_cast<size_t>(tr + 1));
  std::vector<uint32_t> ci(static_cast<size_t>(m->nnz));
  std::vector<uint16_t> ti(static_cast<size_t>(m->nnz));
  BG_CUDA(cudaMemcpy(rp.data(), m->rp(), rp.size() * 8, cudaMemcpyDeviceToHost));
  if (m->nnz) {
    BG_CUDA(cudaMemcpy(ci.data(), m->ci(), ci.size() * 4, cudaMemcpyDeviceToHost));
    BG_CUDA(cudaMemcpy(ti.data(), m->ti(), ti.size() * 2, cudaMemcpyDeviceToHost));
  }
  auto e = std::make_unique<bg_edges>();
  for (int64_t r = 0; r < tr; ++r)
    for (uint64_t t = rp[static_cast<size_t>(r)]; t < rp[static_cast<size_t>(r) + 1]; ++t) {
      const int64_t jb = 4 * static_cast<int64_t>(ci[t]);
      uint32_t tb = ti[t];
      while (tb) {
        const int rc = 15 - __builtin_ctz(tb);
        tb &= tb - 1;
        e->src.push_back(4 * r + (rc >> 2));
        e->dst.push_back(jb + (rc & 3));
      }
    }
  // the header is authoritative for the node count (trailing isolated nodes)
  if (forced < 0) forced = std::max(m->rows, m->cols);
  finish(*e, path, forced, undirected);
  return e;
}

void need(const void* p, const char* what) {
  if (!p) fail(std::string("null ") + what);
}

std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error(path + ": cannot open");
  return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

}  // namespace
}  // namespace bg

using namespace bg;

extern "C" {

int bg_read_edge_list(const char* text, size_t len, const char* name, int64_t forced_nodes, int undirected,
                      bg_edges** out) {
  return guard([&] {
    need(out, "output");
    if (!text && len) fail("read_edge_list: null text");
    *out = edge_list(text ? text : "", len, name ? name : "", forced_nodes, undirected != 0).release();
  });
}

int bg_read_matrix_market(const char* text, size_t len, const char* name, int undirected, bg_edges** out) {
  return guard([&] {
    need(out, "output");
    if (!text && len) fail("read_matrix_market: null text");
    *out = matrix_market(text ? text : "", len, name ? name : "", undirected != 0).release();
  });
}

// ref: load_graph (graphio.cpp:157-176)
int bg_load_graph(const char* path, int64_t forced_nodes, int undirected, bg_edges** out) {
  return guard([&] {
    need(out, "output");
    need(path, "path");
    const std::string p(path);
    std::string text = slurp(p);
    if (text.size() >= 4 && std::memcmp(text.data(), "FRDC", 4) == 0) {
      *out = frdc_edges(p, text, forced_nodes, undirected != 0).release();
      return;
    }
    if (text.rfind("%%MatrixMarket", 0) == 0) {
      *out = matrix_market(text.data(), text.size(), p, undirected != 0).release();
      return;
    }
    *out = edge_list(text.data(), text.size(), p, forced_nodes, undirected != 0).release();
  });
}

int bg_edges_info(const bg_edges* e, int64_t* node_count, int64_t* n_edges, const int64_t** src,
                  const int64_t** dst, const double** weights, int64_t* n_weights) {
  return guard([&] {
    need(e, "edges");
    if (node_count) *node_count = e->node_count;
    if (n_edges) *n_edges = static_cast<int64_t>(e->src.size());
    if (src) *src = e->src.data();
    if (dst) *dst = e->dst.data();
    if (weights) *weights = e->weights.data();
    if (n_weights) *n_weights = static_cast<int64_t>(e->weights.size());
  });
}

void bg_edges_destroy(bg_edges* e) { delete e; }

}  // extern "C"
