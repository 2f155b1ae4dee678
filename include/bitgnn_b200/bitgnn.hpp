// bitgnn_b200/bitgnn.hpp -- header-only C++ host API over the C ABI
// (include/bitgnn_b200.h), mirroring the reference operator API of
// /root/reference/proj/include/bitgnn (kernels.hpp, graphops.hpp,
// bitdense.hpp, bitsparse.hpp) so a caller of bitgnn:: can switch by changing
// the namespace.  Names, argument meaning and error behaviour follow the
// reference:
//   * value types own host storage (ref: bitdense.hpp:18-107, bitsparse.hpp:26-60);
//   * contract violations throw std::invalid_argument, layer failures
//     std::runtime_error("layer i (kind): ..."), trace misuse std::logic_error
//     (ref: kernels.cpp:17, graphops.cpp:476-479), with the reference's messages;
//   * ops are pure; every computation runs on the B200 (no CPU fallback).
// Each host-typed op uploads its operands, runs the sm_100a kernels and
// downloads the result (drop-in semantics).  For device-resident serving use
// GraphBundle (built on device once) and Model (weights resident, CUDA-graph
// captured forward on device pointers).
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <istream>
#include <iterator>
#include <string>
#include <string_view>
#include <utility>
#include <variant>
#include <vector>

#include "../bitgnn_b200.h"

namespace bitgnn_b200 {

using Real = float;

// ---- errors -----------------------------------------------------------------
namespace detail {
inline void check(int status) {
  if (status == BG_OK) return;
  const std::string msg = bg_last_error();
  switch (status) {
    case BG_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case BG_LOGIC_ERROR: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);  // BG_RUNTIME_ERROR, BG_CUDA_ERROR
  }
}

// RAII device allocation through the C ABI (no CUDA headers needed).
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t bytes) : bytes_(bytes) { check(bg_device_alloc(bytes, &p_)); }
  DeviceBuffer(const void* host, size_t bytes) : DeviceBuffer(bytes) {
    if (bytes) check(bg_memcpy(p_, host, bytes, BG_COPY_H2D, nullptr));
  }
  ~DeviceBuffer() {
    if (p_) bg_device_free(p_);
  }
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), bytes_(o.bytes_) {}
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(bytes_, o.bytes_);
    return *this;
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  void* get() const { return p_; }
  template <class T>
  T* as() const { return static_cast<T*>(p_); }
  size_t bytes() const { return bytes_; }
  void download(void* host) const {
    if (bytes_) check(bg_memcpy(host, p_, bytes_, BG_COPY_D2H, nullptr));
  }

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
};
}  // namespace detail

// ---- enums (ref: kernels.hpp:15-17, bitdense.hpp:15-16,130, graphops.hpp:44-55) ----
enum class Precision : uint8_t { F = BG_F, B = BG_B };
enum class KernelOp : uint8_t { BMM = BG_BMM, BSpMM = BG_BSPMM, ADD = BG_ADD, CONCAT = BG_CONCAT };
enum class BitSemantics { ZeroOne = BG_ZERO_ONE, PlusMinus = BG_PLUS_MINUS };
enum class Axis { Row = BG_AXIS_ROW, Col = BG_AXIS_COL };
enum class TrinaryStrategy { IfElse = BG_IF_ELSE, AndAndNot = BG_AND_ANDNOT, TwoAndMinusPopc = BG_TWO_AND_MINUS_POPC };
enum class LayerKind {
  GcnConv = BG_LAYER_GCN,
  SageConv = BG_LAYER_SAGE,
  GraphConv = BG_LAYER_GRAPHCONV,
  FullyConnected = BG_LAYER_FC,
  Aggregate = BG_LAYER_AGGREGATE,
  Relu = BG_LAYER_RELU,
  BatchNorm = BG_LAYER_BATCHNORM,
  Softmax = BG_LAYER_SOFTMAX,
  Binarize = BG_LAYER_BINARIZE,
  Scale = BG_LAYER_SCALE
};

// ref: KernelVariant (kernels.hpp:23-33)
struct KernelVariant {
  KernelOp op = KernelOp::BMM;
  Precision in1 = Precision::B, in2 = Precision::B, out = Precision::B;

  bg_variant c() const {
    return bg_variant{static_cast<int32_t>(op), static_cast<int32_t>(in1), static_cast<int32_t>(in2),
                      static_cast<int32_t>(out)};
  }
  static KernelVariant from_c(bg_variant v) {
    return KernelVariant{static_cast<KernelOp>(v.op), static_cast<Precision>(v.in1),
                         static_cast<Precision>(v.in2), static_cast<Precision>(v.out)};
  }
  bool valid() const { return bg_variant_valid(c()) == 1; }
  std::string name() const {
    char buf[32];
    detail::check(bg_variant_name(c(), buf, sizeof buf));
    return buf;
  }
  static KernelVariant parse(std::string_view text) {
    const std::string t(text);
    bg_variant v{};
    detail::check(bg_variant_parse(t.c_str(), &v));
    return from_c(v);
  }
  bool operator==(const KernelVariant&) const = default;
};

// ---- value types (host storage; ref: bitdense.hpp:18-107) -------------------
class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(int64_t rows, int64_t cols, Real fill = 0)
      : rows_(rows), cols_(cols), data_(static_cast<size_t>(rows * cols), fill) {}
  int64_t rows() const { return rows_; }
  int64_t cols() const { return cols_; }
  Real& at(int64_t i, int64_t j) { return data_[static_cast<size_t>(i * cols_ + j)]; }
  Real at(int64_t i, int64_t j) const { return data_[static_cast<size_t>(i * cols_ + j)]; }
  Real* row(int64_t i) { return data_.data() + i * cols_; }
  const Real* row(int64_t i) const { return data_.data() + i * cols_; }
  Real* data() { return data_.data(); }
  const Real* data() const { return data_.data(); }
  size_t payload_bytes() const { return data_.size() * sizeof(Real); }
  bool operator==(const DenseMatrix&) const = default;

 private:
  int64_t rows_ = 0, cols_ = 0;
  std::vector<Real> data_;
};

class ScaleVector {
 public:
  ScaleVector() = default;
  // ref: ScaleVector ctor (bitdense.cpp:41-47): entries must be > 0
  ScaleVector(Axis axis, std::vector<Real> v) : axis_(axis), v_(std::move(v)) {
    for (Real x : v_)
      if (!(x > 0)) throw std::invalid_argument("ScaleVector: entries must be strictly positive");
  }
  Axis axis() const { return axis_; }
  int64_t size() const { return static_cast<int64_t>(v_.size()); }
  Real operator[](int64_t i) const { return v_[static_cast<size_t>(i)]; }
  const std::vector<Real>& values() const { return v_; }
  size_t payload_bytes() const { return v_.size() * sizeof(Real); }

 private:
  Axis axis_ = Axis::Row;
  std::vector<Real> v_;
};

class BitDenseMatrix {
 public:
  BitDenseMatrix() = default;
  BitDenseMatrix(int64_t rows, int64_t cols, BitSemantics sem, int word_bits = 32)
      : rows_(rows), cols_(cols), word_bits_(word_bits), sem_(sem) {
    if (word_bits != 32 && word_bits != 64)
      throw std::invalid_argument("BitDenseMatrix: word_bits must be 32 or 64");
    data_.assign(static_cast<size_t>(rows * storage_words_per_row()), 0u);
  }
  int64_t rows() const { return rows_; }
  int64_t cols() const { return cols_; }
  int word_bits() const { return word_bits_; }
  BitSemantics semantics() const { return sem_; }
  void set_semantics(BitSemantics s) { sem_ = s; }
  int64_t words_per_row() const { return (cols_ + word_bits_ - 1) / word_bits_; }
  int64_t storage_words_per_row() const { return words_per_row() * (word_bits_ / 32); }
  bool bit(int64_t i, int64_t j) const {
    return (data_[static_cast<size_t>(i * storage_words_per_row() + j / 32)] >> (31 - (j & 31))) & 1u;
  }
  void set_bit(int64_t i, int64_t j, bool v) {
    uint32_t& w = data_[static_cast<size_t>(i * storage_words_per_row() + j / 32)];
    const uint32_t m = 1u << (31 - (j & 31));
    w = v ? (w | m) : (w & ~m);
  }
  uint32_t* data() { return data_.data(); }
  const uint32_t* data() const { return data_.data(); }
  size_t payload_bytes() const { return data_.size() * sizeof(uint32_t); }
  bool operator==(const BitDenseMatrix&) const = default;

 private:
  int64_t rows_ = 0, cols_ = 0;
  int word_bits_ = 32;
  BitSemantics sem_ = BitSemantics::ZeroOne;
  std::vector<uint32_t> data_;
};

// ref: BitOperand / MatOperand (kernels.hpp:37-42)
struct BitOperand {
  BitDenseMatrix bits;
  std::optional<ScaleVector> scale;
};
using MatOperand = std::variant<DenseMatrix, BitOperand>;

inline Precision operand_precision(const MatOperand& m) {
  return std::holds_alternative<DenseMatrix>(m) ? Precision::F : Precision::B;
}
inline int64_t operand_rows(const MatOperand& m) {
  return std::visit([](const auto& x) {
    if constexpr (std::is_same_v<std::decay_t<decltype(x)>, DenseMatrix>) return x.rows();
    else return x.bits.rows();
  }, m);
}
inline int64_t operand_cols(const MatOperand& m) {
  return std::visit([](const auto& x) {
    if constexpr (std::is_same_v<std::decay_t<decltype(x)>, DenseMatrix>) return x.cols();
    else return x.bits.cols();
  }, m);
}

// ref: EdgeList (bitsparse.hpp:16-20)
struct EdgeList {
  int64_t node_count = 0;
  std::vector<std::pair<int64_t, int64_t>> edges;  // (src, dst), directed
  std::vector<double> weights;                     // ignored for structure
};

// ref: FrdcMatrix (bitsparse.hpp:26-60), host arrays.  Validation of the
// reference constructor (bitsparse.cpp:40-70) runs when the matrix is handed
// to a device op (bg_frdc_from_host), with the same messages.
class FrdcMatrix {
 public:
  static constexpr int kTileDim = 4;
  FrdcMatrix() : row_ptr_(1, 0) {}
  FrdcMatrix(int64_t node_rows, int64_t node_cols, std::vector<uint64_t> row_ptr,
             std::vector<uint32_t> col_ind, std::vector<uint16_t> tiles)
      : node_rows_(node_rows), node_cols_(node_cols), row_ptr_(std::move(row_ptr)),
        col_ind_(std::move(col_ind)), tiles_(std::move(tiles)) {}
  int64_t node_rows() const { return node_rows_; }
  int64_t node_cols() const { return node_cols_; }
  int64_t tile_rows() const { return (node_rows_ + kTileDim - 1) / kTileDim; }
  int64_t tile_cols() const { return (node_cols_ + kTileDim - 1) / kTileDim; }
  int64_t nnz_tiles() const { return static_cast<int64_t>(tiles_.size()); }
  const std::vector<uint64_t>& row_ptr() const { return row_ptr_; }
  const std::vector<uint32_t>& col_ind() const { return col_ind_; }
  const std::vector<uint16_t>& tiles() const { return tiles_; }
  std::vector<uint16_t>& mutable_tiles() { return tiles_; }
  size_t payload_bytes() const { return row_ptr_.size() * 8 + col_ind_.size() * 4 + tiles_.size() * 2; }
  bool operator==(const FrdcMatrix&) const = default;

 private:
  int64_t node_rows_ = 0, node_cols_ = 0;
  std::vector<uint64_t> row_ptr_;
  std::vector<uint32_t> col_ind_;
  std::vector<uint16_t> tiles_;
};

// ---- device-resident adjacency ----------------------------------------------
namespace detail {
struct FrdcDeleter {
  void operator()(bg_frdc* m) const { bg_frdc_destroy(m); }
};
using FrdcHandle = std::unique_ptr<bg_frdc, FrdcDeleter>;

inline FrdcHandle upload(const FrdcMatrix& m) {
  bg_frdc* h = nullptr;
  check(bg_frdc_from_host(m.node_rows(), m.node_cols(), m.row_ptr().data(), m.col_ind().data(),
                          m.tiles().data(), m.nnz_tiles(), &h, nullptr));
  return FrdcHandle(h);
}

inline FrdcMatrix download(const bg_frdc* h) {
  bg_frdc_info info{};
  check(bg_frdc_info_get(h, &info));
  std::vector<uint64_t> rp(static_cast<size_t>(info.tile_rows + 1));
  std::vector<uint32_t> ci(static_cast<size_t>(info.nnz_tiles));
  std::vector<uint16_t> ti(static_cast<size_t>(info.nnz_tiles));
  check(bg_frdc_download(h, rp.data(), ci.data(), ti.data()));
  return FrdcMatrix(info.node_rows, info.node_cols, std::move(rp), std::move(ci), std::move(ti));
}

// ref: FrdcFile / write_frdc / read_frdc (bitsparse.hpp:92-106): the container
// bytes are produced and parsed by the library (reads go straight to the
// device); I/O and format faults rethrow as std::runtime_error.
struct FrdcFile {
  FrdcMatrix matrix;
  int word_bits = 32;
};

inline void write_frdc(const std::string& path, const FrdcMatrix& m, int word_bits = 32) {
  FrdcHandle h = upload(m);
  check(bg_frdc_write_file(h.get(), word_bits, path.c_str()));
}

inline FrdcFile read_frdc(const std::string& path) {
  bg_frdc* h = nullptr;
  int wb = 32;
  check(bg_frdc_read_file(path.c_str(), &h, &wb, nullptr));
  FrdcHandle owned(h);
  return {download(owned.get()), wb};
}

struct Edges {
  DeviceBuffer src, dst;
  int64_t n = 0, e = 0;
};
inline Edges upload(const EdgeList& el) {
  std::vector<int64_t> s(el.edges.size()), d(el.edges.size());
  for (size_t k = 0; k < el.edges.size(); ++k) {
    s[k] = el.edges[k].first;
    d[k] = el.edges[k].second;
  }
  Edges r;
  r.n = el.node_count;
  r.e = static_cast<int64_t>(s.size());
  r.src = DeviceBuffer(s.data(), s.size() * 8);
  r.dst = DeviceBuffer(d.data(), d.size() * 8);
  return r;
}

// A MatOperand staged in device memory as a bg_mat.
struct DeviceOperand {
  DeviceBuffer data, scale;
  bg_mat m{};
};
inline DeviceOperand upload(const MatOperand& x) {
  DeviceOperand d;
  if (const auto* f = std::get_if<DenseMatrix>(&x)) {
    d.m.precision = BG_F;
    d.m.word_bits = 32;
    d.m.rows = f->rows();
    d.m.cols = f->cols();
    d.data = DeviceBuffer(f->data(), f->payload_bytes());
  } else {
    const auto& b = std::get<BitOperand>(x);
    d.m.precision = BG_B;
    d.m.word_bits = b.bits.word_bits();
    d.m.semantics = static_cast<int32_t>(b.bits.semantics());
    d.m.rows = b.bits.rows();
    d.m.cols = b.bits.cols();
    d.data = DeviceBuffer(b.bits.data(), b.bits.payload_bytes());
    if (b.scale) {
      d.m.scale_axis = static_cast<int32_t>(b.scale->axis());
      d.scale = DeviceBuffer(b.scale->values().data(), b.scale->payload_bytes());
      d.m.scale = d.scale.as<float>();
    }
  }
  d.m.data = d.data.get();
  return d;
}
// Allocate a result operand described by `desc` (shape/precision/word_bits).
inline DeviceOperand allocate(const bg_mat& desc) {
  DeviceOperand d;
  d.m = desc;
  d.m.scale = nullptr;
  const size_t bytes = desc.precision == BG_F
                           ? static_cast<size_t>(desc.rows * desc.cols) * 4
                           : static_cast<size_t>(desc.rows * bg_storage_words_per_row(desc.cols, desc.word_bits)) * 4;
  d.data = DeviceBuffer(bytes);
  d.m.data = d.data.get();
  return d;
}
inline MatOperand download(const DeviceOperand& d) {
  if (d.m.precision == BG_F) {
    DenseMatrix out(d.m.rows, d.m.cols);
    d.data.download(out.data());
    return out;
  }
  BitOperand out{BitDenseMatrix(d.m.rows, d.m.cols, static_cast<BitSemantics>(d.m.semantics), d.m.word_bits),
                 std::nullopt};
  d.data.download(out.bits.data());
  return out;
}
inline int strategy_code(std::optional<TrinaryStrategy> s) {
  return s ? static_cast<int>(*s) : BG_STRATEGY_DEFAULT;
}
}  // namespace detail

// ---- bitdense ops (ref: bitdense.hpp:110-141) -------------------------------
inline BitDenseMatrix binarize(const DenseMatrix& m, int word_bits = 32) {
  BitDenseMatrix out(m.rows(), m.cols(), BitSemantics::PlusMinus, word_bits);
  detail::DeviceBuffer x(m.data(), m.payload_bytes()), o(out.payload_bytes());
  detail::check(bg_binarize(x.as<float>(), m.rows(), m.cols(), word_bits, o.as<uint32_t>(), nullptr));
  o.download(out.data());
  return out;
}

inline std::pair<BitDenseMatrix, ScaleVector> binarize_with_scale(const DenseMatrix& m, Axis axis,
                                                                  int word_bits = 32) {
  BitDenseMatrix bits(m.rows(), m.cols(), BitSemantics::PlusMinus, word_bits);
  const int64_t n = axis == Axis::Row ? m.rows() : m.cols();
  std::vector<Real> sc(static_cast<size_t>(n));
  detail::DeviceBuffer x(m.data(), m.payload_bytes()), o(bits.payload_bytes()), s(sc.size() * 4);
  detail::check(bg_binarize_with_scale(x.as<float>(), m.rows(), m.cols(), static_cast<int>(axis), word_bits,
                                       o.as<uint32_t>(), s.as<float>(), nullptr));
  o.download(bits.data());
  s.download(sc.data());
  return {std::move(bits), ScaleVector(axis, std::move(sc))};
}

inline DenseMatrix unpack(const BitDenseMatrix& m) {
  DenseMatrix out(m.rows(), m.cols());
  detail::DeviceBuffer b(m.data(), m.payload_bytes()), o(out.payload_bytes());
  detail::check(bg_unpack(b.as<uint32_t>(), m.rows(), m.cols(), m.word_bits(), static_cast<int>(m.semantics()),
                          o.as<float>(), nullptr));
  o.download(out.data());
  return out;
}

inline BitDenseMatrix transpose(const BitDenseMatrix& m) {
  BitDenseMatrix out(m.cols(), m.rows(), m.semantics(), m.word_bits());
  detail::DeviceBuffer b(m.data(), m.payload_bytes()), o(out.payload_bytes());
  detail::check(bg_transpose(b.as<uint32_t>(), m.rows(), m.cols(), m.word_bits(), o.as<uint32_t>(), nullptr));
  o.download(out.data());
  return out;
}

// ---- bitsparse (ref: bitsparse.hpp:74) ---------------------------------------
inline FrdcMatrix frdc_from_edges(const EdgeList& e, bool add_self_loops) {
  auto d = detail::upload(e);
  bg_frdc* h = nullptr;
  detail::check(bg_frdc_from_edges(d.src.as<int64_t>(), d.dst.as<int64_t>(), d.e, d.n, add_self_loops ? 1 : 0,
                                   &h, nullptr));
  detail::FrdcHandle owned(h);
  return detail::download(owned.get());
}

// ref: TileSet (bitsparse.hpp:62-71): the gather unit of Algorithm 1.
struct TileSet {
  static constexpr uint32_t kPadCol = BG_TILESET_PAD_COL;
  int ts = 8;
  std::array<uint64_t, 4> rows{};
  std::array<uint32_t, 16> cols{};
};

// ref: tileset_count (bitsparse.cpp:129-134)
inline int64_t tileset_count(const FrdcMatrix& m, int64_t tile_row, int word_bits = 32) {
  auto h = detail::upload(m);
  int64_t n = 0;
  detail::check(bg_tileset_count(h.get(), tile_row, word_bits, &n));
  return n;
}

// ref: gather_tileset (bitsparse.cpp:136-160); std::invalid_argument with the
// reference's messages.
inline TileSet gather_tileset(const FrdcMatrix& m, int64_t tile_row, int64_t set_index, int word_bits = 32) {
  auto h = detail::upload(m);
  bg_tileset t{};
  detail::check(bg_gather_tileset(h.get(), tile_row, set_index, word_bits, &t));
  TileSet out;
  out.ts = t.ts;
  for (int i = 0; i < 4; ++i) out.rows[static_cast<size_t>(i)] = t.rows[i];
  for (int i = 0; i < 16; ++i) out.cols[static_cast<size_t>(i)] = t.cols[i];
  return out;
}

// ref: frdc_to_dense (bitsparse.cpp:114-127)
inline BitDenseMatrix frdc_to_dense(const FrdcMatrix& m, int word_bits = 32) {
  BitDenseMatrix out(m.node_rows(), m.node_cols(), BitSemantics::ZeroOne, word_bits);
  auto h = detail::upload(m);
  detail::DeviceBuffer d(out.payload_bytes());
  detail::check(bg_frdc_to_dense(h.get(), word_bits, d.as<uint32_t>(), nullptr));
  d.download(out.data());
  return out;
}

// ref: FrdcStats / frdc_stats (bitsparse.hpp:83-90)
struct FrdcStats {
  uint64_t nnz_tiles = 0, nnz_bits = 0, bytes = 0;
  double fill_ratio = 0;
};
inline FrdcStats frdc_stats(const FrdcMatrix& m) {
  auto h = detail::upload(m);
  bg_frdc_stats s{};
  detail::check(bg_frdc_stats_get(h.get(), &s));
  return {s.nnz_tiles, s.nnz_bits, s.bytes, s.fill_ratio};
}

// ref: AdjacencyOperand (kernels.hpp:47-57): non-owning views.
struct AdjacencyOperand {
  const FrdcMatrix* structure = nullptr;
  const ScaleVector* row_scale = nullptr;
  const ScaleVector* col_scale = nullptr;
  bool factorized() const { return row_scale != nullptr; }
};

// ---- kernel families (ref: kernels.hpp:63-97) -------------------------------
inline MatOperand bmm(const KernelVariant& v, const MatOperand& a, const MatOperand& w, int word_bits = 32) {
  auto da = detail::upload(a), dw = detail::upload(w);
  bg_mat od{};
  detail::check(bg_bmm_out_desc(v.c(), &da.m, &dw.m, word_bits, &od));
  auto out = detail::allocate(od);
  detail::check(bg_bmm(v.c(), &da.m, &dw.m, word_bits, &out.m, nullptr));
  return detail::download(out);
}

inline MatOperand bspmm(const KernelVariant& v, const AdjacencyOperand& adj, const MatOperand& x,
                        std::optional<TrinaryStrategy> strategy = std::nullopt, int word_bits = 32) {
  if (!adj.structure) throw std::invalid_argument("bspmm: adjacency has no structure");
  auto A = detail::upload(*adj.structure);
  detail::DeviceBuffer rs, cs;
  if (adj.row_scale) rs = detail::DeviceBuffer(adj.row_scale->values().data(), adj.row_scale->payload_bytes());
  if (adj.col_scale) cs = detail::DeviceBuffer(adj.col_scale->values().data(), adj.col_scale->payload_bytes());
  auto dx = detail::upload(x);
  bg_mat od{};
  detail::check(bg_bspmm_out_desc(v.c(), A.get(), &dx.m, word_bits, &od));
  auto out = detail::allocate(od);
  detail::check(bg_bspmm(v.c(), A.get(), adj.row_scale ? rs.as<float>() : nullptr,
                         adj.col_scale ? cs.as<float>() : nullptr, &dx.m, detail::strategy_code(strategy),
                         word_bits, &out.m, nullptr));
  return detail::download(out);
}

namespace detail {
// Result descriptor of ADD / CONCAT (ref: kernels.cpp:593-668): rows of a,
// cols of a (ADD) or a+b (CONCAT), precision v.out, packing width of a.
inline bg_mat glue_desc(const KernelVariant& v, const bg_mat& a, const bg_mat& b, bool concat) {
  bg_mat o{};
  o.precision = static_cast<int32_t>(v.out);
  o.rows = a.rows;
  o.cols = concat ? a.cols + b.cols : a.cols;
  o.word_bits = a.precision == BG_B ? a.word_bits : 32;
  o.semantics = BG_PLUS_MINUS;
  return o;
}
}  // namespace detail

inline MatOperand add(const KernelVariant& v, const MatOperand& a, const MatOperand& b) {
  auto da = detail::upload(a), db = detail::upload(b);
  auto out = detail::allocate(detail::glue_desc(v, da.m, db.m, false));
  detail::check(bg_add(v.c(), &da.m, &db.m, &out.m, nullptr));
  return detail::download(out);
}

inline MatOperand concat(const KernelVariant& v, const MatOperand& a, const MatOperand& b) {
  auto da = detail::upload(a), db = detail::upload(b);
  auto out = detail::allocate(detail::glue_desc(v, da.m, db.m, true));
  detail::check(bg_concat(v.c(), &da.m, &db.m, &out.m, nullptr));
  return detail::download(out);
}

inline DenseMatrix dense_mm(const DenseMatrix& a, const DenseMatrix& w) {
  if (a.cols() != w.rows()) throw std::invalid_argument("dense_mm: inner dimensions differ");
  DenseMatrix out(a.rows(), w.cols());
  detail::DeviceBuffer da(a.data(), a.payload_bytes()), dw(w.data(), w.payload_bytes()), o(out.payload_bytes());
  detail::check(bg_dense_mm(da.as<float>(), dw.as<float>(), a.rows(), a.cols(), w.cols(), o.as<float>(), nullptr));
  o.download(out.data());
  return out;
}

inline BitDenseMatrix bin(const DenseMatrix& x, int word_bits = 32) { return binarize(x, word_bits); }

inline DenseMatrix scl(const DenseMatrix& x, const ScaleVector& row, const ScaleVector& col) {
  DenseMatrix out(x.rows(), x.cols());
  detail::DeviceBuffer dx(x.data(), x.payload_bytes()), r(row.values().data(), row.payload_bytes()),
      c(col.values().data(), col.payload_bytes()), o(out.payload_bytes());
  if (row.size() != x.rows() || col.size() != x.cols())
    throw std::invalid_argument("scl: scale lengths do not match the matrix");
  detail::check(bg_scl(dx.as<float>(), x.rows(), x.cols(), r.as<float>(), c.as<float>(), o.as<float>(), nullptr));
  o.download(out.data());
  return out;
}

inline DenseMatrix softmax_rows(const DenseMatrix& x) {
  DenseMatrix out(x.rows(), x.cols());
  detail::DeviceBuffer dx(x.data(), x.payload_bytes()), o(out.payload_bytes());
  detail::check(bg_softmax_rows(dx.as<float>(), x.rows(), x.cols(), o.as<float>(), nullptr));
  o.download(out.data());
  return out;
}

// ref: BatchNormParams / batchnorm_infer (graphops.hpp:57-59, graphops.cpp:337-355)
struct BatchNormParams {
  std::vector<Real> gamma, beta, mean, sigma;
};

inline DenseMatrix batchnorm_infer(const DenseMatrix& x, const BatchNormParams& p) {
  const size_t c = static_cast<size_t>(x.cols());
  if (p.gamma.size() != c || p.beta.size() != c || p.mean.size() != c || p.sigma.size() != c)
    throw std::invalid_argument("batchnorm: parameter length != cols");
  DenseMatrix out(x.rows(), x.cols());
  detail::DeviceBuffer dx(x.data(), x.payload_bytes()), g(p.gamma.data(), c * 4), b(p.beta.data(), c * 4),
      m(p.mean.data(), c * 4), s(p.sigma.data(), c * 4), o(out.payload_bytes());
  detail::check(bg_batchnorm_infer(dx.as<float>(), x.rows(), x.cols(), g.as<float>(), b.as<float>(), m.as<float>(),
                                   s.as<float>(), o.as<float>(), nullptr));
  o.download(out.data());
  return out;
}

// ref: FusedPlan / fused_mm_spmm (kernels.hpp:88-97)
struct FusedPlan {
  KernelVariant mm;
  KernelVariant spmm;
};

inline MatOperand fused_mm_spmm(const FusedPlan& plan, const MatOperand& x, const MatOperand& w,
                                const AdjacencyOperand& adj,
                                std::optional<TrinaryStrategy> strategy = std::nullopt) {
  if (!adj.structure) throw std::invalid_argument("fused_mm_spmm: adjacency has no structure");
  auto A = detail::upload(*adj.structure);
  detail::DeviceBuffer rs, cs;
  if (adj.row_scale) rs = detail::DeviceBuffer(adj.row_scale->values().data(), adj.row_scale->payload_bytes());
  if (adj.col_scale) cs = detail::DeviceBuffer(adj.col_scale->values().data(), adj.col_scale->payload_bytes());
  auto dx = detail::upload(x), dw = detail::upload(w);
  bg_mat mid{}, od{};
  detail::check(bg_bmm_out_desc(plan.mm.c(), &dx.m, &dw.m, dx.m.word_bits, &mid));
  detail::check(bg_bspmm_out_desc(plan.spmm.c(), A.get(), &mid, mid.word_bits, &od));
  auto out = detail::allocate(od);
  detail::check(bg_fused_mm_spmm(plan.mm.c(), plan.spmm.c(), &dx.m, &dw.m, A.get(),
                                 adj.row_scale ? rs.as<float>() : nullptr, adj.col_scale ? cs.as<float>() : nullptr,
                                 detail::strategy_code(strategy), &out.m, nullptr));
  return detail::download(out);
}

// ---- graph bundle (ref: GraphBundle / prepare_graph, graphops.hpp:27-40) ------
// Device-resident and immutable; the host arrays are downloaded on request.
class GraphBundle {
 public:
  explicit GraphBundle(bg_graph* g) : g_(g) {}
  ~GraphBundle() {
    if (g_) bg_graph_destroy(g_);
  }
  GraphBundle(const GraphBundle&) = delete;
  GraphBundle& operator=(const GraphBundle&) = delete;
  const bg_graph* handle() const { return g_; }
  bg_graph* mutable_handle() const { return g_; }  // fault-injection hooks only
  int64_t node_count() const { return info().n; }
  FrdcMatrix structure() const { return detail::download(info().structure); }  // A + I
  FrdcMatrix raw() const { return detail::download(info().raw); }              // A, loop-free
  ScaleVector norm_row() const { return scale(info().norm, Axis::Row); }
  ScaleVector norm_col() const { return scale(info().norm, Axis::Col); }
  ScaleVector mean_row() const { return scale(info().mean_row, Axis::Row); }
  std::vector<int64_t> neighbor_count() const {
    std::vector<int64_t> v(static_cast<size_t>(node_count()));
    detail::check(bg_memcpy(v.data(), info().neighbor_count, v.size() * 8, BG_COPY_D2H, nullptr));
    return v;
  }
  std::pair<int64_t, int64_t> partition_rows(int world_size, int rank) const {
    int64_t b = 0, e = 0;
    detail::check(bg_partition_rows(g_, world_size, rank, &b, &e));
    return {b, e};
  }

 private:
  bg_graph_info info() const {
    bg_graph_info i{};
    detail::check(bg_graph_info_get(g_, &i));
    return i;
  }
  ScaleVector scale(const float* dev, Axis axis) const {
    std::vector<Real> v(static_cast<size_t>(node_count()));
    detail::check(bg_memcpy(v.data(), dev, v.size() * 4, BG_COPY_D2H, nullptr));
    return ScaleVector(axis, std::move(v));
  }
  bg_graph* g_ = nullptr;
};

inline std::shared_ptr<const GraphBundle> prepare_graph(const EdgeList& e) {
  auto d = detail::upload(e);
  bg_graph* g = nullptr;
  detail::check(bg_prepare_graph(d.src.as<int64_t>(), d.dst.as<int64_t>(), d.e, d.n, &g, nullptr));
  return std::make_shared<const GraphBundle>(g);
}

// ---- models (ref: LayerSpec / ModelSpec / RunTrace / run_model, graphops.hpp:61-133) ----
// ref: layer_kind_name (graphops.cpp:119-133)
inline const char* layer_kind_name(LayerKind k) {
  switch (k) {
    case LayerKind::GcnConv: return "gcn_conv";
    case LayerKind::SageConv: return "sage_conv";
    case LayerKind::GraphConv: return "graph_conv";
    case LayerKind::FullyConnected: return "fc";
    case LayerKind::Aggregate: return "aggregate";
    case LayerKind::Relu: return "relu";
    case LayerKind::BatchNorm: return "batchnorm";
    case LayerKind::Softmax: return "softmax";
    case LayerKind::Binarize: return "binarize";
    case LayerKind::Scale: return "scale";
  }
  return "?";
}

struct LayerSpec {
  LayerKind kind = LayerKind::FullyConnected;
  std::vector<KernelVariant> plan;
  std::shared_ptr<const DenseMatrix> w1, w2;
  std::optional<BatchNormParams> bn;
  std::optional<ScaleVector> scale_row, scale_col;
  bool relu = false;
};

struct ModelSpec {
  std::vector<LayerSpec> layers;
  Precision input_precision = Precision::F;
  std::shared_ptr<const GraphBundle> graph;
  std::optional<TrinaryStrategy> strategy;
  int word_bits = 32;
};

struct RunTrace {
  struct Point {
    std::string label;
    BitDenseMatrix bits;
  };
  std::vector<Point> points;
  DenseMatrix logits;
};

struct KernelTiming {
  std::string label;
  int64_t ns;
};

namespace detail {
inline std::vector<bg_layer_desc> describe(const ModelSpec& m) {
  std::vector<bg_layer_desc> out(m.layers.size());
  for (size_t i = 0; i < m.layers.size(); ++i) {
    const LayerSpec& l = m.layers[i];
    bg_layer_desc& d = out[i];
    std::memset(&d, 0, sizeof d);
    d.kind = static_cast<int32_t>(l.kind);
    if (l.plan.size() > 4) throw std::invalid_argument("layer plan has more than 4 slots");
    d.n_plan = static_cast<int32_t>(l.plan.size());
    for (size_t k = 0; k < l.plan.size(); ++k) d.plan[k] = l.plan[k].c();
    if (l.w1) {
      d.w1 = l.w1->data();
      d.w1_rows = l.w1->rows();
      d.w1_cols = l.w1->cols();
    }
    if (l.w2) {
      d.w2 = l.w2->data();
      d.w2_rows = l.w2->rows();
      d.w2_cols = l.w2->cols();
    }
    d.relu = l.relu ? 1 : 0;
    if (l.bn) {
      d.bn_gamma = l.bn->gamma.data();
      d.bn_beta = l.bn->beta.data();
      d.bn_mean = l.bn->mean.data();
      d.bn_sigma = l.bn->sigma.data();
      d.bn_len = static_cast<int64_t>(l.bn->gamma.size());
    }
    if (l.scale_row) {
      d.scale_row = l.scale_row->values().data();
      d.scale_row_len = l.scale_row->size();
    }
    if (l.scale_col) {
      d.scale_col = l.scale_col->values().data();
      d.scale_col_len = l.scale_col->size();
    }
  }
  return out;
}
}  // namespace detail

// ref: validate_model (graphops.cpp:245-268): the problems, empty when well formed.
inline std::vector<std::string> validate_model(const ModelSpec& m) {
  auto d = detail::describe(m);
  std::vector<char> buf(1 << 16);
  const int n = bg_validate_model(m.graph ? 1 : 0, static_cast<int>(m.input_precision), d.data(),
                                  static_cast<int>(d.size()), buf.data(), buf.size());
  std::vector<std::string> out;
  if (n <= 0) return out;
  std::string all(buf.data());
  size_t p = 0;
  while (p <= all.size()) {
    const size_t q = all.find('\n', p);
    const std::string line = all.substr(p, q == std::string::npos ? std::string::npos : q - p);
    if (!line.empty()) out.push_back(line);
    if (q == std::string::npos) break;
    p = q + 1;
  }
  return out;
}

// ref: rewrite_eliminate_scl (graphops.cpp:357-368): a Scale node directly
// ahead of a Binarize is dropped (positive factors move no value across the
// sign threshold); every other layer is kept in order.
inline ModelSpec rewrite_eliminate_scl(const ModelSpec& m) {
  ModelSpec out = m;
  out.layers.clear();
  for (size_t i = 0; i < m.layers.size(); ++i) {
    if (m.layers[i].kind == LayerKind::Scale && i + 1 < m.layers.size() &&
        m.layers[i + 1].kind == LayerKind::Binarize)
      continue;
    out.layers.push_back(m.layers[i]);
  }
  return out;
}

// ---- single layers (ref: LayerHooks / gcn_layer / sage_layer / graphconv_layer,
// graphops.hpp:88-105) ----------------------------------------------------------
// record_bits sees every BIN point of the layer, in the reference's order and
// with its labels (prefix + "mm.bin_in", ...); record_ns is not called (per-op
// device times come from Model::run with timings).
struct LayerHooks {
  std::function<void(const std::string&, const BitDenseMatrix&)> record_bits;
  std::function<void(const std::string&, int64_t)> record_ns;
};

namespace detail {
inline MatOperand layer_call(int kind, const MatOperand& x, const LayerSpec& l, const GraphBundle& g,
                             std::optional<TrinaryStrategy> strategy, const LayerHooks* hooks,
                             const std::string& prefix, int word_bits) {
  ModelSpec one;
  one.layers.push_back(l);
  auto descs = describe(one);
  auto dx = upload(x);
  bg_mat od{};
  check(bg_layer_out_desc(kind, descs.data(), &dx.m, word_bits, &od));
  auto out = allocate(od);
  bg_trace* t = nullptr;
  const bool want_bits = hooks && hooks->record_bits;
  if (want_bits) check(bg_trace_create(&t));
  std::unique_ptr<bg_trace, void (*)(bg_trace*)> owned(t, bg_trace_destroy);
  auto fn = kind == BG_LAYER_GCN ? bg_gcn_layer : kind == BG_LAYER_SAGE ? bg_sage_layer : bg_graphconv_layer;
  check(fn(&dx.m, descs.data(), g.handle(), strategy_code(strategy), t, prefix.c_str(), word_bits, &out.m,
           nullptr));
  if (want_bits) {
    const int n = bg_trace_size(t);
    for (int i = 0; i < n; ++i) {
      const char* label = nullptr;
      int64_t r = 0, c = 0;
      int wb = 32;
      const uint32_t* bits = nullptr;
      check(bg_trace_point(t, i, &label, &r, &c, &wb, &bits));
      BitDenseMatrix b(r, c, BitSemantics::PlusMinus, wb);
      check(bg_memcpy(b.data(), bits, b.payload_bytes(), BG_COPY_D2H, nullptr));
      hooks->record_bits(label, b);
    }
  }
  return download(out);
}
}  // namespace detail

// ref: gcn_layer (graphops.cpp:270-285)
inline MatOperand gcn_layer(const MatOperand& x, const LayerSpec& l, const GraphBundle& g,
                            std::optional<TrinaryStrategy> strategy = std::nullopt, const LayerHooks* hooks = nullptr,
                            const std::string& prefix = "", int word_bits = 32) {
  return detail::layer_call(BG_LAYER_GCN, x, l, g, strategy, hooks, prefix, word_bits);
}
// ref: sage_layer (graphops.cpp:325-329)
inline MatOperand sage_layer(const MatOperand& x, const LayerSpec& l, const GraphBundle& g,
                             std::optional<TrinaryStrategy> strategy = std::nullopt, const LayerHooks* hooks = nullptr,
                             const std::string& prefix = "", int word_bits = 32) {
  return detail::layer_call(BG_LAYER_SAGE, x, l, g, strategy, hooks, prefix, word_bits);
}
// ref: graphconv_layer (graphops.cpp:331-335)
inline MatOperand graphconv_layer(const MatOperand& x, const LayerSpec& l, const GraphBundle& g,
                                  std::optional<TrinaryStrategy> strategy = std::nullopt,
                                  const LayerHooks* hooks = nullptr, const std::string& prefix = "",
                                  int word_bits = 32) {
  return detail::layer_call(BG_LAYER_GRAPHCONV, x, l, g, strategy, hooks, prefix, word_bits);
}

// ---- graph readers (ref: graphio.hpp:11-24) ----------------------------------
namespace detail {
inline EdgeList take_edges(bg_edges* h) {
  struct Guard {
    bg_edges* h;
    ~Guard() { bg_edges_destroy(h); }
  } g{h};
  int64_t n = 0, m = 0, nw = 0;
  const int64_t *src = nullptr, *dst = nullptr;
  const double* w = nullptr;
  check(bg_edges_info(h, &n, &m, &src, &dst, &w, &nw));
  EdgeList e;
  e.node_count = n;
  e.edges.reserve(static_cast<size_t>(m));
  for (int64_t k = 0; k < m; ++k) e.edges.emplace_back(src[k], dst[k]);
  e.weights.assign(w, w + nw);
  return e;
}
}  // namespace detail

// Whitespace "src dst [weight]" pairs, 0-based; '#'/'%' comments.
inline EdgeList read_edge_list(std::istream& in, const std::string& name, int64_t forced_nodes = -1,
                               bool undirected = false) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  bg_edges* h = nullptr;
  detail::check(bg_read_edge_list(text.data(), text.size(), name.c_str(), forced_nodes, undirected ? 1 : 0, &h));
  return detail::take_edges(h);
}

// MatrixMarket coordinate (pattern/real/integer, general/symmetric).
inline EdgeList read_matrix_market(std::istream& in, const std::string& name, bool undirected = false) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  bg_edges* h = nullptr;
  detail::check(bg_read_matrix_market(text.data(), text.size(), name.c_str(), undirected ? 1 : 0, &h));
  return detail::take_edges(h);
}

// Sniffs the file: FRDC container, MatrixMarket, else an edge list.
inline EdgeList load_graph(const std::string& path, int64_t forced_nodes = -1, bool undirected = false) {
  bg_edges* h = nullptr;
  detail::check(bg_load_graph(path.c_str(), forced_nodes, undirected ? 1 : 0, &h));
  return detail::take_edges(h);
}

// A device-resident model: weights binarized once, forward captured as one
// CUDA graph after its first run.  The serving entry point.
class Model {
 public:
  explicit Model(const ModelSpec& spec, void* stream = nullptr) : spec_(spec) {
    auto d = detail::describe(spec);
    detail::check(bg_model_create(spec.graph ? spec.graph->handle() : nullptr, static_cast<int>(spec.input_precision),
                                  detail::strategy_code(spec.strategy), spec.word_bits, d.data(),
                                  static_cast<int>(d.size()), &m_, stream));
  }
  ~Model() {
    if (m_) bg_model_destroy(m_);
  }
  Model(const Model&) = delete;
  Model& operator=(const Model&) = delete;
  bg_model* handle() const { return m_; }
  int64_t output_cols() const {
    int64_t c = 0;
    detail::check(bg_model_output_cols(m_, &c));
    return c;
  }
  void set_graph_capture(bool on) { detail::check(bg_model_set_graph_capture(m_, on ? 1 : 0)); }

  // Device pointers: x0 (rows x cols fp32), out/logits (rows x output_cols; logits may be null).
  void forward_device(const float* x0, int64_t rows, int64_t cols, float* out, float* logits,
                      void* stream = nullptr) {
    bg_mat x{};
    x.precision = BG_F;
    x.word_bits = 32;
    x.rows = rows;
    x.cols = cols;
    x.data = const_cast<float*>(x0);
    detail::check(bg_model_forward(m_, &x, out, logits, stream));
  }

  // Host in, host out (H2D, forward, D2H).
  DenseMatrix forward(const DenseMatrix& x, DenseMatrix* logits = nullptr, void* stream = nullptr) {
    DenseMatrix out(x.rows(), output_cols());
    if (logits) *logits = DenseMatrix(x.rows(), output_cols());
    detail::check(bg_model_forward_host(m_, x.data(), x.rows(), x.cols(), out.data(),
                                        logits ? logits->data() : nullptr, stream));
    return out;
  }

  // ref: run_model (graphops.cpp:390-484) with optional trace / timings.
  DenseMatrix run(const MatOperand& x0, RunTrace* trace = nullptr, std::vector<KernelTiming>* timings = nullptr) {
    auto dx = detail::upload(x0);
    const int64_t rows = dx.m.rows, oc = output_cols();
    detail::DeviceBuffer out(static_cast<size_t>(rows * oc) * 4), lg(static_cast<size_t>(rows * oc) * 4);
    if (trace) {
      bg_trace* t = nullptr;
      detail::check(bg_trace_create(&t));
      std::unique_ptr<bg_trace, void (*)(bg_trace*)> owned(t, bg_trace_destroy);
      detail::check(bg_model_forward_traced(m_, &dx.m, out.as<float>(), lg.as<float>(), t, nullptr));
      trace->points.clear();
      const int n = bg_trace_size(t);
      for (int i = 0; i < n; ++i) {
        const char* label = nullptr;
        int64_t r = 0, c = 0;
        int wb = 32;
        const uint32_t* bits = nullptr;
        detail::check(bg_trace_point(t, i, &label, &r, &c, &wb, &bits));
        RunTrace::Point p{label, BitDenseMatrix(r, c, BitSemantics::PlusMinus, wb)};
        detail::check(bg_memcpy(p.bits.data(), bits, p.bits.payload_bytes(), BG_COPY_D2H, nullptr));
        trace->points.push_back(std::move(p));
      }
      trace->logits = DenseMatrix(rows, oc);
      lg.download(trace->logits.data());
    }
    if (timings) {
      std::vector<bg_kernel_timing> kt(256);
      int n = 0;
      detail::check(bg_model_forward_timed(m_, &dx.m, out.as<float>(), lg.as<float>(), kt.data(),
                                           static_cast<int>(kt.size()), &n, nullptr));
      timings->clear();
      for (int i = 0; i < n; ++i) timings->push_back({kt[static_cast<size_t>(i)].label,
                                                     static_cast<int64_t>(kt[static_cast<size_t>(i)].ms * 1e6)});
    }
    if (!trace && !timings) detail::check(bg_model_forward(m_, &dx.m, out.as<float>(), lg.as<float>(), nullptr));
    DenseMatrix result(rows, oc);
    out.download(result.data());
    return result;
  }

 private:
  ModelSpec spec_;  // keeps the graph alive
  bg_model* m_ = nullptr;
};

// ref: run_model (graphops.hpp:132-133): build, run once, return the output.
inline DenseMatrix run_model(const ModelSpec& m, const MatOperand& x0, RunTrace* trace = nullptr,
                             std::vector<KernelTiming>* timings = nullptr) {
  Model model(m);
  return model.run(x0, trace, timings);
}

}  // namespace bitgnn_b200
