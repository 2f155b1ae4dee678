// FRDC container I/O (ref: write_frdc / read_frdc, bitsparse.cpp:171-222;
// layout bitsparse.hpp:92-96).  Little-endian, byte-identical to the
// reference writer:
//   "FRDC" | u32 version=1 | u8 tile_dim=4 | u8 word_bits | u16 reserved=0 |
//   u64 node_rows | u64 node_cols | u64 nnz_tiles |
//   u64 row_ptr[tile_rows+1] | u32 col_ind[nnz] | u16 tiles[nnz]
// Reading goes straight into pinned host staging and then to the device
// (frdc_from_host: the reference's FrdcMatrix validation, then async upload);
// writing downloads the device arrays once.  Errors carry the reference's
// messages and exception classes (runtime_error for I/O and format faults).
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "ops.cuh"

namespace bg {
namespace {

constexpr size_t kHeader = 4 + 4 + 1 + 1 + 2 + 8 + 8 + 8;  // 36 bytes

// Byte source over a memory buffer or a FILE*, with the reference's
// truncation error (get_bytes, bitsparse.cpp:30-36).
struct Source {
  const uint8_t* buf = nullptr;
  size_t len = 0, pos = 0;
  FILE* f = nullptr;
  void read(void* dst, size_t n) {
    if (f) {
      if (n && std::fread(dst, 1, n, f) != n) throw std::runtime_error("FRDC: truncated file");
      return;
    }
    if (len - pos < n) throw std::runtime_error("FRDC: truncated file");
    std::memcpy(dst, buf + pos, n);
    pos += n;
  }
  // Bytes left in the source (a non-seekable file reports "unbounded").
  uint64_t remaining() {
    if (!f) return len - pos;
    const long here = std::ftell(f);
    if (here < 0 || std::fseek(f, 0, SEEK_END) != 0) return UINT64_MAX;
    const long end = std::ftell(f);
    std::fseek(f, here, SEEK_SET);
    return end >= here ? static_cast<uint64_t>(end - here) : 0;
  }
  uint64_t get(int n) {
    uint8_t b[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    read(b, static_cast<size_t>(n));
    uint64_t v = 0;
    for (int i = 0; i < n; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
    return v;
  }
};

struct Pinned {
  void* p = nullptr;
  explicit Pinned(size_t n) {
    if (n) BG_CUDA(cudaMallocHost(&p, n));
  }
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
  Pinned(const Pinned&) = delete;
  Pinned& operator=(const Pinned&) = delete;
};

// ref: read_frdc(std::istream&), bitsparse.cpp:197-216 (same checks, same order)
std::unique_ptr<bg_frdc> read_container(Source& in, int* word_bits, cudaStream_t s) {
  char magic[4];
  try {
    in.read(magic, 4);
  } catch (const std::runtime_error&) {
    throw std::runtime_error("FRDC: bad magic");
  }
  if (std::memcmp(magic, "FRDC", 4) != 0) throw std::runtime_error("FRDC: bad magic");
  if (in.get(4) != 1) throw std::runtime_error("FRDC: unsupported version");
  if (in.get(1) != 4) throw std::runtime_error("FRDC: unsupported tile_dim");
  const int wb = static_cast<int>(in.get(1));
  if (wb != 32 && wb != 64) throw std::runtime_error("FRDC: bad word_bits");
  if (in.get(2) != 0) throw std::runtime_error("FRDC: nonzero reserved field");
  const auto node_rows = static_cast<int64_t>(in.get(8));
  const auto node_cols = static_cast<int64_t>(in.get(8));
  const uint64_t nnz = in.get(8);
  if (node_rows < 0 || node_cols < 0) fail("FRDC: negative dimension");
  const int64_t tile_rows = node_rows / 4 + (node_rows % 4 != 0);
  // The header's sizes are untrusted: the arrays they declare must fit in
  // what is left of the source before anything is allocated (checked without
  // overflow; the reference's reader runs out of bytes there too).
  const uint64_t left = in.remaining();
  const uint64_t rp_words = static_cast<uint64_t>(tile_rows) + 1;
  if (rp_words > left / 8 || nnz > (left - rp_words * 8) / 6) throw std::runtime_error("FRDC: truncated file");
  // x86-64 and the GPU are little-endian: the arrays are read as-is
  const size_t rp_bytes = static_cast<size_t>(rp_words) * 8, ci_bytes = static_cast<size_t>(nnz) * 4,
               ti_bytes = static_cast<size_t>(nnz) * 2;
  Pinned rp(rp_bytes), ci(ci_bytes), ti(ti_bytes);
  in.read(rp.p, rp_bytes);
  in.read(ci.p, ci_bytes);
  in.read(ti.p, ti_bytes);
  auto m = frdc_from_host(node_rows, node_cols, static_cast<const uint64_t*>(rp.p),
                          static_cast<const uint32_t*>(ci.p), static_cast<const uint16_t*>(ti.p),
                          static_cast<int64_t>(nnz), s);
  BG_CUDA(cudaStreamSynchronize(s));  // staging buffers are released on return
  if (word_bits) *word_bits = wb;
  return m;
}

void put(uint8_t*& o, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) *o++ = static_cast<uint8_t>((v >> (8 * i)) & 0xFF);
}

size_t container_bytes(const bg_frdc& m) {
  return kHeader + static_cast<size_t>(m.tile_rows + 1) * 8 + static_cast<size_t>(m.nnz) * 6;
}

// ref: write_frdc(std::ostream&, ...), bitsparse.cpp:171-186
void write_container(const bg_frdc& m, int word_bits, uint8_t* out) {
  uint8_t* o = out;
  std::memcpy(o, "FRDC", 4);
  o += 4;
  put(o, 1, 4);  // version
  put(o, 4, 1);  // tile_dim
  put(o, static_cast<uint64_t>(word_bits), 1);
  put(o, 0, 2);  // reserved
  put(o, static_cast<uint64_t>(m.rows), 8);
  put(o, static_cast<uint64_t>(m.cols), 8);
  put(o, static_cast<uint64_t>(m.nnz), 8);
  BG_CUDA(cudaMemcpy(o, m.row_ptr.p, static_cast<size_t>(m.tile_rows + 1) * 8, cudaMemcpyDeviceToHost));
  o += static_cast<size_t>(m.tile_rows + 1) * 8;
  if (m.nnz) {
    BG_CUDA(cudaMemcpy(o, m.col_ind.p, static_cast<size_t>(m.nnz) * 4, cudaMemcpyDeviceToHost));
    o += static_cast<size_t>(m.nnz) * 4;
    BG_CUDA(cudaMemcpy(o, m.tiles.p, static_cast<size_t>(m.nnz) * 2, cudaMemcpyDeviceToHost));
  }
}

void check_word_bits(int word_bits) {
  if (word_bits != 32 && word_bits != 64) fail("write_frdc: word_bits must be 32 or 64");
}

}  // namespace

size_t frdc_container_bytes(const bg_frdc& m) { return container_bytes(m); }

void frdc_serialize(const bg_frdc& m, int word_bits, void* buf) {
  check_word_bits(word_bits);
  write_container(m, word_bits, static_cast<uint8_t*>(buf));
}

std::unique_ptr<bg_frdc> frdc_deserialize(const void* buf, size_t len, int* word_bits, cudaStream_t s) {
  Source in;
  in.buf = static_cast<const uint8_t*>(buf);
  in.len = len;
  return read_container(in, word_bits, s);
}

void frdc_write_file(const bg_frdc& m, int word_bits, const char* path) {
  check_word_bits(word_bits);
  const std::string p = path ? path : "";
  std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(p.c_str(), "wb"), &std::fclose);
  if (!f) throw std::runtime_error("write_frdc: cannot open " + p);
  const size_t n = container_bytes(m);
  Pinned staging(n);
  write_container(m, word_bits, static_cast<uint8_t*>(staging.p));
  if (std::fwrite(staging.p, 1, n, f.get()) != n) throw std::runtime_error("write_frdc: write failed");
}

std::unique_ptr<bg_frdc> frdc_read_file(const char* path, int* word_bits, cudaStream_t s) {
  const std::string p = path ? path : "";
  std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(p.c_str(), "rb"), &std::fclose);
  if (!f) throw std::runtime_error("read_frdc: cannot open " + p);
  Source in;
  in.f = f.get();
  return read_container(in, word_bits, s);
}

}  // namespace bg
