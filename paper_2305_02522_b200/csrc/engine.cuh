// Engine internals: operand views, workspace pool, operator dispatch with the
// reference's validation, and the device-resident model.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "ops.cuh"

namespace bg {

// Device operand view (ref: MatOperand, kernels.hpp:37-42).
struct Op {
  int prec = BG_F;
  int64_t rows = 0, cols = 0;
  int wb = 32;
  int sem = BG_PLUS_MINUS;
  float* f = nullptr;
  uint32_t* bits = nullptr;
  const float* scale = nullptr;
  int scale_axis = BG_AXIS_ROW;
  // An F operand held as its bit pattern (packed.cu): value = bit ? pval : 0,
  // bits in the packed layout at width wb.  Only the model executor makes
  // and reads these; everything else sees materialized fp32.
  float pval = 0.0f;
  bool packed() const { return prec == BG_F && pval != 0.0f && bits && !f; }
  size_t bytes() const {
    return prec == BG_F && !packed() ? static_cast<size_t>(rows * cols) * 4
                                     : static_cast<size_t>(rows * spw(cols, wb)) * 4;
  }
};

Op op_from_mat(const bg_mat* m);
void op_to_mat(const Op& o, bg_mat* m);

// Deterministic bump pool: the same call sequence gets the same buffers, so a
// forward can be captured once and replayed as a CUDA graph.
// gen changes whenever a slot is (re)allocated: a CUDA graph captured over the
// pool's pointers is only valid while gen is unchanged.
struct Pool {
  std::vector<DevBuf> bufs;
  size_t next = 0;
  uint64_t gen = 0;
  void reset() { next = 0; }
  void* get(size_t bytes);
};

std::string variant_name(bg_variant v);
bool variant_valid(bg_variant v);
bg_variant variant_parse(const std::string& text);
const char* layer_kind_name(int kind);

// Ops with the reference's checks.  Outputs come from `pool`.
// wt_cache/scale_cache: optional pre-binarized transposed weight bits and
// column scales for w (the model precomputes them once).
struct WeightCache {
  const uint32_t* wbits = nullptr;  // w rows x spw(cols) (for traces)
  const uint32_t* wt = nullptr;     // cols x spw(rows)
  const float* scale = nullptr;     // column scales
  const float* f = nullptr;         // fp32 weights (MM.FFF)
  int64_t rows = 0, cols = 0;
  int wb = 32;
};
// Row chunks of an operand that arrives (or must leave) piecewise: chunk c
// covers rows [bounds[c], bounds[c+1]); ready[c] is recorded when it is there.
struct RowChunks {
  int n = 0;
  const int64_t* bounds = nullptr;
  const cudaEvent_t* ready = nullptr;
};
// in_chunks: an fp32 activation still being copied in; the MM waits for each
// chunk's event and runs on it (B outputs only: no row scales are needed).
Op run_bmm(bg_variant v, const Op& a, const Op* w, const WeightCache* wc, int word_bits, Pool& pool,
           cudaStream_t s, const RowChunks* in_chunks = nullptr);
Op run_bspmm(bg_variant v, const bg_frdc* adj, const float* rs, const float* cs, const Op& x,
             int word_bits, Pool& pool, cudaStream_t s);
// fuse_relu: apply the layer's ReLU inside the kernel when the result is F
Op run_add(bg_variant v, const Op& a, const Op& b, Pool& pool, cudaStream_t s, bool fuse_relu = false);
// ReLU(ADD.BBF(a, b)) = 2 (a AND b), returned packed (pval 2); the checks of run_add
Op run_add_relu_packed(bg_variant v, const Op& a, const Op& b, Pool& pool, cudaStream_t s);
// A packed F operand as fp32 (any other operand unchanged)
Op materialize(const Op& x, Pool& pool, cudaStream_t s);
Op run_concat(bg_variant v, const Op& a, const Op& b, Pool& pool, cudaStream_t s);

// Output shapes (for caller allocation through the C ABI).
Op bmm_out_desc(bg_variant v, const Op& a, const Op& w, int word_bits);
Op bspmm_out_desc(bg_variant v, const bg_frdc* adj, const Op& x, int word_bits);

}  // namespace bg
