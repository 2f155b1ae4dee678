// Engine-versus-reference verification on the device (ref: verify_model's
// comparison and VerifyReport, runreport.cpp:51-135, runreport.hpp:13-25).
//
// The caller supplies the reference side (BIN points as packed bits and the
// logits in double, e.g. from the dense oracle or the reference engine); the
// engine side is a device trace.  Everything is compared where it lives:
//   * BIN points: per u32 word, popc of (engine ^ reference) over the valid
//     columns; the first mismatch is the smallest row-major bit index
//     (atomicMin), taken over points in trace order as the reference does;
//   * logits: max |e - o| / max(1, |o|) in double (non-negative doubles order
//     like their bit patterns, so atomicMax on the bits);
//   * argmax: the engine's first row maximum (argmax_row, runreport.cpp:27-33)
//     agrees when the reference value there equals the reference row maximum
//     (exact ties in the reference accept any of the tied classes).
#include <cstring>
#include <string>
#include <vector>

#include "engine.cuh"
#include "model.cuh"

namespace bg {
namespace {

__global__ void k_bits_cmp(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, int64_t rows,
                           int64_t words, int64_t cols, unsigned long long* __restrict__ mism,
                           unsigned long long* __restrict__ first) {
  const int64_t total = rows * words;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = k / words, c0 = 32 * (k - i * words);
    if (c0 >= cols) continue;  // padding word of a 64-bit row
    const uint32_t mask = c0 + 32 <= cols ? 0xFFFFFFFFu : tail_mask32(cols - c0);
    const uint32_t x = (a[k] ^ b[k]) & mask;
    if (x) {
      atomicAdd(mism, static_cast<unsigned long long>(__popc(x)));
      atomicMin(first, static_cast<unsigned long long>(i * cols + c0 + __clz(x)));
    }
  }
}

__global__ void k_logits_cmp(const float* __restrict__ e, const double* __restrict__ o, int64_t rows,
                             int64_t cols, unsigned long long* __restrict__ max_rel,
                             unsigned long long* __restrict__ agree) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float* er = e + i * cols;
    const double* orow = o + i * cols;
    double rel = 0.0;
    int64_t pick = 0;
    double omax = cols ? orow[0] : 0.0;
    for (int64_t j = 0; j < cols; ++j) {
      const double ev = static_cast<double>(er[j]), ov = orow[j];
      rel = fmax(rel, fabs(ev - ov) / fmax(1.0, fabs(ov)));
      if (j && er[j] > er[pick]) pick = j;
      omax = fmax(omax, ov);
    }
    if (rel != rel) rel = __longlong_as_double(0x7FF0000000000000LL);  // NaN compares as +inf
    atomicMax(max_rel, static_cast<unsigned long long>(__double_as_longlong(rel)));
    if (cols == 0 || orow[pick] == omax) atomicAdd(agree, 1ull);
  }
}

int grid_of(int64_t n) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 8LL * sm_count())));
}

}  // namespace

void verify_trace(const bg_trace& eng, const float* elog, int64_t rows, int64_t cols, const bg_ref_point* ref,
                  int n_ref, const double* ref_logits, int64_t ref_rows, int64_t ref_cols, int compare_bits,
                  double tol, bg_verify_report* r, cudaStream_t s) {
  std::memset(r, 0, sizeof *r);
  r->tolerance = tol;
  r->first_mismatch_row = r->first_mismatch_col = -1;
  DevBuf acc(32);  // mismatches, first index, max_rel bits, agree
  if (compare_bits) {
    // ref: runreport.cpp:71-106 (shape and label checks are logic errors)
    if (static_cast<int>(eng.pts.size()) != n_ref)
      throw std::logic_error("verify: engine and reference disagree on trace shape (" +
                             std::to_string(eng.pts.size()) + " vs " + std::to_string(n_ref) + " points)");
    r->bin_points = n_ref;
    DevBuf rb;
    for (int p = 0; p < n_ref; ++p) {
      const TracePoint& ep = eng.pts[static_cast<size_t>(p)];
      const bg_ref_point& op = ref[p];
      const std::string olabel = op.label ? op.label : "";
      if (ep.label != olabel || ep.rows != op.rows || ep.cols != op.cols)
        throw std::logic_error("verify: trace point " + std::to_string(p) + " misaligned (" + ep.label + " vs " +
                               olabel + ")");
      r->bin_values += ep.rows * ep.cols;
      if (op.word_bits != ep.wb) fail("verify: reference point " + olabel + " has another word width");
      const int64_t words = spw(ep.cols, ep.wb);
      const size_t bytes = static_cast<size_t>(ep.rows * words) * 4;
      if (!bytes) continue;
      if (!op.bits) fail("verify: reference point " + olabel + " has no bits");
      if (rb.bytes < bytes) rb.alloc(bytes);
      BG_CUDA(cudaMemcpyAsync(rb.p, op.bits, bytes, cudaMemcpyHostToDevice, s));
      unsigned long long init[2] = {0ull, ~0ull};
      BG_CUDA(cudaMemcpyAsync(acc.p, init, 16, cudaMemcpyHostToDevice, s));
      k_bits_cmp<<<grid_of(ep.rows * words), 256, 0, s>>>(ep.bits.as<uint32_t>(), rb.as<uint32_t>(), ep.rows,
                                                           words, ep.cols, acc.as<unsigned long long>(),
                                                           acc.as<unsigned long long>() + 1);
      BG_LAUNCH_CHECK();
      unsigned long long got[2];
      BG_CUDA(cudaMemcpyAsync(got, acc.p, 16, cudaMemcpyDeviceToHost, s));
      BG_CUDA(cudaStreamSynchronize(s));
      if (got[0]) {
        if (r->bin_mismatches == 0) {
          std::strncpy(r->first_mismatch_label, ep.label.c_str(), sizeof r->first_mismatch_label - 1);
          r->first_mismatch_row = static_cast<int64_t>(got[1] / static_cast<unsigned long long>(ep.cols));
          r->first_mismatch_col = static_cast<int64_t>(got[1] % static_cast<unsigned long long>(ep.cols));
        }
        r->bin_mismatches += static_cast<int64_t>(got[0]);
      }
    }
  }
  // ref: runreport.cpp:108-133
  if (rows != ref_rows || cols != ref_cols || rows < 0 || cols < 0)
    throw std::logic_error("verify: logit shapes disagree");
  DevBuf olog(static_cast<size_t>(std::max<int64_t>(rows * cols, 1)) * 8);
  if (rows * cols) {
    if (!elog || !ref_logits) fail("verify: missing logits");
    BG_CUDA(cudaMemcpyAsync(olog.p, ref_logits, static_cast<size_t>(rows * cols) * 8, cudaMemcpyHostToDevice, s));
  }
  BG_CUDA(cudaMemsetAsync(static_cast<char*>(acc.p) + 16, 0, 16, s));
  if (rows)
    k_logits_cmp<<<grid_of(rows), 256, 0, s>>>(elog, olog.as<double>(), rows, cols,
                                               acc.as<unsigned long long>() + 2, acc.as<unsigned long long>() + 3);
  BG_LAUNCH_CHECK();
  unsigned long long got[2];
  BG_CUDA(cudaMemcpyAsync(got, static_cast<char*>(acc.p) + 16, 16, cudaMemcpyDeviceToHost, s));
  BG_CUDA(cudaStreamSynchronize(s));
  std::memcpy(&r->max_rel_logit_error, &got[0], 8);
  r->argmax_agreement = rows ? static_cast<double>(got[1]) / static_cast<double>(rows) : 1.0;
  r->pass = r->bin_mismatches == 0 && r->argmax_agreement == 1.0 && r->max_rel_logit_error <= r->tolerance;
}

}  // namespace bg

using namespace bg;

extern "C" {

int bg_verify_trace(const bg_trace* engine, const float* engine_logits, int64_t rows, int64_t cols,
                    const bg_ref_point* ref, int n_ref, const double* ref_logits, int compare_bits,
                    double tolerance, bg_verify_report* out, bg_stream stream) {
  return guard([&] {
    if (!engine || !out) fail("verify: null argument");
    if (n_ref && !ref) fail("verify: null reference points");
    verify_trace(*engine, engine_logits, rows, cols, ref, n_ref, ref_logits, rows, cols, compare_bits, tolerance,
                 out, S(stream));
  });
}

int bg_model_verify(bg_model* m, const bg_mat* x0, const bg_ref_point* ref, int n_ref, const double* ref_logits,
                    int64_t ref_rows, int64_t ref_cols, int compare_bits, double tolerance,
                    bg_verify_report* out, bg_stream stream) {
  return guard([&] {
    if (!m || !x0 || !out) fail("verify: null argument");
    cudaStream_t s = S(stream);
    const Op x = op_from_mat(x0);
    bg_trace t;
    DevBuf o, lg;
    // run_model with a RunTrace: logits = the input of the final softmax
    // (graphops.cpp:457-459); the output width is known after one forward
    int64_t oc = -1;
    for (const auto& l : m->layers)
      if (l.info.has_w1) oc = l.w1.cols;
    if (oc < 0) oc = x.cols;  // no weighted layer: elementwise chain keeps the width
    const size_t bytes = static_cast<size_t>(std::max<int64_t>(x.rows * oc, 1)) * 4;
    o.alloc(bytes);
    lg.alloc(bytes);
    forward_impl(*m, x, o.as<float>(), lg.as<float>(), &t, nullptr, s);
    BG_CUDA(cudaStreamSynchronize(s));
    verify_trace(t, lg.as<float>(), x.rows, oc, ref, n_ref, ref_logits, ref_rows, ref_cols, compare_bits,
                 tolerance, out, s);
  });
}

}  // extern "C"
