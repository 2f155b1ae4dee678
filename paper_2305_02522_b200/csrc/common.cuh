// Shared internals of the B200 binary-GNN library: error plumbing, device
// buffers, launch helpers, bit utilities.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <utility>

#include "bitgnn_b200.h"

namespace bg {

// Thrown for device failures; mapped to BG_CUDA_ERROR.
struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

#define BG_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::bg::cuda_error(std::string("CUDA error: ") + cudaGetErrorString(e_) +     \
                             " at " __FILE__ ":" + std::to_string(__LINE__));           \
  } while (0)

#define BG_LAUNCH_CHECK() BG_CUDA(cudaGetLastError())

// Runs f and converts exceptions into status codes + bg_last_error().
template <class F>
int guard(F&& f) {
  try {
    f();
    return BG_OK;
  } catch (const cuda_error& e) {
    set_last_error(e.what());
    return BG_CUDA_ERROR;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return BG_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    set_last_error(e.what());
    return BG_LOGIC_ERROR;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return BG_RUNTIME_ERROR;
  } catch (...) {
    set_last_error("unknown error");
    return BG_RUNTIME_ERROR;
  }
}

[[noreturn]] inline void fail(const std::string& m) { throw std::invalid_argument(m); }

inline cudaStream_t S(bg_stream s) { return static_cast<cudaStream_t>(s); }

inline int64_t spw(int64_t cols, int wb) { return (cols + wb - 1) / wb * (wb / 32); }

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Owning device allocation.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(size_t n) { alloc(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr, o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(bytes, o.bytes);
    return *this;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void alloc(size_t n) {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = n;
    if (n) BG_CUDA(cudaMalloc(&p, n));
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

int sm_count();

// ---- device helpers ---------------------------------------------------- //
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Valid-bit mask of the last u32 word of an n-bit row (MSB-first).
__host__ __device__ __forceinline__ uint32_t tail_mask32(int64_t n) {
  const int rem = static_cast<int>(n & 31);
  return rem == 0 ? 0xFFFFFFFFu : (0xFFFFFFFFu << (32 - rem));
}

template <class T>
__device__ __forceinline__ T ldg(const T* p) {
  return __ldg(p);
}

// exp(d) for d <= 0 in double: Cody-Waite reduction d = n ln2 + r, |r| <=
// ln2/2, degree-13 Taylor polynomial (truncation < 5e-18 relative, Estrin
// scheme), scale by
// 2^n.  Within an ulp of libm's exp, far below the float rounding of the
// probabilities.
__device__ __forceinline__ double exp_nonpos(double d) {
  if (!(d > -745.2)) return d != d ? d : 0.0;  // NaN propagates (as libm's exp); underflow, -inf -> 0
  const double n = rint(d * 1.4426950408889634);
  double r = fma(n, -6.93147180369123816490e-01, d);
  r = fma(n, -1.90821492927058770002e-10, r);
  // Estrin evaluation of sum_{i<=13} r^i / i!: dependency depth 5 instead of
  // Horner's 14 (the kernels using it are FP64-latency-bound)
  const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
  const double a0 = fma(r, 1.0, 1.0), a1 = fma(r, 1.0 / 6.0, 0.5), a2 = fma(r, 1.0 / 120.0, 1.0 / 24.0),
               a3 = fma(r, 1.0 / 5040.0, 1.0 / 720.0), a4 = fma(r, 1.0 / 362880.0, 1.0 / 40320.0),
               a5 = fma(r, 1.0 / 39916800.0, 1.0 / 3628800.0), a6 = fma(r, 1.0 / 6227020800.0, 1.0 / 479001600.0);
  const double b0 = fma(a1, r2, a0), b1 = fma(a3, r2, a2), b2 = fma(a5, r2, a4);
  const double d0 = fma(b1, r4, b0), d1 = fma(a6, r4, b2);
  const double p = fma(d1, r8, d0);
  const int ni = static_cast<int>(n);
  if (ni >= -1022) return p * __longlong_as_double(static_cast<long long>(ni + 1023) << 52);
  return ldexp(p, ni);  // subnormal results
}

}  // namespace bg
