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

// exp(d) for d <= 0 in double (the probabilities' exp, graphops.cpp:372-386):
// d = (64 k + j) ln2/64 + r with |r| <= ln2/128 (Cody-Waite, n*hi exact for
// |n| < 2^21), exp(r) by a degree-6 Taylor polynomial (truncation 3e-20),
// times 2^(j/64) from a correctly rounded table, times 2^k.  Within an ulp
// of libm's exp, far below the float rounding of the probabilities; 12 FP64
// operations instead of the 20 of a full-range polynomial (the FP64 exp is
// what bounds the softmax on B200, ncu).
__device__ const double kExp2J64[64] = {
    1.0, 1.0108892860517005, 1.0218971486541166, 1.0330248790212284,
    1.0442737824274138, 1.0556451783605572, 1.0671404006768237, 1.0787607977571199,
    1.0905077326652577, 1.102382583307841, 1.1143867425958924, 1.1265216186082418,
    1.1387886347566916, 1.1511892299529827, 1.1637248587775775, 1.1763969916502812,
    1.189207115002721, 1.202156731452703, 1.215247359980469, 1.22848053610687,
    1.241857812073484, 1.255380757024691, 1.2690509571917332, 1.2828700160787783,
    1.2968395546510096, 1.3109612115247644, 1.3252366431597413, 1.339667524053303,
    1.3542555469368927, 1.3690024229745905, 1.383909881963832, 1.3989796725383112,
    1.4142135623730951, 1.42961333839197, 1.4451808069770467, 1.460917794180647,
    1.4768261459394993, 1.4929077282912648, 1.5091644275934228, 1.5255981507445384,
    1.5422108254079407, 1.559004400237837, 1.5759808451078865, 1.593142151342267,
    1.6104903319492543, 1.6280274218573478, 1.645755478153965, 1.6636765803267364,
    1.681792830507429, 1.7001063537185235, 1.718619298122478, 1.7373338352737062,
    1.7562521603732995, 1.7753764925265212, 1.7947090750031072, 1.8142521755003989,
    1.8340080864093424, 1.8539791250833855, 1.8741676341103, 1.8945759815869656,
    1.9152065613971474, 1.9360617934922943, 1.9571441241754002, 1.978456026387951,
};
__device__ __forceinline__ double exp_nonpos(double d) {
  if (!(d > -745.2)) return d != d ? d : 0.0;  // NaN propagates (as libm's exp); underflow, -inf -> 0
  const double n = rint(d * 92.33248261689366);  // 64 / ln2
  double r = fma(n, -0.010830423794686794, d);  // ln2/64, high 32 bits
  r = fma(n, -9.015623511786383e-10, r);        // ln2/64, low part
  double p = fma(r, 1.0 / 720.0, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int ni = static_cast<int>(n);
  const int k = ni >> 6;  // floor(n / 64)
  p *= __ldg(&kExp2J64[ni & 63]);
  if (k >= -1022) return p * __longlong_as_double(static_cast<long long>(k + 1023) << 52);
  return ldexp(p, k);  // subnormal results
}

}  // namespace bg
