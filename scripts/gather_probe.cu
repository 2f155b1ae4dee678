// Probe: how fast can 115 M random 64-byte records be gathered from an
// L2-resident 15 MB table on one B200?  The layer-1 aggregation of the
// Reddit GCN is one such gather per adjacency bit.
//   ldg    : LDG.128, four lanes per record (the current kernel's access)
//   bulk   : cp.async.bulk (UBLKCP) of each 64 B record into shared memory
//   gather4: cp.async.bulk.tensor.2d tile::gather4 (4 records per TMA op)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe gather_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t err_ = (x);                                                               \
    if (err_ != cudaSuccess) {                                                            \
      std::printf("CUDA %s at %d\n", cudaGetErrorString(err_), __LINE__);                 \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

constexpr int kRec = 64;  // bytes per record

__global__ void k_ldg(const uint4* __restrict__ rec, const uint32_t* __restrict__ idx, int64_t e,
                      uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  uint32_t acc = 0;
  for (int64_t b = warp * 32; b < e; b += warps * 32) {
    const uint32_t my = b + lane < e ? __ldg(idx + b + lane) : 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // 8 records per step, 4 steps per 32 edges
      const uint32_t j = __shfl_sync(0xFFFFFFFFu, my, 8 * k + (lane >> 2));
      const uint4 v = __ldg(rec + static_cast<int64_t>(j) * 4 + (lane & 3));
      acc ^= v.x + v.y + v.z + v.w;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// records of RB bytes (16/32/64), RB/16 lanes per record
template <int RB>
__global__ void k_ldg_sz(const uint4* __restrict__ rec, const uint32_t* __restrict__ idx, int64_t e,
                         uint32_t* __restrict__ out) {
  constexpr int LPR = RB / 16, RPI = 32 / LPR;  // lanes per record, records per instruction
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  uint32_t acc = 0;
  for (int64_t b = warp * 32; b < e; b += warps * 32) {
    const uint32_t my = b + lane < e ? __ldg(idx + b + lane) : 0;
#pragma unroll
    for (int k = 0; k < 32 / RPI; ++k) {
      const uint32_t j = __shfl_sync(0xFFFFFFFFu, my, RPI * k + lane / LPR);
      const uint4 v = __ldg(rec + static_cast<int64_t>(j) * LPR + (lane % LPR));
      acc ^= v.x + v.y + v.z + v.w;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(
          smem_u32(m)),
      "r"(parity)
      : "memory");
}

constexpr int kStages = 4;
constexpr int kWarps = 4;

// One warp per stream of edges, a ring of kStages x 32 records per warp.
template <int MODE>  // 0: one bulk copy per record, 1: gather4
__global__ void __launch_bounds__(kWarps * 32) k_tma(const uint4* __restrict__ rec, const __grid_constant__ CUtensorMap tm,
                                                     const uint32_t* __restrict__ idx, int64_t e,
                                                     uint32_t* __restrict__ out) {
  __shared__ __align__(128) uint4 ring[kWarps][kStages][32 * 4];
  __shared__ __align__(8) uint64_t bar[kWarps][kStages];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0)
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[w][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t warp = blockIdx.x * static_cast<int64_t>(kWarps) + w;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * kWarps;
  uint32_t acc = 0;
  const int64_t nb = (e + 31) / 32;
  auto issue = [&](int64_t batch, int s) {
    const int64_t b = batch * 32;
    const uint32_t my = b + lane < e ? __ldg(idx + b + lane) : 0;
    if (lane == 0) mbar_expect(&bar[w][s], 32 * kRec);
    __syncwarp();
    if (MODE == 0) {
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(&ring[w][s][lane * 4])),
          "l"(rec + static_cast<int64_t>(my) * 4), "r"(kRec), "r"(smem_u32(&bar[w][s]))
          : "memory");
    } else {
      const uint32_t j0 = __shfl_sync(0xFFFFFFFFu, my, (lane & 7) * 4 + 0);
      const uint32_t j1 = __shfl_sync(0xFFFFFFFFu, my, (lane & 7) * 4 + 1);
      const uint32_t j2 = __shfl_sync(0xFFFFFFFFu, my, (lane & 7) * 4 + 2);
      const uint32_t j3 = __shfl_sync(0xFFFFFFFFu, my, (lane & 7) * 4 + 3);
      if (lane < 8)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(&ring[w][s][lane * 16])),
            "l"(&tm), "r"(0), "r"(j0), "r"(j1), "r"(j2), "r"(j3), "r"(smem_u32(&bar[w][s]))
            : "memory");
    }
  };
  int64_t my_batches = 0;
  for (int64_t bt = warp; bt < nb; bt += warps) ++my_batches;
  for (int s = 0; s < kStages && s < my_batches; ++s) issue(warp + s * warps, s);
  for (int64_t t = 0; t < my_batches; ++t) {
    const int s = static_cast<int>(t % kStages);
    mbar_wait(&bar[w][s], static_cast<uint32_t>((t / kStages) & 1));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 v = ring[w][s][k * 32 + lane];
      acc ^= v.x + v.y + v.z + v.w;
    }
    __syncwarp();
    if (t + kStages < my_batches) issue(warp + (t + kStages) * warps, s);
  }
  if (acc == 0x12345678u) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int64_t n = 232966, e = 114727589;
  std::vector<uint32_t> h(static_cast<size_t>(e));
  std::mt19937 g(1);
  for (auto& v : h) v = g() % static_cast<uint32_t>(n);
  uint4* rec;
  uint32_t *idx, *out;
  CK(cudaMalloc(&rec, n * kRec));
  CK(cudaMemset(rec, 1, n * kRec));
  CK(cudaMalloc(&idx, e * 4));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemcpy(idx, h.data(), e * 4, cudaMemcpyHostToDevice));
  // tensor map: n rows x 16 u32 columns, box 16 x 1 (gather4 loads 4 such rows)
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  CUtensorMap tmh;
  cuuint64_t dims[2] = {16, static_cast<cuuint64_t>(n)}, strides[1] = {kRec};
  cuuint32_t box[2] = {16, 1}, es[2] = {1, 1};
  CUresult r = reinterpret_cast<EncodeFn>(fn)(&tmh, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, rec, dims, strides, box, es,
                                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  std::printf("encode: %d\n", static_cast<int>(r));
  CUtensorMap* tm;
  CK(cudaMalloc(&tm, sizeof tmh));
  CK(cudaMemcpy(tm, &tmh, sizeof tmh, cudaMemcpyHostToDevice));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto time = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    const int reps = 10;
    for (int i = 0; i < reps; ++i) launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    ms /= reps;
    std::printf("%-10s %.4f ms  %.1f Grec/s  %.0f GB/s\n", name, ms, e / (ms * 1e-3) / 1e9,
                e * double(kRec) / (ms * 1e-3) / 1e9);
  };
  for (int occ : {4, 8, 16})
    time(occ == 4 ? "ldg x4" : occ == 8 ? "ldg x8" : "ldg x16",
         [&] { k_ldg<<<sms * occ, 256>>>(rec, idx, e, out); });
  time("ldg16 x8", [&] { k_ldg_sz<16><<<sms * 8, 256>>>(rec, idx, e, out); });
  time("ldg32 x8", [&] { k_ldg_sz<32><<<sms * 8, 256>>>(rec, idx, e, out); });
  time("ldg64 x8", [&] { k_ldg_sz<64><<<sms * 8, 256>>>(rec, idx, e, out); });
  time("ldg32 x16", [&] { k_ldg_sz<32><<<sms * 16, 256>>>(rec, idx, e, out); });
  for (int occ : {4, 8, 16}) {
    time(occ == 4 ? "bulk x4" : occ == 8 ? "bulk x8" : "bulk x16",
         [&] { k_tma<0><<<sms * occ, kWarps * 32>>>(rec, tmh, idx, e, out); });
    if (r == CUDA_SUCCESS)
      time(occ == 4 ? "gath4 x4" : occ == 8 ? "gath4 x8" : "gath4 x16",
           [&] { k_tma<1><<<sms * occ, kWarps * 32>>>(rec, tmh, idx, e, out); });
  }
  CK(cudaGetLastError());
  return 0;
}
