// Is the windowed bit-SpMM's operand stream (every CTA bulk-copies the whole
// 3.7 MB operand into shared memory, 64 KB at a time) limited per SM or by
// L2?  Each CTA streams the buffer `reps` times through a 3-slot ring; the
// aggregate L2->SM rate at 148 / 74 / 37 CTAs answers it.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/bulk_l2_probe scripts/bulk_l2_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void k_stream(const uint8_t* src, uint32_t bytes, int reps, int* sink) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t bar[3];
  constexpr uint32_t kSlot = 64 * 1024;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 3; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint32_t n = bytes / kSlot;
  const uint32_t total = n * reps;
  if (threadIdx.x == 0) {
    for (uint32_t u = 0; u < total; ++u) {
      const int s = u % 3;
      if (u >= 3) {  // wait for the slot's previous copy
        const uint32_t par = ((u / 3) - 1) & 1;
        asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(sa(&bar[s])), "r"(par));
      }
      const uint8_t* g = src + static_cast<uint64_t>(u % n) * kSlot;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(kSlot));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(ring + s * kSlot)), "l"(g), "r"(kSlot), "r"(sa(&bar[s])) : "memory");
    }
    for (uint32_t u = total > 3 ? total - 3 : 0; u < total; ++u) {
      const int s = u % 3;
      const uint32_t par = (u / 3) & 1;
      asm volatile("{\n .reg .pred p;\n W2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W2;\n}\n" ::"r"(sa(&bar[s])), "r"(par));
    }
    sink[blockIdx.x] = ring[blockIdx.x % 1000];
  }
}

int main() {
  const uint32_t bytes = 57 * 64 * 1024;  // ~3.7 MB: Reddit's packed operand
  uint8_t* src; int* sink;
  cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
  cudaMalloc(&sink, 4096 * 4);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 64 * 1024);
  for (int grid : {148, 74, 37, 16}) {
    const int reps = 4;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k_stream<<<grid, 32, 3 * 64 * 1024>>>(src, bytes, reps, sink);
    cudaEventRecord(a);
    k_stream<<<grid, 32, 3 * 64 * 1024>>>(src, bytes, reps, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double tot = static_cast<double>(bytes) * reps * grid;
    printf("CTAs %3d: %.3f ms, aggregate %.0f GB/s, per SM %.1f GB/s\n", grid, ms, tot / ms / 1e6, tot / ms / 1e6 / grid);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
