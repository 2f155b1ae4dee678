// Probe: how does sm_100a serve an LDS.128 whose 32 lanes hit various
// 16-byte bank groups (addr/16 mod 8)?  Read the ncu counters
// l1tex__data_pipe_lsu_wavefronts_mem_shared / _bank_conflicts per kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_bank_probe lds_bank_probe.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
template <int PAT>
__global__ void k(uint32_t* out, int iters) {
  __shared__ uint4 buf[2048];
  const int lane = threadIdx.x & 31;
  int rec;
  switch (PAT) {
    case 0: rec = lane; break;                           // consecutive: 4 ideal
    case 1: rec = lane * 8; break;                       // all bank group 0
    case 2: rec = (lane & 7) + 64 * (lane >> 3); break;  // each quarter covers 8 groups
    case 3: rec = (lane >> 2) + 64 * (lane & 3); break;  // group = lane/4: quarters have 2 groups x 4
    case 4: rec = (lane & 7) * 9 + 256 * (lane >> 3); break;  // quarter perfect, scattered
    case 5: rec = (lane < 16) ? 7 : lane; break;         // half broadcast
    default: rec = ((lane * 37) % 32) * 8 + (lane & 7); break;
  }
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
  uint32_t acc = 0;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const uint4 v = lds128(base + 16u * ((rec + (it & 1) * 1024) & 2047));
    acc += v.x ^ v.y ^ v.z ^ v.w ^ it;
  }
  if (acc == 0x1234567u) out[0] = acc;
}
int main() {
  uint32_t* o;
  cudaMalloc(&o, 4);
  k<0><<<1, 32>>>(o, 1000);
  k<1><<<1, 32>>>(o, 1000);
  k<2><<<1, 32>>>(o, 1000);
  k<3><<<1, 32>>>(o, 1000);
  k<4><<<1, 32>>>(o, 1000);
  k<5><<<1, 32>>>(o, 1000);
  cudaDeviceSynchronize();
  printf("done\n");
}
