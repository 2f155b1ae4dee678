// Column-windowed bit-SpMM (BSpMM.BBB / BBF, ref kernels.cpp:254-333 and the
// emit loop :438-465): out(i,k) = 2*#{j in N(i): x_jk = 1} - deg_i.
//
// Why: the per-edge gather of a 16-byte packed neighbour row from L2 costs one
// L1TEX wavefront per edge (ncu: k_sl_bb runs at 87% of L1TEX throughput), so
// a dense graph is bound at ~1 edge/clk/SM no matter how the loads are shaped.
// Here the packed operand is streamed through shared memory instead, one
// column window of Wn node rows at a time (cp.async.bulk + mbarrier, double
// buffered), and each edge becomes one 16-byte LDS.  The CTA owns a block of
// T node rows, one per thread, whose bit-sliced counters stay in registers
// for the whole sweep over the windows.  Counting is order-free integer work,
// so the result equals the reference's TwoAndMinusPopc/IfElse/AndAndNot
// strategies bit for bit.
//
// Adjacency layout (bg_frdc::Windows, ops.cuh): per (row block, window,
// warp) an ELL segment of u16 window-local columns, 4 per lane per group, so a
// warp's loop count is uniform and every entry load is a coalesced 8-byte
// load; padding entries point at a zero record stored after the window.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "ops.cuh"
#include "tilewalk.cuh"
#include "async.cuh"

namespace bg {
namespace {

// Window buffers share 221 KB of shared memory (13824 records); Wn + 1 a
// multiple of 8 keeps the bank group of a record the same in every buffer
// (k_win_bankorder).  2 buffers -> Wn = 6911.
constexpr int kWinSmemRecords = 13824;
constexpr int kWinMaxBuf = 4;
constexpr int kWinDefaultBuffers = 2;
constexpr int kWinRec = 16;
constexpr int kWinMaxThreads = 576;  // 18 warps: <= 112 registers per thread             // bytes per packed node row (4 u32 words)

__device__ __forceinline__ uint2 ld_nc_v2(const uint2* p) {
  uint2 v;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

// ---- view construction (build once) -----------------------------------------

// Thread per node row: entries per window (u16, row-major rows x nw).
__global__ void k_win_count(const uint64_t* __restrict__ srp, const uint32_t* __restrict__ sl,
                            int64_t rows, int Wn, int nw, uint16_t* __restrict__ cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  uint16_t* c = cnt + i * nw;
  int cur = -1;
  uint32_t run = 0;
  for_each_col(srp, sl, i, [&](uint32_t col) {
    const int w = static_cast<int>(col / static_cast<uint32_t>(Wn));
    if (w != cur) {
      if (cur >= 0) c[cur] = static_cast<uint16_t>(run);
      cur = w;
      run = 0;
    }
    ++run;
  });
  if (cur >= 0) c[cur] = static_cast<uint16_t>(run);
}

// Thread per segment: ELL groups = ceil(max entries of the warp's rows / 4).
__global__ void k_win_seglen(const uint16_t* __restrict__ cnt, int64_t rows, int T, int nw,
                             int64_t nseg, uint32_t* __restrict__ len) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s > nseg) return;
  if (s == nseg) {
    len[s] = 0;
    return;
  }
  const int nwarps = T / 32;
  const int64_t b = s / (static_cast<int64_t>(nw) * nwarps);
  const int64_t r = s % (static_cast<int64_t>(nw) * nwarps);
  const int w = static_cast<int>(r / nwarps), v = static_cast<int>(r % nwarps);
  uint32_t k = 0;
  for (int l = 0; l < 32; ++l) {
    const int64_t i = b * T + v * 32 + l;
    if (i < rows) k = max(k, static_cast<uint32_t>(cnt[i * nw + w]));
  }
  len[s] = (k + 3) / 4;
}

__global__ void k_fill_u16(uint16_t* __restrict__ p, int64_t n, uint16_t v) {
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[t] = v;
}

// Thread per node row: scatter its columns into the ELL slots of its lane.
__global__ void k_win_fill(const uint64_t* __restrict__ srp, const uint32_t* __restrict__ sl,
                           int64_t rows, int T, int Wn, int nw, const uint32_t* __restrict__ seg,
                           uint16_t* __restrict__ ell) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int nwarps = T / 32;
  const int64_t b = i / T;
  const int v = static_cast<int>((i % T) / 32), lane = static_cast<int>(i % 32);
  int cur = -1;
  uint32_t k = 0;
  uint64_t base = 0;
  for_each_col(srp, sl, i, [&](uint32_t col) {
    const int w = static_cast<int>(col / static_cast<uint32_t>(Wn));
    if (w != cur) {
      cur = w;
      k = 0;
      base = static_cast<uint64_t>(seg[(b * nw + w) * nwarps + v]) * 128 + lane * 4;
    }
    ell[base + (k >> 2) * 128 + (k & 3)] = static_cast<uint16_t>(col - static_cast<uint32_t>(w) * Wn);
    ++k;
  });
}

// Bank-aware slot order (build once).  An LDS.128 is served per quarter warp
// (8 lanes, 128 bytes): lanes of a quarter whose records sit in the same
// 16-byte bank group (record index mod 8, the window stride being a multiple
// of 8 records) and differ in address cost an extra wavefront each.  Counting
// is order-free, so each lane's entries may be permuted freely: thread per
// (segment, quarter) fills slot k greedily with, per lane, an entry of a bank
// group no other lane of the quarter uses in that slot (looking a bounded
// distance ahead in the lane's list).
__global__ void k_win_bankorder(const uint32_t* __restrict__ seg, int64_t nseg, int Wn,
                                uint16_t* __restrict__ ell) {
  constexpr int kLook = 48;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nseg * 4) return;
  const int64_t s = t >> 2;
  const int q = static_cast<int>(t & 3);
  const uint64_t base = static_cast<uint64_t>(seg[s]) * 128;
  const uint32_t K = (seg[s + 1] - seg[s]) * 4;
  if (K == 0) return;
  auto at = [&](int l, uint32_t k) -> uint16_t& {
    return ell[base + (k >> 2) * 128 + (8 * q + l) * 4 + (k & 3)];
  };
  uint32_t cnt[8];
  for (int l = 0; l < 8; ++l) {
    uint32_t c = 0;
    while (c < K && at(l, c) != Wn) ++c;
    cnt[l] = c;
  }
  const uint32_t sent_bit = 1u << (Wn & 7);
  for (uint32_t k = 0; k < K; ++k) {
    uint32_t used = 0;
    for (int l = 0; l < 8; ++l)
      if (cnt[l] <= k) used |= sent_bit;
    for (int l = 0; l < 8; ++l) {
      if (cnt[l] <= k) continue;
      const uint32_t end = min(cnt[l], k + kLook);
      uint32_t pick = k;
      for (uint32_t j = k; j < end; ++j)
        if (!((used >> (at(l, j) & 7u)) & 1u)) {
          pick = j;
          break;
        }
      const uint16_t e = at(l, pick);
      if (pick != k) {
        at(l, pick) = at(l, k);
        at(l, k) = e;
      }
      used |= 1u << (e & 7u);
    }
  }
}

// ---- the aggregation kernel ---------------------------------------------------

// Harley-Seal over 8 words into planes P[0..2]; returns the weight-8 carry.
template <int NP>
__device__ __forceinline__ uint32_t hs8_low(uint32_t (&P)[NP], const uint32_t (&x)[8]) {
  uint32_t t1, t2, f1, f2, e, s;
  s = P[0] ^ x[0] ^ x[1]; t1 = maj3(P[0], x[0], x[1]); P[0] = s;
  s = P[0] ^ x[2] ^ x[3]; t2 = maj3(P[0], x[2], x[3]); P[0] = s;
  s = P[1] ^ t1 ^ t2;     f1 = maj3(P[1], t1, t2);     P[1] = s;
  s = P[0] ^ x[4] ^ x[5]; t1 = maj3(P[0], x[4], x[5]); P[0] = s;
  s = P[0] ^ x[6] ^ x[7]; t2 = maj3(P[0], x[6], x[7]); P[0] = s;
  s = P[1] ^ t1 ^ t2;     f2 = maj3(P[1], t1, t2);     P[1] = s;
  s = P[2] ^ f1 ^ f2;     e = maj3(P[2], f1, f2);      P[2] = s;
  return e;
}

// Ripple a carry word of weight 2^q0 into planes q0.. (counts stay < 2^NP).
template <int NP>
__device__ __forceinline__ void ripple(uint32_t (&P)[NP], uint32_t c, int q0) {
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    if (q < q0) continue;
    const uint32_t nq = P[q] ^ c;
    c &= P[q];
    P[q] = nq;
  }
}

template <int NP, bool OUTB>
__global__ void __launch_bounds__(NP <= 10 ? kWinMaxThreads : 480, 1)
    k_win_bb(const uint32_t* __restrict__ seg, const uint16_t* __restrict__ ell, int nw, int Wn, int nbuf,
             int64_t rows, int64_t row0, int64_t row1, int b0, int b1,
             const int32_t* __restrict__ degree, const uint4* __restrict__ x, int64_t f,
             uint32_t* __restrict__ out_bits, float* __restrict__ out_f) {
  static_assert(NP >= 5, "two-level Harley-Seal needs planes 0..4");
  extern __shared__ __align__(16) uint4 sbuf[];  // nbuf windows of (Wn + 1) records
  __shared__ __align__(8) uint64_t full[kWinMaxBuf];
  __shared__ uint32_t done[kWinMaxBuf];  // warps finished with each buffer (monotone)
  const int tid = threadIdx.x, T = blockDim.x, nwarps = T >> 5, warp = tid >> 5, lane = tid & 31;
  const int stride = Wn + 1;
  if (tid < nbuf) {
    sbuf[tid * stride + Wn] = make_uint4(0u, 0u, 0u, 0u);  // padding target
    done[tid] = 0;
    mbar_init(&full[tid], 1);
  }
  if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int mine = b1 - b0 - static_cast<int>(blockIdx.x);
  const int nblk = mine > 0 ? (mine + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x) : 0;
  const int nsteps = nblk * nw;
  auto issue = [&](int step) {
    const int w = step % nw, buf = step % nbuf;
    const int64_t n0 = static_cast<int64_t>(w) * Wn;
    const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(Wn), rows - n0)) * kWinRec;
    mbar_expect_tx(&full[buf], bytes);
    bulk_g2s(sbuf + buf * stride, x + n0, bytes, &full[buf]);
  };
  if (tid == 0)
    for (int k = 0; k < nbuf && k < nsteps; ++k) issue(k);
  auto seg_of = [&](int step) -> int64_t {
    const int bi = step / nw, w = step - bi * nw;
    const int b = b0 + static_cast<int>(blockIdx.x) + bi * static_cast<int>(gridDim.x);
    return (static_cast<int64_t>(b) * nw + w) * nwarps + warp;
  };
  const uint32_t sent = static_cast<uint32_t>(Wn) | (static_cast<uint32_t>(Wn) << 16);
  const uint2 sent2 = make_uint2(sent, sent);
  const uint2* ell2 = reinterpret_cast<const uint2*>(ell) + lane;
  const uint32_t sbase = smem_addr(sbuf);
  auto ld_group = [&](uint32_t g, uint32_t g1) { return g < g1 ? ld_nc_v2(ell2 + static_cast<size_t>(g) * 32) : sent2; };
  uint32_t P[4][NP];
  // 8 entries (two ELL groups): 8 LDS.128, Harley-Seal into planes 0..2 of
  // every word, weight-8 carries out
  auto batch = [&](uint32_t wbase, uint2 a, uint2 c, uint32_t (&e)[4]) {
    const uint32_t pk[4] = {a.x, a.y, c.x, c.y};
    uint4 v[8];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const uint32_t lo = wbase + ((pk[m] & 0xFFFFu) << 4);
      const uint32_t hi = wbase + ((pk[m] >> 16) << 4);
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v[2 * m].x), "=r"(v[2 * m].y), "=r"(v[2 * m].z), "=r"(v[2 * m].w)
                   : "r"(lo));
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v[2 * m + 1].x), "=r"(v[2 * m + 1].y), "=r"(v[2 * m + 1].z), "=r"(v[2 * m + 1].w)
                   : "r"(hi));
    }
    uint32_t xw[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) xw[m] = v[m].x;
    e[0] = hs8_low<NP>(P[0], xw);
#pragma unroll
    for (int m = 0; m < 8; ++m) xw[m] = v[m].y;
    e[1] = hs8_low<NP>(P[1], xw);
#pragma unroll
    for (int m = 0; m < 8; ++m) xw[m] = v[m].z;
    e[2] = hs8_low<NP>(P[2], xw);
#pragma unroll
    for (int m = 0; m < 8; ++m) xw[m] = v[m].w;
    e[3] = hs8_low<NP>(P[3], xw);
  };
  // the current step's first four ELL groups, prefetched a step ahead
  uint32_t g0 = 0, g1 = 0;
  uint2 q0 = sent2, q1 = sent2, q2 = sent2, q3 = sent2;
  if (nsteps > 0) {
    const int64_t s0 = seg_of(0);
    g0 = __ldg(seg + s0);
    g1 = __ldg(seg + s0 + 1);
    q0 = ld_group(g0, g1);
    q1 = ld_group(g0 + 1, g1);
    q2 = ld_group(g0 + 2, g1);
    q3 = ld_group(g0 + 3, g1);
  }
  for (int step = 0; step < nsteps; ++step) {
    const int w = step % nw, buf = step % nbuf;
    if (w == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < NP; ++p) P[q][p] = 0u;
    }
    uint32_t ng0 = 0, ng1 = 0;  // segment bounds of the next step
    if (step + 1 < nsteps) {
      const int64_t sn = seg_of(step + 1);
      ng0 = __ldg(seg + sn);
      ng1 = __ldg(seg + sn + 1);
    }
    mbar_wait(&full[buf], static_cast<uint32_t>(step / nbuf) & 1u);
    const uint32_t wbase = sbase + static_cast<uint32_t>(buf * stride) * kWinRec;
    uint32_t g = g0;
    for (; g + 4 <= g1; g += 4) {
      const uint2 n0 = ld_group(g + 4, g1), n1 = ld_group(g + 5, g1);
      const uint2 n2 = ld_group(g + 6, g1), n3 = ld_group(g + 7, g1);
      uint32_t eA[4], eB[4];
      batch(wbase, q0, q1, eA);
      batch(wbase, q2, q3, eB);
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // two weight-8 carries: CSA into plane 3, ripple from 4
        const uint32_t s3 = P[q][3] ^ eA[q] ^ eB[q];
        const uint32_t cy = maj3(P[q][3], eA[q], eB[q]);
        P[q][3] = s3;
        ripple<NP>(P[q], cy, 4);
      }
      q0 = n0;
      q1 = n1;
      q2 = n2;
      q3 = n3;
    }
    if (g < g1) {  // 1..3 groups left (the rest of q0..q3 is padding)
      uint32_t eA[4];
      batch(wbase, q0, q1, eA);
#pragma unroll
      for (int q = 0; q < 4; ++q) ripple<NP>(P[q], eA[q], 3);
      if (g + 2 < g1) {
        batch(wbase, q2, q3, eA);
#pragma unroll
        for (int q = 0; q < 4; ++q) ripple<NP>(P[q], eA[q], 3);
      }
    }
    // prefetch the next step's first groups, then release this buffer; the
    // last warp out refills it with the window nbuf steps ahead
    q0 = ld_group(ng0, ng1);
    q1 = ld_group(ng0 + 1, ng1);
    q2 = ld_group(ng0 + 2, ng1);
    q3 = ld_group(ng0 + 3, ng1);
    g0 = ng0;
    g1 = ng1;
    __syncwarp();
    if (lane == 0) {
      const uint32_t prev = atomicAdd(&done[buf], 1u);
      if (prev + 1 == static_cast<uint32_t>(nwarps) * static_cast<uint32_t>(step / nbuf + 1) &&
          step + nbuf < nsteps) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(step + nbuf);
      }
    }
    if (w == nw - 1) {
      const int bi = step / nw;
      const int b = b0 + static_cast<int>(blockIdx.x) + bi * static_cast<int>(gridDim.x);
      const int64_t i = static_cast<int64_t>(b) * T + tid;
      if (i >= row0 && i < row1) {
        const uint32_t deg = static_cast<uint32_t>(__ldg(degree + i));
        if (OUTB) {
          uint32_t o[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            // cnt >= ceil(deg/2)  <=>  2*cnt - deg >= 0   (kernels.cpp:440-454)
            uint32_t ge = planes_ge<NP>(P[q], (deg + 1) >> 1);
            if (32 * (q + 1) > f) ge &= (32 * q >= f) ? 0u : tail_mask32(f);
            o[q] = ge;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) out_bits[i * 4 + q] = o[q];
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            for (int bb = 0; bb < 32; ++bb) {
              const int64_t k = 32 * q + bb;
              if (k >= f) break;
              out_f[i * f + k] = static_cast<float>(2 * static_cast<int64_t>(plane_count<NP>(P[q], bb)) -
                                                    static_cast<int64_t>(deg));
            }
        }
      }
    }
  }
}

bool window_forced() { return aggregation_mode() == BG_AGG_WINDOW; }

size_t win_smem_bytes(int Wn, int nbuf) { return static_cast<size_t>(nbuf) * static_cast<size_t>(Wn + 1) * kWinRec; }

int win_buffers() {
  static const int v = [] {
    const char* e = std::getenv("BG_WINDOW_BUFFERS");
    const int n = e && *e ? std::atoi(e) : kWinDefaultBuffers;
    return std::max(1, std::min(n, kWinMaxBuf));
  }();
  return v;
}

// Largest block (multiple of 32 threads) the kernel instance can run with the
// given dynamic shared memory, one CTA per SM.
template <class K>
int max_threads(K kern, size_t smem) {
  BG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int t = 1024;
  for (; t >= 32; t -= 32) {
    int nb = 0;
    BG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, t, smem));
    if (nb >= 1) break;
  }
  if (t < 32) fail("window_bb: kernel does not fit on an SM");
  return t;
}

void build_windows(bg_frdc& A, int T, int Wn, cudaStream_t s) {
  auto& W = A.win;
  if (W.T == T && W.Wn == Wn) return;
  frdc_slivers(A, s);
  const int64_t rows = A.rows;
  const int nw = static_cast<int>(cdiv(A.cols, Wn));
  const int nb = static_cast<int>(cdiv(rows, T));
  const int64_t nseg = static_cast<int64_t>(nb) * nw * (T / 32);
  DevBuf cnt(static_cast<size_t>(std::max<int64_t>(rows * nw, 1)) * 2);
  DevBuf len(static_cast<size_t>(nseg + 1) * 4);
  W.seg.alloc(static_cast<size_t>(nseg + 1) * 4);
  BG_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes, s));
  if (rows > 0)
    k_win_count<<<static_cast<unsigned>(cdiv(rows, 256)), 256, 0, s>>>(A.srp(), A.sl(), rows, Wn, nw,
                                                                       cnt.as<uint16_t>());
  BG_LAUNCH_CHECK();
  k_win_seglen<<<static_cast<unsigned>(cdiv(nseg + 1, 256)), 256, 0, s>>>(cnt.as<uint16_t>(), rows, T, nw,
                                                                          nseg, len.as<uint32_t>());
  BG_LAUNCH_CHECK();
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, len.as<uint32_t>(), W.seg.as<uint32_t>(),
                                static_cast<int>(nseg + 1), s);
  DevBuf tmp(std::max<size_t>(tmp_bytes, 1));
  cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, len.as<uint32_t>(), W.seg.as<uint32_t>(),
                                static_cast<int>(nseg + 1), s);
  BG_LAUNCH_CHECK();
  uint32_t groups = 0;
  BG_CUDA(cudaMemcpyAsync(&groups, W.seg.as<uint32_t>() + nseg, 4, cudaMemcpyDeviceToHost, s));
  BG_CUDA(cudaStreamSynchronize(s));
  const int64_t n16 = static_cast<int64_t>(groups) * 128;
  W.ell.alloc(static_cast<size_t>(std::max<int64_t>(n16, 8)) * 2);
  k_fill_u16<<<static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(cdiv(n16, 256), 65536))), 256, 0, s>>>(
      W.ell.as<uint16_t>(), n16, static_cast<uint16_t>(Wn));
  BG_LAUNCH_CHECK();
  if (rows > 0)
    k_win_fill<<<static_cast<unsigned>(cdiv(rows, 256)), 256, 0, s>>>(A.srp(), A.sl(), rows, T, Wn, nw,
                                                                      W.seg.as<uint32_t>(), W.ell.as<uint16_t>());
  BG_LAUNCH_CHECK();
  if (nseg > 0)
    k_win_bankorder<<<static_cast<unsigned>(cdiv(nseg * 4, 128)), 128, 0, s>>>(W.seg.as<uint32_t>(), nseg, Wn,
                                                                              W.ell.as<uint16_t>());
  BG_LAUNCH_CHECK();
  BG_CUDA(cudaStreamSynchronize(s));
  W.T = T;
  W.Wn = Wn;
  W.nw = nw;
  W.nb = nb;
}

template <int NP, bool OUTB>
bool launch_win(bg_frdc& A, const uint32_t* x, int64_t f, uint32_t* ob, float* of, int64_t r0,
                int64_t r1, cudaStream_t s) {
  auto kern = k_win_bb<NP, OUTB>;
  const int sms = sm_count();
  const int nbuf = win_buffers();
  const int wmax = kWinSmemRecords / nbuf / 8 * 8 - 1;
  const int Wn = std::max(1, std::min<int>(window_nodes_setting() > 0 ? std::min(window_nodes_setting(), wmax) : wmax,
                                           static_cast<int>(A.cols)));
  static const int tmax = max_threads(kern, static_cast<size_t>(kWinSmemRecords) * kWinRec);  // per instance
  const int64_t waves = std::max<int64_t>(1, cdiv(A.rows, static_cast<int64_t>(sms) * tmax));
  const int T = static_cast<int>(std::min<int64_t>(
      tmax, cdiv(cdiv(A.rows, static_cast<int64_t>(sms) * waves), 32) * 32));
  if (!window_forced()) {
    // cost model: bytes streamed into shared memory per adjacency bit vs the
    // ~32-byte L2 sector an edge gather costs
    const double streamed = static_cast<double>(waves) * sms * static_cast<double>(A.cols) * kWinRec;
    if (A.nnz_bits < (int64_t{1} << 22) || streamed > 20.0 * static_cast<double>(A.nnz_bits)) return false;
  }
  build_windows(A, T, Wn, s);
  const auto& W = A.win;
  const int b0 = static_cast<int>(r0 / T), b1 = static_cast<int>(cdiv(r1, T));
  const int grid = std::min(sms, b1 - b0);
  kern<<<grid, T, win_smem_bytes(Wn, nbuf), s>>>(W.seg.as<uint32_t>(), W.ell.as<uint16_t>(), W.nw, W.Wn, nbuf, A.rows,
                                           r0, r1, b0, b1, A.deg(), reinterpret_cast<const uint4*>(x), f, ob,
                                           of);
  BG_LAUNCH_CHECK();
  return true;
}

template <bool OUTB>
bool launch_win_np(bg_frdc& A, const uint32_t* x, int64_t f, uint32_t* ob, float* of, int64_t r0,
                   int64_t r1, cudaStream_t s) {
  const int64_t d = A.max_deg;
  if (d < (1 << 6)) return launch_win<6, OUTB>(A, x, f, ob, of, r0, r1, s);
  if (d < (1 << 8)) return launch_win<8, OUTB>(A, x, f, ob, of, r0, r1, s);
  if (d < (1 << 10)) return launch_win<10, OUTB>(A, x, f, ob, of, r0, r1, s);
  if (d < (1 << 12)) return launch_win<12, OUTB>(A, x, f, ob, of, r0, r1, s);
  return false;
}

}  // namespace

bool window_bb(bg_frdc& A, const uint32_t* x, int64_t f, int wb, uint32_t* out_bits, float* out_f,
               cudaStream_t s, int64_t r0, int64_t r1) {
  if (spw(f, wb) != 4 || A.rows != A.cols || A.rows == 0 || r1 <= r0) return false;
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0) return false;
  const int mode = aggregation_mode();
  if (mode == BG_AGG_SLIVERS || mode == BG_AGG_TILES) return false;
  if (out_bits) return launch_win_np<true>(A, x, f, out_bits, nullptr, r0, r1, s);
  return launch_win_np<false>(A, x, f, nullptr, out_f, r0, r1, s);
}

}  // namespace bg
