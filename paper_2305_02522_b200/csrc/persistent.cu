// Whole-forward persistent kernel for small graphs (the
// paper's cooperative-launch cross-layer fusion).
//
// On Cora/PubMed-size graphs every layer is a few microseconds of work, so a
// forward of separate kernels is bound by their launch and ramp latencies.
// Here ONE cooperative launch (one CTA per SM, all co-resident) runs the whole
// binary GCN chain of run_model (graphops.cpp:390-484) with a grid barrier
// between layers:
//   * MM.FBB / MM.BBB (kernels.cpp:140-176): warp per node row; the row is
//     binarized with a ballot per 32 columns (x >= 0, MSB first,
//     bitdense.cpp:71-88) into the warp's shared words, lane c owns output
//     columns c, c+32, ...: dot = K - 2 popc(a ^ w_c), bit = dot >= 0;
//   * BSpMM.BBB (kernels.cpp:254-333, :440-454): warp per node row, lane b
//     owns output bits b, b+32, ...: counts over the row's neighbours,
//     bit = 2 cnt - deg >= 0;
//   * MM.BBF + BSpMM.FBF + softmax (kernels.cpp:179-190, :512-555,
//     graphops.cpp:372-386): warp per row, lane k owns class k: the
//     neighbours j in ascending order (walk_tile_row, kernels.cpp:218-234),
//     y_jk = float((1 * dot_jk) * beta_k) recomputed from h_j, d_k += y_jk in
//     double, logit float(d_k); then max, the sequential double sum of
//     exp(x - max) over the classes, float(exp / sum).
// Every accumulation is the reference's (integers exact, the double sums in
// its order), so the results equal the layer-by-layer forward bit for bit.
#include <cstdio>
#include <cstdlib>

#include "engine.cuh"
#include "model.cuh"
#include "tilewalk.cuh"

namespace bg {
namespace {

constexpr int kPWarps = 16;           // 512 threads per CTA
constexpr int kPMaxWords = 64;        // K <= 2048 (u32 words of a binarized input row)
constexpr int kPMaxHidden = 128;      // hidden bits per row (4 u32 words)
constexpr int kPMaxClasses = 32;      // lane per class
constexpr int kPMaxLayers = 8;
constexpr int64_t kPMaxNodes = 1 << 17;
constexpr int64_t kPMaxBits = int64_t{1} << 22;

struct PLayer {
  int kind;  // 0: MM (F or B input) -> B, then BSpMM.BBB;  1: MM.BBF + BSpMM.FBF (last)
  int kin, kout;
  int in_f;  // layer input is the fp32 model input
  const uint32_t* wt;  // kout x spw(kin) transposed +-1 weight bits
  const float* beta;   // kout column scales (kind 1)
};

struct PArgs {
  int nl;
  PLayer l[kPMaxLayers];
  int64_t n;
  int wb;
  const float* xf;      // model input, fp32 (first layer in_f)
  const uint32_t* xb;   // or packed bits
  const uint64_t* rp;   // A + I
  const uint32_t* ci;
  const uint16_t* ti;
  const int32_t* deg;
  uint32_t* hbuf[2];    // ping-pong packed activations, n x spw(kPMaxHidden) words
  uint32_t* gbar;       // grid barrier: count, generation
  float* logits;        // may be null
  float* probs;
  unsigned long long* stamps;  // debug (BG_PERSISTENT_STAMPS): globaltimer per block and phase
};

__device__ __forceinline__ void stamp(const PArgs& a, int ph) {
  if (a.stamps && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.stamps[blockIdx.x * 32 + ph] = t;
  }
}

__device__ __forceinline__ void grid_barrier(uint32_t* bar, uint32_t nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile uint32_t* gen = bar + 1;
    const uint32_t g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ int pspw(int cols, int wb) { return (cols + wb - 1) / wb * (wb / 32); }

// Visits the neighbours j of node row i in ascending column order.
template <class F>
__device__ __forceinline__ void for_neighbours(const PArgs& a, int64_t i, F f) {
  const int64_t t = i >> 2;
  const int sh = 12 - 4 * static_cast<int>(i & 3);
  for (uint64_t k = a.rp[t]; k < a.rp[t + 1]; ++k) {
    const uint32_t nib = (static_cast<uint32_t>(a.ti[k]) >> sh) & 0xFu;
    if (!nib) continue;
    const int64_t j0 = 4 * static_cast<int64_t>(a.ci[k]);
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (nib & (8u >> c)) f(j0 + c);
  }
}

constexpr int kPPlanes = 12;        // bit-sliced neighbour counts: max degree < 4096

__global__ void __launch_bounds__(kPWarps * 32, 1) k_persistent_gcn(const PArgs a) {
  __shared__ uint32_t wsm[kPMaxHidden * kPMaxWords];   // the layer's weights (32 KB max)
  __shared__ uint32_t rowbits[kPWarps][kPMaxWords];     // a warp's binarized input row
  __shared__ float bsm[kPMaxClasses];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kPWarps + wib, nw = static_cast<int64_t>(gridDim.x) * kPWarps;
  // thread-per-row phases: rows spread over every SM first (row i on block
  // i % grid), so a small graph's rows do not pile onto a few SMs
  const int64_t gt = static_cast<int64_t>(threadIdx.x) * gridDim.x + blockIdx.x;
  const int64_t nt = static_cast<int64_t>(gridDim.x) * blockDim.x;
  constexpr int hw = 4;  // row pitch of the activation buffers (u32 words, 16-byte rows)
  int cur = 0;           // hbuf holding the current activation
  int ph = 0;
  stamp(a, ph++);
  for (int li = 0; li < a.nl; ++li) {
    const PLayer& L = a.l[li];
    const int kw = pspw(L.kin, a.wb), ow = pspw(L.kout, a.wb);
    for (int t = threadIdx.x; t < L.kout * kw; t += blockDim.x) wsm[t] = __ldg(L.wt + t);
    if (L.kind == 1 && static_cast<int>(threadIdx.x) < L.kout) bsm[threadIdx.x] = __ldg(L.beta + threadIdx.x);
    __syncthreads();
    if (L.kind == 0) {
      uint32_t* hout = a.hbuf[cur ^ 1];
      if (L.in_f) {
        // ---- MM.FBB: warp per row, the whole row's loads in flight at once ----
        for (int64_t i = gw; i < a.n; i += nw) {
          const float* xr = a.xf + i * L.kin;
          float v[kPMaxWords];
#pragma unroll
          for (int u = 0; u < kPMaxWords; ++u) {
            const int col = 32 * u + lane;
            v[u] = (u < kw && col < L.kin) ? __ldg(xr + col) : -1.0f;
          }
#pragma unroll
          for (int u = 0; u < kPMaxWords; ++u) {
            if (u >= kw) break;
            const uint32_t b = __brev(__ballot_sync(0xFFFFFFFFu, 32 * u + lane < L.kin && v[u] >= 0.0f));
            if (lane == 0) rowbits[wib][u] = b;  // x >= 0 -> 1, MSB first; padding words 0
          }
          __syncwarp();
          // lane c: columns c, c+32, c+64, c+96 in one pass over the row words
          int pc[4] = {0, 0, 0, 0};
          const uint32_t* wl = wsm + lane * kw;
#pragma unroll 4
          for (int w = 0; w < kw; ++w) {
            const uint32_t x = rowbits[wib][w];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (32 * q + lane < L.kout) pc[q] += __popc(x ^ wl[32 * q * kw + w]);
          }
          uint32_t outw[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)  // pm1_dot_words >= 0 (kernels.cpp:30-41, :166-171)
            outw[q] = __brev(__ballot_sync(0xFFFFFFFFu, 32 * q + lane < L.kout && L.kin - 2 * pc[q] >= 0));
          if (lane < hw) hout[i * hw + lane] = lane < ow ? outw[lane] : 0u;
          __syncwarp();
        }
      } else {
        // ---- MM.BBB: thread per row (K <= 128: at most 4 input words) --------
        const uint32_t* hin = li == 0 ? a.xb : a.hbuf[cur];
        const int64_t pitch = li == 0 ? kw : hw;
        for (int64_t i = gt; i < a.n; i += nt) {
          uint32_t r[4];
#pragma unroll
          for (int w = 0; w < 4; ++w) r[w] = w < kw ? hin[i * pitch + w] : 0u;
          uint32_t outw[4] = {0u, 0u, 0u, 0u};
          for (int col = 0; col < L.kout; ++col) {
            int pc = 0;
#pragma unroll
            for (int w = 0; w < 4; ++w)
              if (w < kw) pc += __popc(r[w] ^ wsm[col * kw + w]);
            if (L.kin - 2 * pc >= 0) outw[col >> 5] |= 0x80000000u >> (col & 31);
          }
          *reinterpret_cast<uint4*>(hout + i * hw) = make_uint4(outw[0], outw[1], outw[2], outw[3]);
        }
      }
      stamp(a, ph++);
      grid_barrier(a.gbar, gridDim.x);
      stamp(a, ph++);
      // ---- BSpMM.BBB over A + I: 8 lanes per row (4 rows per warp) ------------
      // lane g of a row owns output bits [16g, 16g + 16): bit-sliced counts of
      // those bits over the neighbours; every neighbour's word is loaded by the
      // lanes that need it, all loads of a pass (<= 32 neighbours) in flight
      const uint32_t* hx = a.hbuf[cur ^ 1];
      uint32_t* hy = a.hbuf[cur];
      const int g = lane & 7, grp = lane >> 3;
      const unsigned gmask = 0xFFu << (8 * grp);
      for (int64_t ib = 4 * gw; ib < a.n; ib += 4 * nw) {
        const int64_t i = ib + grp;
        const bool row_ok = i < a.n;
        uint32_t P[kPPlanes];
#pragma unroll
        for (int p = 0; p < kPPlanes; ++p) P[p] = 0u;
        uint64_t k0 = 0, k1 = 0;
        if (row_ok) {
          k0 = a.rp[i >> 2];
          k1 = a.rp[(i >> 2) + 1];
        }
        const int sh = 12 - 4 * static_cast<int>(i & 3);
        const int wsel = g >> 1, hsh = (g & 1) ? 0 : 16;  // this lane's 16 bits of a row
        for (uint64_t kb = k0; kb < k1; kb += 8) {         // uniform within the group
          const uint64_t k = kb + g;
          uint32_t nib = 0;
          int64_t j0 = 0;
          if (k < k1) {
            nib = (static_cast<uint32_t>(a.ti[k]) >> sh) & 0xFu;
            j0 = 4 * static_cast<int64_t>(a.ci[k]);
          }
          uint32_t xs[32];
          int nx = 0;
#pragma unroll
          for (int src = 0; src < 8; ++src) {  // every neighbour of the pass, in turn
            const uint32_t sn = __shfl_sync(gmask, nib, src, 8);
            const int64_t sj = __shfl_sync(gmask, j0, src, 8);
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (sn & (8u >> c)) xs[nx++] = hx[(sj + c) * hw + wsel];
          }
          for (int t = 0; t < nx; ++t) {
            uint32_t c = (xs[t] >> hsh) & 0xFFFFu;
#pragma unroll
            for (int p = 0; p < kPPlanes; ++p) {
              const uint32_t u = P[p] & c;
              P[p] ^= c;
              c = u;
            }
          }
        }
        // cnt >= ceil(deg/2)  <=>  2 cnt - deg >= 0  (kernels.cpp:440-454)
        const uint32_t half = row_ok ? static_cast<uint32_t>(a.deg[i] + 1) >> 1 : 0u;
        uint32_t ge = planes_ge<kPPlanes>(P, half) & 0xFFFFu;  // bit b <-> output bit 16g + 15 - b
        const int c0 = 16 * g;
        if (c0 + 16 > L.kout) ge &= c0 >= L.kout ? 0u : (0xFFFFu << (c0 + 16 - L.kout)) & 0xFFFFu;
        const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, ge, 1);
        if (row_ok && !(g & 1)) {  // lanes 2w, 2w+1 hold word w's high and low halves
          const int w = g >> 1;
          hy[i * hw + w] = w < ow ? (ge << 16) | other : 0u;
        }
      }
      stamp(a, ph++);
      grid_barrier(a.gbar, gridDim.x);
      stamp(a, ph++);
    } else {
      // ---- MM.BBF + BSpMM.FBF + softmax ----------------------------------------
      const uint4* h = reinterpret_cast<const uint4*>(a.hbuf[cur]);
      const int C = L.kout;
      if (C <= 8) {
        // 8 lanes per row (4 rows per warp), lane k = class k: the pass's
        // neighbours (tiles in order, bits in order: ascending j) are loaded by
        // their tile's lane and handed round with shuffles
        const int g = lane & 7, grp = lane >> 3;
        const unsigned gmask = 0xFFu << (8 * grp);
        const bool live = g < C;
        const double bk = static_cast<double>(bsm[live ? g : 0]);
        uint32_t wk[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) wk[w] = (live && w < kw) ? wsm[g * kw + w] : 0u;
        for (int64_t ib = 4 * gw; ib < a.n; ib += 4 * nw) {
          const int64_t i = ib + grp;
          const bool row_ok = i < a.n;
          uint64_t k0 = 0, k1 = 0;
          if (row_ok) {
            k0 = a.rp[i >> 2];
            k1 = a.rp[(i >> 2) + 1];
          }
          const int sh = 12 - 4 * static_cast<int>(i & 3);
          double d = 0.0;
          for (uint64_t kb = k0; kb < k1; kb += 8) {
            const uint64_t k = kb + g;
            uint32_t nib = 0;
            uint4 hv[4] = {};
            if (k < k1) {
              nib = (static_cast<uint32_t>(a.ti[k]) >> sh) & 0xFu;
              const int64_t j0 = 4 * static_cast<int64_t>(a.ci[k]);
#pragma unroll
              for (int c = 0; c < 4; ++c)
                if (nib & (8u >> c)) hv[c] = h[j0 + c];
            }
#pragma unroll
            for (int src = 0; src < 8; ++src) {
              const uint32_t sn = __shfl_sync(gmask, nib, src, 8);
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                if (!(sn & (8u >> c))) continue;  // uniform in the group
                const uint32_t x0 = __shfl_sync(gmask, hv[c].x, src, 8), x1 = __shfl_sync(gmask, hv[c].y, src, 8);
                const uint32_t x2 = __shfl_sync(gmask, hv[c].z, src, 8), x3 = __shfl_sync(gmask, hv[c].w, src, 8);
                const int pc = __popc(x0 ^ wk[0]) + __popc(x1 ^ wk[1]) + __popc(x2 ^ wk[2]) + __popc(x3 ^ wk[3]);
                // x_jk = float((1 * dot) * beta_k) (MM.BBF, alpha = 1); d_k += 1 * x_jk
                const float y = __double2float_rn(__dmul_rn(static_cast<double>(L.kin - 2 * pc), bk));
                d = __dadd_rn(d, static_cast<double>(y));
              }
            }
          }
          const float x = __double2float_rn(d);  // float(1 * d) (kernels.cpp:549)
          float mx = live ? x : -INFINITY;
#pragma unroll
          for (int o = 4; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o, 8));
          const double e = live ? exp(static_cast<double>(x) - static_cast<double>(mx)) : 0.0;
          double sum = 0.0;  // sequential, class order (graphops.cpp:380)
          for (int k = 0; k < C; ++k) sum = __dadd_rn(sum, __shfl_sync(0xFFFFFFFFu, e, k, 8));
          if (live && row_ok) {
            if (a.logits) a.logits[i * C + g] = x;
            a.probs[i * C + g] = __double2float_rn(__ddiv_rn(e, sum));
          }
        }
      } else {
        // warp per row, lane per class
        const bool live = lane < C;
        const double beta = live ? static_cast<double>(bsm[lane]) : 0.0;
        for (int64_t i = gw; i < a.n; i += nw) {
          double d = 0.0;
          for_neighbours(a, i, [&](int64_t j) {
            const uint4 v = h[j];
            const uint32_t x[4] = {v.x, v.y, v.z, v.w};
            if (!live) return;
            int pc = 0;
#pragma unroll
            for (int w = 0; w < 4; ++w)
              if (w < kw) pc += __popc(x[w] ^ wsm[lane * kw + w]);
            const float y = __double2float_rn(__dmul_rn(static_cast<double>(L.kin - 2 * pc), beta));
            d = __dadd_rn(d, static_cast<double>(y));
          });
          const float x = __double2float_rn(d);
          float mx = live ? x : -INFINITY;
#pragma unroll
          for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
          const double e = live ? exp(static_cast<double>(x) - static_cast<double>(mx)) : 0.0;
          double sum = 0.0;  // sequential, class order (graphops.cpp:380)
          for (int k = 0; k < C; ++k) sum = __dadd_rn(sum, __shfl_sync(0xFFFFFFFFu, e, k));
          if (live) {
            if (a.logits) a.logits[i * C + lane] = x;
            a.probs[i * C + lane] = __double2float_rn(__ddiv_rn(e, sum));
          }
        }
      }
    }
    __syncthreads();  // wsm reused by the next layer
  }
  stamp(a, ph++);
}

}  // namespace

namespace {
bool g_persistent_forced = false;
}
bool persistent_forced() { return g_persistent_forced; }
void set_persistent_forced(bool on) { g_persistent_forced = on; }

// The chain run_model would execute, when it is one of the shapes above on a
// small graph; false otherwise (the layer-by-layer forward runs).
bool persistent_forward(bg_model& m, const Op& x0, float* out, float* logits, cudaStream_t s) {
  if (!m.graph || !m.graph->structure || !out || m.graph->row0 != 0) return false;
  // Opt-in (BG_PERSISTENT=1): measured on B200 it does not beat the captured
  // layer-by-layer forward (Cora 45 vs 25 us, PubMed 152 vs 54 us): the time
  // is the fp32 row stream of the first product and the per-row latency
  // chains of each phase, not the launches a CUDA graph already hides.
  static const bool enabled = [] {
    const char* e = std::getenv("BG_PERSISTENT");
    return e && std::atoi(e) == 1;
  }();
  if (!enabled && !persistent_forced()) return false;
  const bg_frdc& A = *m.graph->structure;
  const int64_t n = m.graph->n;
  if (A.rows != n || A.cols != n || n == 0 || n > kPMaxNodes || A.nnz_bits > kPMaxBits ||
      A.max_deg >= (int64_t{1} << kPPlanes))
    return false;
  if (x0.rows != n || x0.scale || x0.packed()) return false;
  if (x0.prec == BG_B && (x0.sem != BG_PLUS_MINUS || x0.wb != m.wb)) return false;
  const size_t nl = m.layers.size();
  if (nl < 2 || nl - 1 > static_cast<size_t>(kPMaxLayers) || m.layers[nl - 1].info.kind != BG_LAYER_SOFTMAX)
    return false;
  PArgs a{};
  a.nl = static_cast<int>(nl - 1);
  a.n = n;
  a.wb = m.wb;
  int64_t kin = x0.cols;
  for (size_t i = 0; i + 1 < nl; ++i) {
    const ModelLayer& l = m.layers[i];
    if (l.info.kind != BG_LAYER_GCN || l.info.plan.size() != 2 || l.w1.rows != kin || l.w1.wb != m.wb) return false;
    const bg_variant mm = l.info.plan[0], sp = l.info.plan[1];
    const bool last = i + 2 == nl;
    const bool first_f = i == 0 && x0.prec == BG_F;
    PLayer& L = a.l[i];
    L.kin = static_cast<int>(kin);
    L.kout = static_cast<int>(l.w1.cols);
    L.in_f = first_f;
    L.wt = l.w1.wt.as<uint32_t>();
    L.beta = l.w1.scale.as<float>();
    if (spw(kin, m.wb) > kPMaxWords || L.kout * spw(kin, m.wb) > kPMaxHidden * kPMaxWords) return false;
    const bool mm_b = mm.op == BG_BMM && mm.in2 == BG_B && mm.out == BG_B && (mm.in1 == (first_f ? BG_F : BG_B));
    const bool sp_b = sp.op == BG_BSPMM && sp.in1 == BG_B && sp.in2 == BG_B && sp.out == BG_B;
    const bool mm_f = mm.op == BG_BMM && mm.in1 == BG_B && mm.in2 == BG_B && mm.out == BG_F && !first_f;
    const bool sp_f = sp.op == BG_BSPMM && sp.in1 == BG_F && sp.in2 == BG_B && sp.out == BG_F;
    if (!last && mm_b && sp_b && L.kout <= kPMaxHidden) L.kind = 0;
    else if (last && mm_f && sp_f && !l.relu && L.kout <= kPMaxClasses && kin <= kPMaxHidden) L.kind = 1;
    else return false;
    kin = l.w1.cols;
  }
  if (a.l[a.nl - 1].kind != 1) return false;
  // workspace: two activation buffers and the grid barrier, from the pool
  // (same call sequence every forward -> capturable)
  const size_t hb = static_cast<size_t>(n) * spw(kPMaxHidden, 32) * 4;
  a.hbuf[0] = static_cast<uint32_t*>(m.pool.get(hb));
  a.hbuf[1] = static_cast<uint32_t*>(m.pool.get(hb));
  a.gbar = static_cast<uint32_t*>(m.pool.get(8));
  BG_CUDA(cudaMemsetAsync(a.gbar, 0, 8, s));
  a.xf = x0.prec == BG_F ? x0.f : nullptr;
  a.xb = x0.prec == BG_B ? x0.bits : nullptr;
  a.rp = A.rp();
  a.ci = A.ci();
  a.ti = A.ti();
  a.deg = A.deg();
  a.logits = logits;
  a.probs = out;
  static unsigned long long* dbg = [] {
    unsigned long long* p = nullptr;
    if (const char* e = std::getenv("BG_PERSISTENT_STAMPS"); e && std::atoi(e) == 1)
      BG_CUDA(cudaMalloc(&p, 148 * 32 * 8));
    return p;
  }();
  a.stamps = dbg;
  static int grid = [] {
    int nb = 0;
    BG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_persistent_gcn, kPWarps * 32, 0));
    return nb >= 1 ? sm_count() : 0;
  }();
  if (grid == 0) return false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kPWarps * 32);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (the grid barrier)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BG_CUDA(cudaLaunchKernelEx(&cfg, k_persistent_gcn, a));
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  BG_CUDA(cudaStreamIsCapturing(s, &cap));
  if (dbg && cap == cudaStreamCaptureStatusNone) {  // debug: per-phase spans (min/max over blocks), us
    unsigned long long h[148 * 32];
    BG_CUDA(cudaMemcpyAsync(h, dbg, sizeof h, cudaMemcpyDeviceToHost, s));
    BG_CUDA(cudaStreamSynchronize(s));
    const int nph = 2 + 4 * (a.nl - 1);
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < grid; ++b) t0 = std::min(t0, h[b * 32]);
    std::fprintf(stderr, "[persistent]");
    for (int p = 1; p < nph; ++p) {
      unsigned long long mx = 0, mn = ~0ull;
      for (int b = 0; b < grid; ++b) mx = std::max(mx, h[b * 32 + p] - t0), mn = std::min(mn, h[b * 32 + p] - t0);
      std::fprintf(stderr, " p%d %.1f/%.1f", p, mn / 1e3, mx / 1e3);
    }
    std::fprintf(stderr, "\n");
  }
  return true;
}

}  // namespace bg
