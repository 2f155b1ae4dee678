// Binary sparse aggregation over FRDC 4x4 bit tiles (ref: bspmm,
// kernels.cpp:413-556).
//
// Integer path (BBB / BBF, kernels.cpp:254-465): out(i,k) = 2*cnt(i,k) - deg(i)
// with cnt = #{j in N(i): x_jk = 1}; BBB keeps the sign bit (>= 0).
//
//   One warp per tile row.  The warp streams the tile row's col_ind/tiles
//   with coalesced loads (one tile per lane), counting-sorts the set bits by
//   local node row into four shared-memory rings (a packed 4x8-bit warp scan
//   gives every lane its slots), and drains each ring in batches of 8 edges
//   per slot lane.  Lane (slot s, word g) gathers word g of 8 neighbour rows
//   and adds them into bit-sliced (vertical) counters with a Harley-Seal
//   carry-save tree: ~4 LOP3 per gathered word, no per-feature unpacking.
//   At the end the slot lanes are summed with a bit-sliced butterfly and the
//   BBB threshold cnt >= ceil(deg/2) is evaluated plane-wise, producing the
//   packed output word directly (north-star item 4: no unpacked round trip).
//
// Real-valued path (FBF/FFF/FBB/FFB and BFF/BFB, kernels.cpp:467-555): one
// warp per node row walks its neighbours in ascending column order (ballot
// over the tile chunk, then ascending lane, then ascending local column --
// the order of walk_tile_row, :218-234) and accumulates in double, lanes over
// features, so every output is bit-identical to the reference's sequential sum.
#include <algorithm>

#include "ops.cuh"
#include "tilewalk.cuh"

namespace bg {
namespace {

constexpr int kBBWarps = 8;

// G = word lanes (power of two), S = 32/G slot lanes, NP planes per lane.
template <int G, int NP, bool OUTB>
__global__ void __launch_bounds__(kBBWarps * 32)
    k_bspmm_bb(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ ci,
               const uint16_t* __restrict__ ti, int64_t tr0, int64_t trows, int64_t rows,
               const int32_t* __restrict__ degree, const uint32_t* __restrict__ x, int64_t xspw,
               int64_t f, uint32_t* __restrict__ out_bits, float* __restrict__ out_f, const FEpi ep) {
  constexpr int S = 32 / G;
  constexpr int B = 8 * S;  // edges per drained batch
  constexpr int LOGS = S == 1 ? 0 : S == 2 ? 1 : S == 4 ? 2 : S == 8 ? 3 : S == 16 ? 4 : 5;
  constexpr int NQ = NP + LOGS;  // planes after the slot reduction
  __shared__ uint32_t ring_all[kBBWarps][4][kRing];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane % G, slot = lane / G;
  const int64_t word = static_cast<int64_t>(blockIdx.y) * G + g;
  const bool word_ok = word < xspw;
  uint32_t(*ring)[kRing] = ring_all[warp];
  // Lanes past the row's last word gather word 0 and discard it, so the
  // batch loop below needs no per-load predicate.
  const uint32_t* xw = x + (word_ok ? word : 0);
  const uint32_t xstride = static_cast<uint32_t>(xspw);
  (void)degree;

  for (int64_t tr = tr0 + static_cast<int64_t>(blockIdx.x) * kBBWarps + warp; tr < trows;
       tr += static_cast<int64_t>(gridDim.x) * kBBWarps) {
    uint32_t P[4][NP];
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int q = 0; q < NP; ++q) P[n][q] = 0;

    auto drain = [&](auto nc, uint32_t h, uint32_t cnt) {
      constexpr int n = decltype(nc)::value;
      uint32_t xv[8];
      if (cnt == static_cast<uint32_t>(B)) {
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const uint32_t j = ring[n][(h + slot + S * m) & (kRing - 1)];
          xv[m] = __ldg(xw + j * xstride);
        }
      } else {
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const uint32_t e = static_cast<uint32_t>(slot + S * m);
          xv[m] = 0;
          if (e < cnt) xv[m] = __ldg(xw + ring[n][(h + e) & (kRing - 1)] * xstride);
        }
      }
      hs_add8<NP>(P[n], xv);
    };
    uint32_t fill[4];
    walk_tile_row<B>(rp, ci, ti, tr, ring, fill, drain);

    // Slot reduction and epilogue per node row.
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      uint32_t Q[NQ];
      slot_reduce<G, NP, NQ>(P[n], Q);
      const int64_t row = 4 * tr + n;
      if (row >= rows || !word_ok) continue;
      const uint32_t deg = fill[n];
      if (OUTB) {
        // cnt >= ceil(deg/2)  <=>  2*cnt - deg >= 0   (kernels.cpp:440-454)
        uint32_t ge = planes_ge<NQ>(Q, (deg + 1) >> 1);
        if (32 * (word + 1) > f) ge &= (32 * word >= f) ? 0u : tail_mask32(f);
        if (slot == 0) out_bits[row * xspw + word] = ge;
      } else if (ep.bits) {  // every slot lane holds the totals: one packs the word
        if (slot == 0)
          fepi_store_word(ep, out_f, row, f, word, [&](int b) {
            return static_cast<float>(2 * static_cast<int64_t>(plane_count<NQ>(Q, b)) - static_cast<int64_t>(deg));
          });
      } else {
        for (int b = slot; b < 32; b += S) {
          const int64_t k = 32 * word + b;
          if (k >= f) break;
          out_f[row * f + k] = fepi_apply(
              ep, static_cast<float>(2 * static_cast<int64_t>(plane_count<NQ>(Q, b)) - static_cast<int64_t>(deg)), k);
        }
      }
    }
  }
}

template <int G, int NP, bool OUTB>
void launch_bb(const bg_frdc& A, const uint32_t* x, int64_t f, int64_t xspw, uint32_t* ob,
               float* of, int64_t t0, int64_t t1, cudaStream_t s) {
  const int64_t groups = cdiv(xspw, G);
  const int64_t blocks = std::max<int64_t>(
      1, std::min<int64_t>(cdiv(t1 - t0, kBBWarps), static_cast<int64_t>(sm_count()) * 64));
  dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>(groups));
  k_bspmm_bb<G, NP, OUTB><<<grid, kBBWarps * 32, 0, s>>>(A.rp(), A.ci(), A.ti(), t0, t1,
                                                         A.rows, A.deg(), x, xspw, f, ob, of, current_fepi());
  BG_LAUNCH_CHECK();
}

template <int G, bool OUTB>
void launch_bb_np(const bg_frdc& A, const uint32_t* x, int64_t f, int64_t xspw, uint32_t* ob,
                  float* of, int64_t t0, int64_t t1, cudaStream_t s) {
  constexpr int S = 32 / G;
  // The ring deals a row's edges round-robin to the S slot lanes in batches
  // of 8 each, so a lane's counters see at most ceil(deg/(8S))*8 edges.
  const int64_t per_lane = (A.max_deg + 8 * S - 1) / (8 * S) * 8;
  if (per_lane < (1 << 7)) return launch_bb<G, 7, OUTB>(A, x, f, xspw, ob, of, t0, t1, s);
  if (per_lane < (1 << 10)) return launch_bb<G, 10, OUTB>(A, x, f, xspw, ob, of, t0, t1, s);
  if (per_lane < (1 << 13)) return launch_bb<G, 13, OUTB>(A, x, f, xspw, ob, of, t0, t1, s);
  if (per_lane < (1 << 16)) return launch_bb<G, 16, OUTB>(A, x, f, xspw, ob, of, t0, t1, s);
  if (per_lane < (1 << 20)) return launch_bb<G, 20, OUTB>(A, x, f, xspw, ob, of, t0, t1, s);
  if (per_lane < (1 << 26)) return launch_bb<G, 26, OUTB>(A, x, f, xspw, ob, of, t0, t1, s);
  fail("bspmm: node degree " + std::to_string(A.max_deg) + " exceeds the counter range");
}

// ---- real-valued walk ------------------------------------------------------
template <int M, bool XBITS, bool OUTB>
__global__ void __launch_bounds__(256)
    k_bspmm_f(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ ci,
              const uint16_t* __restrict__ ti, int64_t rows, const float* __restrict__ xf,
              const uint32_t* __restrict__ xb, int64_t xspw, const float* __restrict__ rs,
              const float* __restrict__ cs, int64_t f, int64_t ospw,
              uint32_t* __restrict__ out_bits, float* __restrict__ out_f, int64_t row0, const FEpi ep) {
  const int64_t i = row0 + ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  if (i >= rows) return;
  const int lane = threadIdx.x & 31;
  const int64_t fbase = static_cast<int64_t>(blockIdx.y) * 32 * M;
  const int64_t tr = i >> 2;
  const int shift = 12 - 4 * static_cast<int>(i & 3);
  double d[M];
#pragma unroll
  for (int m = 0; m < M; ++m) d[m] = 0.0;
  const uint64_t t1 = rp[tr + 1];
  for (uint64_t base = rp[tr]; base < t1; base += 32) {
    const uint64_t t = base + lane;
    uint32_t nib = 0, col = 0;
    if (t < t1) {
      nib = (__ldg(ti + t) >> shift) & 0xFu;
      col = __ldg(ci + t);
    }
    uint32_t mask = __ballot_sync(0xFFFFFFFFu, nib != 0);
    while (mask) {
      const int L = __ffs(mask) - 1;
      mask &= mask - 1;
      const uint32_t nl = __shfl_sync(0xFFFFFFFFu, nib, L);
      const uint32_t cl = __shfl_sync(0xFFFFFFFFu, col, L);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (!(nl & (8u >> c))) continue;
        const int64_t j = 4 * static_cast<int64_t>(cl) + c;
        const double w = cs ? static_cast<double>(__ldg(cs + j)) : 1.0;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const int64_t k = fbase + 32 * m + lane;
          if (k < f) {
            if (XBITS) {
              const uint32_t bit = (__ldg(xb + j * xspw + (k >> 5)) >> (31 - (k & 31))) & 1u;
              d[m] = __dadd_rn(d[m], bit ? w : -w);
            } else {
              d[m] = __dadd_rn(d[m], __dmul_rn(w, static_cast<double>(__ldg(xf + j * f + k))));
            }
          }
        }
      }
    }
  }
  const double si = rs ? static_cast<double>(rs[i]) : 1.0;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int64_t k = fbase + 32 * m + lane;
    const double v = __dmul_rn(si, d[m]);
    if (OUTB) {
      const uint32_t word = __brev(__ballot_sync(0xFFFFFFFFu, k < f && v >= 0.0));
      const int64_t w = (fbase >> 5) + m;
      if (lane == 0 && w < ospw) out_bits[i * ospw + w] = word;
    } else {
      fepi_store_lane(ep, out_f, i, f, k, __double2float_rn(v));
    }
  }
  if (OUTB && lane == 0 && blockIdx.y == gridDim.y - 1)
    for (int64_t w = (f + 31) / 32; w < ospw; ++w) out_bits[i * ospw + w] = 0;
}

template <int M, bool XBITS, bool OUTB>
void launch_f(const bg_frdc& A, const SpmmFArgs& a, int64_t row0, int64_t row1, cudaStream_t s) {
  const int64_t passes = cdiv(a.f, 32 * M);
  dim3 grid(static_cast<unsigned>(cdiv((row1 - row0) * 32, 256)), static_cast<unsigned>(passes));
  const int64_t xspw = XBITS ? spw(a.f, a.xwb) : 0;
  const int64_t ospw = OUTB ? spw(a.f, a.owb) : 0;
  k_bspmm_f<M, XBITS, OUTB><<<grid, 256, 0, s>>>(A.rp(), A.ci(), A.ti(), row1, a.x_f, a.x_bits,
                                                 xspw, a.row_scale, a.col_scale, a.f, ospw,
                                                 a.out_bits, a.out_f, row0, current_fepi());
  BG_LAUNCH_CHECK();
}

template <bool XBITS, bool OUTB>
void launch_f_m(const bg_frdc& A, const SpmmFArgs& a, int64_t r0, int64_t r1, cudaStream_t s) {
  if (a.f <= 32) launch_f<1, XBITS, OUTB>(A, a, r0, r1, s);
  else if (a.f <= 64) launch_f<2, XBITS, OUTB>(A, a, r0, r1, s);
  else launch_f<4, XBITS, OUTB>(A, a, r0, r1, s);
}

}  // namespace

void bspmm_bb(const bg_frdc& A, const uint32_t* x, int64_t f, int wb, uint32_t* out_bits,
              float* out_f, cudaStream_t s, int64_t row0, int64_t row1) {
  if (use_slivers()) return sliver_bb(const_cast<bg_frdc&>(A), x, f, wb, out_bits, out_f, s, row0, row1);
  if (row1 < 0) row1 = A.rows;
  const int64_t t0 = row0 / 4, t1 = (row1 + 3) / 4;
  if (A.rows == 0 || t1 <= t0) return;
  const int64_t xspw = spw(f, wb);
  if (xspw == 0) {
    return;
  }
  const bool ob = out_bits != nullptr;
  if (xspw <= 4) {
    if (ob) launch_bb_np<4, true>(A, x, f, xspw, out_bits, out_f, t0, t1, s);
    else launch_bb_np<4, false>(A, x, f, xspw, out_bits, out_f, t0, t1, s);
  } else if (xspw <= 8) {
    if (ob) launch_bb_np<8, true>(A, x, f, xspw, out_bits, out_f, t0, t1, s);
    else launch_bb_np<8, false>(A, x, f, xspw, out_bits, out_f, t0, t1, s);
  } else if (xspw <= 16) {
    if (ob) launch_bb_np<16, true>(A, x, f, xspw, out_bits, out_f, t0, t1, s);
    else launch_bb_np<16, false>(A, x, f, xspw, out_bits, out_f, t0, t1, s);
  } else {
    if (ob) launch_bb_np<32, true>(A, x, f, xspw, out_bits, out_f, t0, t1, s);
    else launch_bb_np<32, false>(A, x, f, xspw, out_bits, out_f, t0, t1, s);
  }
}

void bspmm_f(const bg_frdc& A, const SpmmFArgs& a, cudaStream_t s, int64_t row0, int64_t row1) {
  if (use_slivers()) return sliver_f(const_cast<bg_frdc&>(A), a, s, row0, row1);
  if (row1 < 0) row1 = A.rows;
  if (A.rows == 0 || a.f == 0 || row1 <= row0) return;
  const bool xb = a.x_bits != nullptr, ob = a.out_bits != nullptr;
  if (xb && ob) launch_f_m<true, true>(A, a, row0, row1, s);
  else if (xb) launch_f_m<true, false>(A, a, row0, row1, s);
  else if (ob) launch_f_m<false, true>(A, a, row0, row1, s);
  else launch_f_m<false, false>(A, a, row0, row1, s);
}

}  // namespace bg
