// Row-sharded multi-GPU forward (one process per GPU).
//
// Nodes are split into contiguous tile-row ranges balanced by FRDC tiles
// (bg_partition_bounds).  Every rank holds the whole graph and the weights and
// computes its own node rows of every layer; the only exchange is the one the
// algorithm needs: before each neighbour aggregation the rank's rows of the
// aggregated operand (packed activations for the binary plans: 16 B per node
// at hidden 128) are all-gathered over NVLink with NCCL (a group of in-place
// broadcasts, so uneven row ranges need no padding).  Row partitioning does not
// change any per-row accumulation order, so every shard count produces output
// bit-identical to the single-GPU forward.
//
// "Virtual" mode (no communicator) computes every rank's range in one process
// on one device, exercising exactly the per-range kernels and exchange points;
// the tests use it to check the sharded path on a single B200.
#include <dlfcn.h>
#include <nccl.h>  // types and signatures only: NCCL is loaded lazily (see nccl())

#include <algorithm>
#include <cstring>
#include <vector>

#include "engine.cuh"
#include "model.cuh"

namespace bg {
namespace {

// NCCL is resolved at first use with dlopen("libnccl.so.2"): inside a torch
// process that returns the NCCL torch already loaded (same soname), and a
// plain C++ host gets the system library.  Linking it at load time instead
// would pin whichever NCCL the dynamic linker found first for the whole
// process.
struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return r;
    r.get_unique_id = reinterpret_cast<decltype(r.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    r.comm_init_rank = reinterpret_cast<decltype(r.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    r.comm_destroy = reinterpret_cast<decltype(r.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    r.group_start = reinterpret_cast<decltype(r.group_start)>(dlsym(h, "ncclGroupStart"));
    r.group_end = reinterpret_cast<decltype(r.group_end)>(dlsym(h, "ncclGroupEnd"));
    r.broadcast = reinterpret_cast<decltype(r.broadcast)>(dlsym(h, "ncclBroadcast"));
    r.error_string = reinterpret_cast<decltype(r.error_string)>(dlsym(h, "ncclGetErrorString"));
    return r;
  }();
  if (!n.get_unique_id || !n.comm_init_rank || !n.broadcast)
    throw std::runtime_error("NCCL (libnccl.so.2) is not available");
  return n;
}

}  // namespace
}  // namespace bg

struct bg_comm {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;
  // External exchange (bg_comm_create_external): a host callback in place of
  // NCCL, e.g. a host-staged all-gather over another transport.
  bg_allgather_fn ext = nullptr;
  void* ext_ctx = nullptr;
  ~bg_comm() {
    if (comm && !ext) bg::nccl().comm_destroy(comm);
  }
};

namespace bg {
namespace {

#define BG_NCCL(call)                                                                       \
  do {                                                                                      \
    ncclResult_t r_ = (call);                                                               \
    if (r_ != ncclSuccess)                                                                  \
      throw ::bg::cuda_error(std::string("NCCL error: ") + ::bg::nccl().error_string(r_) +  \
                             " at " __FILE__ ":" + std::to_string(__LINE__));               \
  } while (0)

// Per-op CUDA-event timing of the sharded forward (bench.py's kernel table at
// N > 1); labels follow the single-GPU forward, plus "layerI.allgather".
using EventList = std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>>;
struct Timer {
  EventList* ev = nullptr;
  cudaStream_t s = nullptr;
  void begin(const std::string& label) {
    if (!ev) return;
    cudaEvent_t a, b;
    BG_CUDA(cudaEventCreate(&a));
    BG_CUDA(cudaEventCreate(&b));
    BG_CUDA(cudaEventRecord(a, s));
    ev->push_back({label, {a, b}});
  }
  void end() {
    if (ev) BG_CUDA(cudaEventRecord(ev->back().second.second, s));
  }
};

struct Shard {
  bg_model& m;
  const std::vector<int64_t>& bounds;  // world + 1 node-row boundaries
  std::vector<std::pair<int64_t, int64_t>> ranges;  // ranges computed by this process
  int64_t off;                         // node row of the model graph's first FRDC row (a shard's row0)
  bg_comm* comm;                       // null: virtual ranks in one process
  cudaStream_t s;
  Timer tm;
  std::string prefix;  // "layerI." of the layer being run

  // Make rows [bounds[q], bounds[q+1]) of a full-size buffer valid on every rank.
  void allgather(void* buf, int64_t row_bytes) {
    if (!comm) return;
    tm.begin(prefix + "allgather");
    if (comm->ext) {  // the callback runs on the host once this rank's rows are produced
      BG_CUDA(cudaStreamSynchronize(s));
      const int rc = comm->ext(comm->ext_ctx, buf, row_bytes, bounds.data(), comm->world, comm->rank, s);
      if (rc) throw std::runtime_error("sharded forward: external all-gather failed (" + std::to_string(rc) + ")");
      tm.end();
      return;
    }
    BG_NCCL(nccl().group_start());
    for (int q = 0; q < comm->world; ++q) {
      const int64_t r0 = bounds[q], r1 = bounds[q + 1];
      if (r1 <= r0) continue;
      char* p = static_cast<char*>(buf) + r0 * row_bytes;
      BG_NCCL(nccl().broadcast(p, p, static_cast<size_t>((r1 - r0) * row_bytes), ncclUint8, q,
                            comm->comm, s));
    }
    BG_NCCL(nccl().group_end());
    tm.end();
  }

  int64_t row_bytes(const Op& o) const {
    return o.prec == BG_F ? o.cols * 4 : spw(o.cols, o.wb) * 4;
  }

  Op alloc_like(int prec, int64_t cols, int wb) {
    Op o;
    o.prec = prec;
    o.rows = m.graph->n;
    o.cols = cols;
    o.wb = wb;
    if (prec == BG_F) o.f = static_cast<float*>(m.pool.get(o.bytes()));
    else o.bits = static_cast<uint32_t*>(m.pool.get(o.bytes()));
    return o;
  }

  // Both MMs of a SAGE / GraphConv layer as one paired F->B product on this
  // process's rows (the input read once); false when they do not pair.
  bool mm_pair(ModelLayer& l, const Op& x, Op& hs, Op& hn) {
    const bg_variant p0 = l.info.plan[0], p1 = l.info.plan[1];
    auto fb = [](bg_variant v) { return v.op == BG_BMM && v.in1 == BG_F && v.out == BG_B; };
    if (!fb(p0) || !fb(p1) || x.prec != BG_F || x.scale) return false;
    if (l.w1.rows != l.w2.rows || l.w1.cols != l.w2.cols || l.w1.wb != m.wb || l.w2.wb != m.wb ||
        x.cols != l.w1.rows)
      return false;
    const int64_t n = l.w1.cols, ospw = spw(n, m.wb);
    const uint32_t* wtp = paired_weights(l, m.wb, s);
    Op a = alloc_like(BG_B, n, m.wb), b = alloc_like(BG_B, n, m.wb);
    tm.begin(prefix + "mm_pair[" + variant_name(p0) + "]");
    bool first = true;
    for (auto [r0, r1] : ranges) {
      if (r1 <= r0) continue;
      BmmArgs k;
      k.rows = r1 - r0;
      k.k = x.cols;
      k.n = k.n2 = n;
      k.wb = m.wb;
      k.wt = wtp;
      k.a_f = x.f + r0 * x.cols;
      k.out_bits = a.bits + r0 * ospw;
      k.out_bits2 = b.bits + r0 * ospw;
      if (!bmm_pair(k, s)) {
        if (first) {  // nothing launched: the caller runs the two products
          tm.end();
          if (tm.ev) {
            cudaEventDestroy(tm.ev->back().second.first);
            cudaEventDestroy(tm.ev->back().second.second);
            tm.ev->pop_back();
          }
          return false;
        }
        BmmArgs one = k;  // a later range the pair kernels do not take
        one.out_bits2 = nullptr;
        one.n2 = 0;
        one.wt = l.w1.wt.as<uint32_t>();
        bmm(one, s);
        one.wt = l.w2.wt.as<uint32_t>();
        one.out_bits = k.out_bits2;
        bmm(one, s);
      }
      first = false;
    }
    tm.end();
    hs = a;
    hn = b;
    return true;
  }

  // ref: run_mm_slot on rows [r0, r1) (row-local).
  Op mm(bg_variant v, const Op& x, const WeightDev& w, const std::string& label) {
    tm.begin(prefix + label + "[" + variant_name(v) + "]");
    Op o = mm_impl(v, x, w);
    tm.end();
    return o;
  }
  Op mm_impl(bg_variant v, const Op& x, const WeightDev& w) {
    if (v.in1 == BG_F && v.in2 == BG_F && v.out == BG_F) fail("sharded forward: MM.FFF not supported");
    if (v.in1 == BG_B && x.wb != w.wb) fail("bmm: operand word widths disagree");
    if (x.cols != w.rows) fail("bmm: inner dimensions disagree");
    const int wb = w.wb;
    Op out = alloc_like(v.out, w.cols, wb);
    float* alpha_all = nullptr;
    if (v.in1 == BG_F && v.out == BG_F)
      alpha_all = static_cast<float*>(m.pool.get(static_cast<size_t>(x.rows) * 4));
    for (auto [r0, r1] : ranges) {
      if (r1 <= r0) continue;
      BmmArgs k;
      k.rows = r1 - r0;
      k.k = x.cols;
      k.n = w.cols;
      k.wb = wb;
      k.wt = w.wt.as<uint32_t>();
      if (v.in1 == BG_F) {
        k.a_f = x.f + r0 * x.cols;
        if (alpha_all) {
          l1_scales(k.a_f, k.rows, x.cols, BG_AXIS_ROW, alpha_all + r0, s);
          k.alpha = alpha_all + r0;
        }
      } else {
        k.a_bits = x.bits + r0 * spw(x.cols, x.wb);
        k.alpha = x.scale ? x.scale + r0 : nullptr;
      }
      if (v.out == BG_B) {
        k.out_bits = out.bits + r0 * spw(w.cols, wb);
      } else {
        k.out_f = out.f + r0 * w.cols;
        k.beta = w.scale.as<float>();
      }
      bmm(k, s);
    }
    return out;
  }

  Op spmm(bg_variant v, const bg_frdc* A, const float* rs, const float* cs, const Op& x,
          bool& x_full) {
    if (!x_full) {
      allgather(x.prec == BG_F ? static_cast<void*>(x.f) : static_cast<void*>(x.bits), row_bytes(x));
      x_full = true;
    }
    tm.begin(prefix + "spmm[" + variant_name(v) + "]");
    Op out = alloc_like(v.out, x.cols, v.in1 == BG_B ? x.wb : m.wb);
    // FRDC rows are local (rows r - off of a shard); outputs and row scales
    // are indexed by node row, so their bases move by off rows
    const int64_t orow = out.prec == BG_F ? out.cols : spw(out.cols, out.wb);
    uint32_t* obits = out.bits ? out.bits + off * orow : nullptr;
    float* of = out.f ? out.f + off * orow : nullptr;
    for (auto [r0, r1] : ranges) {
      if (r1 <= r0) continue;
      if (v.in1 == BG_B && v.in2 == BG_B) {
        bspmm_bb(*A, x.bits, x.cols, x.wb, obits, of, s, r0 - off, r1 - off);
      } else {
        SpmmFArgs a;
        a.f = x.cols;
        if (v.in1 == BG_B) {
          a.x_bits = x.bits;
          a.xwb = x.wb;
        } else {
          a.x_f = x.f;
        }
        a.row_scale = v.in2 == BG_F && rs ? rs + off : nullptr;
        a.col_scale = v.in2 == BG_F ? cs : nullptr;
        a.out_bits = obits;
        a.owb = out.wb;
        a.out_f = of;
        bspmm_f(*A, a, s, r0 - off, r1 - off);
      }
    }
    tm.end();
    return out;
  }

  // fuse_relu: the layer's ReLU inside the F-output ADD kernel
  Op add(bg_variant v, const Op& a, const Op& b, bool fuse_relu) {
    tm.begin(prefix + "add[" + variant_name(v) + "]");
    Op out = alloc_like(v.out, a.cols, a.wb);
    for (auto [r0, r1] : ranges) {
      if (r1 <= r0) continue;
      if (v.in1 == BG_F) {
        add_fff(a.f + r0 * a.cols, b.f + r0 * b.cols, (r1 - r0) * a.cols, out.f + r0 * a.cols, s, fuse_relu);
      } else if (v.out == BG_B) {
        const int64_t w = spw(a.cols, a.wb);
        add_bbb(a.bits + r0 * w, b.bits + r0 * w, (r1 - r0) * w, out.bits + r0 * w, s);
      } else {
        const int64_t w = spw(a.cols, a.wb);
        add_bbf(a.bits + r0 * w, b.bits + r0 * w, r1 - r0, a.cols, a.wb, out.f + r0 * a.cols, s, fuse_relu);
      }
    }
    tm.end();
    return out;
  }

  void relu_rows(Op& x) {
    if (x.prec != BG_F) return;
    tm.begin(prefix + "relu");
    for (auto [r0, r1] : ranges)
      if (r1 > r0) relu(x.f + r0 * x.cols, (r1 - r0) * x.cols, s);
    tm.end();
  }
};

void forward_sharded(bg_model& m, const Op& x0, const std::vector<int64_t>& bounds, int world,
                     int rank, bg_comm* comm, float* out_base, float* logits_base, cudaStream_t s,
                     EventList* timing = nullptr) {
  if (!m.graph) fail("sharded forward: model carries no graph");
  const int64_t n = m.graph->n;
  if (static_cast<int>(bounds.size()) != world + 1 || bounds.front() != 0 || bounds.back() != n)
    fail("sharded forward: bounds must run from 0 to the node count");
  for (int q = 0; q < world; ++q)
    if (bounds[q] > bounds[q + 1] || (bounds[q] % 4 != 0))
      fail("sharded forward: bounds must be non-decreasing tile-row (multiple of 4) offsets");
  if (x0.prec != m.input_prec) fail("model input tag does not match the provided operand");
  {
    std::vector<std::string> errors = validate_model(true, m.input_prec, m.infos);
    if (!errors.empty()) fail("invalid model: " + errors.front());
  }
  m.pool.reset();
  Shard sh{m, bounds, {}, m.graph->row0, comm, s, Timer{timing, s}, ""};
  if (comm) sh.ranges.push_back({bounds[rank], bounds[rank + 1]});
  else
    for (int q = 0; q < world; ++q) sh.ranges.push_back({bounds[q], bounds[q + 1]});
  // the model's graph (whole, or this rank's shard) must hold every range
  for (auto [r0, r1] : sh.ranges)
    if (r1 > r0 && (r0 < m.graph->row0 || r1 > m.graph->row0 + m.graph->structure->rows ||
                    r1 > m.graph->row0 + m.graph->raw->rows))
      fail("sharded forward: the model's graph does not hold node rows [" + std::to_string(r0) + ", " +
           std::to_string(r1) + ")");

  Op cur = x0;
  bool cur_full = comm == nullptr;  // virtual mode: every range is computed here
  const size_t nl = m.layers.size();
  float* probs_done = nullptr;
  for (size_t i = 0; i < nl; ++i) {
    ModelLayer& l = m.layers[i];
    sh.prefix = "layer" + std::to_string(i) + ".";
    try {
      switch (l.info.kind) {
        case BG_LAYER_GCN: {
          const bg_variant mm = l.info.plan[0], sp = l.info.plan[1];
          const bg_frdc& A = *m.graph->structure;
          const bool fused = mm.in1 == BG_B && mm.in2 == BG_B && mm.out == BG_F &&
                             sp.in1 == BG_F && sp.in2 == BG_B && sp.out == BG_F && !l.relu &&
                             cur.prec == BG_B && cur.sem == BG_PLUS_MINUS && !cur.scale && cur.wb == m.wb &&
                             cur.cols == l.w1.rows && cur.rows == A.cols &&
                             gcn1_fused_supported(A, cur.cols, cur.wb, l.w1.cols);
          if (fused) {
            if (comm && cur.bits == x0.bits) {
              // the caller's rank-local input (read through a shifted base):
              // gather into a full-size buffer, never into the caller's memory
              Op full = sh.alloc_like(BG_B, cur.cols, cur.wb);
              const int64_t rb = sh.row_bytes(cur), r0 = bounds[rank], r1 = bounds[rank + 1];
              if (r1 > r0)
                BG_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(full.bits) + r0 * rb,
                                        reinterpret_cast<const char*>(cur.bits) + r0 * rb,
                                        static_cast<size_t>((r1 - r0) * rb), cudaMemcpyDeviceToDevice, s));
              full.sem = cur.sem;
              cur = full;
              cur_full = false;
            }
            if (!cur_full) {
              sh.allgather(cur.bits, sh.row_bytes(cur));
              cur_full = true;
            }
            auto* recs = static_cast<uint32_t*>(m.pool.get(static_cast<size_t>(n + 1) * 64));  // + zero record
            sh.tm.begin(sh.prefix + "mm[" + variant_name(mm) + "]");
            gcn1_records(cur.bits, n, cur.cols, cur.wb, l.w1.wt.as<uint32_t>(), l.w1.scale.as<float>(),
                         l.w1.cols, recs, s);
            sh.tm.end();
            Op o = sh.alloc_like(BG_F, l.w1.cols, m.wb);
            float* probs = nullptr;
            if (i + 1 < nl && m.layers[i + 1].info.kind == BG_LAYER_SOFTMAX)
              probs = (i + 2 == nl && out_base) ? out_base : static_cast<float*>(m.pool.get(o.bytes()));
            sh.tm.begin(sh.prefix + "spmm[" + variant_name(sp) + "]");
            const int64_t C = l.w1.cols, off = sh.off;
            for (auto [r0, r1] : sh.ranges)
              if (r1 > r0)
                gcn1_aggregate(A, recs, cur.cols, cur.wb, l.w1.wt.as<uint32_t>(), l.w1.scale.as<float>(), C,
                               o.f + off * C, probs ? probs + off * C : nullptr, s, r0 - off, r1 - off);
            sh.tm.end();
            probs_done = probs;
            cur = o;
            cur_full = comm == nullptr;
            break;
          }
          Op h = sh.mm(mm, cur, l.w1, "mm");
          bool h_full = comm == nullptr;
          const bool fac = sp.in2 == BG_F;
          cur = sh.spmm(sp, &A, fac ? m.graph->norm.as<float>() : nullptr,
                        fac ? m.graph->norm.as<float>() : nullptr, h, h_full);
          cur_full = comm == nullptr;
          if (l.relu) sh.relu_rows(cur);
          break;
        }
        case BG_LAYER_SAGE:
        case BG_LAYER_GRAPHCONV: {
          const bool mean = l.info.kind == BG_LAYER_SAGE;
          Op hs, hn;
          if (!sh.mm_pair(l, cur, hs, hn)) {
            hs = sh.mm(l.info.plan[0], cur, l.w1, "mm_self");
            hn = sh.mm(l.info.plan[1], cur, l.w2, "mm_neigh");
          }
          bool hn_full = comm == nullptr;
          const bg_variant sp = l.info.plan[2];
          const bool fac = sp.in2 == BG_F;
          const float* rs = fac ? (mean ? m.graph->mean_row.as<float>() : m.graph->ones.as<float>()) : nullptr;
          const float* cs = fac ? m.graph->ones.as<float>() : nullptr;
          Op agg = sh.spmm(sp, m.graph->raw.get(), rs, cs, hn, hn_full);
          if (mean && sp.in2 == BG_B && sp.out == BG_F)
            for (auto [r0, r1] : sh.ranges)
              if (r1 > r0)
                scale_rows_double(agg.f + r0 * agg.cols, r1 - r0, agg.cols,
                                  m.graph->neighbor_count.as<int64_t>() + r0, s);
          cur = sh.add(l.info.plan[3], hs, agg, l.relu && l.info.plan[3].out == BG_F);
          cur_full = comm == nullptr;
          break;
        }
        case BG_LAYER_FC:
          cur = sh.mm(l.info.plan[0], cur, l.w1, "mm");
          cur_full = comm == nullptr;
          if (l.relu) sh.relu_rows(cur);
          break;
        case BG_LAYER_RELU:
          if (cur.f == x0.f) fail("sharded forward: a leading ReLU layer is not supported");
          sh.relu_rows(cur);
          break;
        case BG_LAYER_SOFTMAX: {
          if (logits_base)
            for (auto [r0, r1] : sh.ranges)
              if (r1 > r0)
                BG_CUDA(cudaMemcpyAsync(logits_base + r0 * cur.cols, cur.f + r0 * cur.cols,
                                        static_cast<size_t>((r1 - r0) * cur.cols) * 4,
                                        cudaMemcpyDeviceToDevice, s));
          float* dst = (i + 1 == nl && out_base) ? out_base : static_cast<float*>(m.pool.get(cur.bytes()));
          if (probs_done && i == nl - 1 && probs_done == out_base) {
            // already produced by the fused aggregation epilogue (an empty
            // timed span keeps the label list of the 1-GPU forward)
            sh.tm.begin(sh.prefix + "softmax");
            sh.tm.end();
          } else {
            sh.tm.begin(sh.prefix + "softmax");
            for (auto [r0, r1] : sh.ranges)
              if (r1 > r0) softmax_rows(cur.f + r0 * cur.cols, r1 - r0, cur.cols, dst + r0 * cur.cols, s);
            sh.tm.end();
          }
          cur.f = dst;
          break;
        }
        default:
          fail(std::string("sharded forward: layer kind ") + layer_kind_name(l.info.kind) +
               " is not supported");
      }
    } catch (const cuda_error&) {
      throw;
    } catch (const std::exception& e) {
      throw std::runtime_error("layer " + std::to_string(i) + " (" + layer_kind_name(l.info.kind) +
                               "): " + e.what());
    }
  }
  if (cur.prec != BG_F) fail("model output must be full precision");
  const bool last_softmax = nl && m.layers[nl - 1].info.kind == BG_LAYER_SOFTMAX;
  for (auto [r0, r1] : sh.ranges) {
    if (r1 <= r0) continue;
    const size_t bytes = static_cast<size_t>((r1 - r0) * cur.cols) * 4;
    if (out_base && cur.f != out_base)
      BG_CUDA(cudaMemcpyAsync(out_base + r0 * cur.cols, cur.f + r0 * cur.cols, bytes,
                              cudaMemcpyDeviceToDevice, s));
    if (logits_base && !last_softmax)
      BG_CUDA(cudaMemcpyAsync(logits_base + r0 * cur.cols, cur.f + r0 * cur.cols, bytes,
                              cudaMemcpyDeviceToDevice, s));
  }
}

}  // namespace
}  // namespace bg

namespace bg {
namespace {
void sharded_entry(bg_model* m, bg_comm* comm, const bg_mat* x, const int64_t* bounds, int world, int rank,
                   float* out, float* logits, bg_stream stream, EventList* timing) {
  {
    if (!m || !x || !bounds) fail("sharded forward: null argument");
    if (comm && (comm->world != world || comm->rank != rank))
      fail("sharded forward: communicator does not match world/rank");
    if (rank < 0 || rank >= world) fail("sharded forward: bad rank");
    std::vector<int64_t> b(bounds, bounds + world + 1);
    Op x0 = op_from_mat(x);
    const int64_t r0 = b[rank], r1 = b[rank + 1];
    int64_t oc = 0;
    for (const auto& l : m->layers)
      if (l.info.has_w1) oc = l.w1.cols;
    float* out_base = out;
    float* log_base = logits;
    if (comm) {
      // x and out hold this rank's rows only: index them through shifted bases
      if (x0.rows != r1 - r0) fail("sharded forward: x must hold this rank's rows");
      if (x0.prec == BG_F) x0.f -= r0 * x0.cols;
      else x0.bits -= r0 * spw(x0.cols, x0.wb);
      x0.rows = m->graph ? m->graph->n : x0.rows;
      if (out) out_base = out - r0 * oc;
      if (logits) log_base = logits - r0 * oc;
    }
    forward_sharded(*m, x0, b, world, rank, comm, out_base, log_base, S(stream), timing);
  }
}
}  // namespace
}  // namespace bg

using namespace bg;

extern "C" {

int bg_partition_bounds(const uint64_t* rp, int64_t tile_rows, int64_t n, int world,
                        int64_t* bounds) {
  return guard([&] {
    if (world < 1) fail("partition: world size must be positive");
    if (!rp || !bounds) fail("partition: null pointer");
    const uint64_t total = rp[tile_rows];
    bounds[0] = 0;
    for (int k = 1; k < world; ++k) {
      const uint64_t target = (total * static_cast<uint64_t>(k) + world - 1) / world;
      const int64_t t = std::lower_bound(rp, rp + tile_rows + 1, target) - rp;
      bounds[k] = std::max<int64_t>(bounds[k - 1], std::min<int64_t>(4 * t, n));
      bounds[k] -= bounds[k] % 4;
      bounds[k] = std::max<int64_t>(bounds[k - 1], bounds[k]);
    }
    bounds[world] = n;
  });
}

int bg_comm_unique_id(uint8_t* out, size_t len) {
  return guard([&] {
    if (!out || len < sizeof(ncclUniqueId)) fail("unique id buffer too small");
    ncclUniqueId id;
    BG_NCCL(nccl().get_unique_id(&id));
    std::memcpy(out, &id, sizeof id);
  });
}

int bg_comm_create(int world, int rank, const uint8_t* id, size_t len, bg_comm** out) {
  return guard([&] {
    if (!out || !id || len < sizeof(ncclUniqueId)) fail("bad communicator arguments");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    auto c = std::make_unique<bg_comm>();
    c->world = world;
    c->rank = rank;
    BG_NCCL(nccl().comm_init_rank(&c->comm, world, uid, rank));
    *out = c.release();
  });
}

void bg_comm_destroy(bg_comm* c) { delete c; }

int bg_comm_create_external(int world, int rank, bg_allgather_fn fn, void* ctx, bg_comm** out) {
  return guard([&] {
    if (!out || !fn) fail("bad communicator arguments");
    if (world < 1 || rank < 0 || rank >= world) fail("partition: bad rank/world size");
    auto c = std::make_unique<bg_comm>();
    c->world = world;
    c->rank = rank;
    c->ext = fn;
    c->ext_ctx = ctx;
    *out = c.release();
  });
}

int bg_graph_shard(const bg_graph* g, int64_t row_begin, int64_t row_end, bg_graph** out, bg_stream stream) {
  return guard([&] {
    if (!g || !out) fail("graph shard: null argument");
    *out = graph_shard(*g, row_begin, row_end, S(stream)).release();
  });
}

int bg_model_forward_sharded(bg_model* m, bg_comm* comm, const bg_mat* x, const int64_t* bounds,
                             int world, int rank, float* out, float* logits, bg_stream stream) {
  return guard([&] {
    auto run = [&] { sharded_entry(m, comm, x, bounds, world, rank, out, logits, stream, nullptr); };
    cudaStream_t st = S(stream);
    // An NCCL exchange is stream-ordered and capturable: the forward replays
    // as one CUDA graph (kernels + broadcasts) like bg_model_forward.  The
    // external exchange runs host code mid-forward and is never captured.
    if (!m || !x || !bounds || !comm || comm->ext || !m->capture || st == nullptr) {
      run();
      return;
    }
    bg_model::Key k;
    k.x = x->data;
    k.rows = x->rows;
    k.cols = x->cols;
    k.prec = x->precision;
    k.wb = x->word_bits;
    k.out = out;
    k.logits = logits;
    k.s = st;
    uint64_t h = reinterpret_cast<uintptr_t>(comm) * 0x9E3779B97F4A7C15ull ^ static_cast<uint64_t>(world * 131 + rank);
    for (int q = 0; q <= world; ++q) h = h * 1000003ull ^ static_cast<uint64_t>(bounds[q]);
    k.extra = h;
    run_captured(*m, m->sharded, k, st, run);
  });
}

int bg_model_forward_sharded_timed(bg_model* m, bg_comm* comm, const bg_mat* x, const int64_t* bounds,
                                   int world, int rank, float* out, bg_kernel_timing* timings, int cap, int* n,
                                   bg_stream stream) {
  EventList ev;
  const int rc = guard([&] {
    sharded_entry(m, comm, x, bounds, world, rank, out, nullptr, stream, &ev);
    BG_CUDA(cudaStreamSynchronize(S(stream)));
    int k = 0;
    for (const auto& e : ev) {
      if (k >= cap) break;
      float ms = 0.0f;
      BG_CUDA(cudaEventElapsedTime(&ms, e.second.first, e.second.second));
      std::memset(timings[k].label, 0, sizeof timings[k].label);
      std::strncpy(timings[k].label, e.first.c_str(), sizeof timings[k].label - 1);
      timings[k].ms = ms;
      ++k;
    }
    if (n) *n = k;
  });
  for (auto& e : ev) {
    cudaEventDestroy(e.second.first);
    cudaEventDestroy(e.second.second);
  }
  return rc;
}

}  // extern "C"

