// Model / trace objects behind the C ABI handles.
#pragma once

#include <functional>
#include <string>
#include <utility>
#include <vector>

#include "engine.cuh"

namespace bg {

struct LayerInfo {
  int kind = BG_LAYER_FC;
  std::vector<bg_variant> plan;
  bool has_w1 = false, has_w2 = false, has_bn = false, has_scale = false;
};

struct WeightDev {
  int64_t rows = 0, cols = 0;
  int wb = 32;
  DevBuf f, bits, scale, wt;
  void upload(const float* host, int64_t r, int64_t c, int wb, cudaStream_t s);
  WeightCache cache() const;
};

struct ModelLayer {
  LayerInfo info;
  bool relu = false;
  WeightDev w1, w2;
  DevBuf wt_pair;  // W1 | zero pad to a 32-column boundary | W2, transposed bits (paired FBB)
  DevBuf bn_g, bn_b, bn_m, bn_s;
  int64_t bn_len = 0;
  DevBuf sr, sc;
  int64_t sr_len = 0, sc_len = 0;
};

struct TracePoint {
  std::string label;
  int64_t rows = 0, cols = 0;
  int wb = 32;
  DevBuf bits;
};

int layer_output_precision(const LayerInfo& l, int in, std::vector<std::string>* errors);
std::vector<std::string> validate_model(bool has_graph, int input_prec,
                                        const std::vector<LayerInfo>& layers);
LayerInfo layer_info(const bg_layer_desc& d);

// The paired-product weight layout of a SAGE / GraphConv layer (W1 | pad | W2).
const uint32_t* paired_weights(ModelLayer& l, int wb, cudaStream_t s);

}  // namespace bg

struct bg_trace {
  std::vector<bg::TracePoint> pts;
};

struct bg_model {
  const bg_graph* graph = nullptr;
  int input_prec = BG_F;
  int strategy = -1;
  int wb = 32;
  std::vector<bg::LayerInfo> infos;
  std::vector<bg::ModelLayer> layers;
  bg::Pool pool;
  int64_t last_out_cols = -1;
  // CUDA-graph replay of a forward bound to fixed buffers (bg_model_forward,
  // and the NCCL-sharded forward): one slot each.
  bool capture = true;
  struct Key {
    const void* x = nullptr;
    int64_t rows = 0, cols = 0;
    int prec = 0, wb = 0;
    float* out = nullptr;
    float* logits = nullptr;
    cudaStream_t s = nullptr;
    uint64_t agg_gen = 0;    // aggregation layout settings the graph was recorded with
    uint64_t pool_gen = 0;   // pool allocation state the graph's pointers come from
    uint64_t graph_gen = 0;  // FRDC views the graph's pointers come from
    uint64_t extra = 0;      // sharded: communicator, rank and bounds
    bool operator==(const Key& o) const {
      return x == o.x && rows == o.rows && cols == o.cols && prec == o.prec && wb == o.wb &&
             out == o.out && logits == o.logits && s == o.s && agg_gen == o.agg_gen &&
             pool_gen == o.pool_gen && graph_gen == o.graph_gen && extra == o.extra;
    }
  };
  struct CaptureSlot {
    Key key;
    cudaGraphExec_t exec = nullptr;
    void reset() {
      if (exec) cudaGraphExecDestroy(exec);
      exec = nullptr;
      key = Key{};
    }
    ~CaptureSlot() { reset(); }
  };
  CaptureSlot fwd, sharded;
  // Buffers of the host-pointer entry point.
  bg::DevBuf hx, hout, hlog;
  cudaStream_t copy_stream = nullptr;    // H2D / D2H of the host entry point
  std::vector<cudaEvent_t> chunk_events;  // 2 x chunks (input landed, output ready)
  ~bg_model() {
    for (cudaEvent_t e : chunk_events) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
  }
};

namespace bg {
// Host-streaming context (bg_model_forward_host): the model input arrives in
// row chunks (in.ready events) and the final output is produced per row chunk
// (out.ready recorded; out_done set when the last layer did so).
struct StreamChunks {
  RowChunks in, out;
  bool out_done = false;
};
// One layer called on its own (ref: gcn_layer / sage_layer / graphconv_layer,
// graphops.cpp:270-335): labels start with `prefix`, the result may be
// binary and is left in the model's pool.
struct LayerCall {
  std::string prefix;
  Op result;
};
// Runs `run` on stream st through the slot's CUDA graph: the first call with
// a binding runs eagerly (sizing the pool, building views), the second
// captures, later ones replay -- re-recorded whenever the key (binding,
// aggregation settings, pool or FRDC-view generation) changes.
uint64_t graph_generation(const bg_graph* g);
void run_captured(bg_model& m, bg_model::CaptureSlot& slot, bg_model::Key k, cudaStream_t st,
                  const std::function<void()>& run);
// persistent.cu: the whole forward as one cooperative kernel for small
// graphs and binary GCN chains; false when not eligible (nothing launched).
bool persistent_forward(bg_model& m, const Op& x0, float* out, float* logits, cudaStream_t s);
bool persistent_forced();             // bg_set_persistent(1)
void set_persistent_forced(bool on);
void forward_impl(bg_model& m, const Op& x0, float* out, float* logits, bg_trace* trace,
                  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>>* timing,
                  cudaStream_t s, StreamChunks* chunks = nullptr, LayerCall* single = nullptr);
}
