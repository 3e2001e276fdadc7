// Pack = K job lanes of one model co-resident on one GPU, plus the launch
// sequence of one training step for all of them.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "models.cuh"
#include "tlk_common.cuh"

namespace tlk {

struct Pack {
  // description
  int model = 0, batch = 0, lanes = 0, max_steps = 0, host_input = 0;
  const ModelDef* def = nullptr;      // MLP / CNN
  GptCfg gcfg{};                       // transformer packs
  std::vector<TensorInfo> tinfo;       // parameter tensors of a lane (all models)
  TensorInfo* tinfo_dev = nullptr;
  int64_t pcount = 0, stride = 0;
  // lane table
  LaneState* lane_dev = nullptr;
  std::vector<LaneState> lane_host;
  // per-lane arenas [lanes, stride]
  float *params = nullptr, *grads = nullptr, *mom1 = nullptr, *mom2 = nullptr;
  uint16_t* wbf = nullptr;
  float* loss = nullptr;       // [lanes, max_steps]
  float* last_loss = nullptr;  // [lanes]
  // inputs
  uint8_t* pixels = nullptr;   // [lanes, batch, 784]
  int32_t* labels = nullptr;   // [lanes, batch]
  uint16_t* x = nullptr;       // [lanes, batch, 784] bf16 (k/256)
  const int8_t* teacher = nullptr;  // [10, 784] (context-owned)
  // model scratch (one allocation, carved by the model's alloc function)
  void* scratch = nullptr;            // host-side struct of device pointers
  void (*scratch_free)(void*) = nullptr;
  void* acts = nullptr;          // activation scratch base (TLK_BUF_ACTS)
  size_t acts_bytes = 0;
  uint16_t* wt = nullptr;       // transposed bf16 weight copies (model specific)
  int64_t wt_stride = 0;
  // all device allocations of this pack, freed on destroy; their bytes are
  // charged to the owning context's budget (tlk_set_mem_limit)
  std::vector<void*> allocs;
  size_t alloc_bytes = 0;
  int64_t* ctx_in_use = nullptr;  // the context's running total
  int64_t ctx_limit = 0;          // 0 = no budget (device memory only)
  // the stream this pack's work is enqueued on: the context stream, or its
  // own (TLK_PACK_OWN_STREAM) so packs of different models run concurrently
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // CUDA graph of one step
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  int launches_per_step = 0;
  // parameter range (floats, within a lane) whose update is fused into its
  // wgrad epilogue (see cnn.cu); the end-of-step optimizer skips it
  int64_t fused_lo = 0, fused_hi = 0;
  // work of a step that runs after its graph, on a stream of its own (CNN:
  // fc1 wgrad + Adam, overlapping the next step's forward; cnn.cu): the
  // runtime launches defer() after every step-graph launch, once the graph's
  // ev_defer_in has fired, and records ev_defer_out after it; the next step
  // graph waits for ev_defer_out where it needs the result, and every API call
  // that exposes pack state first makes the pack stream wait for it (settle)
  int (*defer)(Pack&, cudaStream_t) = nullptr;
  cudaStream_t defer_st = nullptr;
  cudaEvent_t ev_defer_in = nullptr, ev_defer_out = nullptr;
  // side stream + events for concurrent graph branches
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_tail = nullptr;
  // pipelined host-input steps (tlk_step_host_async): a second input slot and
  // the step graph captured against it, a copy stream, per-slot events
  uint8_t* px_alt = nullptr;
  int32_t* lb_alt = nullptr;
  cudaGraph_t hgraph_alt = nullptr, hgraph0 = nullptr;
  cudaGraphExec_t hexec_alt = nullptr, hexec0 = nullptr;
  // per-slot losses written by the head kernel straight into mapped pinned
  // host memory (no D2H copy in the step); copied to the caller's buffer
  // by tlk_step_host_wait
  float* ll_host = nullptr;  // [2][lanes]
  float* hout[2] = {nullptr, nullptr};
  cudaStream_t copy_st = nullptr;
  cudaEvent_t h2d_ev[2] = {nullptr, nullptr}, done_ev[2] = {nullptr, nullptr};
  int64_t host_steps = 0;
  int flags = 0;  // TLK_PACK_* (e.g. write every gradient for tests)
  // one step's host-input blob (tlk_step_host_blob): device segments filled in order
  struct HostSeg {
    void* dst;
    size_t bytes;
  };
  std::vector<HostSeg> host_segs;
  // named internal buffers (tlk_pack_named): activations, statistics, snapshots
  struct Named {
    std::string name;
    void* ptr;
    size_t bytes;
  };
  std::vector<Named> named;
  void name_buf(const std::string& n, void* ptr, size_t bytes) { named.push_back({n, ptr, bytes}); }
  // per-kernel profiling (tlk_profile_step): an event after every launch
  std::vector<cudaEvent_t>* prof = nullptr;
  std::vector<const char*>* prof_names = nullptr;
  void mark(cudaStream_t st, const char* name) {
    if (!prof) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);  // a graph node under capture
    prof->push_back(e);
    prof_names->push_back(name);
  }
};

// Device allocation that records ownership; reports "out of memory" on failure.
int pack_alloc(Pack& p, void** ptr, size_t bytes);

// Model hooks.
int mlp_setup(Pack& p);
int mlp_enqueue_step(Pack& p, cudaStream_t st);
int cnn_setup(Pack& p);
int cnn_enqueue_step(Pack& p, cudaStream_t st);
// persistent per-GPU scheduler kernel (cnn_persist.cu): `nsteps` steps of
// every lane in one launch; TLK_PACK_PERSISTENT (or TLK_CNN_PERSIST=1)
bool cnn_persist_enabled(const Pack& p);
int cnn_persist_enqueue(Pack& p, cudaStream_t st, int nsteps);
int gpt_setup(Pack& p);
int gpt_enqueue_step(Pack& p, cudaStream_t st);
int resnet_setup(Pack& p);
int resnet_enqueue_step(Pack& p, cudaStream_t st);
// (count, fan_in) and init kind of every ResNet-18 tensor (oracle/resnet.py order)
void resnet_tensor_list(std::vector<std::pair<int64_t, int>>& cnt_fan, std::vector<int>& kinds);
std::vector<TensorInfo> model_tensors(int model, const GptCfg& c);

// Common kernels (kernels.cu).

int enqueue_inputs(Pack& p, cudaStream_t st);  // datagen (or host-input convert)
int enqueue_head(Pack& p, cudaStream_t st, const uint16_t* h, int hidden, int64_t w_off,
                 int64_t b_off, uint16_t* dz_prev, int64_t db_prev_off);
int enqueue_optimizer(Pack& p, cudaStream_t st);
int enqueue_optimizer_range(Pack& p, cudaStream_t st, int64_t lo, int64_t hi, bool complement,
                            const char* name);
int enqueue_end_step(Pack& p, cudaStream_t st);
int enqueue_lane_init(Pack& p, int lane, cudaStream_t st);
int enqueue_datagen_raw(uint64_t seed, int step, int batch, const int8_t* teacher, uint8_t* px,
                        int32_t* labels, cudaStream_t st);
int build_teacher(int8_t** dev_out);

}  // namespace tlk
