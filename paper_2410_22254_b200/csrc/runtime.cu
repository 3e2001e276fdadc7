// libtlk C ABI: contexts (one per GPU), packs of K job lanes, graph-captured
// steps, host-buffer end-to-end steps, result readback.  See include/tlk.h.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <utility>

#include "pack.cuh"

namespace tlk {

// ------------------------------------------------------------ errors --------
static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation)
    return fail(TLK_EOOM, "out of memory: %s (%s)", what, cudaGetErrorString(e));
  return fail(TLK_ECUDA, "CUDA error %s at %s", cudaGetErrorString(e), what);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("TLK_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

int pack_alloc(Pack& p, void** ptr, size_t bytes) {
  if (!bytes) bytes = 16;
  if (p.ctx_in_use && p.ctx_limit > 0 && *p.ctx_in_use + int64_t(bytes) > p.ctx_limit)
    return fail(TLK_EOOM,
                "out of memory: pack allocation of %zu bytes exceeds the context budget "
                "(%lld of %lld bytes in use)",
                bytes, (long long)*p.ctx_in_use, (long long)p.ctx_limit);
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(TLK_EOOM, "out of memory: pack allocation of %zu bytes failed (%s)", bytes,
                cudaGetErrorString(e));
  }
  p.allocs.push_back(*ptr);
  p.alloc_bytes += bytes;
  if (p.ctx_in_use) *p.ctx_in_use += int64_t(bytes);
  return TLK_OK;
}

}  // namespace tlk

using namespace tlk;

struct tlk_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int8_t* teacher = nullptr;
  std::vector<std::unique_ptr<Pack>> packs;  // destroyed packs leave a null entry (ids stay stable)
  int64_t mem_in_use = 0;  // bytes held by live packs
  int64_t mem_limit = 0;   // admission budget (0 = device memory only)
};

namespace {

void destroy_pack(Pack& p) {
  if (p.copy_st) cudaStreamDestroy(p.copy_st);
  for (int k = 0; k < 2; ++k) {
    if (p.h2d_ev[k]) cudaEventDestroy(p.h2d_ev[k]);
    if (p.done_ev[k]) cudaEventDestroy(p.done_ev[k]);
  }
  if (p.defer_st) {
    cudaStreamSynchronize(p.defer_st);
    cudaStreamDestroy(p.defer_st);
    cudaEventDestroy(p.ev_defer_in);
    cudaEventDestroy(p.ev_defer_out);
    p.defer_st = nullptr;
    p.defer = nullptr;
  }
  if (p.hexec_alt) cudaGraphExecDestroy(p.hexec_alt);
  if (p.hgraph_alt) cudaGraphDestroy(p.hgraph_alt);
  if (p.hexec0) cudaGraphExecDestroy(p.hexec0);
  if (p.hgraph0) cudaGraphDestroy(p.hgraph0);
  if (p.ll_host) cudaFreeHost(p.ll_host);
  if (p.side) cudaStreamDestroy(p.side);
  if (p.ev_fork) cudaEventDestroy(p.ev_fork);
  if (p.ev_join) cudaEventDestroy(p.ev_join);
  if (p.ev_tail) cudaEventDestroy(p.ev_tail);
  if (p.graph_exec) cudaGraphExecDestroy(p.graph_exec);
  if (p.graph) cudaGraphDestroy(p.graph);
  for (void* a : p.allocs) cudaFree(a);
  p.allocs.clear();
  if (p.ctx_in_use) *p.ctx_in_use -= int64_t(p.alloc_bytes);
  p.alloc_bytes = 0;
  if (p.own_stream && p.stream) cudaStreamDestroy(p.stream);
  p.stream = nullptr;
  if (p.scratch && p.scratch_free) p.scratch_free(p.scratch);
  p.scratch = nullptr;
}

int get_pack(tlk_ctx* ctx, int32_t id, Pack** out) {
  TLK_CHECK(ctx, TLK_EINVAL, "null context");
  TLK_CHECK(id >= 0 && id < int32_t(ctx->packs.size()) && ctx->packs[id], TLK_EINVAL,
            "bad pack id %d", id);
  TLK_CUDA(cudaSetDevice(ctx->device));
  *out = ctx->packs[id].get();
  return TLK_OK;
}

int enqueue_step(Pack& p, cudaStream_t st) {
  switch (p.model) {
    case TLK_MODEL_MLP: return mlp_enqueue_step(p, st);
    case TLK_MODEL_CNN: return cnn_enqueue_step(p, st);
    case TLK_MODEL_XFORMER:
    case TLK_MODEL_GPT: return gpt_enqueue_step(p, st);
    case TLK_MODEL_RESNET18: return resnet_enqueue_step(p, st);
  }
  return fail(TLK_EINVAL, "unknown model %d", p.model);
}

int capture_step(Pack& p, cudaStream_t st, cudaGraph_t* graph, cudaGraphExec_t* exec) {
  TLK_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  int rc = enqueue_step(p, st);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(st, &g);
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  TLK_CUDA(e);
  *graph = g;
  TLK_CUDA(cudaGraphInstantiate(exec, g, 0));
  return TLK_OK;
}

int ensure_graph(Pack& p, cudaStream_t st) {
  if (p.graph_exec) return TLK_OK;
  return capture_step(p, st, &p.graph, &p.graph_exec);
}

// Second input slot + the step graph captured against it (inputs are kernel
// arguments of the captured graph), copy stream and per-slot events.
int ensure_host_pipeline(Pack& p, cudaStream_t st) {
  int rc = ensure_graph(p, st);
  if (rc || p.hexec_alt) return rc;
  const size_t L = size_t(p.lanes), B = size_t(p.batch);
  void* v = nullptr;
  if ((rc = pack_alloc(p, &v, L * B * 784))) return rc;
  p.px_alt = static_cast<uint8_t*>(v);
  if ((rc = pack_alloc(p, &v, L * B * 4))) return rc;
  p.lb_alt = static_cast<int32_t*>(v);
  TLK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p.ll_host), 2 * L * 4, cudaHostAllocMapped));
  float* ll_dev = nullptr;
  TLK_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ll_dev), p.ll_host, 0));
  float* const last_loss = p.last_loss;
  p.last_loss = ll_dev;  // slot 0: device inputs of the regular graph, losses to host slot 0
  rc = capture_step(p, st, &p.hgraph0, &p.hexec0);
  if (!rc) {
    p.last_loss = ll_dev + L;
    std::swap(p.pixels, p.px_alt);
    std::swap(p.labels, p.lb_alt);
    rc = capture_step(p, st, &p.hgraph_alt, &p.hexec_alt);
    std::swap(p.pixels, p.px_alt);
    std::swap(p.labels, p.lb_alt);
  }
  p.last_loss = last_loss;
  if (rc) return rc;
  TLK_CUDA(cudaStreamCreateWithFlags(&p.copy_st, cudaStreamNonBlocking));
  for (int k = 0; k < 2; ++k) {
    TLK_CUDA(cudaEventCreateWithFlags(&p.h2d_ev[k], cudaEventDisableTiming));
    TLK_CUDA(cudaEventCreateWithFlags(&p.done_ev[k], cudaEventDisableTiming));
  }
  return TLK_OK;
}

// Launch one step graph, then the step's deferred work (Pack::defer) on the
// pack's defer stream once the graph's ev_defer_in has fired.
int launch_step(Pack& p, cudaGraphExec_t g) {
  TLK_CUDA(cudaGraphLaunch(g, p.stream));
  if (!p.defer) return TLK_OK;
  TLK_CUDA(cudaStreamWaitEvent(p.defer_st, p.ev_defer_in, 0));
  int rc = p.defer(p, p.defer_st);
  if (rc) return rc;
  TLK_CUDA(cudaEventRecord(p.ev_defer_out, p.defer_st));
  return TLK_OK;
}

// Make the pack stream wait for the last step's deferred work: from here on
// the pack's parameters / optimizer state are those after every launched step.
int settle(Pack& p) {
  if (p.defer) TLK_CUDA(cudaStreamWaitEvent(p.stream, p.ev_defer_out, 0));
  return TLK_OK;
}

int upload_lane(tlk_ctx* ctx, Pack& p, int lane) {
  TLK_CUDA(cudaMemcpyAsync(p.lane_dev + lane, &p.lane_host[lane], sizeof(LaneState),
                           cudaMemcpyHostToDevice, p.stream));
  return TLK_OK;
}

}  // namespace

extern "C" {

int tlk_abi_version(void) { return TLK_ABI_VERSION; }
const char* tlk_last_error(void) { return g_err; }

static void fill_info(int model, const GptCfg& c, int batch, tlk_model_info* out) {
  const auto ts = model_tensors(model, c);
  out->param_count = 0;
  for (const auto& t : ts) out->param_count += t.count;
  out->param_stride = ts.empty() ? 0 : round_up(ts.back().off + ts.back().count, PARAM_ALIGN);
  out->num_tensors = int32_t(ts.size());
  if (is_gpt(model)) {  // 6 x (matmul params + attention) per token, x T tokens per sample
    const int64_t d = c.d, T = c.T;
    const int64_t mm = 12 * d * d * c.layers + int64_t(c.V) * d;
    out->flops_per_sample = 6 * T * (mm + int64_t(c.layers) * T * d);
  } else if (model == TLK_MODEL_RESNET18) {  // 6 x conv/fc MACs per sample
    int64_t macs = 32LL * 32 * 64 * 27 + 5120;
    const int C[4] = {64, 128, 256, 512};
    int cin = 64, res = 32;
    for (int s = 0; s < 4; ++s)
      for (int b = 0; b < 2; ++b) {
        const int ci = b == 0 ? cin : C[s], ho = (b == 0 && s > 0) ? res / 2 : res;
        macs += int64_t(ho) * ho * C[s] * 9 * ci + int64_t(ho) * ho * C[s] * 9 * C[s];
        if (b == 0 && s > 0) macs += int64_t(ho) * ho * C[s] * ci;
        res = ho;
        if (b == 1) cin = C[s];
      }
    out->flops_per_sample = 6 * macs;
  } else {
    out->flops_per_sample = 6 * model_def(model)->macs_per_sample;
  }
  (void)batch;
}

int tlk_model_query(int32_t model, int32_t batch, tlk_model_info* out) {
  TLK_CHECK(out && (model_def(model) || is_gpt(model) || model == TLK_MODEL_RESNET18), TLK_EINVAL,
            "unknown model %d", model);
  fill_info(model, gpt_default(model), batch, out);
  return TLK_OK;
}

int tlk_model_tensor(int32_t model, int32_t t, int64_t* offset, int64_t* count, int32_t* fan_in) {
  TLK_CHECK(model_def(model) || is_gpt(model) || model == TLK_MODEL_RESNET18, TLK_EINVAL,
            "unknown model %d", model);
  const auto ts = model_tensors(model, gpt_default(model));
  TLK_CHECK(t >= 0 && t < int32_t(ts.size()), TLK_EINVAL, "bad tensor %d", t);
  if (offset) *offset = ts[t].off;
  if (count) *count = ts[t].count;
  if (fan_in) *fan_in = ts[t].fan_in;
  return TLK_OK;
}

int tlk_open(int32_t device, tlk_ctx** out) {
  TLK_CHECK(out, TLK_EINVAL, "null out");
  int n = 0;
  TLK_CUDA(cudaGetDeviceCount(&n));
  TLK_CHECK(device >= 0 && device < n, TLK_EINVAL, "device %d not visible (%d devices)", device,
            n);
  TLK_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  TLK_CUDA(cudaGetDeviceProperties(&prop, device));
  TLK_CHECK(prop.major == 10 && prop.minor == 0, TLK_ESTATE,
            "libtlk is built for sm_100a (B200); device %d is sm_%d%d", device, prop.major,
            prop.minor);
  auto ctx = std::make_unique<tlk_ctx>();
  ctx->device = device;
  TLK_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  int rc = build_teacher(&ctx->teacher);
  if (rc) return rc;
  *out = ctx.release();
  return TLK_OK;
}

int tlk_close(tlk_ctx* ctx) {
  if (!ctx) return TLK_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& p : ctx->packs)
    if (p) {
      cudaStreamSynchronize(p->stream);
      destroy_pack(*p);
    }
  if (ctx->teacher) cudaFree(ctx->teacher);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return TLK_OK;
}

int tlk_sync(tlk_ctx* ctx) {
  TLK_CHECK(ctx, TLK_EINVAL, "null context");
  TLK_CUDA(cudaSetDevice(ctx->device));
  TLK_CUDA(cudaStreamSynchronize(ctx->stream));
  for (auto& p : ctx->packs)
    if (p && p->defer) {
      TLK_CUDA(cudaStreamSynchronize(p->defer_st));
      if (int rc = settle(*p)) return rc;
    }
  for (auto& p : ctx->packs)
    if (p && p->own_stream) TLK_CUDA(cudaStreamSynchronize(p->stream));
  return TLK_OK;
}

int tlk_set_mem_limit(tlk_ctx* ctx, int64_t bytes) {
  TLK_CHECK(ctx && bytes >= 0, TLK_EINVAL, "bad arguments");
  ctx->mem_limit = bytes;
  for (auto& p : ctx->packs)
    if (p) p->ctx_limit = bytes;
  return TLK_OK;
}

int tlk_mem_in_use(tlk_ctx* ctx, int64_t* bytes) {
  TLK_CHECK(ctx && bytes, TLK_EINVAL, "null argument");
  *bytes = ctx->mem_in_use;
  return TLK_OK;
}

int tlk_pack_destroy(tlk_ctx* ctx, int32_t pack) {
  TLK_CHECK(ctx, TLK_EINVAL, "null context");
  TLK_CHECK(pack >= 0 && pack < int32_t(ctx->packs.size()) && ctx->packs[pack], TLK_EINVAL,
            "bad pack id %d", pack);
  TLK_CUDA(cudaSetDevice(ctx->device));
  Pack& p = *ctx->packs[pack];
  TLK_CUDA(cudaStreamSynchronize(p.stream));
  destroy_pack(p);
  ctx->packs[pack].reset();
  return TLK_OK;
}

int tlk_pack_stream(tlk_ctx* ctx, int32_t pack, void** stream) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  TLK_CHECK(stream, TLK_EINVAL, "null argument");
  *stream = p->stream;
  return TLK_OK;
}

int tlk_stream(tlk_ctx* ctx, void** stream) {
  TLK_CHECK(ctx && stream, TLK_EINVAL, "null argument");
  *stream = ctx->stream;
  return TLK_OK;
}

int tlk_pack_create(tlk_ctx* ctx, const tlk_pack_desc* desc, int32_t* pack_id) {
  TLK_CHECK(ctx && desc && pack_id, TLK_EINVAL, "null argument");
  const ModelDef* d = model_def(desc->model);
  const bool gpt = is_gpt(desc->model), rn = desc->model == TLK_MODEL_RESNET18;
  TLK_CHECK(d || gpt || rn, TLK_EINVAL, "unknown model %d", desc->model);
  TLK_CHECK(desc->lanes >= 1 && desc->lanes <= 4096, TLK_EINVAL, "lanes must be 1..4096");
  if (rn)
    TLK_CHECK(desc->batch >= 8 && desc->batch <= 512 && desc->batch % 8 == 0, TLK_EINVAL,
              "resnet18 packs: batch a multiple of 8 in [8, 512]");
  else if (!gpt)
    TLK_CHECK(desc->batch >= 8 && desc->batch <= 64 && desc->batch % 8 == 0, TLK_EINVAL,
              "batch must be a multiple of 8 in [8, 64] (got %d)", desc->batch);
  else
    TLK_CHECK(desc->batch >= 1 && desc->batch <= 4096, TLK_EINVAL, "transformer packs: batch in [1, 4096]");
  GptCfg gc = gpt_default(desc->model);
  if (gpt) {
    if (desc->layers > 0) gc.layers = desc->layers;
    if (desc->d_model > 0) gc.d = desc->d_model;
    if (desc->heads > 0) gc.heads = desc->heads;
    if (desc->seq_len > 0) gc.T = desc->seq_len;
    if (desc->vocab > 0) gc.V = desc->vocab;
  }
  TLK_CHECK(desc->max_steps >= 1, TLK_EINVAL, "max_steps must be >= 1");
  TLK_CUDA(cudaSetDevice(ctx->device));
  auto p = std::make_unique<Pack>();
  p->model = desc->model;
  p->batch = desc->batch;
  p->lanes = desc->lanes;
  p->max_steps = desc->max_steps;
  p->host_input = desc->host_input;
  p->flags = desc->flags;
  p->def = d;
  p->gcfg = gc;
  p->tinfo = model_tensors(desc->model, gc);
  {
    tlk_model_info mi;
    fill_info(desc->model, gc, desc->batch, &mi);
    p->pcount = mi.param_count;
    p->stride = mi.param_stride;
  }
  p->teacher = ctx->teacher;
  p->ctx_in_use = &ctx->mem_in_use;
  p->ctx_limit = ctx->mem_limit;
  if (desc->flags & TLK_PACK_OWN_STREAM) {
    TLK_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    p->own_stream = true;
  } else {
    p->stream = ctx->stream;
  }
  const size_t L = size_t(p->lanes), S = size_t(p->stride), B = size_t(p->batch);
  int rc = 0;
  void* v = nullptr;
  auto grab = [&](size_t bytes) -> void* {
    if (rc) return nullptr;
    rc = pack_alloc(*p, &v, bytes);
    return rc ? nullptr : v;
  };
  p->lane_dev = static_cast<LaneState*>(grab(L * sizeof(LaneState)));
  p->params = static_cast<float*>(grab(L * S * 4));
  p->grads = static_cast<float*>(grab(L * S * 4));
  p->mom1 = static_cast<float*>(grab(L * S * 4));
  p->mom2 = static_cast<float*>(grab(L * S * 4));
  p->wbf = static_cast<uint16_t*>(grab(L * S * 2));
  p->loss = static_cast<float*>(grab(L * size_t(p->max_steps) * 4));
  p->last_loss = static_cast<float*>(grab(L * 4));
  p->pixels = static_cast<uint8_t*>(grab(L * B * 784));
  p->labels = static_cast<int32_t*>(grab(L * B * 4));
  p->x = static_cast<uint16_t*>(grab(L * B * 784 * 2));
  p->tinfo_dev = static_cast<TensorInfo*>(grab(p->tinfo.size() * sizeof(TensorInfo)));
  if (!rc) {
    const cudaError_t e = cudaMemcpy(p->tinfo_dev, p->tinfo.data(),
                                     p->tinfo.size() * sizeof(TensorInfo), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) rc = cuda_fail(e, "tensor table upload");
  }
  if (!rc)
    rc = p->model == TLK_MODEL_MLP        ? mlp_setup(*p)
         : p->model == TLK_MODEL_CNN      ? cnn_setup(*p)
         : p->model == TLK_MODEL_RESNET18 ? resnet_setup(*p)
                                          : gpt_setup(*p);
  if (rc) {
    destroy_pack(*p);
    return rc;
  }
  if (p->host_segs.empty())  // MLP / CNN: u8 pixels [lanes][batch][784], then int32 labels [lanes][batch]
    p->host_segs = {{p->pixels, L * B * 784}, {p->labels, L * B * 4}};
  TLK_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
  TLK_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
  TLK_CUDA(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
  TLK_CUDA(cudaEventCreateWithFlags(&p->ev_tail, cudaEventDisableTiming));
  p->lane_host.assign(L, LaneState{});
  TLK_CUDA(cudaMemsetAsync(p->lane_dev, 0, L * sizeof(LaneState), p->stream));
  TLK_CUDA(cudaMemsetAsync(p->loss, 0, L * size_t(p->max_steps) * 4, p->stream));
  TLK_CUDA(cudaMemsetAsync(p->params, 0, L * S * 4, p->stream));
  TLK_CUDA(cudaMemsetAsync(p->grads, 0, L * S * 4, p->stream));
  TLK_CUDA(cudaStreamSynchronize(p->stream));
  ctx->packs.push_back(std::move(p));
  *pack_id = int32_t(ctx->packs.size() - 1);
  return TLK_OK;
}

int tlk_lane_load(tlk_ctx* ctx, int32_t pack, int32_t lane, const tlk_job_desc* job) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  if ((rc = settle(*p))) return rc;
  TLK_CHECK(job && lane >= 0 && lane < p->lanes, TLK_EINVAL, "bad lane %d", lane);
  TLK_CHECK(job->steps >= 1 && job->steps <= p->max_steps, TLK_EINVAL,
            "steps %d outside 1..max_steps=%d", job->steps, p->max_steps);
  TLK_CHECK(job->optimizer == TLK_OPT_ADAM || job->optimizer == TLK_OPT_ADAMW ||
                job->optimizer == TLK_OPT_SGD,
            TLK_EINVAL, "unknown optimizer %d", job->optimizer);
  TLK_CHECK(job->lr > 0.0f && job->eps > 0.0f, TLK_EINVAL, "lr and eps must be positive");
  LaneState s{};
  s.active = 1;
  s.steps_done = 0;
  s.steps = job->steps;
  s.optimizer = job->optimizer;
  s.lr = job->lr;
  s.beta1 = job->beta1;
  s.beta2 = job->beta2;
  s.eps = job->eps;
  s.wd = job->weight_decay;
  s.momentum = job->momentum;
  s.seed = job->seed;
  s.b1t = 1.0;
  s.b2t = 1.0;
  p->lane_host[lane] = s;
  if ((rc = enqueue_lane_init(*p, lane, p->stream))) return rc;
  TLK_CUDA(cudaMemsetAsync(p->loss + size_t(lane) * p->max_steps, 0, size_t(p->max_steps) * 4,
                           p->stream));
  return upload_lane(ctx, *p, lane);
}

int tlk_lane_release(tlk_ctx* ctx, int32_t pack, int32_t lane) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  if ((rc = settle(*p))) return rc;
  TLK_CHECK(lane >= 0 && lane < p->lanes, TLK_EINVAL, "bad lane %d", lane);
  TLK_CUDA(cudaMemcpyAsync(&p->lane_host[lane], p->lane_dev + lane, sizeof(LaneState),
                           cudaMemcpyDeviceToHost, p->stream));
  TLK_CUDA(cudaStreamSynchronize(p->stream));
  p->lane_host[lane].active = 0;
  return upload_lane(ctx, *p, lane);
}

int tlk_run(tlk_ctx* ctx, int32_t pack, int32_t steps) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  TLK_CHECK(steps >= 0, TLK_EINVAL, "steps must be >= 0");
  TLK_CHECK(!p->host_input, TLK_ESTATE, "host-input pack: use tlk_step_host");
  if (p->model == TLK_MODEL_CNN && cnn_persist_enabled(*p)) {
    // the persistent scheduler kernel runs up to PERSIST_CHUNK steps of every
    // lane per launch: lanes overlap across steps, no launch chain at all
    constexpr int PERSIST_CHUNK = 64;
    for (int done = 0; done < steps; done += PERSIST_CHUNK)
      if ((rc = cnn_persist_enqueue(*p, p->stream, std::min(PERSIST_CHUNK, steps - done)))) return rc;
    return TLK_OK;
  }
  if ((rc = ensure_graph(*p, p->stream))) return rc;
  for (int i = 0; i < steps; ++i)
    if ((rc = launch_step(*p, p->graph_exec))) return rc;
  return settle(*p);  // a run ends with every step complete
}

int tlk_step_host(tlk_ctx* ctx, int32_t pack, const uint8_t* pixels, const int32_t* labels,
                  float* losses_out) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  TLK_CHECK(p->host_input, TLK_ESTATE, "pack was created without host_input");
  TLK_CHECK(pixels && labels, TLK_EINVAL, "null input buffers");
  const size_t L = size_t(p->lanes), B = size_t(p->batch);
  TLK_CUDA(cudaMemcpyAsync(p->pixels, pixels, L * B * 784, cudaMemcpyHostToDevice, p->stream));
  TLK_CUDA(cudaMemcpyAsync(p->labels, labels, L * B * 4, cudaMemcpyHostToDevice, p->stream));
  if ((rc = ensure_graph(*p, p->stream))) return rc;
  if ((rc = launch_step(*p, p->graph_exec)) || (rc = settle(*p))) return rc;
  if (losses_out) {
    TLK_CUDA(cudaMemcpyAsync(losses_out, p->last_loss, L * 4, cudaMemcpyDeviceToHost,
                             p->stream));
    TLK_CUDA(cudaStreamSynchronize(p->stream));
  }
  return TLK_OK;
}

int tlk_pack_host_input_bytes(tlk_ctx* ctx, int32_t pack, int64_t* bytes) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  TLK_CHECK(bytes, TLK_EINVAL, "null argument");
  int64_t n = 0;
  for (const auto& sg : p->host_segs) n += int64_t(sg.bytes);
  *bytes = n;
  return TLK_OK;
}

int tlk_step_host_blob(tlk_ctx* ctx, int32_t pack, const void* blob, int64_t bytes, float* losses_out) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  TLK_CHECK(p->host_input, TLK_ESTATE, "pack was created without host_input");
  int64_t need = 0;
  for (const auto& sg : p->host_segs) need += int64_t(sg.bytes);
  TLK_CHECK(blob && bytes == need, TLK_EINVAL, "host input blob of %lld bytes, the pack takes %lld",
            (long long)bytes, (long long)need);
  const char* src = static_cast<const char*>(blob);
  for (const auto& sg : p->host_segs) {
    TLK_CUDA(cudaMemcpyAsync(sg.dst, src, sg.bytes, cudaMemcpyHostToDevice, p->stream));
    src += sg.bytes;
  }
  if ((rc = ensure_graph(*p, p->stream))) return rc;
  if ((rc = launch_step(*p, p->graph_exec)) || (rc = settle(*p))) return rc;
  if (losses_out)
    TLK_CUDA(cudaMemcpyAsync(losses_out, p->last_loss, size_t(p->lanes) * 4, cudaMemcpyDeviceToHost, p->stream));
  TLK_CUDA(cudaStreamSynchronize(p->stream));
  return TLK_OK;
}

// Pipelined host-input step: step k uses input slot k & 1.  The copy stream
// waits until step k-2 (the slot's previous user) has finished, copies the
// inputs, and the compute stream waits for that copy, replays the slot's
// graph and copies the losses back; nothing blocks the caller, so step k+1's
// H2D overlaps step k's kernels.  tlk_step_host_wait(ticket) returns once the
// step's losses are in losses_out (valid for the two newest tickets).
int tlk_step_host_async(tlk_ctx* ctx, int32_t pack, const uint8_t* pixels, const int32_t* labels,
                        float* losses_out, int64_t* ticket) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  TLK_CHECK(p->host_input, TLK_ESTATE, "pack was created without host_input");
  TLK_CHECK(pixels && labels && losses_out && ticket, TLK_EINVAL, "null buffers");
  if ((rc = ensure_host_pipeline(*p, p->stream))) return rc;
  const int s = int(p->host_steps & 1);
  const size_t L = size_t(p->lanes), B = size_t(p->batch);
  if (p->host_steps >= 2) TLK_CUDA(cudaStreamWaitEvent(p->copy_st, p->done_ev[s], 0));
  TLK_CUDA(cudaMemcpyAsync(s ? p->px_alt : p->pixels, pixels, L * B * 784, cudaMemcpyHostToDevice, p->copy_st));
  TLK_CUDA(cudaMemcpyAsync(s ? p->lb_alt : p->labels, labels, L * B * 4, cudaMemcpyHostToDevice, p->copy_st));
  TLK_CUDA(cudaEventRecord(p->h2d_ev[s], p->copy_st));
  TLK_CUDA(cudaStreamWaitEvent(p->stream, p->h2d_ev[s], 0));
  // (the deferred work of the step stays in flight: the next step's graph
  // waits for it where it must, tlk_sync and the lane calls settle it)
  if ((rc = launch_step(*p, s ? p->hexec_alt : p->hexec0))) return rc;
  TLK_CUDA(cudaEventRecord(p->done_ev[s], p->stream));
  p->hout[s] = losses_out;  // filled from the mapped slot by tlk_step_host_wait
  *ticket = p->host_steps++;
  return TLK_OK;
}

int tlk_step_host_wait(tlk_ctx* ctx, int32_t pack, int64_t ticket) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  TLK_CHECK(ticket >= 0 && ticket < p->host_steps && ticket + 2 >= p->host_steps, TLK_EINVAL,
            "ticket %lld is not one of the two newest host steps", (long long)ticket);
  const int s = int(ticket & 1);
  TLK_CUDA(cudaEventSynchronize(p->done_ev[s]));
  // the step's head kernel wrote the losses into mapped host slot s (visible
  // once the step has completed); slot s is next written by step ticket + 2,
  // which cannot have been enqueued while this ticket is still waitable
  if (p->hout[s]) {
    std::memcpy(p->hout[s], p->ll_host + size_t(s) * p->lanes, size_t(p->lanes) * 4);
    p->hout[s] = nullptr;
  }
  return TLK_OK;
}

int tlk_lane_status_get(tlk_ctx* ctx, int32_t pack, int32_t lane, tlk_lane_status* out) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  TLK_CHECK(out && lane >= 0 && lane < p->lanes, TLK_EINVAL, "bad lane %d", lane);
  LaneState s;
  TLK_CUDA(cudaMemcpyAsync(&s, p->lane_dev + lane, sizeof(s), cudaMemcpyDeviceToHost,
                           p->stream));
  TLK_CUDA(cudaStreamSynchronize(p->stream));
  out->active = s.active;
  out->steps_done = s.steps_done;
  out->steps = s.steps;
  out->error = 0;
  return TLK_OK;
}

int tlk_lane_losses(tlk_ctx* ctx, int32_t pack, int32_t lane, float* host, int32_t n) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  TLK_CHECK(host && lane >= 0 && lane < p->lanes && n >= 0 && n <= p->max_steps, TLK_EINVAL,
            "bad lane/n");
  TLK_CUDA(cudaMemcpyAsync(host, p->loss + size_t(lane) * p->max_steps, size_t(n) * 4,
                           cudaMemcpyDeviceToHost, p->stream));
  TLK_CUDA(cudaStreamSynchronize(p->stream));
  return TLK_OK;
}

int tlk_lane_params(tlk_ctx* ctx, int32_t pack, int32_t lane, float* host, int64_t n) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  if ((rc = settle(*p))) return rc;
  TLK_CHECK(host && lane >= 0 && lane < p->lanes && n >= 0 && n <= p->stride, TLK_EINVAL,
            "bad lane/n");
  TLK_CUDA(cudaMemcpyAsync(host, p->params + size_t(lane) * p->stride, size_t(n) * 4,
                           cudaMemcpyDeviceToHost, p->stream));
  TLK_CUDA(cudaStreamSynchronize(p->stream));
  return TLK_OK;
}

int tlk_pack_tensor(tlk_ctx* ctx, int32_t pack, int32_t which, void** dev_ptr, int64_t* bytes) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  if ((rc = settle(*p))) return rc;
  TLK_CHECK(dev_ptr && bytes, TLK_EINVAL, "null argument");
  const int64_t L = p->lanes, S = p->stride, B = p->batch;
  switch (which) {
    case TLK_BUF_PARAMS: *dev_ptr = p->params; *bytes = L * S * 4; break;
    case TLK_BUF_GRADS: *dev_ptr = p->grads; *bytes = L * S * 4; break;
    case TLK_BUF_MOM1: *dev_ptr = p->mom1; *bytes = L * S * 4; break;
    case TLK_BUF_MOM2: *dev_ptr = p->mom2; *bytes = L * S * 4; break;
    case TLK_BUF_WBF16: *dev_ptr = p->wbf; *bytes = L * S * 2; break;
    case TLK_BUF_LOSS: *dev_ptr = p->loss; *bytes = L * int64_t(p->max_steps) * 4; break;
    case TLK_BUF_PIXELS: *dev_ptr = p->pixels; *bytes = L * B * 784; break;
    case TLK_BUF_LABELS: *dev_ptr = p->labels; *bytes = L * B * 4; break;
    case TLK_BUF_ACTS: *dev_ptr = p->acts; *bytes = int64_t(p->acts_bytes); break;
    default: return fail(TLK_EINVAL, "unknown buffer %d", which);
  }
  return TLK_OK;
}

int tlk_pack_named(tlk_ctx* ctx, int32_t pack, const char* name, void** dev_ptr, int64_t* bytes) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  if ((rc = settle(*p))) return rc;
  TLK_CHECK(name && dev_ptr && bytes, TLK_EINVAL, "null argument");
  for (const auto& nb : p->named)
    if (nb.name == name) {
      *dev_ptr = nb.ptr;
      *bytes = int64_t(nb.bytes);
      return TLK_OK;
    }
  return fail(TLK_EINVAL, "pack has no buffer named '%s'", name);
}

int tlk_pack_info(tlk_ctx* ctx, int32_t pack, tlk_model_info* out) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  TLK_CHECK(out, TLK_EINVAL, "null argument");
  fill_info(p->model, p->gcfg, p->batch, out);
  return TLK_OK;
}

int tlk_pack_launches_per_step(tlk_ctx* ctx, int32_t pack, int32_t* n) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  TLK_CHECK(n, TLK_EINVAL, "null argument");
  *n = p->launches_per_step;
  return TLK_OK;
}

int tlk_profile_step(tlk_ctx* ctx, int32_t pack, int32_t iters, float* ms, char* names,
                     int32_t names_len, int32_t max_n, int32_t* n_out) {
  Pack* p = nullptr;
  int rc = get_pack(ctx, pack, &p);
  if (rc) return rc;
  if ((rc = settle(*p))) return rc;
  TLK_CHECK(iters >= 1 && ms && n_out && max_n > 0, TLK_EINVAL, "bad arguments");
  TLK_CHECK(!p->host_input, TLK_ESTATE, "profile needs a device-input pack");
  // One step captured with an event node after every kernel, replayed
  // `iters` times: device-side durations without host launch gaps.
  std::vector<cudaEvent_t> ev;
  std::vector<const char*> nm;
  cudaEvent_t start;
  TLK_CUDA(cudaEventCreate(&start));
  TLK_CUDA(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
  cudaEventRecordWithFlags(start, p->stream, cudaEventRecordExternal);
  p->prof = &ev;
  p->prof_names = &nm;
  rc = enqueue_step(*p, p->stream);
  p->prof = nullptr;
  p->prof_names = nullptr;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(p->stream, &g);
  if (rc) return rc;
  TLK_CUDA(e);
  cudaGraphExec_t ge = nullptr;
  TLK_CUDA(cudaGraphInstantiate(&ge, g, 0));
  std::vector<double> acc(ev.size(), 0.0);
  for (int it = 0; it < iters; ++it) {
    TLK_CUDA(cudaGraphLaunch(ge, p->stream));
    TLK_CUDA(cudaStreamSynchronize(p->stream));
    cudaEvent_t prev = start;
    for (size_t k = 0; k < ev.size(); ++k) {
      float t = 0.f;
      cudaEventElapsedTime(&t, prev, ev[k]);
      acc[k] += t;
      prev = ev[k];
    }
  }
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaEventDestroy(start);
  for (auto x : ev) cudaEventDestroy(x);
  const int n = int(acc.size()) < max_n ? int(acc.size()) : max_n;
  std::string joined;
  for (int k = 0; k < n; ++k) {
    ms[k] = float(acc[k] / iters);
    joined += nm[k];
    if (k + 1 < n) joined += ",";
  }
  if (names && names_len > 0) {
    std::strncpy(names, joined.c_str(), size_t(names_len) - 1);
    names[names_len - 1] = 0;
  }
  *n_out = n;
  return TLK_OK;
}

int tlk_selftest_datagen(uint64_t seed, int32_t step, int32_t batch, uint8_t* pixels_dev,
                         int32_t* labels_dev, void* stream) {
  TLK_CHECK(pixels_dev && labels_dev && batch > 0, TLK_EINVAL, "bad arguments");
  static int8_t* teacher = nullptr;
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> g(mu);
    if (!teacher) {
      int rc = build_teacher(&teacher);
      if (rc) return rc;
    }
  }
  return enqueue_datagen_raw(seed, step, batch, teacher, pixels_dev, labels_dev,
                             static_cast<cudaStream_t>(stream));
}

}  // extern "C"
