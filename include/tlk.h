/*
 * tlk.h -- C ABI of the B200 packed-jobs runtime (libtlk.so).
 *
 * The reference (trilaunch, pure Python) runs every task as an opaque child
 * process: `_spawn(argv, env, timeout_s, log_dir, task_id)`
 * (/root/reference/pkg/src/trilaunch/executor.py:105-141), called once per
 * task from each slot thread's queue loop (executor.py:192-213).  K slots
 * pinned to one GPU (core.py:147-179) therefore become K CUDA contexts that
 * the driver time-slices.  This ABI replaces that per-task seam for training
 * tasks: one context per GPU holds a *pack* of K job lanes (one per slot
 * pinned to that GPU) whose forward, backward and optimizer steps run as
 * grouped sm_100a kernels -- one launch per layer-phase for all K lanes.
 *
 * Plain C types only (no torch types): the Python host binds it with ctypes
 * (paper_2410_22254_b200/runtime.py).  All functions return 0 on success or a
 * negative TLK_E* code; tlk_last_error() gives the thread-local message.  An
 * allocation failure reports TLK_EOOM with "out of memory" in the message so
 * the reference's classify_failure (executor.py:95-102) flags oom_flag.
 */
#ifndef TLK_H_
#define TLK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLK_ABI_VERSION 1

/* error codes */
#define TLK_OK 0
#define TLK_EINVAL (-1)  /* bad argument */
#define TLK_ECUDA (-2)   /* CUDA runtime error */
#define TLK_EOOM (-3)    /* device allocation failed ("out of memory") */
#define TLK_ESTATE (-4)  /* call not valid in the current state */

/* job models (the training tasks the paper packs) */
#define TLK_MODEL_MLP 1 /* MNIST MLP 784-512-512-10, ReLU */
#define TLK_MODEL_CNN 2 /* MNIST CNN: conv3x3(1->32) conv3x3(32->64) maxpool2 fc(9216->128) fc(128->10) */
#define TLK_MODEL_XFORMER 3 /* 2-layer pre-LN transformer, d=256, 4 heads, T=128, byte vocab (config 4) */
#define TLK_MODEL_GPT 4     /* tiny-GPT, 6 layers, d=384, 6 heads, T=256, vocab 65 (config 5) */
#define TLK_MODEL_RESNET18 5 /* ResNet-18 CIFAR variant, 3x32x32 inputs, batch-stat BN (config 3) */

/* optimizers */
#define TLK_OPT_ADAM 1
#define TLK_OPT_ADAMW 2
#define TLK_OPT_SGD 3 /* SGD with (optional) momentum */

/* buffers a pack exports for zero-copy tensor handoff (tlk_pack_tensor) */
#define TLK_BUF_PARAMS 0  /* fp32 [lanes, param_stride] master weights   */
#define TLK_BUF_GRADS 1   /* fp32 [lanes, param_stride]                  */
#define TLK_BUF_MOM1 2    /* fp32 [lanes, param_stride] Adam m / SGD buf */
#define TLK_BUF_MOM2 3    /* fp32 [lanes, param_stride] Adam v           */
#define TLK_BUF_WBF16 4   /* bf16 [lanes, param_stride] GEMM operand copy */
#define TLK_BUF_LOSS 5    /* fp32 [lanes, max_steps] per-step mean loss  */
#define TLK_BUF_PIXELS 6  /* u8   [lanes, batch, 784] current input batch */
#define TLK_BUF_LABELS 7  /* i32  [lanes, batch] current labels          */
#define TLK_BUF_ACTS 8    /* model activation scratch (debug/tests; layout per model) */

typedef struct tlk_ctx tlk_ctx;

/* One training task = one lane.  Parsed by the host from the task argv
 * (`python -m paper_2410_22254_b200.job --model cnn --seed 3 ...`). */
typedef struct {
  int64_t task_id;
  int32_t slot_index;
  int32_t steps;       /* optimizer steps to run */
  int32_t optimizer;   /* TLK_OPT_* */
  float lr, beta1, beta2, eps, weight_decay, momentum;
  uint64_t seed;       /* init + data stream */
} tlk_job_desc;

typedef struct {
  int32_t model;      /* TLK_MODEL_* (all lanes of a pack share it) */
  int32_t batch;      /* per-lane batch */
  int32_t lanes;      /* K co-resident jobs */
  int32_t max_steps;  /* loss-curve capacity per lane */
  int32_t host_input; /* 1: inputs come from tlk_step_host, 0: synthesised on device */
  int32_t flags;      /* TLK_PACK_* */
  /* transformer packs: 0 = the model's default */
  int32_t layers, d_model, heads, seq_len, vocab;
} tlk_pack_desc;

/* pack flags */
#define TLK_PACK_WRITE_ALL_GRADS 1 /* also store gradients whose optimizer update is fused
                                      into a wgrad epilogue (tests/inspection) */
#define TLK_PACK_SNAPSHOTS 2       /* keep per-layer copies of intermediate gradients
                                      (layer-local parity tests; ResNet packs) */
#define TLK_PACK_PERSISTENT 8      /* CNN packs: run steps on the persistent per-GPU scheduler
                                      kernel (one launch per chunk of steps, device work
                                      queue, per-lane dependency counters) instead of the
                                      per-phase kernel graph; bit-identical results */
#define TLK_PACK_OWN_STREAM 4      /* the pack gets its own CUDA stream (tlk_pack_stream), so
                                      packs of different models on one GPU run concurrently;
                                      default: the context stream */

typedef struct {
  int64_t param_count;   /* real parameters per job */
  int64_t param_stride;  /* padded per-lane stride of the fp32 arenas */
  int64_t flops_per_sample;  /* 3 x 2 x MACs (fwd + dgrad + wgrad) */
  int32_t num_tensors;
} tlk_model_info;

typedef struct {
  int32_t active;      /* 1 while steps_done < steps */
  int32_t steps_done;
  int32_t steps;
  int32_t error;       /* 0 or TLK_E* */
} tlk_lane_status;

/* -- library -------------------------------------------------------------- */
int tlk_abi_version(void);
const char* tlk_last_error(void);
int tlk_model_query(int32_t model, int32_t batch, tlk_model_info* out);
/* offset (in floats) and element count of tensor `t` inside a lane's arena */
int tlk_model_tensor(int32_t model, int32_t t, int64_t* offset, int64_t* count, int32_t* fan_in);

/* -- context: one per GPU (replaces one CUDA context per child process) ---- */
int tlk_open(int32_t device, tlk_ctx** out);
int tlk_close(tlk_ctx* ctx);
/* waits for the context stream and every pack stream */
int tlk_sync(tlk_ctx* ctx);
/* Admission budget for pack memory on this context (0 = device memory only).
 * A pack allocation that would exceed it fails with TLK_EOOM ("out of
 * memory"), like a device allocation failure: the host admits tasks against
 * it (the reference simulator's per-device capacity, sim.py:388-402). */
int tlk_set_mem_limit(tlk_ctx* ctx, int64_t bytes);
/* bytes currently held by the context's live packs */
int tlk_mem_in_use(tlk_ctx* ctx, int64_t* bytes);
/* the context's CUDA stream (cudaStream_t), for event timing by the host */
int tlk_stream(tlk_ctx* ctx, void** stream);

/* -- packs: K lanes of one model ------------------------------------------ */
int tlk_pack_create(tlk_ctx* ctx, const tlk_pack_desc* desc, int32_t* pack_id);
/* Free every device resource of a pack (waits for its stream first); the id
 * becomes invalid.  The reference frees a task's GPU memory when its process
 * exits; the packed host destroys a pack once none of its lanes is in use. */
int tlk_pack_destroy(tlk_ctx* ctx, int32_t pack);
/* the stream the pack's work is enqueued on (cudaStream_t) */
int tlk_pack_stream(tlk_ctx* ctx, int32_t pack, void** stream);
/* (Re)load a lane with a task: device-side init of weights/state from seed.
 * Replaces spawning the task's process (executor.py:199 -> _spawn). */
int tlk_lane_load(tlk_ctx* ctx, int32_t pack, int32_t lane, const tlk_job_desc* job);
int tlk_lane_release(tlk_ctx* ctx, int32_t pack, int32_t lane);
/* Advance every active lane by up to `steps` steps (asynchronous). */
int tlk_run(tlk_ctx* ctx, int32_t pack, int32_t steps);
/* End-to-end step from HOST buffers: H2D of u8 pixels [lanes,batch,784] and
 * i32 labels [lanes,batch], one step, D2H of the per-lane losses [lanes]. */
int tlk_step_host(tlk_ctx* ctx, int32_t pack, const uint8_t* pixels, const int32_t* labels,
                  float* losses_out);
/* Pipelined form of tlk_step_host: enqueues the step and returns at once.
 * Step k uses device input slot k & 1: its H2D copy (on a copy stream) waits
 * only for step k-2, so it overlaps step k-1's kernels.  pixels / labels must
 * stay valid (and should be pinned) until the copy is done, losses_out until
 * tlk_step_host_wait(ticket) returns; only the two newest tickets can be
 * waited on.  The step writes its losses into mapped pinned host memory (one
 * slot per input slot, no D2H copy in the stream); tlk_step_host_wait copies
 * them into losses_out.  Do not interleave with tlk_step_host without
 * waiting first. */
/* Bytes of one step's host-input blob of a host_input pack, and the step
 * from such a blob (H2D copies into the model's input buffers on the pack
 * stream, one step, D2H of the per-lane losses [lanes], synchronous).
 * Layouts (lanes outermost):
 *   MLP / CNN: u8 pixels [lanes][batch][784], int32 labels [lanes][batch]
 *   transformer / tiny-GPT: int32 tokens [lanes][batch][T + 1] (inputs
 *     tokens[:, :-1], targets tokens[:, 1:])
 *   ResNet-18: bf16 images [lanes][batch][32][32][3] (NHWC), int32 labels
 *     [lanes][batch] */
int tlk_pack_host_input_bytes(tlk_ctx* ctx, int32_t pack, int64_t* bytes);
int tlk_step_host_blob(tlk_ctx* ctx, int32_t pack, const void* blob, int64_t bytes, float* losses_out);
int tlk_step_host_async(tlk_ctx* ctx, int32_t pack, const uint8_t* pixels, const int32_t* labels,
                        float* losses_out, int64_t* ticket);
int tlk_step_host_wait(tlk_ctx* ctx, int32_t pack, int64_t ticket);
int tlk_lane_status_get(tlk_ctx* ctx, int32_t pack, int32_t lane, tlk_lane_status* out);
int tlk_lane_losses(tlk_ctx* ctx, int32_t pack, int32_t lane, float* host, int32_t n);
int tlk_lane_params(tlk_ctx* ctx, int32_t pack, int32_t lane, float* host, int64_t n);
/* Device pointer + size of a pack buffer (TLK_BUF_*), for zero-copy tensors. */
int tlk_pack_tensor(tlk_ctx* ctx, int32_t pack, int32_t which, void** dev_ptr, int64_t* bytes);
/* Device pointer + size of a named model-internal buffer (activations, BN
   statistics, gradient snapshots; names per model, e.g. "conv3.y"), all
   lanes [lanes, ...].  TLK_EINVAL for unknown names. */
int tlk_pack_named(tlk_ctx* ctx, int32_t pack, const char* name, void** dev_ptr, int64_t* bytes);
/* Parameter layout of this pack's lanes (depends on the transformer config). */
int tlk_pack_info(tlk_ctx* ctx, int32_t pack, tlk_model_info* out);
/* Number of kernels one tlk_run step launches for this pack. */
int tlk_pack_launches_per_step(tlk_ctx* ctx, int32_t pack, int32_t* n);

/* Per-kernel device time of one step: runs `iters` un-graphed steps with a CUDA
 * event after every launch; ms[k] = mean duration of launch k, names =
 * comma-separated kernel names.  Advances the lanes like tlk_run. */
int tlk_profile_step(tlk_ctx* ctx, int32_t pack, int32_t iters, float* ms, char* names,
                     int32_t names_len, int32_t max_n, int32_t* n_out);

/* -- self-test hooks (used by tests/ only) --------------------------------- */
/* C[b] = A[b] * B[b]^T on the tcgen05 path.  A is [M,K] (a_mn=0) or [K,M]
 * (a_mn=1); B is [N,K] (b_mn=0) or [K,N] (b_mn=1); bf16 in, fp32 C [M,N]. */
int tlk_selftest_gemm(int32_t a_mn, int32_t b_mn, int32_t bn, const void* A, const void* B,
                      float* C, int32_t batch, int32_t M, int32_t N, int32_t K, void* stream);
/* Counter RNG + synthetic data generator, for bit-exact checks vs the oracle. */
int tlk_selftest_datagen(uint64_t seed, int32_t step, int32_t batch, uint8_t* pixels_dev,
                         int32_t* labels_dev, void* stream);
/* The packed optimizer update (straight-line fast-path sqrt/div) against the
 * library-intrinsic formulation on n random states of the given TLK_OPT_*
 * kind; *mismatches = elements whose p, m or v differ in any bit. */
int tlk_selftest_optimizer(int32_t kind, uint64_t seed, int64_t n, uint64_t* mismatches);
/* In-graph timeline of the CNN step kernels (libtlk built with -DTLK_KTRACE;
 * otherwise TLK_EINVAL).  reset != 0 clears it; else copies n >= 288 values:
 * [step mod 8][kernel id 0..11][earliest CTA entry, earliest end of the PDL
 * wait, latest warp exit], %globaltimer ns (tools/cnn_timeline.py). */
int tlk_cnn_ktrace(int32_t reset, uint64_t* out, int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* TLK_H_ */
