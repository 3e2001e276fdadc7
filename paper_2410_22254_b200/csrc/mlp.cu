// MNIST MLP 784-512-512-10 pack: one training step for every lane.
//
// Batch 64 (the configs): mlp2.cu, two launches per step.  Other batch sizes
// (and TLK_MLP_V1=1): 8 kernels, captured once into a CUDA graph:
//   inputs -> fc1 fwd -> fc2 fwd -> head(fc3 + CE + bwd) -> fc2 wgrad ->
//   fc2 dgrad(+mask, fc1 bias grad) -> fc1 wgrad -> optimizer (+ end of step)
#include <cstdlib>

#include "linear.cuh"
#include "pack.cuh"

namespace tlk {
namespace {

struct MlpScratch {
  uint16_t *h1, *h2, *dz1, *dz2;  // [lanes][batch][512] bf16
};

}  // namespace

bool mlp2_enabled(const Pack& p);
int mlp2_enqueue_step(Pack& p, cudaStream_t st, uint16_t* h1, uint16_t* h2, uint16_t* dz1, uint16_t* dz2);

int mlp_setup(Pack& p) {
  const size_t n = size_t(p.lanes) * p.batch * 512 * sizeof(uint16_t);
  void* base = nullptr;
  int rc = pack_alloc(p, &base, 4 * n);
  if (rc) return rc;
  auto* s = new MlpScratch{static_cast<uint16_t*>(base),
                           reinterpret_cast<uint16_t*>(static_cast<char*>(base) + n),
                           reinterpret_cast<uint16_t*>(static_cast<char*>(base) + 2 * n),
                           reinterpret_cast<uint16_t*>(static_cast<char*>(base) + 3 * n)};
  p.acts = base;
  p.acts_bytes = 4 * n;
  p.scratch = s;
  p.scratch_free = [](void* q) { delete static_cast<MlpScratch*>(q); };
  p.launches_per_step = mlp2_enabled(p) ? 2 : 8;
  if (getenv("TLK_MLP_TRACE") && getenv("TLK_MLP_TRACE")[0] == '1') {  // mlp2.cu phase timeline
    void* tb = nullptr;
    if ((rc = pack_alloc(p, &tb, 4 * 32 * 8))) return rc;
    TLK_CUDA(cudaMemset(tb, 0, 4 * 32 * 8));
    p.name_buf("mlp.trace", tb, 4 * 32 * 8);
  }
  return TLK_OK;
}

int mlp_enqueue_step(Pack& p, cudaStream_t st) {
  const MlpScratch& s = *static_cast<MlpScratch*>(p.scratch);
  const ModelDef& d = *p.def;
  const int B = p.batch, L = p.lanes;
  const int64_t act = int64_t(B) * 512;
  const int64_t o_w1 = tensor_offset(d, 0), o_b1 = tensor_offset(d, 1);
  const int64_t o_w2 = tensor_offset(d, 2), o_b2 = tensor_offset(d, 3);
  const int64_t o_w3 = tensor_offset(d, 4), o_b3 = tensor_offset(d, 5);
  if (mlp2_enabled(p)) return mlp2_enqueue_step(p, st, s.h1, s.h2, s.dz1, s.dz2);  // mlp2.cu: 2 launches
  int rc;
  if ((rc = enqueue_inputs(p, st))) return rc;

  LinFwd f1{p.lane_dev, p.wbf, p.params, p.stride, o_w1, o_b1, p.x, int64_t(B) * 784, s.h1, act,
            512, 784, B};
  TLK_CUDA(launch_gemm(f1, dim3(512 / GEMM_BM, (B + 63) / 64, L), st));
  p.mark(st, "fc1_fwd");
  LinFwd f2{p.lane_dev, p.wbf, p.params, p.stride, o_w2, o_b2, s.h1, act, s.h2, act, 512, 512, B};
  TLK_CUDA(launch_gemm(f2, dim3(512 / GEMM_BM, (B + 63) / 64, L), st));
  p.mark(st, "fc2_fwd");

  if ((rc = enqueue_head(p, st, s.h2, 512, o_w3, o_b3, s.dz2, o_b2))) return rc;

  LinWgrad g2{p.lane_dev, s.dz2, act, s.h1, act, p.grads, p.stride, o_w2, 512, 512, B};
  TLK_CUDA(launch_gemm(g2, dim3(512 / GEMM_BM, 512 / LinWgrad::BN, L), st));
  p.mark(st, "fc2_wgrad");
  LinDgrad d2{p.lane_dev, p.wbf, p.stride, o_w2, s.dz2, act, s.h1, s.dz1, act, p.grads, o_b1,
              512, 512, B};
  TLK_CUDA(launch_gemm(d2, dim3(512 / GEMM_BM, 1, L), st));
  p.mark(st, "fc2_dgrad");
  LinWgrad g1{p.lane_dev, s.dz1, act, p.x, int64_t(B) * 784, p.grads, p.stride, o_w1,
              512, 784, B};
  TLK_CUDA(launch_gemm(g1, dim3(512 / GEMM_BM, (784 + LinWgrad::BN - 1) / LinWgrad::BN, L), st));
  p.mark(st, "fc1_wgrad");

  if ((rc = enqueue_optimizer(p, st))) return rc;
  return enqueue_end_step(p, st);
}

}  // namespace tlk
