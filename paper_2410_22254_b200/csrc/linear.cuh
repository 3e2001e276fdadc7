// Linear-layer GEMM problems for the grouped tcgen05 kernel (all lanes of a
// pack in one launch; blockIdx.z = lane [x k-split]).
//
//   LinFwd    Y[b,o]   = bf16(relu(sum_i W[o,i] X[b,i] + bias[o]))
//             computed transposed (M = out features, N = batch) so the
//             tiny batch sits in UMMA N and the weight rows fill M = 128.
//   LinWgrad  dW[o,i]  = sum_b dZ[b,o] X[b,i]             (fp32 into grads)
//             M = out, N = in, K = batch; both operands MN-major.
//   LinDgrad  dZp[b,i] = bf16(sum_o W[o,i] dZ[b,o] * [Hp[b,i] > 0]),
//             db_prev[i] = sum_b dZp[b,i];  M = in, N = batch, K = out,
//             W read MN-major (no transposed copy needed).
#pragma once
#include "models.cuh"
#include "tc_gemm.cuh"

namespace tlk {

struct LaneWork {
  int j, m0, n0, kb_begin, kb_end, split;
};

struct LinFwd {
  static constexpr int BN = 64, STAGES = 4;
  static constexpr bool A_MN = false, B_MN = false;
  static constexpr bool TILE_EPILOGUE = false;
  using Work = LaneWork;
  struct Carry {};
  const LaneState* lanes;
  const uint16_t* W;  // bf16 shadow arena
  const float* bias;  // fp32 master arena
  int64_t pstride, w_off, b_off;
  const uint16_t* X;
  int64_t xst;
  uint16_t* Y;
  int64_t yst;
  int out, in, batch;

  TLK_DEV bool work(Work& w) const {
    w.j = blockIdx.z;
    if (!lanes[w.j].active) return false;
    w.m0 = blockIdx.x * GEMM_BM;
    w.n0 = blockIdx.y * BN;
    w.kb_begin = 0;
    w.kb_end = (in + GEMM_BK - 1) / GEMM_BK;
    w.split = 0;
    return true;
  }
  TLK_DEV const void* zero_src() const { return W; }
  TLK_DEV const void* a_src(const Work& w, int m, int k) const {
    return (m < out && k < in) ? W + w.j * pstride + w_off + int64_t(m) * in + k : nullptr;
  }
  TLK_DEV const void* b_src(const Work& w, int n, int k) const {
    return (n < batch && k < in) ? X + w.j * xst + int64_t(n) * in + k : nullptr;
  }
  TLK_DEV void epilogue(const Work& w, int m, int n0, const float (&v)[32], Carry&) const {
    if (m >= out) return;
    const float bb = bias[w.j * pstride + b_off + m];
    uint16_t* y = Y + w.j * yst + m;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (n0 + i < batch) y[int64_t(n0 + i) * out] = f2bf(fmaxf(v[i] + bb, 0.0f));
  }
  TLK_DEV void finish(const Work&, int, Carry&) const {}
};

struct LinWgrad {
  static constexpr int BN = 128, STAGES = 4;
  static constexpr bool A_MN = true, B_MN = true;
  static constexpr bool TILE_EPILOGUE = false;
  using Work = LaneWork;
  struct Carry {};
  const LaneState* lanes;
  const uint16_t* dZ;  // [lanes][batch][out]
  int64_t dzst;
  const uint16_t* X;   // [lanes][batch][in]
  int64_t xst;
  float* grads;
  int64_t pstride, w_off;
  int out, in, batch;

  TLK_DEV bool work(Work& w) const {
    w.j = blockIdx.z;
    if (!lanes[w.j].active) return false;
    w.m0 = blockIdx.x * GEMM_BM;
    w.n0 = blockIdx.y * BN;
    w.kb_begin = 0;
    w.kb_end = (batch + GEMM_BK - 1) / GEMM_BK;
    w.split = 0;
    return true;
  }
  TLK_DEV const void* zero_src() const { return dZ; }
  TLK_DEV const void* a_src(const Work& w, int m, int k) const {
    return (m < out && k < batch) ? dZ + w.j * dzst + int64_t(k) * out + m : nullptr;
  }
  TLK_DEV const void* b_src(const Work& w, int n, int k) const {
    return (n < in && k < batch) ? X + w.j * xst + int64_t(k) * in + n : nullptr;
  }
  TLK_DEV void epilogue(const Work& w, int m, int n0, const float (&v)[32], Carry&) const {
    if (m >= out || n0 >= in) return;
    float* g = grads + w.j * pstride + w_off + int64_t(m) * in + n0;
    if (n0 + 32 <= in && ((reinterpret_cast<uintptr_t>(g) & 15) == 0)) {
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        *reinterpret_cast<float4*>(g + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (n0 + i < in) g[i] = v[i];
    }
  }
  TLK_DEV void finish(const Work&, int, Carry&) const {}
};

struct LinDgrad {
  static constexpr int BN = 64, STAGES = 4;
  static constexpr bool A_MN = true, B_MN = false;
  static constexpr bool TILE_EPILOGUE = false;
  using Work = LaneWork;
  struct Carry {
    float db;
  };
  const LaneState* lanes;
  const uint16_t* W;  // bf16 shadow arena, tensor [out][in]
  int64_t pstride, w_off;
  const uint16_t* dZ;  // [lanes][batch][out]
  int64_t dzst;
  const uint16_t* Hp;  // previous activation [lanes][batch][in]
  uint16_t* dZp;       // [lanes][batch][in]
  int64_t hst;
  float* grads;
  int64_t db_off;
  int out, in, batch;

  TLK_DEV bool work(Work& w) const {
    w.j = blockIdx.z;
    if (!lanes[w.j].active) return false;
    w.m0 = blockIdx.x * GEMM_BM;
    w.n0 = blockIdx.y * BN;
    w.kb_begin = 0;
    w.kb_end = (out + GEMM_BK - 1) / GEMM_BK;
    w.split = 0;
    return true;
  }
  TLK_DEV const void* zero_src() const { return W; }
  TLK_DEV const void* a_src(const Work& w, int m, int k) const {
    return (m < in && k < out) ? W + w.j * pstride + w_off + int64_t(k) * in + m : nullptr;
  }
  TLK_DEV const void* b_src(const Work& w, int n, int k) const {
    return (n < batch && k < out) ? dZ + w.j * dzst + int64_t(n) * out + k : nullptr;
  }
  TLK_DEV void epilogue(const Work& w, int m, int n0, const float (&v)[32], Carry& c) const {
    if (m >= in) return;
    const uint16_t* hp = Hp + w.j * hst + m;
    uint16_t* dz = dZp + w.j * hst + m;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int n = n0 + i;
      if (n < batch) {
        const uint16_t z = f2bf(bf2f(hp[int64_t(n) * in]) > 0.0f ? v[i] : 0.0f);
        dz[int64_t(n) * in] = z;
        c.db += bf2f(z);
      }
    }
  }
  TLK_DEV void finish(const Work& w, int m, Carry& c) const {
    if (m < in && blockIdx.y == 0 && gridDim.y == 1) grads[w.j * pstride + db_off + m] = c.db;
  }
};

}  // namespace tlk
