// Generic strided GEMM problem for the transformer pack: every operand is
// described by strides, a launch enumerates z = (lane, b, h) batches, and the
// epilogue kind is a runtime (CTA-uniform) switch.  Covers the dense layers
// (rows = tokens), the attention products per (sequence, head), and the
// weight-gradient products (K = tokens).
#pragma once
#include "models.cuh"
#include "tc_gemm.cuh"

namespace tlk {

struct Operand {  // element (mn, k) = base + lane*ls + zb*bs + zh*hs + mn*mn_st + k*k_st
  const uint16_t* base;
  int64_t ls, bs, hs, mn_st, k_st;
  int MN, K;  // bounds (zero fill outside)
};

enum EpiKind : int {
  EPI_BF16 = 0,      // out16 = bf16(acc + bias)
  EPI_BF16_GELU,     // z = acc + bias -> out32 (z); out16 = bf16(gelu_tanh(z))
  EPI_F32,           // out32 = acc
  EPI_RESADD,        // out32 = aux32 + acc + bias
  EPI_GELU_BWD,      // out16 = bf16(acc * gelu'(aux32))
  EPI_SOFTMAX,       // row: out16 = bf16(softmax(acc * scale, causal))
  EPI_SOFTMAX_BWD,   // row: out16 = bf16(P (acc - sum_j P acc) * scale), P = aux16
  EPI_CE,            // row: cross entropy vs targets -> lossrow, out16 = bf16(dlogits)
};

struct Epi {  // out[row][col] = base + lane*ls + zb*bs + zh*hs + row*ld + col
  int kind;
  int rows, cols;  // valid output extent (rows = M, cols = N)
  void* out;
  int64_t ls, bs, hs, ld;
  float* out32b;   // second output (EPI_BF16_GELU: pre-activation z, same indexing)
  const float* bias;  // fp32, + lane * bias_ls
  int64_t bias_ls;
  const void* aux;    // EPI_RESADD / EPI_GELU_BWD: fp32, EPI_SOFTMAX_BWD: bf16 (same indexing)
  float scale;
  int causal;
  const int32_t* targets;  // EPI_CE: [lane][rows] (+ lane*tg_ls)
  int64_t tg_ls;
  float* lossrow;          // EPI_CE: [lane][rows]
  float tokens;            // EPI_CE: dlogits are divided by the token count
};

struct ZWork {
  int j, zb, zh, m0, n0, kb_begin, kb_end, split;
};

TLK_DEV float gelu_tanh(float x, float& t) {
  const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  t = tanhf(u);
  return 0.5f * x * (1.0f + t);
}
TLK_DEV float gelu_tanh_grad(float x) {
  const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  const float t = tanhf(u);
  const float du = 0.7978845608028654f * (1.0f + 3.0f * 0.044715f * x * x);
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * du;
}

template <int BN_, bool AMN, bool BMN, bool ROW>
struct SGemm {
  static constexpr int BN = BN_, STAGES = BN_ >= 256 ? 3 : 4;
  static constexpr bool A_MN = AMN, B_MN = BMN;
  static constexpr bool TILE_EPILOGUE = false;
  static constexpr bool ROW_EPILOGUE = ROW;
  using Work = ZWork;
  struct Carry {};
  const LaneState* lanes;
  Operand a, b;
  Epi e;
  int nb, nh, kblocks;

  TLK_DEV bool work(Work& w) const {
    const int z = blockIdx.z, per = nb * nh;
    w.j = z / per;
    const int r = z % per;
    w.zb = r / nh;
    w.zh = r % nh;
    if (!lanes[w.j].active) return false;
    w.m0 = blockIdx.x * GEMM_BM;
    w.n0 = blockIdx.y * BN;
    w.kb_begin = 0;
    w.kb_end = kblocks;
    w.split = 0;
    return true;
  }
  TLK_DEV const void* zero_src() const { return a.base; }
  TLK_DEV const void* a_src(const Work& w, int m, int k) const {
    if (m >= a.MN || k >= a.K) return nullptr;
    return a.base + w.j * a.ls + w.zb * a.bs + w.zh * a.hs + m * a.mn_st + k * a.k_st;
  }
  TLK_DEV const void* b_src(const Work& w, int n, int k) const {
    if (n >= b.MN || k >= b.K) return nullptr;
    return b.base + w.j * b.ls + w.zb * b.bs + w.zh * b.hs + n * b.mn_st + k * b.k_st;
  }
  TLK_DEV int64_t off(const Work& w, int m, int n) const {
    return w.j * e.ls + w.zb * e.bs + w.zh * e.hs + int64_t(m) * e.ld + n;
  }
  TLK_DEV void epilogue(const Work& w, int m, int n0, const float (&v)[32], Carry&) const {
    if (m >= e.rows || n0 >= e.cols) return;
    const int64_t o = off(w, m, n0);
    const float* bias = e.bias ? e.bias + w.j * e.bias_ls + n0 : nullptr;
    const int nv = min(32, e.cols - n0);
    switch (e.kind) {
      case EPI_BF16: {
        uint16_t* out = static_cast<uint16_t*>(e.out) + o;
        for (int i = 0; i < nv; ++i) out[i] = f2bf(v[i] + (bias ? bias[i] : 0.f));
        break;
      }
      case EPI_BF16_GELU: {
        uint16_t* out = static_cast<uint16_t*>(e.out) + o;
        float* zo = e.out32b + o;
        for (int i = 0; i < nv; ++i) {
          const float z = v[i] + (bias ? bias[i] : 0.f);
          float t;
          zo[i] = z;
          out[i] = f2bf(gelu_tanh(z, t));
        }
        break;
      }
      case EPI_F32: {
        float* out = static_cast<float*>(e.out) + o;
        for (int i = 0; i < nv; ++i) out[i] = v[i];
        break;
      }
      case EPI_RESADD: {
        float* out = static_cast<float*>(e.out) + o;
        const float* res = static_cast<const float*>(e.aux) + o;
        for (int i = 0; i < nv; ++i) out[i] = res[i] + (v[i] + (bias ? bias[i] : 0.f));
        break;
      }
      case EPI_GELU_BWD: {
        uint16_t* out = static_cast<uint16_t*>(e.out) + o;
        const float* z = static_cast<const float*>(e.aux) + o;
        for (int i = 0; i < nv; ++i) out[i] = f2bf(v[i] * gelu_tanh_grad(z[i]));
        break;
      }
      default:
        break;
    }
  }
  TLK_DEV void finish(const Work&, int, Carry&) const {}

  // whole-row epilogues: taddr = this warp's TMEM lane quarter, column 0
  TLK_DEV void row_epilogue(const Work& w, int m, uint32_t taddr) const {
    const bool live = m < e.rows;
    const int ncols = e.cols;
    const int lim = e.causal ? min(ncols, m + 1) : ncols;  // valid columns of this row
    float v[32];
    if (e.kind == EPI_SOFTMAX) {
      float mx = -INFINITY;
      for (int c0 = 0; c0 < BN; c0 += 32) {
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < lim) mx = fmaxf(mx, v[i] * e.scale);
      }
      float s = 0.f;
      for (int c0 = 0; c0 < BN; c0 += 32) {
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < lim) s += expf(v[i] * e.scale - mx);
      }
      uint16_t* out = static_cast<uint16_t*>(e.out) + off(w, m, 0);
      for (int c0 = 0; c0 < BN; c0 += 32) {
        tmem_ld32(taddr + c0, v);
        if (!live || c0 >= ncols) continue;
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float p0 = (c0 + i < lim) ? expf(v[i] * e.scale - mx) / s : 0.f;
          const float p1 = (c0 + i + 1 < lim) ? expf(v[i + 1] * e.scale - mx) / s : 0.f;
          pk[i / 2] = pack_bf2(p0, p1);
        }
        uint4* o4 = reinterpret_cast<uint4*>(out + c0);
#pragma unroll
        for (int q = 0; q < 4; ++q) o4[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
      }
    } else if (e.kind == EPI_SOFTMAX_BWD) {
      const uint16_t* P = static_cast<const uint16_t*>(e.aux) + off(w, m, 0);
      float dsum = 0.f;
      for (int c0 = 0; c0 < BN; c0 += 32) {
        tmem_ld32(taddr + c0, v);
        if (!live) continue;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < ncols) dsum += bf2f(P[c0 + i]) * v[i];
      }
      uint16_t* out = static_cast<uint16_t*>(e.out) + off(w, m, 0);
      for (int c0 = 0; c0 < BN; c0 += 32) {
        tmem_ld32(taddr + c0, v);
        if (!live || c0 >= ncols) continue;
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float a0 = bf2f(P[c0 + i]) * (v[i] - dsum) * e.scale;
          const float a1 = bf2f(P[c0 + i + 1]) * (v[i + 1] - dsum) * e.scale;
          pk[i / 2] = pack_bf2(a0, a1);
        }
        uint4* o4 = reinterpret_cast<uint4*>(out + c0);
#pragma unroll
        for (int q = 0; q < 4; ++q) o4[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
      }
    } else if (e.kind == EPI_CE) {
      const int y = live ? e.targets[w.j * e.tg_ls + m] : 0;
      float mx = -INFINITY, ly = 0.f;
      for (int c0 = 0; c0 < BN; c0 += 32) {
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < ncols) {
            mx = fmaxf(mx, v[i]);
            if (c0 + i == y) ly = v[i];
          }
      }
      float s = 0.f;
      for (int c0 = 0; c0 < BN; c0 += 32) {
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < ncols) s += expf(v[i] - mx);
      }
      if (live) e.lossrow[w.j * int64_t(e.rows) + m] = (mx + logf(s)) - ly;
      uint16_t* out = static_cast<uint16_t*>(e.out) + off(w, m, 0);
      for (int c0 = 0; c0 < BN; c0 += 32) {
        tmem_ld32(taddr + c0, v);
        if (!live) continue;
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float d0 = 0.f, d1 = 0.f;
          if (c0 + i < ncols) d0 = (expf(v[i] - mx) / s - (c0 + i == y ? 1.f : 0.f)) / e.tokens;
          if (c0 + i + 1 < ncols)
            d1 = (expf(v[i + 1] - mx) / s - (c0 + i + 1 == y ? 1.f : 0.f)) / e.tokens;
          pk[i / 2] = pack_bf2(d0, d1);
        }
        uint4* o4 = reinterpret_cast<uint4*>(out + c0);
#pragma unroll
        for (int q = 0; q < 4; ++q) o4[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
      }
    }
  }
};

}  // namespace tlk
