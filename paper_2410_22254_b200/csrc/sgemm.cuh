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

// tanh on the SFU (MUFU.TANH, max rel. error ~2^-11): both GELU outputs are
// rounded to bf16 (2^-8), so the hardware approximation is below the
// storage precision.  z itself stays exact fp32.
TLK_DEV float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// e^x on the SFU (ex2.approx; ~2 ulp): softmax / CE probabilities are stored
// as bf16; the CE loss value itself uses logf of the (fp32) sum.
TLK_DEV float exp_fast(float x) { return exp2f(x * 1.4426950408889634f); }

TLK_DEV float gelu_tanh(float x, float& t) {
  const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  t = tanh_fast(u);
  return 0.5f * x * (1.0f + t);
}
TLK_DEV float gelu_tanh_grad(float x) {
  const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  const float t = tanh_fast(u);
  const float du = 0.7978845608028654f * (1.0f + 3.0f * 0.044715f * x * x);
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * du;
}

template <int BN_, bool AMN, bool BMN, bool ROW>
struct SGemm {
  // 3 stages at BN=128 (97 KB) / 4 at BN=64 (97 KB): two CTAs per SM, so one
  // CTA's epilogue overlaps the other's mainloop
  static constexpr int BN = BN_, STAGES = BN_ >= 128 ? 3 : 4;
  static constexpr bool EPILOGUE4 = true;
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

  // fp32 aux operand (residual / pre-activation) of 4 columns, fetched ahead
  // of the TMEM read so that the loads are in flight together
  TLK_DEV float4 aux4(const Work& w, int m, int n) const {
    if ((e.kind != EPI_RESADD && e.kind != EPI_GELU_BWD) || m >= e.rows || n + 4 > e.cols)
      return make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t o = off(w, m, n);
    if (o & 3) return make_float4(0.f, 0.f, 0.f, 0.f);
    return *reinterpret_cast<const float4*>(static_cast<const float*>(e.aux) + o);
  }

  // 4 consecutive columns n..n+3 of row m (lanes of a warp cover whole rows);
  // a = aux4(w, m, n)
  TLK_DEV void epilogue4(const Work& w, int m, int n, float x0, float x1, float x2, float x3,
                         float4 a) const {
    if (m >= e.rows || n >= e.cols) return;
    const int64_t o = off(w, m, n);
    float v[4] = {x0, x1, x2, x3};
    if (e.bias && (e.kind == EPI_BF16 || e.kind == EPI_BF16_GELU || e.kind == EPI_RESADD)) {
      const float* bias = e.bias + w.j * e.bias_ls + n;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (n + i < e.cols) v[i] += bias[i];
    }
    const bool vec = n + 4 <= e.cols && (o & 3) == 0;
    switch (e.kind) {
      case EPI_BF16: {
        uint16_t* out = static_cast<uint16_t*>(e.out) + o;
        if (vec) {
          *reinterpret_cast<uint2*>(out) = make_uint2(pack_bf2(v[0], v[1]), pack_bf2(v[2], v[3]));
        } else {
          for (int i = 0; i < 4 && n + i < e.cols; ++i) out[i] = f2bf(v[i]);
        }
        break;
      }
      case EPI_BF16_GELU: {
        uint16_t* out = static_cast<uint16_t*>(e.out) + o;
        float* zo = e.out32b + o;
        float g[4], t;
#pragma unroll
        for (int i = 0; i < 4; ++i) g[i] = gelu_tanh(v[i], t);
        if (vec) {
          *reinterpret_cast<float4*>(zo) = make_float4(v[0], v[1], v[2], v[3]);
          *reinterpret_cast<uint2*>(out) = make_uint2(pack_bf2(g[0], g[1]), pack_bf2(g[2], g[3]));
        } else {
          for (int i = 0; i < 4 && n + i < e.cols; ++i) {
            zo[i] = v[i];
            out[i] = f2bf(g[i]);
          }
        }
        break;
      }
      case EPI_F32: {
        float* out = static_cast<float*>(e.out) + o;
        if (vec) {
          *reinterpret_cast<float4*>(out) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
          for (int i = 0; i < 4 && n + i < e.cols; ++i) out[i] = v[i];
        }
        break;
      }
      case EPI_RESADD: {
        float* out = static_cast<float*>(e.out) + o;
        const float* res = static_cast<const float*>(e.aux) + o;
        if (vec) {
          const float4 r = a;
          *reinterpret_cast<float4*>(out) = make_float4(r.x + v[0], r.y + v[1], r.z + v[2], r.w + v[3]);
        } else {
          for (int i = 0; i < 4 && n + i < e.cols; ++i) out[i] = res[i] + v[i];
        }
        break;
      }
      case EPI_GELU_BWD: {
        uint16_t* out = static_cast<uint16_t*>(e.out) + o;
        const float* z = static_cast<const float*>(e.aux) + o;
        if (vec) {
          const float4 zz = a;
          *reinterpret_cast<uint2*>(out) =
              make_uint2(pack_bf2(v[0] * gelu_tanh_grad(zz.x), v[1] * gelu_tanh_grad(zz.y)),
                         pack_bf2(v[2] * gelu_tanh_grad(zz.z), v[3] * gelu_tanh_grad(zz.w)));
        } else {
          for (int i = 0; i < 4 && n + i < e.cols; ++i) out[i] = f2bf(v[i] * gelu_tanh_grad(z[i]));
        }
        break;
      }
      default:
        break;
    }
  }

  // whole-row epilogues: thread = row m (= warp row base + lane), taddr = this
  // warp's TMEM lane quarter at column 0, buf = the warp's 32 x 33 fp32
  // staging buffer.  Row-major bf16 tiles (P, dS, dlogits) move through `buf`
  // so that global loads/stores are coalesced along rows (a warp covers 4
  // rows x 32 columns per instruction).  Causal rows skip the 32-column
  // chunks that lie entirely above the diagonal for the whole warp: those
  // entries of P / dS are never written and stay zero from the pack's
  // initial memset (nothing else writes these buffers).
  TLK_DEV void store_chunk(const Work& w, int row0, int c0, float* buf, int lane) const {
    __syncwarp();
    const int rsub = lane >> 3, c4 = (lane & 7) * 4;
    uint16_t* out = static_cast<uint16_t*>(e.out);
#pragma unroll 4
    for (int r0 = 0; r0 < 32; r0 += 4) {
      const int r = r0 + rsub, m = row0 + r, n = c0 + c4;
      if (m < e.rows && n < e.cols) {
        const float* x = buf + r * 33 + c4;
        uint16_t* o = out + off(w, m, n);
        if (n + 4 <= e.cols) {
          *reinterpret_cast<uint2*>(o) = make_uint2(pack_bf2(x[0], x[1]), pack_bf2(x[2], x[3]));
        } else {
          for (int i = 0; i < 4 && n + i < e.cols; ++i) o[i] = f2bf(x[i]);
        }
      }
    }
    __syncwarp();
  }
  // buf[r][c] <- bf16 aux tile (rows row0.., columns c0..c0+32), 0 outside
  TLK_DEV void load_chunk(const Work& w, int row0, int c0, float* buf, int lane) const {
    __syncwarp();
    const int rsub = lane >> 3, c4 = (lane & 7) * 4;
    const uint16_t* src = static_cast<const uint16_t*>(e.aux);
#pragma unroll 4
    for (int r0 = 0; r0 < 32; r0 += 4) {
      const int r = r0 + rsub, m = row0 + r, n = c0 + c4;
      float* x = buf + r * 33 + c4;
      if (m < e.rows && n + 4 <= e.cols) {
        const uint2 u = *reinterpret_cast<const uint2*>(src + off(w, m, n));
        x[0] = __uint_as_float(u.x << 16);
        x[1] = __uint_as_float(u.x & 0xffff0000u);
        x[2] = __uint_as_float(u.y << 16);
        x[3] = __uint_as_float(u.y & 0xffff0000u);
      } else {
        for (int i = 0; i < 4; ++i) x[i] = (m < e.rows && n + i < e.cols) ? bf2f(src[off(w, m, n + i)]) : 0.f;
      }
    }
    __syncwarp();
  }

  TLK_DEV void row_epilogue(const Work& w, int m, uint32_t taddr, float* buf, int lane) const {
    const bool live = m < e.rows;
    const int ncols = e.cols;
    const int row0 = m - lane;
    const int lim = e.causal ? min(ncols, m + 1) : ncols;            // valid columns of this row
    const int wlim = e.causal ? min(ncols, row0 + 32) : ncols;       // warp-uniform chunk bound
    float v[32];
    if (e.kind == EPI_SOFTMAX) {
      float mx = -INFINITY;
      for (int c0 = 0; c0 < wlim; c0 += 32) {
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < lim) mx = fmaxf(mx, v[i] * e.scale);
      }
      float s = 0.f;
      for (int c0 = 0; c0 < wlim; c0 += 32) {
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < lim) s += exp_fast(v[i] * e.scale - mx);
      }
      const float inv = 1.f / s;
      for (int c0 = 0; c0 < wlim; c0 += 32) {
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          buf[lane * 33 + i] = (c0 + i < lim) ? exp_fast(v[i] * e.scale - mx) * inv : 0.f;
        store_chunk(w, row0, c0, buf, lane);
      }
    } else if (e.kind == EPI_SOFTMAX_BWD) {
      float dsum = 0.f;
      for (int c0 = 0; c0 < wlim; c0 += 32) {
        load_chunk(w, row0, c0, buf, lane);
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < ncols) dsum += buf[lane * 33 + i] * v[i];
      }
      for (int c0 = 0; c0 < wlim; c0 += 32) {
        load_chunk(w, row0, c0, buf, lane);
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) buf[lane * 33 + i] = buf[lane * 33 + i] * (v[i] - dsum) * e.scale;
        store_chunk(w, row0, c0, buf, lane);
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
          if (c0 + i < ncols) s += exp_fast(v[i] - mx);
      }
      if (live) e.lossrow[w.j * int64_t(e.rows) + m] = (mx + logf(s)) - ly;
      // dlogits over the padded width (zeros in the padding columns)
      const float inv = 1.f / s, invt = 1.f / e.tokens;
      for (int c0 = 0; c0 < BN; c0 += 32) {
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          buf[lane * 33 + i] =
              (c0 + i < ncols) ? (exp_fast(v[i] - mx) * inv - (c0 + i == y ? 1.f : 0.f)) * invt : 0.f;
        store_chunk_padded(w, row0, c0, buf, lane);
      }
    }
  }
  // dlogits rows are Vp wide (ld): the padding columns are written as zeros
  TLK_DEV void store_chunk_padded(const Work& w, int row0, int c0, float* buf, int lane) const {
    __syncwarp();
    const int rsub = lane >> 3, c4 = (lane & 7) * 4;
    uint16_t* out = static_cast<uint16_t*>(e.out);
#pragma unroll 4
    for (int r0 = 0; r0 < 32; r0 += 4) {
      const int r = r0 + rsub, m = row0 + r, n = c0 + c4;
      if (m < e.rows && n < e.ld) {
        const float* x = buf + r * 33 + c4;
        *reinterpret_cast<uint2*>(out + off(w, m, n)) =
            make_uint2(pack_bf2(x[0], x[1]), pack_bf2(x[2], x[3]));
      }
    }
    __syncwarp();
  }
};

}  // namespace tlk
