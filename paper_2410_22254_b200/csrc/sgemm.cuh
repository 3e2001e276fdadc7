// Strided GEMM problems of the transformer pack and their fused epilogues.
// Every operand is described by strides, a launch enumerates z = (lane, b, h)
// batches, and the epilogue kind is a launch-uniform switch resolved once per
// tile into a specialised routine.  Covers the dense layers (rows = tokens),
// the attention products per (sequence, head), and the weight-gradient
// products (K = tokens).  The mainloop lives in tgemm.cuh.
#pragma once
#include "models.cuh"
#include "tc_gemm.cuh"
#include "tma.cuh"

namespace tlk {

struct Operand {  // element (mn, k) = base + lane*ls + zb*bs + zh*hs + mn*mn_st + k*k_st
  const uint16_t* base;
  int64_t ls, bs, hs, mn_st, k_st;
  int MN, K;  // bounds (zero fill outside)
};

enum EpiKind : int {
  EPI_BF16 = 0,      // out16 = bf16(acc + bias)
  EPI_BF16_GELU,     // z = acc + bias -> out2 = bf16(z); out16 = bf16(gelu_tanh(z))
  EPI_F32,           // out32 = acc
  EPI_RESADD,        // out32 = aux32 + acc + bias
  EPI_GELU_BWD,      // out16 = bf16(acc * gelu'(aux16))
  EPI_SOFTMAX,       // row: out16 = bf16(softmax(acc * scale, causal))
  EPI_SOFTMAX_BWD,   // row: out16 = bf16(P (acc - D) * scale), P = aux16, D = rowvec
  EPI_CE,            // row: cross entropy vs targets -> lossrow, out16 = bf16(dlogits)
  EPI_BF16_ROWDOT,   // out16 = bf16(acc); rowout[row, head] = sum_c out16 * aux16 (TMA path, 64-col parts)
};

struct Epi {  // out[row][col] = base + lane*ls + zb*bs + zh*hs + row*ld + col
  int kind;
  int rows, cols;  // valid output extent (rows = M, cols = N)
  void* out;
  int64_t ls, bs, hs, ld;
  uint16_t* out2;  // second output (EPI_BF16_GELU: bf16 pre-activation z, same indexing)
  const float* bias;  // fp32, + lane * bias_ls
  int64_t bias_ls;
  const void* aux;    // EPI_RESADD: fp32, EPI_GELU_BWD / EPI_SOFTMAX_BWD: bf16 (same indexing)
  float scale;
  int causal;
  int causal_k;  // A is causal in (row, k): 1 -> only k <= row, 2 -> only k >= row (transposed P / dS);
                 // the all-zero k-blocks are skipped (adding exact zeros: same bits)
  const int32_t* targets;  // EPI_CE: [lane][rows] (+ lane*tg_ls)
  int64_t tg_ls;
  float* lossrow;          // EPI_CE: [lane][rows]
  float tokens;            // EPI_CE: dlogits are divided by the token count
  const float* rowvec;     // EPI_SOFTMAX_BWD: D[row] at lane*rv_ls + zb*rv_bs + zh*rv_hs + row
  float* rowout;           // EPI_BF16_ROWDOT: [lane][row / rv_T][head][row % rv_T], head = column / 64
  int rv_T, rv_H;
  int64_t rv_ls, rv_bs, rv_hs;
  float* colpart;          // EPI_GELU_BWD / EPI_BF16 (optional): column sums of the stored bf16
  int64_t cp_ls;           //   output per 32-row block (bias-gradient partials):
  int cp_cols, cp_col0;    //   [lane][(zb * rows + row) / 32][cp_cols], column cp_col0 + zh*hs + n
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
TLK_DEV float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
TLK_DEV float exp_fast(float x) { return ex2_approx(x * 1.4426950408889634f); }

// gelu(x) = 0.5 x (1 + tanh(u)), u = c0 x + c1 x^3, written as FMA chains
// (x^2 once; 0.5 folded into the final FMA).
constexpr float GELU_C0 = 0.7978845608028654f, GELU_C1 = 0.7978845608028654f * 0.044715f;
TLK_DEV float gelu_tanh(float x, float& t) {
  const float x2 = x * x;
  t = tanh_fast(x * fmaf(x2, GELU_C1, GELU_C0));
  const float h = 0.5f * x;
  return fmaf(h, t, h);
}
// y * gelu'(x) = 0.5 y (1 + t + x du (1 - t^2)),  du = c0 + 3 c1 x^2
TLK_DEV float gelu_bwd_mul(float y, float x) {
  const float x2 = x * x;
  const float t = tanh_fast(x * fmaf(x2, GELU_C1, GELU_C0));
  const float xd = x * fmaf(x2, 3.0f * GELU_C1, GELU_C0);
  const float q = fmaf(xd, fmaf(-t, t, 1.0f), t);
  const float hy = 0.5f * y;
  return fmaf(hy, q, hy);
}

// the same two functions on f32x2 pairs (bit-identical per lane: the FMA
// chains are the scalar ones, with -(3 c1 x^2 + c0) and t^2 - 1 carrying the
// signs so that no negation instruction is needed)
TLK_DEV f2 gelu2(f2 x) {
  const f2 x2 = f2_mul(x, x);
  const f2 u = f2_mul(x, f2_fma(x2, f2_make(GELU_C1, GELU_C1), f2_make(GELU_C0, GELU_C0)));
  const f2 t = f2_make(tanh_fast(f2_lo(u)), tanh_fast(f2_hi(u)));
  const f2 h = f2_mul(x, f2_make(0.5f, 0.5f));
  return f2_fma(h, t, h);
}
TLK_DEV f2 gelu_bwd_mul2(f2 y, f2 x) {
  const f2 x2 = f2_mul(x, x);
  const f2 u = f2_mul(x, f2_fma(x2, f2_make(GELU_C1, GELU_C1), f2_make(GELU_C0, GELU_C0)));
  const f2 t = f2_make(tanh_fast(f2_lo(u)), tanh_fast(f2_hi(u)));
  const f2 xdn = f2_mul(x, f2_fma(x2, f2_make(-3.0f * GELU_C1, -3.0f * GELU_C1), f2_make(-GELU_C0, -GELU_C0)));
  const f2 q = f2_fma(xdn, f2_fma(t, t, f2_make(-1.0f, -1.0f)), t);
  const f2 hy = f2_mul(y, f2_make(0.5f, 0.5f));
  return f2_fma(hy, q, hy);
}

// Epilogue state of one launch + the per-kind tile routines.  A warp owns 32
// accumulator rows (its TMEM lane quarter); `buf` is its 32 x 33 fp32 smem
// staging buffer.  TMEM gives each thread one ROW, global memory wants a warp
// to cover whole rows, so every 32 x 32 chunk is transposed through `buf` and
// then written 4 rows x 32 columns per warp instruction (8-byte bf16 / 16-byte
// fp32 vectors per lane).  Host-side contract (checked in gpt.cu): cols, ld
// and all z strides are multiples of 4 elements, bases 16-byte aligned.
struct EpiOps {
  const LaneState* lanes;
  Epi e;
  int nb, nh, kblocks;

  TLK_DEV int64_t off(const ZWork& w, int m, int n) const {
    return w.j * e.ls + w.zb * e.bs + w.zh * e.hs + int64_t(m) * e.ld + n;
  }

  // ---- dense (per-element) epilogues -------------------------------------
  // NP column parts: part p of the two warps sharing a TMEM lane quarter
  // takes the 32-column chunks [p NC/NP, (p+1) NC/NP) of the tile
  template <int KIND, int BN, int NP = 1>
  TLK_DEV void tile4(const ZWork& w, uint32_t tq, int row0, float* buf, int lane, int part = 0) const {
    constexpr int NC = BN / 32;
    const int cc0 = part * (NC / NP), cc1 = cc0 + NC / NP;
    const int rsub = lane >> 3, c4 = (lane & 7) * 4;
    const int64_t step = 4 * e.ld;
    const int64_t o0 = off(w, row0 + rsub, w.n0 + c4);
    constexpr bool BIAS = KIND == EPI_BF16 || KIND == EPI_BF16_GELU || KIND == EPI_RESADD;
    constexpr bool AUX = KIND == EPI_RESADD || KIND == EPI_GELU_BWD;
    const float* bias = (BIAS && e.bias) ? e.bias + w.j * e.bias_ls : nullptr;
    // aux rows of chunk cc + 1 are fetched while chunk cc is processed
    float4 ax[8], nx[8];
    auto fetch = [&](int cc, float4 (&dst)[8]) {
      const int n = w.n0 + cc * 32 + c4;
      if constexpr (KIND == EPI_GELU_BWD) {  // bf16 pre-activation
        const uint16_t* a = static_cast<const uint16_t*>(e.aux) + o0 + cc * 32;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint2 u = (n < e.cols && row0 + 4 * k + rsub < e.rows) ? *reinterpret_cast<const uint2*>(a + k * step)
                                                                       : make_uint2(0u, 0u);
          dst[k] = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                               __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
        }
      } else {
        const float* a = static_cast<const float*>(e.aux) + o0 + cc * 32;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          dst[k] = (n < e.cols && row0 + 4 * k + rsub < e.rows) ? *reinterpret_cast<const float4*>(a + k * step)
                                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    // one warp per lane quarter (NP == 1): the next chunk's aux rows are in
    // flight during this chunk; with two (NP == 2, 96-register budget) the
    // chunk's own aux rows are issued before its TMEM load and staging
    if constexpr (AUX && NP == 1) fetch(cc0, nx);
#pragma unroll 1
    for (int cc = cc0; cc < cc1; ++cc) {
      const int n = w.n0 + cc * 32 + c4;
      const bool col_ok = n < e.cols;
      const int64_t o = o0 + cc * 32;
      if constexpr (AUX) {
        if constexpr (NP == 1) {
#pragma unroll
          for (int k = 0; k < 8; ++k) ax[k] = nx[k];
          if (cc + 1 < cc1) fetch(cc + 1, nx);
        } else {
          fetch(cc, ax);
        }
      }
      float4 bb = make_float4(0.f, 0.f, 0.f, 0.f);
      if (bias && col_ok) bb = make_float4(bias[n], bias[n + 1], bias[n + 2], bias[n + 3]);
      float cs[4] = {0.f, 0.f, 0.f, 0.f};  // EPI_GELU_BWD column partials
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {  // two 16-column TMEM loads: fewer live registers
        float v[16];
        tmem_ld16(tq + cc * 32 + hf * 16, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) buf[lane * 33 + hf * 16 + i] = v[i];
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int r = 4 * k + rsub;
        if (!col_ok || row0 + r >= e.rows) continue;
        const float* x = buf + r * 33 + c4;
        float y0 = x[0], y1 = x[1], y2 = x[2], y3 = x[3];
        if constexpr (BIAS) {
          y0 += bb.x;
          y1 += bb.y;
          y2 += bb.z;
          y3 += bb.w;
        }
        const int64_t oo = o + k * step;
        if constexpr (KIND == EPI_BF16) {
          const uint32_t lo = pack_bf2(y0, y1), hi = pack_bf2(y2, y3);
          *reinterpret_cast<uint2*>(static_cast<uint16_t*>(e.out) + oo) = make_uint2(lo, hi);
          cs[0] += __uint_as_float(lo << 16);
          cs[1] += __uint_as_float(lo & 0xffff0000u);
          cs[2] += __uint_as_float(hi << 16);
          cs[3] += __uint_as_float(hi & 0xffff0000u);
        } else if constexpr (KIND == EPI_BF16_GELU) {
          float t;
          *reinterpret_cast<uint2*>(e.out2 + oo) = make_uint2(pack_bf2(y0, y1), pack_bf2(y2, y3));
          const float g0 = gelu_tanh(y0, t), g1 = gelu_tanh(y1, t), g2 = gelu_tanh(y2, t),
                      g3 = gelu_tanh(y3, t);
          *reinterpret_cast<uint2*>(static_cast<uint16_t*>(e.out) + oo) =
              make_uint2(pack_bf2(g0, g1), pack_bf2(g2, g3));
        } else if constexpr (KIND == EPI_F32) {
          *reinterpret_cast<float4*>(static_cast<float*>(e.out) + oo) = make_float4(y0, y1, y2, y3);
        } else if constexpr (KIND == EPI_RESADD) {
          const float4 r4 = ax[k];
          *reinterpret_cast<float4*>(static_cast<float*>(e.out) + oo) =
              make_float4(r4.x + y0, r4.y + y1, r4.z + y2, r4.w + y3);
        } else if constexpr (KIND == EPI_GELU_BWD) {
          const float4 z = ax[k];
          const uint32_t lo = pack_bf2(gelu_bwd_mul(y0, z.x), gelu_bwd_mul(y1, z.y));
          const uint32_t hi = pack_bf2(gelu_bwd_mul(y2, z.z), gelu_bwd_mul(y3, z.w));
          *reinterpret_cast<uint2*>(static_cast<uint16_t*>(e.out) + oo) = make_uint2(lo, hi);
          cs[0] += __uint_as_float(lo << 16);
          cs[1] += __uint_as_float(lo & 0xffff0000u);
          cs[2] += __uint_as_float(hi << 16);
          cs[3] += __uint_as_float(hi & 0xffff0000u);
        }
      }
      if constexpr (KIND == EPI_GELU_BWD || KIND == EPI_BF16) {
        // column sums of this warp's 32 rows of the stored (bf16) values:
        // lanes l, l+8, l+16, l+24 hold the same 4 columns (fixed xor order)
        if (e.colpart) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            cs[i] += __shfl_xor_sync(0xffffffffu, cs[i], 8);
            cs[i] += __shfl_xor_sync(0xffffffffu, cs[i], 16);
          }
          if (rsub == 0 && col_ok && row0 < e.rows) {  // rows past e.rows belong to the next z
            const int64_t frow = int64_t(w.zb) * (e.bs / e.ld) + row0;  // row within the lane
            const int pc = e.cp_cols ? e.cp_cols : e.cols;
            *reinterpret_cast<float4*>(e.colpart + w.j * e.cp_ls + (frow >> 5) * pc + e.cp_col0 + w.zh * e.hs + n) =
                make_float4(cs[0], cs[1], cs[2], cs[3]);
          }
        }
      }
      __syncwarp();
    }
  }

  // ---- TMA-staged dense epilogues (thread = accumulator row) ---------------
  // tile4 transposes every 32 x 32 chunk through `buf` so that global stores
  // coalesce; here each thread keeps its TMEM row, works on 16-column chunks
  // in registers and writes them (one or two 16 B vectors per 8 columns) into
  // a per-warp 2 KB staging tile laid out in the TMA swizzle of a {16, 32}
  // box, which one lane stores with cp.async.bulk.tensor.  The aux operand
  // (GELU' input, residual) is TMA-loaded into the same tile one chunk ahead
  // and overwritten in place, NB - 1 chunks ahead (NB tiles per warp, ring
  // position `cnt`);
  // rows / columns past the tensor are clipped by TMA, so there are no
  // per-element bounds checks.  Bias-gradient column partials are summed
  // from the staged bf16 tile.
  template <int KIND>
  static constexpr int tma_ob() {
    return (KIND == EPI_F32 || KIND == EPI_RESADD) ? 4 : 2;
  }
  template <int KIND>
  static constexpr uint32_t tma_aux_bytes() {
    return (KIND == EPI_GELU_BWD || KIND == EPI_BF16_ROWDOT) ? 32 * 16 * 2 : KIND == EPI_RESADD ? 32 * 16 * 4 : 0;
  }
  // byte offset of 16 B vector c of row r in a swizzled {16, 32} box tile
  template <int OB>
  TLK_DEV static uint32_t sw_off(int r, int c) {
    if constexpr (OB == 2)
      return uint32_t(r * 32 + ((c ^ ((r >> 2) & 1)) << 4));  // SWIZZLE_32B
    else
      return uint32_t(r * 64 + ((c ^ ((r >> 1) & 3)) << 4));  // SWIZZLE_64B
  }
  TLK_DEV bool tma_live(const ZWork& w, int row0, int n) const { return row0 < e.rows && n < e.cols; }

  // issue the aux load of the warp's first chunk of a tile (before its TMEM wait)
  template <int KIND, int BN, int NP, int TB, int NB>
  TLK_DEV void tma_pre(const ZWork& w, int row0, int lane, int part, uint32_t stg, uint64_t* abar, uint32_t cnt,
                       const CUtensorMap* ma) const {
    if constexpr (tma_aux_bytes<KIND>() > 0) {
      if (lane == 0) {
        const int c0 = part * (BN / 16 / NP);
        bulk_wait_read<1>();  // stores that last read these buffers are done
#pragma unroll
        for (int k = 0; k < NB - 1; ++k) {
          const int n = w.n0 + (c0 + k) * 16;
          if (k < BN / 16 / NP && tma_live(w, row0, n)) {
            const uint32_t b = (cnt + k) % NB;
            mbar_expect_tx(&abar[b], tma_aux_bytes<KIND>());
            tma_load_5d(stg + b * TB, ma, n, row0, w.zh, w.zb, w.j, &abar[b]);
          }
        }
      }
    }
  }

  template <int KIND, int BN, int NP, int TB, int NB>
  TLK_DEV void tile_tma(const ZWork& w, uint32_t tq, int row0, int lane, int part, uint8_t* stg_p, uint64_t* abar,
                        uint32_t& cnt, const CUtensorMap* mo, const CUtensorMap* mo2, const CUtensorMap* ma) const {
    constexpr int NC = BN / 16;
    constexpr uint32_t AUXB = tma_aux_bytes<KIND>();
    constexpr bool BIAS = KIND == EPI_BF16 || KIND == EPI_BF16_GELU || KIND == EPI_RESADD;
    constexpr bool CP = KIND == EPI_GELU_BWD || KIND == EPI_BF16;
    static_assert(TB >= (KIND == EPI_BF16_GELU || tma_ob<KIND>() == 4 ? 2048 : 1024), "staging tile too small");
    const int cc0 = part * (NC / NP), cc1 = cc0 + NC / NP;
    const float* bias = (BIAS && e.bias) ? e.bias + w.j * e.bias_ls : nullptr;
    const uint32_t stg = smem_u32(stg_p);
    f2 dot = f2_make(0.f, 0.f);  // EPI_BF16_ROWDOT: this part's head (even, odd columns)
    // bias-gradient partials of this warp's 32-row block (per tile)
    float* cpb = nullptr;
    bool cp_full = true;
    if constexpr (CP) {
      if (e.colpart) {
        const int64_t frow = int64_t(w.zb) * (e.bs / e.ld) + row0;  // row within the lane
        const int pc = e.cp_cols ? e.cp_cols : e.cols;
        cpb = e.colpart + w.j * e.cp_ls + (frow >> 5) * pc + e.cp_col0 + w.zh * e.hs;
        cp_full = row0 + 32 <= e.rows;
      }
    }
#pragma unroll 1
    for (int cc = cc0; cc < cc1; ++cc) {
      const int n = w.n0 + cc * 16;
      if (!tma_live(w, row0, n)) break;  // warp-uniform: the rest of the row block is outside too
      const uint32_t b = cnt % NB;
      uint8_t* bp = stg_p + b * TB;
      f2 a[8];
      {
        float v[16];
        tmem_ld16(tq + cc * 16, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = f2_make(v[2 * i], v[2 * i + 1]);
      }
      if (bias) {
        const float4* b4 = reinterpret_cast<const float4*>(bias + n);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 x = b4[i];
          a[2 * i] = f2_add(a[2 * i], f2_make(x.x, x.y));
          a[2 * i + 1] = f2_add(a[2 * i + 1], f2_make(x.z, x.w));
        }
      }
      if constexpr (AUXB > 0) mbar_wait(&abar[b], (cnt / NB) & 1);
      if constexpr (KIND == EPI_BF16) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
          *reinterpret_cast<uint4*>(bp + sw_off<2>(lane, c)) =
              make_uint4(bf2_from_f2(a[4 * c]), bf2_from_f2(a[4 * c + 1]), bf2_from_f2(a[4 * c + 2]),
                         bf2_from_f2(a[4 * c + 3]));
      } else if constexpr (KIND == EPI_BF16_ROWDOT) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint4* y4 = reinterpret_cast<uint4*>(bp + sw_off<2>(lane, c));
          const uint4 y = *y4;
          const uint4 o = make_uint4(bf2_from_f2(a[4 * c]), bf2_from_f2(a[4 * c + 1]), bf2_from_f2(a[4 * c + 2]),
                                     bf2_from_f2(a[4 * c + 3]));
          *y4 = o;
          dot = f2_fma(f2_from_bf2(o.x), f2_from_bf2(y.x), dot);
          dot = f2_fma(f2_from_bf2(o.y), f2_from_bf2(y.y), dot);
          dot = f2_fma(f2_from_bf2(o.z), f2_from_bf2(y.z), dot);
          dot = f2_fma(f2_from_bf2(o.w), f2_from_bf2(y.w), dot);
        }
      } else if constexpr (KIND == EPI_BF16_GELU) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          *reinterpret_cast<uint4*>(bp + 1024 + sw_off<2>(lane, c)) =
              make_uint4(bf2_from_f2(a[4 * c]), bf2_from_f2(a[4 * c + 1]), bf2_from_f2(a[4 * c + 2]),
                         bf2_from_f2(a[4 * c + 3]));
          *reinterpret_cast<uint4*>(bp + sw_off<2>(lane, c)) =
              make_uint4(bf2_from_f2(gelu2(a[4 * c])), bf2_from_f2(gelu2(a[4 * c + 1])),
                         bf2_from_f2(gelu2(a[4 * c + 2])), bf2_from_f2(gelu2(a[4 * c + 3])));
        }
      } else if constexpr (KIND == EPI_F32) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *reinterpret_cast<ulonglong2*>(bp + sw_off<4>(lane, c)) = make_ulonglong2(a[2 * c], a[2 * c + 1]);
      } else if constexpr (KIND == EPI_RESADD) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          ulonglong2* r = reinterpret_cast<ulonglong2*>(bp + sw_off<4>(lane, c));
          const ulonglong2 r2 = *r;
          *r = make_ulonglong2(f2_add(r2.x, a[2 * c]), f2_add(r2.y, a[2 * c + 1]));
        }
      } else if constexpr (KIND == EPI_GELU_BWD) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint4* z4 = reinterpret_cast<uint4*>(bp + sw_off<2>(lane, c));
          const uint4 z = *z4;
          *z4 = make_uint4(bf2_from_f2(gelu_bwd_mul2(a[4 * c], f2_from_bf2(z.x))),
                           bf2_from_f2(gelu_bwd_mul2(a[4 * c + 1], f2_from_bf2(z.y))),
                           bf2_from_f2(gelu_bwd_mul2(a[4 * c + 2], f2_from_bf2(z.z))),
                           bf2_from_f2(gelu_bwd_mul2(a[4 * c + 3], f2_from_bf2(z.w))));
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if constexpr (CP) {
        if (cpb) {
          // lane = (row group g, column pair cp): rows 8g.. in a rotated order
          // (the four groups hit four different 32 B bank segments)
          const int cp = lane & 7, g = lane >> 3;
          const uint8_t* col = bp + (cp & 3) * 4;
          f2 sum = f2_make(0.f, 0.f);
          if (cp_full) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int r = 8 * g + ((i + g) & 7);
              sum = f2_add(sum, f2_from_bf2(*reinterpret_cast<const uint32_t*>(col + sw_off<2>(r, cp >> 2))));
            }
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int r = 8 * g + ((i + g) & 7);
              const uint32_t u = *reinterpret_cast<const uint32_t*>(col + sw_off<2>(r, cp >> 2));
              sum = f2_add(sum, f2_from_bf2(row0 + r < e.rows ? u : 0u));
            }
          }
          float s0 = f2_lo(sum), s1 = f2_hi(sum);
          s0 += __shfl_xor_sync(0xffffffffu, s0, 8);
          s1 += __shfl_xor_sync(0xffffffffu, s1, 8);
          s0 += __shfl_xor_sync(0xffffffffu, s0, 16);
          s1 += __shfl_xor_sync(0xffffffffu, s1, 16);
          if (lane < 8) *reinterpret_cast<float2*>(cpb + n + 2 * cp) = make_float2(s0, s1);
        }
      }
      if (lane == 0) {
        tma_store_5d(mo, stg + b * TB, n, row0, w.zh, w.zb, w.j);
        if constexpr (KIND == EPI_BF16_GELU) tma_store_5d(mo2, stg + b * TB + 1024, n, row0, w.zh, w.zb, w.j);
        bulk_commit();
        bulk_wait_read<1>();  // only this chunk's store may still read its buffer
        if constexpr (AUXB > 0) {  // aux of chunk cc + NB - 1 into the buffer chunk cc - 1 used
          const int nn = n + (NB - 1) * 16;
          if (cc + NB - 1 < cc1 && tma_live(w, row0, nn)) {
            const uint32_t bn = (cnt + NB - 1) % NB;
            mbar_expect_tx(&abar[bn], AUXB);
            tma_load_5d(stg + bn * TB, ma, nn, row0, w.zh, w.zb, w.j, &abar[bn]);
          }
        }
      }
      __syncwarp();
      ++cnt;
    }
    if constexpr (KIND == EPI_BF16_ROWDOT) {
      const int m = row0 + lane;
      if (m < e.rows && tma_live(w, row0, w.n0 + cc0 * 16)) {
        const int h = (w.n0 + cc0 * 16) >> 6;
        e.rowout[((int64_t(w.j) * (e.rows / e.rv_T) + m / e.rv_T) * e.rv_H + h) * e.rv_T + m % e.rv_T] =
            f2_lo(dot) + f2_hi(dot);
      }
    }
  }

  template <int BN, int NP, int TB, int NB>
  TLK_DEV void tma_pre_any(const ZWork& w, int row0, int lane, int part, uint32_t stg, uint64_t* abar, uint32_t cnt,
                           const CUtensorMap* ma) const {
    if (e.kind == EPI_GELU_BWD) {
      tma_pre<EPI_GELU_BWD, BN, NP, TB, NB>(w, row0, lane, part, stg, abar, cnt, ma);
    } else if (e.kind == EPI_BF16_ROWDOT) {
      if constexpr (BN / NP == 64) tma_pre<EPI_BF16_ROWDOT, BN, NP, TB, NB>(w, row0, lane, part, stg, abar, cnt, ma);
    } else if (e.kind == EPI_RESADD) {
      if constexpr (TB >= 2048) tma_pre<EPI_RESADD, BN, NP, TB, NB>(w, row0, lane, part, stg, abar, cnt, ma);
    }
  }
  template <int BN, int NP, int TB, int NB>
  TLK_DEV void tile_tma_any(const ZWork& w, uint32_t tq, int row0, int lane, int part, uint8_t* stg_p,
                            uint64_t* abar, uint32_t& cnt, const CUtensorMap* mo, const CUtensorMap* mo2,
                            const CUtensorMap* ma) const {
    switch (e.kind) {
      case EPI_BF16: tile_tma<EPI_BF16, BN, NP, TB, NB>(w, tq, row0, lane, part, stg_p, abar, cnt, mo, mo2, ma); break;
      case EPI_BF16_ROWDOT:  // one 64-column head per part warp (host-checked)
        if constexpr (BN / NP == 64)
          tile_tma<EPI_BF16_ROWDOT, BN, NP, TB, NB>(w, tq, row0, lane, part, stg_p, abar, cnt, mo, mo2, ma);
        else
          __trap();
        break;
      case EPI_BF16_GELU:
        if constexpr (TB >= 2048) tile_tma<EPI_BF16_GELU, BN, NP, TB, NB>(w, tq, row0, lane, part, stg_p, abar, cnt, mo, mo2, ma); else __trap();
        break;
      case EPI_F32: if constexpr (TB >= 2048) tile_tma<EPI_F32, BN, NP, TB, NB>(w, tq, row0, lane, part, stg_p, abar, cnt, mo, mo2, ma); else __trap(); break;
      case EPI_RESADD: if constexpr (TB >= 2048) tile_tma<EPI_RESADD, BN, NP, TB, NB>(w, tq, row0, lane, part, stg_p, abar, cnt, mo, mo2, ma); else __trap(); break;
      case EPI_GELU_BWD:
        tile_tma<EPI_GELU_BWD, BN, NP, TB, NB>(w, tq, row0, lane, part, stg_p, abar, cnt, mo, mo2, ma);
        break;
      default: break;
    }
  }

  // ---- whole-row epilogues ------------------------------------------------
  TLK_DEV void fetch_chunk(const uint16_t* p, int64_t step, int row0, uint2 (&u)[8], int lane) const {
    const int rsub = lane >> 3;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      u[k] = (row0 + 4 * k + rsub < e.rows) ? *reinterpret_cast<const uint2*>(p + k * step) : make_uint2(0u, 0u);
  }
  TLK_DEV void deposit_chunk(const uint2 (&u)[8], float* buf, int lane) const {
    const int rsub = lane >> 3, c4 = (lane & 7) * 4;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float* x = buf + (4 * k + rsub) * 33 + c4;
      x[0] = __uint_as_float(u[k].x << 16);
      x[1] = __uint_as_float(u[k].x & 0xffff0000u);
      x[2] = __uint_as_float(u[k].y << 16);
      x[3] = __uint_as_float(u[k].y & 0xffff0000u);
    }
    __syncwarp();
  }
  TLK_DEV void store_chunk(uint16_t* p, int64_t step, int row0, const float* buf, int lane) const {
    const int rsub = lane >> 3, c4 = (lane & 7) * 4;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = 4 * k + rsub;
      if (row0 + r >= e.rows) continue;
      const float* x = buf + r * 33 + c4;
      *reinterpret_cast<uint2*>(p + k * step) = make_uint2(pack_bf2(x[0], x[1]), pack_bf2(x[2], x[3]));
    }
    __syncwarp();
  }

  // Causal rows skip the 32-column chunks that lie entirely above the
  // diagonal for the whole warp: those entries of P / dS are never written
  // and stay zero from the pack's initial memset (nothing else writes them).
  // Row-epilogue tiles span all columns (n0 == 0, BN >= cols).  With NP = 2
  // column parts, two warps share each TMEM lane quarter: part p takes
  // columns [p BN/2, (p+1) BN/2); the row max / sum / target logit of the
  // two parts are exchanged through `xchg` ([3][2][128] floats of this
  // accumulator's group, named barrier `bar` over the group's 8 warps) and
  // combined in part order.
  template <int BN, int NP>
  TLK_DEV void row_tile(const ZWork& w, uint32_t taddr, int row0, float* buf, int lane, int part, float* xchg,
                        int bar) const {
    const int m = row0 + lane, rl = row0 - w.m0 + lane;
    const bool live = m < e.rows;
    const int ncols = e.cols;
    const int lim = e.causal ? min(ncols, m + 1) : ncols;       // valid columns of this row
    const int wlim = e.causal ? min(ncols, row0 + 32) : ncols;  // warp-uniform chunk bound
    const int cbeg = part * (BN / NP), cend = min(cbeg + BN / NP, wlim);
    const int rsub = lane >> 3, c4 = (lane & 7) * 4;
    const int64_t step = 4 * e.ld;
    // combine a per-part row value with the other part's: op(part0, part1)
    auto combine = [&](int slot, float v, auto op) -> float {
      if constexpr (NP == 1) {
        return v;
      } else {
        xchg[(slot * 2 + part) * 128 + rl] = v;
        named_bar_sync(bar, 256);
        const float o = xchg[(slot * 2 + (1 - part)) * 128 + rl];
        return part == 0 ? op(v, o) : op(o, v);
      }
    };
    auto fmax_ = [](float x, float y) { return fmaxf(x, y); };
    auto fadd_ = [](float x, float y) { return x + y; };
    float v[32];
    if (e.kind == EPI_SOFTMAX) {
      // p = 2^(v*k - mx*k), k = scale * log2(e), on the SFU (ex2.approx, ~2
      // ulp; P is stored as bf16).  Only the chunk holding the causal
      // diagonal (or the ragged last chunk) needs per-element bounds checks.
      const float k2 = e.scale * 1.4426950408889634f;
      const int cfull = e.causal ? row0 : (ncols & ~31);  // chunks below cfull are whole for every lane
      float mx = -INFINITY;
      for (int c0 = cbeg; c0 < cend; c0 += 32) {
        tmem_ld32(taddr + c0, v);
        if (c0 < cfull) {
#pragma unroll
          for (int i = 0; i < 32; ++i) mx = fmaxf(mx, v[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c0 + i < lim) mx = fmaxf(mx, v[i]);
        }
      }
      mx = combine(0, mx, fmax_);
      const float mk = mx * k2;
      float s = 0.f;
      for (int c0 = cbeg; c0 < cend; c0 += 32) {
        tmem_ld32(taddr + c0, v);
        if (c0 < cfull) {
#pragma unroll
          for (int i = 0; i < 32; ++i) s += ex2_approx(fmaf(v[i], k2, -mk));
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c0 + i < lim) s += ex2_approx(fmaf(v[i], k2, -mk));
        }
      }
      s = combine(1, s, fadd_);
      const float inv = 1.f / s;
      uint16_t* out = static_cast<uint16_t*>(e.out) + off(w, row0 + rsub, c4);
      for (int c0 = cbeg; c0 < cend; c0 += 32) {
        tmem_ld32(taddr + c0, v);
        if (c0 < cfull) {
#pragma unroll
          for (int i = 0; i < 32; ++i) buf[lane * 33 + i] = ex2_approx(fmaf(v[i], k2, -mk)) * inv;
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            buf[lane * 33 + i] = (c0 + i < lim) ? ex2_approx(fmaf(v[i], k2, -mk)) * inv : 0.f;
        }
        store_chunk(out + c0, step, row0, buf, lane);
      }
    } else if (e.kind == EPI_SOFTMAX_BWD) {
      // one pass: dS = P (dP - D) scale; the next chunk's P rows are fetched
      // before this chunk is processed (two chunks of loads in flight)
      const float D = live ? e.rowvec[w.j * e.rv_ls + w.zb * e.rv_bs + w.zh * e.rv_hs + m] : 0.f;
      const uint16_t* P = static_cast<const uint16_t*>(e.aux) + off(w, row0 + rsub, c4);
      uint16_t* out = static_cast<uint16_t*>(e.out) + off(w, row0 + rsub, c4);
      uint2 nxt[8];
      if (cbeg < cend) fetch_chunk(P + cbeg, step, row0, nxt, lane);
      for (int c0 = cbeg; c0 < cend; c0 += 32) {
        uint2 cur[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) cur[k] = nxt[k];
        if (c0 + 32 < cend) fetch_chunk(P + c0 + 32, step, row0, nxt, lane);
        deposit_chunk(cur, buf, lane);
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) buf[lane * 33 + i] = buf[lane * 33 + i] * (v[i] - D) * e.scale;
        store_chunk(out + c0, step, row0, buf, lane);
      }
    } else if (e.kind == EPI_CE) {
      const int y = live ? e.targets[w.j * e.tg_ls + m] : 0;
      const int ce = min(cbeg + BN / NP, BN);
      float mx = -INFINITY, ly = 0.f;
      for (int c0 = cbeg; c0 < ce; c0 += 32) {
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < ncols) {
            mx = fmaxf(mx, v[i]);
            if (c0 + i == y) ly = v[i];
          }
      }
      mx = combine(0, mx, fmax_);
      ly = combine(2, ly, fadd_);  // exactly one part holds the target logit
      float s = 0.f;
      for (int c0 = cbeg; c0 < ce; c0 += 32) {
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < ncols) s += exp_fast(v[i] - mx);
      }
      s = combine(1, s, fadd_);
      if (live && part == 0) e.lossrow[w.j * int64_t(e.rows) + m] = (mx + logf(s)) - ly;
      // dlogits over the padded width e.ld (zeros in the padding columns)
      const float inv = 1.f / s, invt = 1.f / e.tokens;
      uint16_t* out = static_cast<uint16_t*>(e.out) + off(w, row0 + rsub, c4);
      for (int c0 = cbeg; c0 < ce && c0 < e.ld; c0 += 32) {
        tmem_ld32(taddr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          buf[lane * 33 + i] =
              (c0 + i < ncols) ? (exp_fast(v[i] - mx) * inv - (c0 + i == y ? 1.f : 0.f)) * invt : 0.f;
        store_chunk(out + c0, step, row0, buf, lane);
      }
    }
    if constexpr (NP > 1) named_bar_sync(bar, 256);  // exchange slots reusable by the group's next tile
  }

  template <int BN, int NP = 1>
  TLK_DEV void tile(const ZWork& w, uint32_t tq, int row0, float* buf, int lane, bool row, int part = 0) const {
    if (row) {
      row_tile<BN, 1>(w, tq, row0, buf, lane, 0, nullptr, 0);
      return;
    }
    switch (e.kind) {
      case EPI_BF16: tile4<EPI_BF16, BN, NP>(w, tq, row0, buf, lane, part); break;
      case EPI_BF16_GELU: tile4<EPI_BF16_GELU, BN, NP>(w, tq, row0, buf, lane, part); break;
      case EPI_F32: tile4<EPI_F32, BN, NP>(w, tq, row0, buf, lane, part); break;
      case EPI_RESADD: tile4<EPI_RESADD, BN, NP>(w, tq, row0, buf, lane, part); break;
      case EPI_GELU_BWD: tile4<EPI_GELU_BWD, BN, NP>(w, tq, row0, buf, lane, part); break;
      default: break;
    }
  }
};

}  // namespace tlk
