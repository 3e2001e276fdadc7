// Transformer packs (TLK_MODEL_XFORMER: config 4's 2-layer d=256 model;
// TLK_MODEL_GPT: config 5's tiny-GPT), all lanes per launch.  Restated by
// oracle/gpt.py (see its docstring for the model and the numerics contract).
//
// Per layer forward:  LN1 -> QKV (tcgen05, +bias, bf16) -> S = QK^T per
// (sequence, head) with a softmax row epilogue (scale, causal mask) -> Y = PV
// -> proj (+bias, residual add, fp32) -> LN2 -> FC (+bias, GELU; z kept fp32)
// -> FC2 (+bias, residual add).  Head: LNf -> logits with a cross-entropy row
// epilogue (per-token loss + bf16 dlogits) -> fixed-order loss reduction.
// Backward mirrors it: weight gradients are tcgen05 GEMMs with K = tokens
// (both operands MN-major), dgrads read the weights MN-major (no transposed
// copies), dP gets a softmax-backward row epilogue, LN backward and every
// bias / gain / embedding gradient are deterministic two-stage reductions.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "pack.cuh"
#include "rng.cuh"
#include "sgemm.cuh"
#include "tgemm.cuh"
#include "attn.cuh"

namespace tlk {

constexpr uint32_t STREAM_TOKENS = 3;
__constant__ int kMarkovA[8] = {1, 3, 5, 7, 11, 13, 17, 19};
__constant__ int kMarkovC[8] = {1, 2, 3, 5, 8, 13, 21, 34};

namespace {

struct LayerBufs {
  float *xin, *xmid, *st1, *st2;
  uint16_t* z;  // bf16 GELU pre-activation (the GELU backward evaluates at bf16(z))
  uint16_t *a, *qkv, *P, *y, *m, *f;
  float* stats;  // fused attention: per-query (max * k2, 1 / sum) softmax statistics
};

struct GptBufs {
  GptCfg c;
  int N, Vp, sms;
  unsigned long long* atrace = nullptr;  // TLK_ATTN_TRACE=1: [fwd, bwd][64 tiles][32] event clocks
  bool fused_attn;  // attn.cuh kernels (T = 128 / 256) instead of the P / dS GEMM chain
  int32_t *tokens, *targets;
  std::vector<LayerBufs> L;
  float *xL, *stf, *lossrow;
  uint16_t *xf, *dl;
  // backward scratch (shared by all layers)
  float *dx, *dmm, *D;  // D: softmax-backward row terms [lane][b][h][t]
  uint16_t *dxb, *dz, *dy, *dS, *dqkv;
  float* part;      // reduction partials
  int64_t part_st;  // floats per lane
  // parameter offsets
  std::vector<int64_t> off;  // by tensor index
};

int64_t tensor_off(const Pack& p, int t) { return p.tinfo[t].off; }

// tensor indices (oracle/gpt.py::tensors order)
enum { T_WTE = 0, T_WPE = 1 };
inline int T_LAYER(int l, int k) { return 2 + 12 * l + k; }
enum { K_LN1G, K_LN1B, K_AW, K_AB, K_PW, K_PB, K_LN2G, K_LN2B, K_FW, K_FB, K_F2W, K_F2B };
inline int T_LNFG(const GptCfg& c) { return 2 + 12 * c.layers; }

// ------------------------------------------------------------- tokens -------
__global__ void gpt_tokens_kernel(const LaneState* __restrict__ lanes, int B, int T, int V,
                                  int32_t* __restrict__ tokens, int32_t* __restrict__ targets) {
  pdl_begin();
  const int s = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (s >= B || !lanes[j].active) return;
  const uint64_t key = rng_key(lanes[j].seed, STREAM_TOKENS, uint64_t(lanes[j].steps_done));
  const uint64_t base = uint64_t(s) * (T + 1);
  int32_t* tk = tokens + (int64_t(j) * B + s) * (T + 1);
  int32_t* tg = targets + (int64_t(j) * B + s) * T;
  int t = int(rng_bits(key, base) % uint64_t(V));
  tk[0] = t;
  for (int i = 0; i < T; ++i) {
    const int k = int(rng_bits(key, base + i + 1) >> 61);
    t = (t * kMarkovA[k] + kMarkovC[k]) % V;
    tk[i + 1] = t;
    tg[i] = t;
  }
}

// host-input packs: the tokens came from the host (tlk_step_host_blob);
// targets are the tokens shifted by one
__global__ void gpt_targets_kernel(const LaneState* __restrict__ lanes, int B, int T,
                                   const int32_t* __restrict__ tokens, int32_t* __restrict__ targets) {
  pdl_begin();
  const int s = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (s >= B || !lanes[j].active) return;
  const int32_t* tk = tokens + (int64_t(j) * B + s) * (T + 1);
  int32_t* tg = targets + (int64_t(j) * B + s) * T;
  for (int i = 0; i < T; ++i) tg[i] = tk[i + 1];
}

// x0[row][c] = wte[tok][c] + wpe[t][c]: one warp per row, 8 rows per CTA,
// float4 columns when the arena offsets allow it (`vec`)
__global__ void __launch_bounds__(256) gpt_embed_kernel(const LaneState* __restrict__ lanes, GptCfg c, int B,
                                                        const int32_t* __restrict__ tokens,
                                                        const float* __restrict__ params, int64_t pstride,
                                                        int64_t o_wte, int64_t o_wpe, float* __restrict__ x,
                                                        int vec) {
  pdl_begin();
  const int j = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (!lanes[j].active) return;
  const int row = blockIdx.x * 8 + warp;
  if (row >= B * c.T) return;
  const int b = row / c.T, t = row % c.T;
  const int tok = tokens[(int64_t(j) * B + b) * (c.T + 1) + t];
  const float* P = params + j * pstride;
  const float* we = P + o_wte + int64_t(tok) * c.d;
  const float* pe = P + o_wpe + int64_t(t) * c.d;
  float* xr = x + (int64_t(j) * B * c.T + row) * c.d;
  if (vec) {
    for (int i = lane; i < c.d / 4; i += 32) {
      const float4 u = reinterpret_cast<const float4*>(we)[i], v = reinterpret_cast<const float4*>(pe)[i];
      reinterpret_cast<float4*>(xr)[i] = make_float4(u.x + v.x, u.y + v.y, u.z + v.z, u.w + v.w);
    }
  } else {
    for (int i = lane; i < c.d; i += 32) xr[i] = we[i] + pe[i];
  }
}

// ------------------------------------------------------------- LayerNorm ----
// one warp per row: y = bf16((x - mean) * rstd * g + b); stats = (mean, rstd)
__global__ void __launch_bounds__(256) ln_fwd_kernel(const LaneState* __restrict__ lanes, int N,
                                                     int d, const float* __restrict__ x,
                                                     const float* __restrict__ params,
                                                     int64_t pstride, int64_t og, int64_t ob,
                                                     uint16_t* __restrict__ y,
                                                     float* __restrict__ stats) {
  pdl_begin();
  const int j = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (!lanes[j].active) return;
  const int row = blockIdx.x * 8 + warp;
  if (row >= N) return;
  const float* xr = x + (int64_t(j) * N + row) * d;
  float s = 0.f;
  for (int i = lane; i < d; i += 32) s += xr[i];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mu = s / float(d);
  float q = 0.f;
  for (int i = lane; i < d; i += 32) {
    const float c = xr[i] - mu;
    q += c * c;
  }
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rstd = 1.0f / sqrtf(q / float(d) + 1e-5f);
  const float* g = params + j * pstride + og;
  const float* bb = params + j * pstride + ob;
  uint16_t* yr = y + (int64_t(j) * N + row) * d;
  for (int i = lane; i < d; i += 32) yr[i] = f2bf((xr[i] - mu) * rstd * g[i] + bb[i]);
  if (lane == 0) {
    stats[(int64_t(j) * N + row) * 2] = mu;
    stats[(int64_t(j) * N + row) * 2 + 1] = rstd;
  }
}

// Vector LayerNorm forward (d = 128 KV): lane l owns the float4 columns
// 4 (l + 32 k); a warp normalises LNF_WROWS consecutive rows with the next
// row's loads in flight, gain / bias held in registers, packed bf16 stores.
constexpr int LNF_WROWS = 8;
template <int KV>
__global__ void __launch_bounds__(256) ln_fwd_vec_kernel(const LaneState* __restrict__ lanes, int N,
                                                         const float* __restrict__ x,
                                                         const float* __restrict__ params, int64_t pstride,
                                                         int64_t og, int64_t ob, uint16_t* __restrict__ y,
                                                         float* __restrict__ stats) {
  pdl_begin();
  constexpr int d = 128 * KV;
  const int j = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (!lanes[j].active) return;
  const int row0 = (blockIdx.x * 8 + warp) * LNF_WROWS;
  const int nrows = max(0, min(LNF_WROWS, N - row0));
  if (nrows == 0) return;
  float4 g[KV], bb[KV], cur[KV], nxt[KV];
  const float* gp = params + j * pstride + og;
  const float* bp = params + j * pstride + ob;
  const float* xr = x + (int64_t(j) * N + row0) * d;
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    const int i = 4 * (lane + 32 * k);
    g[k] = *reinterpret_cast<const float4*>(gp + i);
    bb[k] = *reinterpret_cast<const float4*>(bp + i);
    cur[k] = *reinterpret_cast<const float4*>(xr + i);
  }
  for (int r = 0; r < nrows; ++r) {
    if (r + 1 < nrows)
#pragma unroll
      for (int k = 0; k < KV; ++k) nxt[k] = *reinterpret_cast<const float4*>(xr + (r + 1) * d + 4 * (lane + 32 * k));
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < KV; ++k) s += (cur[k].x + cur[k].y) + (cur[k].z + cur[k].w);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mu = s / float(d);
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const float c0 = cur[k].x - mu, c1 = cur[k].y - mu, c2 = cur[k].z - mu, c3 = cur[k].w - mu;
      q += (c0 * c0 + c1 * c1) + (c2 * c2 + c3 * c3);
    }
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float rstd = 1.0f / sqrtf(q / float(d) + 1e-5f);
    uint16_t* yr = y + (int64_t(j) * N + row0 + r) * d;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const float4 v = cur[k];
      *reinterpret_cast<uint2*>(yr + 4 * (lane + 32 * k)) =
          make_uint2(pack_bf2((v.x - mu) * rstd * g[k].x + bb[k].x, (v.y - mu) * rstd * g[k].y + bb[k].y),
                     pack_bf2((v.z - mu) * rstd * g[k].z + bb[k].z, (v.w - mu) * rstd * g[k].w + bb[k].w));
    }
    if (lane == 0)
      *reinterpret_cast<float2*>(stats + (int64_t(j) * N + row0 + r) * 2) = make_float2(mu, rstd);
#pragma unroll
    for (int k = 0; k < KV; ++k) cur[k] = nxt[k];
  }
}

// LayerNorm backward for 64 rows per CTA (8 warps x 8 rows):
//   dxh = dy g; dx = (dxh - mean(dxh) - xh mean(dxh xh)) rstd
//   dxt (fp32 residual grad) = (accumulate ? dxt : 0) + dx; dxb = bf16(dxt)
//   part[lane][blk][0:d] = sum_rows dy xh, part[..][d:2d] = sum_rows dy (fixed order)
// Lane l of a warp owns the float4 columns 4*(l + 32k), k < KV (d = 128 KV);
// the next row's x / dy / dxt are fetched before the current row is reduced,
// so every warp keeps two rows of loads in flight.
// LNB_WARPS warps of LNB_WROWS rows per CTA.  KV = 3 needs ~150 registers
// unconstrained (one CTA, 8 warps of loads per SM); capped at 128 (two CTAs
// per SM, a few spilled values in L1) it runs 10% faster.
#ifndef TLK_LNB_WARPS
#define TLK_LNB_WARPS 8
#endif
constexpr int LNB_WARPS = TLK_LNB_WARPS, LNB_WROWS = 8, LNB_ROWS = LNB_WARPS * LNB_WROWS;
template <int KV>
struct LnRow {
  float4 x[KV], dy[KV], acc[KV];
  float mu, rstd;
};
template <int KV>
TLK_DEV void ln_row_load(LnRow<KV>& r, const float* x, const float* dy, const float* dxt, const float* stats,
                         int64_t ro, int64_t so, int lane, bool acc) {
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    const int i = 4 * (lane + 32 * k);
    r.x[k] = *reinterpret_cast<const float4*>(x + ro + i);
    r.dy[k] = *reinterpret_cast<const float4*>(dy + ro + i);
    r.acc[k] = acc ? *reinterpret_cast<const float4*>(dxt + ro + i) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  r.mu = stats[so];
  r.rstd = stats[so + 1];
}
template <int KV>
__global__ void __launch_bounds__(LNB_WARPS * 32, KV <= 3 ? 2 : 1) ln_bwd_kernel(
    const LaneState* __restrict__ lanes, int N, const float* __restrict__ dy,
    const float* __restrict__ x, const float* __restrict__ stats, const float* __restrict__ params,
    int64_t pstride, int64_t og, float* __restrict__ dxt, uint16_t* __restrict__ dxb, int accumulate,
    float* __restrict__ part, int64_t part_st) {
  pdl_begin();
  constexpr int d = 128 * KV;
  const int j = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (!lanes[j].active) return;
  extern __shared__ float red[];  // [LNB_WARPS][3][d]
  // ag / ab: dgamma / dbeta partials; ax: column sums of the stored bf16 dx
  // (the bias gradient of the GEMM that consumes dxb next)
  float4 g[KV], ag[KV], ab[KV], ax[KV];
  const float* gp = params + j * pstride + og;
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    const int i = 4 * (lane + 32 * k);
    g[k] = make_float4(gp[i], gp[i + 1], gp[i + 2], gp[i + 3]);
    ag[k] = ab[k] = ax[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int row0 = blockIdx.x * LNB_ROWS + warp * LNB_WROWS;
  const int nrows = max(0, min(LNB_WROWS, N - row0));
  LnRow<KV> cur, nxt;
  if (nrows > 0)
    ln_row_load(cur, x, dy, dxt, stats, (int64_t(j) * N + row0) * d, (int64_t(j) * N + row0) * 2, lane,
                accumulate);
  for (int r = 0; r < nrows; ++r) {
    const int row = row0 + r;
    const int64_t ro = (int64_t(j) * N + row) * d;
    if (r + 1 < nrows)
      ln_row_load(nxt, x, dy, dxt, stats, ro + d, (int64_t(j) * N + row + 1) * 2, lane, accumulate);
    float4 xh[KV];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      xh[k] = make_float4((cur.x[k].x - cur.mu) * cur.rstd, (cur.x[k].y - cur.mu) * cur.rstd,
                          (cur.x[k].z - cur.mu) * cur.rstd, (cur.x[k].w - cur.mu) * cur.rstd);
      const float4 dv = cur.dy[k];
      const float h0 = dv.x * g[k].x, h1 = dv.y * g[k].y, h2 = dv.z * g[k].z, h3 = dv.w * g[k].w;
      s1 += h0 + h1 + h2 + h3;
      s2 += h0 * xh[k].x + h1 * xh[k].y + h2 * xh[k].z + h3 * xh[k].w;
      ag[k].x += dv.x * xh[k].x;
      ag[k].y += dv.y * xh[k].y;
      ag[k].z += dv.z * xh[k].z;
      ag[k].w += dv.w * xh[k].w;
      ab[k].x += dv.x;
      ab[k].y += dv.y;
      ab[k].z += dv.z;
      ab[k].w += dv.w;
    }
    for (int o = 16; o; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    const float m1 = s1 / float(d), m2 = s2 / float(d);
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int i = 4 * (lane + 32 * k);
      const float4 dv = cur.dy[k], a = cur.acc[k];
      const float t0 = a.x + (dv.x * g[k].x - m1 - xh[k].x * m2) * cur.rstd;
      const float t1 = a.y + (dv.y * g[k].y - m1 - xh[k].y * m2) * cur.rstd;
      const float t2 = a.z + (dv.z * g[k].z - m1 - xh[k].z * m2) * cur.rstd;
      const float t3 = a.w + (dv.w * g[k].w - m1 - xh[k].w * m2) * cur.rstd;
      *reinterpret_cast<float4*>(dxt + ro + i) = make_float4(t0, t1, t2, t3);
      const uint32_t lo = pack_bf2(t0, t1), hi = pack_bf2(t2, t3);
      *reinterpret_cast<uint2*>(dxb + ro + i) = make_uint2(lo, hi);
      ax[k].x += __uint_as_float(lo << 16);
      ax[k].y += __uint_as_float(lo & 0xffff0000u);
      ax[k].z += __uint_as_float(hi << 16);
      ax[k].w += __uint_as_float(hi & 0xffff0000u);
    }
    cur = nxt;
  }
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    const int i = 4 * (lane + 32 * k);
    *reinterpret_cast<float4*>(red + (warp * 3) * d + i) = ag[k];
    *reinterpret_cast<float4*>(red + (warp * 3 + 1) * d + i) = ab[k];
    *reinterpret_cast<float4*>(red + (warp * 3 + 2) * d + i) = ax[k];
  }
  __syncthreads();
  float* out = part + j * part_st + int64_t(blockIdx.x) * 3 * d;
  for (int i = threadIdx.x; i < 3 * d; i += blockDim.x) {
    const int f = i / d, c = i % d;
    float s = 0.f;
    for (int w = 0; w < LNB_WARPS; ++w) s += red[(w * 3 + f) * d + c];
    out[i] = s;
  }
}

// D[lane][b][h][t] = sum_c dY[t][h*64 + c] Y[t][h*64 + c] (bf16 inputs, fp32,
// c in order): the softmax-backward row term rowsum(P o dP) via the identity
// rowsum(P o dP) = rowsum(dY o Y).  One thread per (token, head).
__global__ void attn_rowdot_kernel(const LaneState* __restrict__ lanes, int N, int T, int H,
                                   const uint16_t* __restrict__ dy, const uint16_t* __restrict__ y,
                                   float* __restrict__ D) {
  pdl_begin();
  const int j = blockIdx.y;
  if (!lanes[j].active) return;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // token * H + h
  if (idx >= N * H) return;
  const int n = idx / H, h = idx % H, d = H * 64;
  const int64_t o = (int64_t(j) * N + n) * d + h * 64;
  const uint4* a = reinterpret_cast<const uint4*>(dy + o);
  const uint4* b = reinterpret_cast<const uint4*>(y + o);
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint4 u = a[q], v = b[q];
    const uint32_t uu[4] = {u.x, u.y, u.z, u.w}, vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      s += __uint_as_float(uu[e] << 16) * __uint_as_float(vv[e] << 16);
      s += __uint_as_float(uu[e] & 0xffff0000u) * __uint_as_float(vv[e] & 0xffff0000u);
    }
  }
  const int bi = n / T, t = n % T;
  D[((int64_t(j) * (N / T) + bi) * H + h) * T + t] = s;
}

// ------------------------------------------------------------- reductions --
// dst0[c] (c < split) / dst1[c - split] = sum_blk part[lane][blk][c], fixed order
__global__ void reduce_parts_kernel(const LaneState* __restrict__ lanes, const float* __restrict__ part,
                                    int64_t part_st, int nblk, int C, float* __restrict__ grads,
                                    int64_t pstride, int64_t off0, int split, int64_t off1, int split2,
                                    int64_t off2) {
  pdl_begin();
  const int c = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (!lanes[j].active || c >= C) return;
  if (c >= split2 && off2 < 0) return;  // third partial set without a target
  const float* p = part + j * part_st + c;
  float s = 0.f;
  for (int b = 0; b < nblk; ++b) s += p[int64_t(b) * C];
  grads[j * pstride + (c < split ? off0 + c : c < split2 ? off1 + (c - split) : off2 + (c - split2))] = s;
}

// Same sum over many partial rows: 8 row groups per 32 columns (group g
// takes rows g, g + 8, ... in order; groups combined in order).
__global__ void __launch_bounds__(256) reduce_parts8_kernel(const LaneState* __restrict__ lanes,
                                                            const float* __restrict__ part, int64_t part_st, int nblk,
                                                            int C, float* __restrict__ grads, int64_t pstride,
                                                            int64_t off) {
  pdl_begin();
  const int cl = threadIdx.x & 31, g = threadIdx.x >> 5, c = blockIdx.x * 32 + cl, j = blockIdx.y;
  if (!lanes[j].active) return;
  __shared__ float sh[8][32];
  float s = 0.f;
  if (c < C) {
    const float* p = part + j * part_st + c;
#pragma unroll 4
    for (int b = g; b < nblk; b += 8) s += p[int64_t(b) * C];
  }
  sh[g][cl] = s;
  __syncthreads();
  if (g == 0 && c < C) {
    float t = sh[0][cl];
    for (int k = 1; k < 8; ++k) t += sh[k][cl];
    grads[j * pstride + off + c] = t;
  }
}

// mean token loss (fixed order) -> loss curve; per-step optimizer scalars
__global__ void __launch_bounds__(512) gpt_loss_kernel(LaneState* __restrict__ lanes, int N,
                                                       const float* __restrict__ lossrow,
                                                       float* __restrict__ loss, int max_steps,
                                                       float* __restrict__ last_loss) {
  pdl_begin();
  const int j = blockIdx.x, tid = threadIdx.x;
  if (!lanes[j].active) return;
  __shared__ float red[512];
  const int per = (N + 511) / 512;
  float s = 0.f;
  for (int r = tid * per; r < min(N, (tid + 1) * per); ++r) s += lossrow[int64_t(j) * N + r];
  red[tid] = s;
  __syncthreads();
  if (tid == 0) {
    float t = 0.f;
    for (int i = 0; i < 512; ++i) t += red[i];
    const float Lm = t / float(N);
    LaneState& ls = lanes[j];
    loss[int64_t(j) * max_steps + ls.steps_done] = Lm;
    last_loss[j] = Lm;
    lane_step_scalars(ls);
  }
}

// Token-embedding gradient for a small vocabulary (V x d fp32 fits shared
// memory): CTA (row chunk, lane) streams its rows of dx once, thread c owns
// float4 column c of every vocabulary row, acc[token][c] += dx[row][c] in row
// order (the next EMT_U rows in flight while a batch is added), and writes
// part[lane][chunk][v][c] (one wave of CTAs: two per SM);
// reduce_parts8 sums the chunks in fixed order.  Every dx row is read once at
// full width (the vocabulary-block kernel below rescans the token list per
// block and keeps only a few loads in flight).
constexpr int EMT_U = 8;
constexpr size_t EMT_SMEM_MAX = 112 * 1024;  // two CTAs per SM
__global__ void __launch_bounds__(128) embed_bwd_tok_kernel(const LaneState* __restrict__ lanes, int N, int d, int V,
                                                            const int32_t* __restrict__ tokens, int T,
                                                            const float* __restrict__ dx, float* __restrict__ part,
                                                            int64_t part_st, int rows_per) {
  pdl_begin();
  extern __shared__ float4 acc4[];  // [V][d / 4]
  const int j = blockIdx.y, tid = threadIdx.x, d4 = d >> 2;
  if (!lanes[j].active) return;
  for (int i = tid; i < V * d4; i += blockDim.x) acc4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  const int r0 = blockIdx.x * rows_per, r1 = min(N, r0 + rows_per);
  if (tid < d4) {
    const float4* g = reinterpret_cast<const float4*>(dx + int64_t(j) * N * d) + tid;
    const int32_t* tk = tokens + int64_t(j) * (N / T) * (T + 1);
    auto tok = [&](int row) { return tk[(row / T) * (T + 1) + row % T]; };
    auto add = [&](int v, const float4& x) {
      if (unsigned(v) < unsigned(V)) {
        float4& a = acc4[v * d4 + tid];
        a.x += x.x, a.y += x.y, a.z += x.z, a.w += x.w;
      }
    };
    // software pipeline: the next EMT_U rows are loaded while this batch is added
    float4 val[EMT_U], nval[EMT_U];
    int v[EMT_U], nv[EMT_U];
    int r = r0;
    const bool full0 = r + EMT_U <= r1;
    if (full0)
#pragma unroll
      for (int u = 0; u < EMT_U; ++u) v[u] = tok(r + u), val[u] = g[int64_t(r + u) * d4];
    while (full0 && r + EMT_U <= r1) {
      const bool more = r + 2 * EMT_U <= r1;
      if (more)
#pragma unroll
        for (int u = 0; u < EMT_U; ++u) nv[u] = tok(r + EMT_U + u), nval[u] = g[int64_t(r + EMT_U + u) * d4];
#pragma unroll
      for (int u = 0; u < EMT_U; ++u) add(v[u], val[u]);
      r += EMT_U;
      if (!more) break;
#pragma unroll
      for (int u = 0; u < EMT_U; ++u) v[u] = nv[u], val[u] = nval[u];
    }
    for (; r < r1; ++r) add(tok(r), g[int64_t(r) * d4]);
    float4* out = reinterpret_cast<float4*>(part + j * part_st + int64_t(blockIdx.x) * V * d) + tid;
    for (int w = 0; w < V; ++w) out[int64_t(w) * d4] = acc4[w * d4 + tid];
  }
}

// Token-embedding gradient by vocabulary row: CTA (vocab block of EMV rows,
// column slice) scans the lane's input tokens in order, compacts the rows
// whose token falls in its block (block-wide scan -> token order), and
// thread c accumulates dx[row][c] into its rows' sums in that order.  Every
// dx row is read once, nothing is staged through partials, and the sums are
// per vocabulary row in token order (deterministic).
constexpr int EMV = 16, EMV_COLS = 128, EMV_CHUNK = 1024;
__global__ void __launch_bounds__(EMV_COLS) embed_bwd_vocab_kernel(const LaneState* __restrict__ lanes, int N, int d,
                                                                   int V, const int32_t* __restrict__ tokens, int T,
                                                                   const float* __restrict__ dx,
                                                                   float* __restrict__ grads, int64_t pstride,
                                                                   int64_t o_wte) {
  pdl_begin();
  const int v0 = blockIdx.x * EMV, c = blockIdx.y * EMV_COLS + threadIdx.x, j = blockIdx.z, tid = threadIdx.x;
  if (!lanes[j].active) return;
  __shared__ float acc[EMV][EMV_COLS];
  __shared__ int list[EMV_CHUNK];
  __shared__ int cnt[EMV_COLS + 1];
  for (int v = 0; v < EMV; ++v) acc[v][tid] = 0.f;
  constexpr int PER = EMV_CHUNK / EMV_COLS;  // tokens checked per thread per chunk
  for (int r0 = 0; r0 < N; r0 += EMV_CHUNK) {
    int mine[PER], m = 0;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int row = r0 + tid * PER + u;
      int v = -1;
      if (row < N) {
        const int b = row / T, t = row % T;
        v = tokens[(int64_t(j) * (N / T) + b) * (T + 1) + t] - v0;
      }
      mine[u] = (v >= 0 && v < EMV) ? (row << 4) | v : -1;
      m += mine[u] >= 0;
    }
    __syncthreads();  // previous chunk's list fully consumed
    cnt[tid + 1] = m;
    if (tid == 0) cnt[0] = 0;
    __syncthreads();
    if (tid == 0)
      for (int k = 1; k <= EMV_COLS; ++k) cnt[k] += cnt[k - 1];  // exclusive offsets, thread order = token order
    __syncthreads();
    int pos = cnt[tid];
#pragma unroll
    for (int u = 0; u < PER; ++u)
      if (mine[u] >= 0) list[pos++] = mine[u];
    __syncthreads();
    const int total = cnt[EMV_COLS];
    if (c < d) {
      const float* g = dx + int64_t(j) * N * d + c;
      int k = 0;
      for (; k + 4 <= total; k += 4) {  // four rows in flight, added in list order
        float val[4];
        int vv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int e = list[k + q];
          vv[q] = e & 15;
          val[q] = g[int64_t(e >> 4) * d];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[vv[q]][tid] += val[q];
      }
      for (; k < total; ++k) {
        const int e = list[k];
        acc[e & 15][tid] += g[int64_t(e >> 4) * d];
      }
    }
  }
  if (c < d)
    for (int v = 0; v < EMV && v0 + v < V; ++v) grads[j * pstride + o_wte + int64_t(v0 + v) * d + c] = acc[v][tid];
}

// dwpe[t][c] = sum_b dx[b*T + t][c] (b in order)
__global__ void wpe_bwd_kernel(const LaneState* __restrict__ lanes, int B, int T, int d,
                               const float* __restrict__ dx, float* __restrict__ grads,
                               int64_t pstride, int64_t o_wpe) {
  pdl_begin();
  const int t = blockIdx.x, j = blockIdx.y;
  if (!lanes[j].active) return;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < B; ++b) s += dx[(int64_t(j) * B * T + int64_t(b) * T + t) * d + c];
    grads[j * pstride + o_wpe + int64_t(t) * d + c] = s;
  }
}

// ------------------------------------------------------------- GEMM glue ---
Operand op(const uint16_t* base, int64_t ls, int64_t bs, int64_t hs, int64_t mn_st, int64_t k_st,
           int MN, int K) {
  return Operand{base, ls, bs, hs, mn_st, k_st, MN, K};
}

// Tensor maps of a dense epilogue's outputs / aux operand ({16 columns, 32
// rows} boxes, SW32 for bf16 rows, SW64 for fp32 rows; dims {cols, rows, h,
// b, lane} over the Epi strides).  `on` stays 0 (per-element tile4 path) for
// layouts the TMA tiles cannot express or when TLK_TMA_EPI=0.
bool tma_epi_usable(const Epi& e) {
  static const bool off = getenv("TLK_TMA_EPI") && getenv("TLK_TMA_EPI")[0] == '0';
  const bool dense = e.kind == EPI_BF16 || e.kind == EPI_BF16_GELU || e.kind == EPI_F32 || e.kind == EPI_RESADD ||
                     e.kind == EPI_GELU_BWD || e.kind == EPI_BF16_ROWDOT;
  const bool f32 = e.kind == EPI_F32 || e.kind == EPI_RESADD;
  const int64_t eb = f32 ? 4 : 2;
  auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  return !off && dense && e.cols % 16 == 0 && (e.ld * eb) % 16 == 0 && (e.hs * eb) % 16 == 0 &&
         (e.bs * eb) % 16 == 0 && (e.ls * eb) % 16 == 0 && al(e.out) && (e.kind != EPI_BF16_GELU || al(e.out2)) &&
         (!(e.kind == EPI_GELU_BWD || e.kind == EPI_RESADD || e.kind == EPI_BF16_ROWDOT) || al(e.aux));
}

int tma_epi_maps(CUtensorMap& mo, CUtensorMap& mo2, CUtensorMap& ma, int& on, const Epi& e, int lanes, int nb,
                 int nh) {
  on = 0;
  if (!tma_epi_usable(e)) return TLK_OK;
  const bool f32 = e.kind == EPI_F32 || e.kind == EPI_RESADD;
  auto mk = [&](CUtensorMap& m, const void* base, bool is_f32) {
    const uint64_t eb = is_f32 ? 4 : 2;
    const uint64_t dims[5] = {uint64_t(e.cols), uint64_t(e.rows), uint64_t(nh), uint64_t(nb), uint64_t(lanes)};
    const uint64_t st[4] = {uint64_t(e.ld) * eb, uint64_t(e.hs) * eb, uint64_t(e.bs) * eb, uint64_t(e.ls) * eb};
    return make_tmap_5d(&m, is_f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, base, dims,
                        st, 16, 32, is_f32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  };
  int rc = mk(mo, e.out, f32);
  if (!rc && e.kind == EPI_BF16_GELU) rc = mk(mo2, e.out2, false);
  if (!rc && (e.kind == EPI_GELU_BWD || e.kind == EPI_RESADD || e.kind == EPI_BF16_ROWDOT))
    rc = mk(ma, e.aux, e.kind == EPI_RESADD);
  if (rc) return rc;
  on = 1;
  return TLK_OK;
}

template <int BN, bool AMN, bool BMN, bool ROW, bool LIGHT = false, bool COMPACT = false>
int gemm(const Pack& p, cudaStream_t st, const Operand& A, const Operand& B, const Epi& e, int M,
         int N, int K, int nb, int nh, const char* name) {
  using G = TGemm<BN, AMN, BMN, ROW, LIGHT, COMPACT>;
  G g{};
  g.g = EpiOps{p.lane_dev, e, nb, nh, (K + GEMM_BK - 1) / GEMM_BK};
  // vector-epilogue contract (sgemm.cuh): 4-element aligned rows and z strides
  TLK_CHECK(e.ld % 4 == 0 && e.ls % 4 == 0 && e.bs % 4 == 0 && e.hs % 4 == 0 &&
                (ROW || e.cols % 4 == 0) && (reinterpret_cast<uintptr_t>(e.out) & 15) == 0,
            TLK_EINVAL, "%s: epilogue layout not 4-element aligned", name);
  TLK_CHECK(!ROW || N <= BN, TLK_EINVAL, "%s: row epilogue needs the whole row in one tile", name);
  int rc = make_operand_map(&g.ta, A, AMN, GEMM_BM, p.lanes, nb, nh);
  if (!rc) rc = make_operand_map(&g.tb, B, BMN, BN, p.lanes, nb, nh);
  if (!rc && !ROW) rc = tma_epi_maps(g.to, g.to2, g.tx, g.tma_epi, e, p.lanes, nb, nh);
  if (rc) return rc;
  TLK_CHECK(!COMPACT || g.tma_epi, TLK_EINVAL, "%s: compact epilogue tiles need the TMA epilogue", name);
  g.mt = (M + GEMM_BM - 1) / GEMM_BM;
  g.nt = (N + BN - 1) / BN;
  g.ntiles = g.mt * g.nt * p.lanes * nb * nh;
  const int sms = static_cast<const GptBufs*>(p.scratch)->sms;
  TLK_CUDA(launch_tgemm(g, sms, st));
  const_cast<Pack&>(p).mark(st, name);
  return TLK_OK;
}

// Dense (non-row-epilogue) GEMMs: the widest N tile that divides N (256,
// 192, else 128).  Wider tiles reuse each A (activation) tile across more
// columns: fewer L2 -> SM bytes per MMA (TLK_GEMM_BN128=1 forces 128).
template <bool AMN, bool BMN>
int gemm_auto(const Pack& p, cudaStream_t st, const Operand& A, const Operand& B, const Epi& e, int M, int N, int K,
              int nb, int nh, const char* name) {
  static const bool narrow = getenv("TLK_GEMM_BN128") && getenv("TLK_GEMM_BN128")[0] == '1';
  if constexpr (!(AMN && BMN)) {
    // bf16-output epilogues on the TMA path: 1 KB staging tiles, one more stage
    if ((e.kind == EPI_BF16 || e.kind == EPI_GELU_BWD) && !narrow && tma_epi_usable(e)) {
      if (N % 256 == 0) return gemm<256, AMN, BMN, false, false, true>(p, st, A, B, e, M, N, K, nb, nh, name);
      if (N % 192 == 0) return gemm<192, AMN, BMN, false, false, true>(p, st, A, B, e, M, N, K, nb, nh, name);
    }
    // plain fp32 output (dgrads): one epilogue warp per lane quarter, deeper pipeline
    if (e.kind == EPI_F32 && !narrow) {
      if (N % 256 == 0) return gemm<256, AMN, BMN, false, true>(p, st, A, B, e, M, N, K, nb, nh, name);
      if (N % 192 == 0) return gemm<192, AMN, BMN, false, true>(p, st, A, B, e, M, N, K, nb, nh, name);
    }
  }
  if (!narrow && N % 256 == 0) return gemm<256, AMN, BMN, false>(p, st, A, B, e, M, N, K, nb, nh, name);
  if (!narrow && N % 192 == 0) return gemm<192, AMN, BMN, false>(p, st, A, B, e, M, N, K, nb, nh, name);
  return gemm<128, AMN, BMN, false>(p, st, A, B, e, M, N, K, nb, nh, name);
}

Epi epi(int kind, int rows, int cols, void* out, int64_t ls, int64_t bs, int64_t hs, int64_t ld) {
  Epi e{};
  e.kind = kind;
  e.rows = rows;
  e.cols = cols;
  e.out = out;
  e.ls = ls;
  e.bs = bs;
  e.hs = hs;
  e.ld = ld;
  e.scale = 1.f;
  return e;
}

// ------------------------------------------------------- fused attention --
// Epilogue descriptors shared by the fused and the unfused attention paths.
Epi attn_y_epi(const GptBufs& b, const LayerBufs& lb) {
  const int64_t T = b.c.T, d = b.c.d, nd = int64_t(b.N) * d;
  return epi(EPI_BF16, int(T), 64, lb.y, nd, T * d, 64, d);
}
Epi attn_dqkv_epi(const GptBufs& b, int which) {  // 0 dq, 1 dk, 2 dv
  const int64_t T = b.c.T, d = b.c.d, nd3 = int64_t(b.N) * 3 * d;
  Epi e = epi(EPI_BF16, int(T), 64, b.dqkv + which * d, nd3, T * 3 * d, 64, 3 * d);
  e.colpart = b.part;  // qkv.b gradient partials
  e.cp_ls = b.part_st;
  e.cp_cols = int(3 * d);
  e.cp_col0 = int(which * d);
  return e;
}

int attn_args(const Pack& p, const GptBufs& b, const LayerBufs& lb, AttnArgs& a) {
  const GptCfg c = b.c;
  const int64_t T = c.T, d = c.d, nd = int64_t(b.N) * d, nd3 = nd * 3;
  a = AttnArgs{};
  int rc = make_operand_map(&a.tq, op(lb.qkv, nd3, T * 3 * d, 64, 3 * d, 1, int(T), 64), false, 128, p.lanes,
                            p.batch, c.heads);
  if (!rc) rc = make_operand_map(&a.tk, op(lb.qkv + d, nd3, T * 3 * d, 64, 3 * d, 1, int(T), 64), false, 128,
                                 p.lanes, p.batch, c.heads);
  if (!rc) rc = make_operand_map(&a.tv, op(lb.qkv + 2 * d, nd3, T * 3 * d, 64, 3 * d, 1, int(T), 64), false, 128,
                                 p.lanes, p.batch, c.heads);
  if (!rc) rc = make_operand_map(&a.tdy, op(b.dy, nd, T * d, 64, d, 1, int(T), 64), false, 128, p.lanes, p.batch,
                                 c.heads);
  if (rc) return rc;
  a.lanes = p.lane_dev;
  a.nb = p.batch;
  a.nh = c.heads;
  a.items = p.lanes * p.batch * c.heads;
  a.scale = 1.0f / sqrtf(64.f);
  a.stats = lb.stats;
  a.D = b.D;
  a.trace = nullptr;
  return TLK_OK;
}

int attn_fwd(const Pack& p, const GptBufs& b, const LayerBufs& lb, cudaStream_t st) {
  AttnArgs a;
  if (int rc = attn_args(p, b, lb, a)) return rc;
  a.ey = attn_y_epi(b, lb);
  a.trace = b.atrace;
  {
    const int64_t T = b.c.T, d = b.c.d, nd = int64_t(b.N) * d;
    if (int rc = make_operand_map(&a.to[0], op(lb.y, nd, T * d, 64, d, 1, int(T), 64), false, 32, p.lanes,
                                  p.batch, b.c.heads))
      return rc;
  }
  TLK_CUDA(b.c.T == 256 ? launch_attn_fwd<2>(a, b.sms, st) : launch_attn_fwd<1>(a, b.sms, st));
  const_cast<Pack&>(p).mark(st, "attn_fwd");
  return TLK_OK;
}

int attn_bwd(const Pack& p, const GptBufs& b, const LayerBufs& lb, cudaStream_t st) {
  AttnArgs a;
  if (int rc = attn_args(p, b, lb, a)) return rc;
  a.edq = attn_dqkv_epi(b, 0);
  a.edk = attn_dqkv_epi(b, 1);
  a.edv = attn_dqkv_epi(b, 2);
  a.trace = b.atrace ? b.atrace + 64 * 32 : nullptr;
  {
    const int64_t T = b.c.T, d = b.c.d, nd3 = int64_t(b.N) * 3 * d;
    for (int i = 0; i < 3; ++i)
      if (int rc = make_operand_map(&a.to[i], op(b.dqkv + i * d, nd3, T * 3 * d, 64, 3 * d, 1, int(T), 64), false,
                                    32, p.lanes, p.batch, b.c.heads))
        return rc;
  }
  TLK_CUDA(b.c.T == 256 ? launch_attn_bwd<2>(a, b.sms, st) : launch_attn_bwd<1>(a, b.sms, st));
  const_cast<Pack&>(p).mark(st, "attn_bwd");
  return TLK_OK;
}

#define TLK_TRY(x)              \
  do {                          \
    int rc_ = (x);              \
    if (rc_) return rc_;        \
  } while (0)

}  // namespace

// ------------------------------------------------------------- setup -------
int gpt_setup(Pack& p) {
  const GptCfg c = p.gcfg;
  TLK_CHECK(c.d % c.heads == 0 && c.d / c.heads == 64, TLK_EINVAL, "gpt: head dim must be 64");
  TLK_CHECK(c.d % 128 == 0 && c.d <= 512, TLK_EINVAL, "gpt: d_model must be a multiple of 128 <= 512");
  TLK_CHECK(c.T == 64 || c.T == 128 || c.T == 256, TLK_EINVAL, "gpt: seq_len must be 64, 128 or 256");
  TLK_CHECK(c.V >= 2 && c.V <= 256, TLK_EINVAL, "gpt: vocab must be in [2, 256]");
  TLK_CHECK((int64_t(p.batch) * c.T) % 256 == 0, TLK_EINVAL, "gpt: batch*seq_len must be a multiple of 256");
  auto* b = new GptBufs{};
  p.scratch = b;
  p.scratch_free = [](void* q) { delete static_cast<GptBufs*>(q); };
  b->c = c;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    b->sms = 148;
    cudaDeviceGetAttribute(&b->sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t L = p.lanes, N = int64_t(p.batch) * c.T, d = c.d, H = c.heads, T = c.T;
  b->N = int(N);
  {
    static const char* f = getenv("TLK_ATTN_FUSED");  // 0: the unfused P / dS GEMM chain
    // attn.cuh lists a CTA's work items in shared memory (ATT_MAX_ITEMS per CTA)
    b->fused_attn = (T == 128 || T == 256) && !(f && f[0] == '0') &&
                    L * p.batch * H <= int64_t(b->sms) * ATT_MAX_ITEMS;
  }
  b->Vp = (c.V + 31) / 32 * 32;
  if (b->Vp > 256) return fail(TLK_EINVAL, "gpt: vocab too large");
  // sizes (bytes) of everything, one allocation
  struct Item {
    void** ptr;
    size_t bytes;
  };
  std::vector<Item> items;
  auto add = [&](void** ptr, size_t bytes) { items.push_back({ptr, (bytes + 255) & ~size_t(255)}); };
  add(reinterpret_cast<void**>(&b->tokens), L * p.batch * (T + 1) * 4);
  add(reinterpret_cast<void**>(&b->targets), L * N * 4);
  b->L.resize(c.layers);
  for (auto& lb : b->L) {
    add(reinterpret_cast<void**>(&lb.xin), L * N * d * 4);
    add(reinterpret_cast<void**>(&lb.xmid), L * N * d * 4);
    add(reinterpret_cast<void**>(&lb.st1), L * N * 2 * 4);
    add(reinterpret_cast<void**>(&lb.st2), L * N * 2 * 4);
    add(reinterpret_cast<void**>(&lb.z), L * N * 4 * d * 2);
    add(reinterpret_cast<void**>(&lb.a), L * N * d * 2);
    add(reinterpret_cast<void**>(&lb.qkv), L * N * 3 * d * 2);
    if (b->fused_attn)
      add(reinterpret_cast<void**>(&lb.stats), L * p.batch * H * T * 2 * 4);
    else
      add(reinterpret_cast<void**>(&lb.P), L * p.batch * H * T * T * 2);
    add(reinterpret_cast<void**>(&lb.y), L * N * d * 2);
    add(reinterpret_cast<void**>(&lb.m), L * N * d * 2);
    add(reinterpret_cast<void**>(&lb.f), L * N * 4 * d * 2);
  }
  add(reinterpret_cast<void**>(&b->xL), L * N * d * 4);
  add(reinterpret_cast<void**>(&b->stf), L * N * 2 * 4);
  add(reinterpret_cast<void**>(&b->lossrow), L * N * 4);
  add(reinterpret_cast<void**>(&b->xf), L * N * d * 2);
  add(reinterpret_cast<void**>(&b->dl), L * N * b->Vp * 2);
  add(reinterpret_cast<void**>(&b->dx), L * N * d * 4);
  add(reinterpret_cast<void**>(&b->dmm), L * N * d * 4);
  add(reinterpret_cast<void**>(&b->dxb), L * N * d * 2);
  add(reinterpret_cast<void**>(&b->dz), L * N * 4 * d * 2);
  add(reinterpret_cast<void**>(&b->dy), L * N * d * 2);
  if (!b->fused_attn) add(reinterpret_cast<void**>(&b->dS), L * p.batch * H * T * T * 2);
  add(reinterpret_cast<void**>(&b->dqkv), L * N * 3 * d * 2);
  add(reinterpret_cast<void**>(&b->D), L * N * H * 4);
  // reduction partials: max of LN-backward (N/LNB_ROWS x 3d) and the GELU' / dq,dk,dv
  // epilogue bias partials (N/32 x 4d, N/32 x 3d)
  const int64_t ps = std::max((N + LNB_ROWS - 1) / LNB_ROWS * 3 * d, int64_t((N + 31) / 32) * 4 * d);
  b->part_st = ps;
  add(reinterpret_cast<void**>(&b->part), L * ps * 4);
  size_t total = 0;
  for (auto& it : items) total += it.bytes;
  void* base = nullptr;
  int rc = pack_alloc(p, &base, total);
  if (rc) return rc;
  TLK_CUDA(cudaMemset(base, 0, total));
  char* cur = static_cast<char*>(base);
  for (auto& it : items) {
    *it.ptr = cur;
    cur += it.bytes;
  }
  p.acts = base;
  p.acts_bytes = total;
  p.launches_per_step = 0;  // counted at capture (mark)
  if (b->fused_attn && getenv("TLK_ATTN_TRACE") && getenv("TLK_ATTN_TRACE")[0] == '1') {
    void* tb = nullptr;
    int rc2 = pack_alloc(p, &tb, 2 * 64 * 32 * 8);
    if (rc2) return rc2;
    TLK_CUDA(cudaMemset(tb, 0, 2 * 64 * 32 * 8));
    b->atrace = static_cast<unsigned long long*>(tb);
    p.name_buf("attn.trace", tb, 2 * 64 * 32 * 8);
  }
  p.host_segs = {{b->tokens, size_t(L) * p.batch * (T + 1) * 4}};  // int32 [lanes][batch][T + 1]
  return TLK_OK;
}

// ------------------------------------------------------------- one step -----
int gpt_enqueue_step(Pack& p, cudaStream_t st) {
  GptBufs& b = *static_cast<GptBufs*>(p.scratch);
  const GptCfg c = b.c;
  const int Lc = p.lanes, B = p.batch, T = c.T, d = c.d, H = c.heads, V = c.V, Vp = b.Vp;
  const int N = b.N, dh = 64;
  const int64_t PS = p.stride;
  const float* PR = p.params;
  const uint16_t* WB = p.wbf;
  float* G = p.grads;
  const int64_t nd = int64_t(N) * d, nd3 = nd * 3, nd4 = nd * 4;
  const int64_t tt = int64_t(T) * T, pl = int64_t(B) * H * tt;  // P per lane
  const float scale = 1.0f / sqrtf(float(dh));
  auto O = [&](int t) { return tensor_off(p, t); };
  const LaneState* LS = p.lane_dev;
  int count = 0;
  auto marked = [&](const char* name) {
    p.mark(st, name);
    ++count;
  };

  if (p.host_input)
    TLK_CUDA(launch(gpt_targets_kernel, dim3((B + 127) / 128, Lc), 128, 0, st, LS, B, T, b.tokens, b.targets));
  else
    TLK_CUDA(launch(gpt_tokens_kernel, dim3((B + 127) / 128, Lc), 128, 0, st, LS, B, T, V, b.tokens, b.targets));
  TLK_CUDA(cudaGetLastError());
  marked("tokens");
  float* x0 = c.layers ? b.L[0].xin : b.xL;
  {
    const int vec = d % 4 == 0 && O(T_WTE) % 4 == 0 && O(T_WPE) % 4 == 0 && PS % 4 == 0 &&
                    (reinterpret_cast<uintptr_t>(PR) & 15) == 0 && (reinterpret_cast<uintptr_t>(x0) & 15) == 0;
    TLK_CUDA(launch(gpt_embed_kernel, dim3((N + 7) / 8, Lc), 256, 0, st, LS, c, B, b.tokens, PR, PS, O(T_WTE),
                    O(T_WPE), x0, vec));
  }
  TLK_CUDA(cudaGetLastError());
  marked("embed");

  auto ln_fwd = [&](const float* x, int64_t og, int64_t ob, uint16_t* y, float* stats) -> int {
    const dim3 gv((N + 8 * LNF_WROWS - 1) / (8 * LNF_WROWS), Lc);
    if (d == 128)
      TLK_CUDA(launch(ln_fwd_vec_kernel<1>, gv, 256, 0, st, LS, N, x, PR, PS, og, ob, y, stats));
    else if (d == 256)
      TLK_CUDA(launch(ln_fwd_vec_kernel<2>, gv, 256, 0, st, LS, N, x, PR, PS, og, ob, y, stats));
    else if (d == 384)
      TLK_CUDA(launch(ln_fwd_vec_kernel<3>, gv, 256, 0, st, LS, N, x, PR, PS, og, ob, y, stats));
    else if (d == 512)
      TLK_CUDA(launch(ln_fwd_vec_kernel<4>, gv, 256, 0, st, LS, N, x, PR, PS, og, ob, y, stats));
    else
      TLK_CUDA(launch(ln_fwd_kernel, dim3((N + 7) / 8, Lc), 256, 0, st, LS, N, d, x, PR, PS, og, ob, y, stats));
    return TLK_OK;
  };
  for (int l = 0; l < c.layers; ++l) {
    LayerBufs& lb = b.L[l];
    float* xnext = (l + 1 < c.layers) ? b.L[l + 1].xin : b.xL;
    TLK_TRY(ln_fwd(lb.xin, O(T_LAYER(l, K_LN1G)), O(T_LAYER(l, K_LN1B)), lb.a, lb.st1));
    TLK_CUDA(cudaGetLastError());
    marked("ln1");
    {  // qkv = a Wqkv^T + b
      Epi e = epi(EPI_BF16, N, 3 * d, lb.qkv, nd3, 0, 0, 3 * d);
      e.bias = PR + O(T_LAYER(l, K_AB));
      e.bias_ls = PS;
      TLK_TRY((gemm_auto<false, false>(p, st, op(lb.a, nd, 0, 0, d, 1, N, d),
                                              op(WB + O(T_LAYER(l, K_AW)), PS, 0, 0, d, 1, 3 * d, d), e,
                                              N, 3 * d, d, 1, 1, "qkv")));
      ++count;
    }
    if (b.fused_attn) {  // Y = softmax(Q K^T / sqrt(dh), causal) V, fused (attn.cuh)
      TLK_TRY(attn_fwd(p, b, lb, st));
      ++count;
    } else {
    {  // P = softmax(Q K^T / sqrt(dh)), per (sequence, head)
      Epi e = epi(EPI_SOFTMAX, T, T, lb.P, pl, int64_t(H) * tt, tt, T);
      e.scale = scale;
      e.causal = 1;
      const Operand A = op(lb.qkv, nd3, int64_t(T) * 3 * d, dh, 3 * d, 1, T, dh);
      const Operand Bk = op(lb.qkv + d, nd3, int64_t(T) * 3 * d, dh, 3 * d, 1, T, dh);
      if (T == 256)
        TLK_TRY((gemm<256, false, false, true>(p, st, A, Bk, e, T, T, dh, B, H, "attn_scores")));
      else if (T == 128)
        TLK_TRY((gemm<128, false, false, true>(p, st, A, Bk, e, T, T, dh, B, H, "attn_scores")));
      else
        TLK_TRY((gemm<64, false, false, true>(p, st, A, Bk, e, T, T, dh, B, H, "attn_scores")));
      ++count;
    }
    {  // y = P V
      Epi e = epi(EPI_BF16, T, dh, lb.y, nd, int64_t(T) * d, dh, d);
      e.causal_k = 1;  // P rows: keys <= query
      TLK_TRY((gemm<64, false, true, false>(
          p, st, op(lb.P, pl, int64_t(H) * tt, tt, T, 1, T, T),
          op(lb.qkv + 2 * d, nd3, int64_t(T) * 3 * d, dh, 1, 3 * d, dh, T), e, T, dh, T, B, H, "attn_pv")));
      ++count;
    }
    }
    {  // xmid = xin + y Wo^T + bo
      Epi e = epi(EPI_RESADD, N, d, lb.xmid, nd, 0, 0, d);
      e.aux = lb.xin;
      e.bias = PR + O(T_LAYER(l, K_PB));
      e.bias_ls = PS;
      TLK_TRY((gemm_auto<false, false>(p, st, op(lb.y, nd, 0, 0, d, 1, N, d),
                                              op(WB + O(T_LAYER(l, K_PW)), PS, 0, 0, d, 1, d, d), e, N,
                                              d, d, 1, 1, "proj")));
      ++count;
    }
    TLK_TRY(ln_fwd(lb.xmid, O(T_LAYER(l, K_LN2G)), O(T_LAYER(l, K_LN2B)), lb.m, lb.st2));
    TLK_CUDA(cudaGetLastError());
    marked("ln2");
    {  // z = m W1^T + b1, f = gelu(z)
      Epi e = epi(EPI_BF16_GELU, N, 4 * d, lb.f, nd4, 0, 0, 4 * d);
      e.out2 = lb.z;
      e.bias = PR + O(T_LAYER(l, K_FB));
      e.bias_ls = PS;
      TLK_TRY((gemm_auto<false, false>(p, st, op(lb.m, nd, 0, 0, d, 1, N, d),
                                              op(WB + O(T_LAYER(l, K_FW)), PS, 0, 0, d, 1, 4 * d, d), e,
                                              N, 4 * d, d, 1, 1, "fc")));
      ++count;
    }
    {  // xnext = xmid + f W2^T + b2
      Epi e = epi(EPI_RESADD, N, d, xnext, nd, 0, 0, d);
      e.aux = lb.xmid;
      e.bias = PR + O(T_LAYER(l, K_F2B));
      e.bias_ls = PS;
      TLK_TRY((gemm_auto<false, false>(p, st, op(lb.f, nd4, 0, 0, 4 * d, 1, N, 4 * d),
                                              op(WB + O(T_LAYER(l, K_F2W)), PS, 0, 0, 4 * d, 1, d, 4 * d),
                                              e, N, d, 4 * d, 1, 1, "fc2")));
      ++count;
    }
  }
  const int tf = T_LNFG(c);
  TLK_TRY(ln_fwd(b.xL, O(tf), O(tf + 1), b.xf, b.stf));
  TLK_CUDA(cudaGetLastError());
  marked("lnf");
  {  // logits -> CE row epilogue: lossrow, dl = (softmax - onehot) / N
    Epi e = epi(EPI_CE, N, V, b.dl, int64_t(N) * Vp, 0, 0, Vp);
    e.targets = b.targets;
    e.tg_ls = N;
    e.lossrow = b.lossrow;
    e.tokens = float(N);
    const Operand A = op(b.xf, nd, 0, 0, d, 1, N, d);
    const Operand Bh = op(WB + O(tf + 2), PS, 0, 0, d, 1, V, d);
    if (Vp <= 64)
      TLK_TRY((gemm<64, false, false, true>(p, st, A, Bh, e, N, Vp, d, 1, 1, "head_ce")));
    else if (Vp <= 96)
      TLK_TRY((gemm<96, false, false, true>(p, st, A, Bh, e, N, Vp, d, 1, 1, "head_ce")));
    else if (Vp <= 128)
      TLK_TRY((gemm<128, false, false, true>(p, st, A, Bh, e, N, Vp, d, 1, 1, "head_ce")));
    else
      TLK_TRY((gemm<256, false, false, true>(p, st, A, Bh, e, N, Vp, d, 1, 1, "head_ce")));
    ++count;
  }
  TLK_CUDA(launch(gpt_loss_kernel, Lc, 512, 0, st, p.lane_dev, N, b.lossrow, p.loss, p.max_steps, p.last_loss));
  TLK_CUDA(cudaGetLastError());
  marked("loss");

  // ---------------------------------------------------------------- backward
  {  // dxf = dl Whead (fp32), dWhead = dl^T xf
    Epi e = epi(EPI_F32, N, d, b.dmm, nd, 0, 0, d);
    TLK_TRY((gemm_auto<false, true>(p, st, op(b.dl, int64_t(N) * Vp, 0, 0, Vp, 1, N, V),
                                           op(WB + O(tf + 2), PS, 0, 0, 1, d, d, V), e, N, d, V, 1, 1,
                                           "head_dgrad")));
    Epi g = epi(EPI_F32, V, d, G + O(tf + 2), PS, 0, 0, d);
    TLK_TRY((gemm_auto<true, true>(p, st, op(b.dl, int64_t(N) * Vp, 0, 0, 1, Vp, V, N),
                                          op(b.xf, nd, 0, 0, 1, d, d, N), g, V, d, N, 1, 1, "head_wgrad")));
    count += 2;
  }
  // bias_t >= 0: the stored dxb's column sums are that tensor's gradient (the
  // bias of the GEMM that consumes dxb next)
  auto ln_bwd = [&](const float* dy, const float* x, const float* stats, int og, int ob, int accumulate,
                    const char* name, int bias_t) -> int {
    const int nblk = (N + LNB_ROWS - 1) / LNB_ROWS;
    const dim3 grid(nblk, Lc);
    const size_t sm = LNB_WARPS * 3 * size_t(d) * 4;
    switch (d / 128) {
      case 1:
        TLK_CUDA(launch(ln_bwd_kernel<1>, grid, LNB_WARPS * 32, sm, st, LS, N, dy, x, stats, PR, PS, O(og), b.dx, b.dxb, accumulate,
                                                b.part, b.part_st));
        break;
      case 2:
        TLK_CUDA(launch(ln_bwd_kernel<2>, grid, LNB_WARPS * 32, sm, st, LS, N, dy, x, stats, PR, PS, O(og), b.dx, b.dxb, accumulate,
                                                b.part, b.part_st));
        break;
      case 3:
        TLK_CUDA(launch(ln_bwd_kernel<3>, grid, LNB_WARPS * 32, sm, st, LS, N, dy, x, stats, PR, PS, O(og), b.dx, b.dxb, accumulate,
                                                b.part, b.part_st));
        break;
      default:
        TLK_CUDA(launch(ln_bwd_kernel<4>, grid, LNB_WARPS * 32, sm, st, LS, N, dy, x, stats, PR, PS, O(og), b.dx, b.dxb, accumulate,
                                                b.part, b.part_st));
        break;
    }
    TLK_CUDA(cudaGetLastError());
    marked(name);
    TLK_CUDA(launch(reduce_parts_kernel, dim3((3 * d + 255) / 256, Lc), 256, 0, st, LS, b.part, b.part_st, nblk, 3 * d,
                    G, PS, O(og), d, O(ob), 2 * d, bias_t >= 0 ? O(bias_t) : int64_t(-1)));
    TLK_CUDA(cudaGetLastError());
    marked("ln_param_grads");
    return TLK_OK;
  };
  TLK_TRY(ln_bwd(b.dmm, b.xL, b.stf, tf, tf + 1, 0, "lnf_bwd", T_LAYER(c.layers - 1, K_F2B)));

  for (int l = c.layers - 1; l >= 0; --l) {
    LayerBufs& lb = b.L[l];
    bool rowdot_fused = false;
    {  // fc2: dW2 = dxb^T f ; db2 ; dz = (dxb W2) * gelu'(z)
      Epi g = epi(EPI_F32, d, 4 * d, G + O(T_LAYER(l, K_F2W)), PS, 0, 0, 4 * d);
      TLK_TRY((gemm_auto<true, true>(p, st, op(b.dxb, nd, 0, 0, 1, d, d, N),
                                            op(lb.f, nd4, 0, 0, 1, 4 * d, 4 * d, N), g, d, 4 * d, N, 1, 1,
                                            "fc2_wgrad")));
      Epi e = epi(EPI_GELU_BWD, N, 4 * d, b.dz, nd4, 0, 0, 4 * d);
      e.aux = lb.z;
      e.colpart = b.part;  // fc.b gradient partials (per 32 rows), summed right below
      e.cp_ls = b.part_st;
      TLK_TRY((gemm_auto<false, true>(p, st, op(b.dxb, nd, 0, 0, d, 1, N, d),
                                             op(WB + O(T_LAYER(l, K_F2W)), PS, 0, 0, 1, 4 * d, 4 * d, d), e,
                                             N, 4 * d, d, 1, 1, "fc2_dgrad")));
      count += 2;
      TLK_CUDA(launch(reduce_parts8_kernel, dim3((4 * d + 31) / 32, Lc), 256, 0, st, LS, b.part, b.part_st,
                      (N + 31) / 32, 4 * d, G, PS, O(T_LAYER(l, K_FB))));
      marked("bias_reduce");
    }
    {  // fc: dW1 = dz^T m ; db1 ; dmm = dz W1 (fp32)
      Epi g = epi(EPI_F32, 4 * d, d, G + O(T_LAYER(l, K_FW)), PS, 0, 0, d);
      TLK_TRY((gemm_auto<true, true>(p, st, op(b.dz, nd4, 0, 0, 1, 4 * d, 4 * d, N),
                                            op(lb.m, nd, 0, 0, 1, d, d, N), g, 4 * d, d, N, 1, 1,
                                            "fc_wgrad")));
      Epi e = epi(EPI_F32, N, d, b.dmm, nd, 0, 0, d);
      TLK_TRY((gemm_auto<false, true>(p, st, op(b.dz, nd4, 0, 0, 4 * d, 1, N, 4 * d),
                                             op(WB + O(T_LAYER(l, K_FW)), PS, 0, 0, 1, d, d, 4 * d), e, N,
                                             d, 4 * d, 1, 1, "fc_dgrad")));
      count += 2;
    }
    TLK_TRY(ln_bwd(b.dmm, lb.xmid, lb.st2, T_LAYER(l, K_LN2G), T_LAYER(l, K_LN2B), 1, "ln2_bwd", T_LAYER(l, K_PB)));
    {  // proj: dWo = dxb^T y ; dbo ; dy = dxb Wo (bf16)
      Epi g = epi(EPI_F32, d, d, G + O(T_LAYER(l, K_PW)), PS, 0, 0, d);
      TLK_TRY((gemm_auto<true, true>(p, st, op(b.dxb, nd, 0, 0, 1, d, d, N),
                                            op(lb.y, nd, 0, 0, 1, d, d, N), g, d, d, N, 1, 1, "proj_wgrad")));
      Epi e = epi(EPI_BF16, N, d, b.dy, nd, 0, 0, d);
      // fused attention: the softmax-backward row term D = rowsum(dY o Y)
      // comes out of this GEMM's epilogue (one 64-column head per epilogue
      // warp, BN = 128); otherwise attn_rowdot_kernel computes it
      Epi er = e;
      er.kind = EPI_BF16_ROWDOT;
      er.aux = lb.y;
      er.rowout = b.D;
      er.rv_T = T;
      er.rv_H = H;
      rowdot_fused = b.fused_attn && tma_epi_usable(er) && d % 128 == 0 && d == 64 * H;
      if (rowdot_fused)
        TLK_TRY((gemm<128, false, true, false, false, true>(p, st, op(b.dxb, nd, 0, 0, d, 1, N, d),
                                                            op(WB + O(T_LAYER(l, K_PW)), PS, 0, 0, 1, d, d, d),
                                                            er, N, d, d, 1, 1, "proj_dgrad")));
      else
        TLK_TRY((gemm_auto<false, true>(p, st, op(b.dxb, nd, 0, 0, d, 1, N, d),
                                               op(WB + O(T_LAYER(l, K_PW)), PS, 0, 0, 1, d, d, d), e, N, d, d,
                                               1, 1, "proj_dgrad")));
      count += 2;
    }
    {  // attention backward per (sequence, head)
      if (!rowdot_fused) {
        TLK_CUDA(launch(attn_rowdot_kernel, dim3((N * H + 255) / 256, Lc), 256, 0, st, LS, N, T, H, b.dy, lb.y,
                        b.D));
        TLK_CUDA(cudaGetLastError());
        marked("attn_rowdot");
      }
      if (b.fused_attn) {  // dS on chip; dQ / dK / dV + qkv.b partials (attn.cuh)
        TLK_TRY(attn_bwd(p, b, lb, st));
        ++count;
      } else {
      Epi e = epi(EPI_SOFTMAX_BWD, T, T, b.dS, pl, int64_t(H) * tt, tt, T);
      e.aux = lb.P;
      e.scale = scale;
      e.rowvec = b.D;
      e.rv_ls = int64_t(N) * H;
      e.rv_bs = int64_t(H) * T;
      e.rv_hs = T;
      const Operand A = op(b.dy, nd, int64_t(T) * d, dh, d, 1, T, dh);
      const Operand Bv = op(lb.qkv + 2 * d, nd3, int64_t(T) * 3 * d, dh, 3 * d, 1, T, dh);
      if (T == 256)
        TLK_TRY((gemm<256, false, false, true>(p, st, A, Bv, e, T, T, dh, B, H, "attn_dp")));
      else if (T == 128)
        TLK_TRY((gemm<128, false, false, true>(p, st, A, Bv, e, T, T, dh, B, H, "attn_dp")));
      else
        TLK_TRY((gemm<64, false, false, true>(p, st, A, Bv, e, T, T, dh, B, H, "attn_dp")));
      // dq = dS K
      Epi eq = epi(EPI_BF16, T, dh, b.dqkv, nd3, int64_t(T) * 3 * d, dh, 3 * d);
      eq.causal_k = 1;
      eq.colpart = b.part;  // qkv.b gradient partials (columns 0 ..)
      eq.cp_ls = b.part_st;
      eq.cp_cols = 3 * d;
      eq.cp_col0 = 0;
      TLK_TRY((gemm<64, false, true, false>(p, st, op(b.dS, pl, int64_t(H) * tt, tt, T, 1, T, T),
                                            op(lb.qkv + d, nd3, int64_t(T) * 3 * d, dh, 1, 3 * d, dh, T), eq,
                                            T, dh, T, B, H, "attn_dq")));
      // dk = dS^T Q
      Epi ek = epi(EPI_BF16, T, dh, b.dqkv + d, nd3, int64_t(T) * 3 * d, dh, 3 * d);
      ek.causal_k = 2;  // dS^T rows = keys: queries >= key
      ek.colpart = b.part;  // qkv.b gradient partials (columns d ..)
      ek.cp_ls = b.part_st;
      ek.cp_cols = 3 * d;
      ek.cp_col0 = d;
      TLK_TRY((gemm<64, true, true, false>(p, st, op(b.dS, pl, int64_t(H) * tt, tt, 1, T, T, T),
                                           op(lb.qkv, nd3, int64_t(T) * 3 * d, dh, 1, 3 * d, dh, T), ek, T,
                                           dh, T, B, H, "attn_dk")));
      // dv = P^T dY
      Epi ev = epi(EPI_BF16, T, dh, b.dqkv + 2 * d, nd3, int64_t(T) * 3 * d, dh, 3 * d);
      ev.causal_k = 2;
      ev.colpart = b.part;  // qkv.b gradient partials (columns 2 * d ..)
      ev.cp_ls = b.part_st;
      ev.cp_cols = 3 * d;
      ev.cp_col0 = 2 * d;
      TLK_TRY((gemm<64, true, true, false>(p, st, op(lb.P, pl, int64_t(H) * tt, tt, 1, T, T, T),
                                           op(b.dy, nd, int64_t(T) * d, dh, 1, d, dh, T), ev, T, dh, T, B,
                                           H, "attn_dv")));
      count += 4;
      }
      TLK_CUDA(launch(reduce_parts8_kernel, dim3((3 * d + 31) / 32, Lc), 256, 0, st, LS, b.part, b.part_st,
                      (N + 31) / 32, 3 * d, G, PS, O(T_LAYER(l, K_AB))));
      marked("bias_reduce");
    }
    {  // qkv: dWqkv = dqkv^T a ; db ; da = dqkv Wqkv (fp32)
      Epi g = epi(EPI_F32, 3 * d, d, G + O(T_LAYER(l, K_AW)), PS, 0, 0, d);
      TLK_TRY((gemm_auto<true, true>(p, st, op(b.dqkv, nd3, 0, 0, 1, 3 * d, 3 * d, N),
                                            op(lb.a, nd, 0, 0, 1, d, d, N), g, 3 * d, d, N, 1, 1,
                                            "qkv_wgrad")));
      Epi e = epi(EPI_F32, N, d, b.dmm, nd, 0, 0, d);
      TLK_TRY((gemm_auto<false, true>(p, st, op(b.dqkv, nd3, 0, 0, 3 * d, 1, N, 3 * d),
                                             op(WB + O(T_LAYER(l, K_AW)), PS, 0, 0, 1, d, d, 3 * d), e, N, d,
                                             3 * d, 1, 1, "qkv_dgrad")));
      count += 2;
    }
    TLK_TRY(ln_bwd(b.dmm, lb.xin, lb.st1, T_LAYER(l, K_LN1G), T_LAYER(l, K_LN1B), 1, "ln1_bwd",
                   l > 0 ? T_LAYER(l - 1, K_F2B) : -1));
  }
  {  // embeddings
    TLK_CHECK(int64_t(N) < (int64_t(1) << 27), TLK_EINVAL, "embedding gradient: %d tokens per lane", N);
    const size_t emt_smem = size_t(V) * d * 4;
    const int emt_chunks = std::min<int64_t>({int64_t(N + 255) / 256, std::max(1, 2 * b.sms / Lc),  // one wave
                                              b.part_st / (int64_t(V) * d)});
    if (d % 4 == 0 && d <= 512 && emt_smem <= EMT_SMEM_MAX && emt_chunks >= 1) {
      static bool emt_configured = false;
      if (!emt_configured) {
        TLK_CUDA(cudaFuncSetAttribute(embed_bwd_tok_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(EMT_SMEM_MAX)));
        emt_configured = true;
      }
      const int rows_per = (N + emt_chunks - 1) / emt_chunks;
      TLK_CUDA(launch(embed_bwd_tok_kernel, dim3((N + rows_per - 1) / rows_per, Lc), 128, emt_smem, st, LS, N, d, V,
                      b.tokens, T, b.dx, b.part, b.part_st, rows_per));
      TLK_CUDA(launch(reduce_parts8_kernel, dim3((V * d + 31) / 32, Lc), 256, 0, st, LS, b.part, b.part_st,
                      (N + rows_per - 1) / rows_per, V * d, G, PS, O(T_WTE)));
      ++count;
    } else {
      TLK_CUDA(launch(embed_bwd_vocab_kernel, dim3((V + EMV - 1) / EMV, (d + EMV_COLS - 1) / EMV_COLS, Lc), EMV_COLS,
                      0, st, LS, N, d, V, b.tokens, T, b.dx, G, PS, O(T_WTE)));
    }
    marked("wte_grad");
    TLK_CUDA(launch(wpe_bwd_kernel, dim3(T, Lc), 128, 0, st, LS, B, T, d, b.dx, G, PS, O(T_WPE)));
    TLK_CUDA(cudaGetLastError());
    marked("wpe");
  }
  TLK_TRY(enqueue_optimizer(p, st));
  ++count;
  p.launches_per_step = count;
  return TLK_OK;
}

}  // namespace tlk
