// ResNet-18 (CIFAR variant) packs: K jobs x batch B per step, every
// convolution of all K lanes in one persistent tcgen05 launch (conv.cuh).
// Numerics restate oracle/resnet.py (bf16 conv operands and outputs, fp32
// accumulation, batch-statistics BatchNorm with centred variance, fp32 head
// and gradients).  Per-lane buffers are NHWC bf16 [lane][B][H][W][C].
//
// One step (all lanes):
//   inputs -> weight transposes (dgrad B operands)
//   stem conv (SIMT, C_in = 3) -> BN stats -> BN+ReLU
//   per BasicBlock: conv1 -> stats -> BN+ReLU ; conv2 -> stats ;
//                   [1x1 s2 conv -> stats] ; BN (+shortcut) + ReLU
//   head (avg-pool, fc, CE, dlogits, d pool) -> loss
//   per block (reverse): BN2(+BNd) backward ; wgrad/dgrad conv2 ; BN1
//                   backward ; wgrad/dgrad conv1 (+ ds) accumulating into the
//                   block-input gradient
//   stem BN backward + stem wgrad (SIMT) -> optimizer
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "conv.cuh"
#include "pack.cuh"
#include "rng.cuh"

namespace tlk {
namespace {

constexpr uint32_t STREAM_RDATA = 4, STREAM_RTEACHER = 5;
constexpr int IMG = 3072;  // 32 x 32 x 3
constexpr float BN_EPS = 1e-5f;

struct ConvL {
  int cin, cout, k, stride;
  int H, W, Ho, Wo;  // input / output resolution
  int t_w, t_g, t_b;  // tensor indices: weight, BN gain, BN bias
  int64_t wt_off;     // transposed weight offset in p.wt (per lane)
  uint16_t* y;        // conv output (bf16, pre-BN)
  float* stats;       // [lane][2][cout] mean, rstd
};

struct Block {
  int c1, c2, cd;          // conv indices (cd = -1: identity shortcut)
  uint16_t *xin, *a1, *o;  // block input, BN1-ReLU output, block output
  float* snapG;            // TLK_PACK_SNAPSHOTS: gradient w.r.t. o (fp32)
};

struct RnBufs {
  int B;
  std::vector<ConvL> conv;  // 0 = stem
  std::vector<Block> blk;
  uint16_t* xin;     // [lane][B][32][32][3]
  uint16_t* a0;      // stem output (post BN-ReLU)
  int8_t* teacher;   // [10][3072]
  float* part;       // stats / reduction partials (per lane part_ls floats)
  int64_t part_ls;
  float* sums;       // BN backward sums [lane][3][512]
  float *G0, *G1, *da;   // fp32 gradients at the largest resolution
  uint16_t *dy, *dyd;    // bf16 BN-backward outputs
  float* wpart;          // wgrad split-K partials
  int64_t wpart_ls;
  float* lossrow;        // [lane][B]
  float* snap_stem;      // TLK_PACK_SNAPSHOTS: gradient w.r.t. a0
  float* stat2;          // BN statistics level-2 records [lane][S][3][C]
  int64_t stat2_ls;
  unsigned* stat_cnt;    // [lane][STAT_MAX_CBLK] arrival counters (zero between launches)
  int sms;
  int64_t act_ls(int H, int W, int C) const { return int64_t(B) * H * W * C; }
};

// ------------------------------------------------------------------ inputs --
__global__ void __launch_bounds__(256) rn_inputs_kernel(const LaneState* __restrict__ lanes, int B,
                                                        const int8_t* __restrict__ teacher,
                                                        uint16_t* __restrict__ x, int32_t* __restrict__ labels) {
  pdl_begin();
  const int b = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  if (!lanes[j].active) return;
  const LaneState& s = lanes[j];
  const uint64_t key = rng_key(s.seed, STREAM_RDATA, uint64_t(s.steps_done));
  long long sc[10];
#pragma unroll
  for (int k = 0; k < 10; ++k) sc[k] = 0;
  uint16_t* xo = x + (int64_t(j) * B + b) * IMG;
  for (int i = tid; i < IMG; i += 256) {
    const uint64_t w = rng_bits(key, uint64_t(b) * IMG + i);
    const int S = int(w & 0xFFFF) + int((w >> 16) & 0xFFFF) + int((w >> 32) & 0xFFFF) + int(w >> 48) - 131070;
    xo[i] = f2bf(__fmul_rn(float(S), 1.0f / 37837.227f));
#pragma unroll
    for (int k = 0; k < 10; ++k) sc[k] += (long long)teacher[k * IMG + i] * S;
  }
  __shared__ long long red[8][10];
  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    long long v = sc[k];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (tid == 0) {
    long long best = 0;
    int arg = 0;
    for (int k = 0; k < 10; ++k) {
      long long v = 0;
      for (int w = 0; w < 8; ++w) v += red[w][k];
      if (k == 0 || v > best) {
        best = v;
        arg = k;
      }
    }
    labels[int64_t(j) * B + b] = arg;
  }
}

// --------------------------------------------------------- weight transpose --
struct WtEntry {
  int64_t src, dst;  // element offsets (src in the bf16 shadow, dst in p.wt)
  int cout, taps, cin, tiles0;  // tiles0 = first 32x32 tile index of this conv
};
struct WtTable {
  WtEntry e[24];
  int n, tiles;
};
// WT[tap][ci][co] = W[co][tap][ci] (bf16), 64x64 tiles through smem (every
// transposed conv has cin, cout multiples of 64): 16-byte loads along ci,
// 16-byte stores along co.
__global__ void __launch_bounds__(256) rn_wt_transpose_kernel(const LaneState* __restrict__ lanes,
                                                              const __grid_constant__ WtTable tab,
                                                              const uint16_t* __restrict__ wbf, int64_t wstride,
                                                              uint16_t* __restrict__ wt, int64_t wt_stride) {
  pdl_begin();
  const int j = blockIdx.y;
  if (!lanes[j].active) return;
  __shared__ uint16_t t[64][72];  // [co][ci], rows padded to 144 B
  int c = 0;
  while (c + 1 < tab.n && tab.e[c + 1].tiles0 <= int(blockIdx.x)) ++c;
  const WtEntry& E = tab.e[c];
  int r = blockIdx.x - E.tiles0;
  const int nci = E.cin / 64, nco = E.cout / 64;
  const int ci_t = r % nci;
  r /= nci;
  const int co_t = r % nco;
  const int tap = r / nco;
  const uint16_t* src = wbf + j * wstride + E.src;
  uint16_t* dst = wt + j * wt_stride + E.dst;
#pragma unroll
  for (int u = 0; u < 2; ++u) {  // 64 rows x 8 chunks of 8 ci
    const int i = threadIdx.x + 256 * u, row = i >> 3, ch = i & 7;
    const int co = co_t * 64 + row;
    *reinterpret_cast<uint4*>(&t[row][ch * 8]) =
        *reinterpret_cast<const uint4*>(src + (int64_t(co) * E.taps + tap) * E.cin + ci_t * 64 + ch * 8);
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 2; ++u) {  // 64 ci rows x 8 chunks of 8 co
    const int i = threadIdx.x + 256 * u, row = i >> 3, ch = i & 7;
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      w[k] = uint32_t(t[ch * 8 + 2 * k][row]) | (uint32_t(t[ch * 8 + 2 * k + 1][row]) << 16);
    const int ci = ci_t * 64 + row;
    *reinterpret_cast<uint4*>(dst + (int64_t(tap) * E.cin + ci) * E.cout + co_t * 64 + ch * 8) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// ---------------------------------------------------------------- stem conv --
// y0[pix][co] = bf16(sum_{kh,kw,ci} x[pix + tap][ci] W[co][kh][kw][ci]); one CTA
// per 128-pixel tile (4 image rows), thread = (channel, quarter of 32 pixels);
// writes the (mean, M2) partial of its 32 pixels like the tensor-core convs.
__global__ void __launch_bounds__(256) rn_stem_fwd_kernel(const LaneState* __restrict__ lanes, int B,
                                                          const uint16_t* __restrict__ x,
                                                          const uint16_t* __restrict__ wbf, int64_t wstride,
                                                          int64_t w_off, uint16_t* __restrict__ y,
                                                          float* __restrict__ part, int64_t part_ls) {
  pdl_begin();
  const int tile = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  if (!lanes[j].active) return;
  __shared__ float xs[6][34][3];
  const int b = tile / 8, r0 = (tile % 8) * 4;  // rows r0..r0+3 of image b
  const uint16_t* xi = x + (int64_t(j) * B + b) * IMG;
  for (int i = tid; i < 6 * 34 * 3; i += 256) {
    const int c = i % 3, xx = (i / 3) % 34, yy = i / 102;
    const int gy = r0 + yy - 1, gx = xx - 1;
    xs[yy][xx][c] = (gy >= 0 && gy < 32 && gx >= 0 && gx < 32) ? bf2f(xi[(gy * 32 + gx) * 3 + c]) : 0.f;
  }
  const int co = tid & 63, q = tid >> 6;
  float w[27];
  const uint16_t* wp = wbf + j * wstride + w_off + co * 27;
#pragma unroll
  for (int t = 0; t < 27; ++t) w[t] = bf2f(wp[t]);
  __syncthreads();
  float v[32];
  const int ry = q;  // quarter q = image row r0 + q (32 pixels)
#pragma unroll 4
  for (int px = 0; px < 32; ++px) {
    float acc = 0.f;
#pragma unroll
    for (int kh = 0; kh < 3; ++kh)
#pragma unroll
      for (int kw = 0; kw < 3; ++kw)
#pragma unroll
        for (int ci = 0; ci < 3; ++ci) acc = fmaf(xs[ry + kh][px + kw][ci], w[(kh * 3 + kw) * 3 + ci], acc);
    v[px] = bf2f(f2bf(acc));
  }
  uint16_t* yo = y + (int64_t(j) * B * 1024 + int64_t(tile) * 128 + q * 32) * 64 + co;
  float s = 0.f;
#pragma unroll
  for (int px = 0; px < 32; ++px) {
    yo[px * 64] = f2bf(v[px]);
    s += v[px];
  }
  const float mean = s * (1.0f / 32.0f);
  float m2 = 0.f;
#pragma unroll
  for (int px = 0; px < 32; ++px) m2 += (v[px] - mean) * (v[px] - mean);
  float* pp = part + j * part_ls + (int64_t(tile) * 4 + q) * 2 * 64 + co;
  pp[0] = mean;
  pp[64] = m2;
}

// -------------------------------------------------------------- BN stats ----
// (mean, M2) partials of 32 rows each [P][2][C] -> stats[lane][2][C] = mean,
// rstd via Chan's pairwise combination in a fixed order.  Grid (C/32, S,
// lanes): CTA s folds partials [s*128, s*128+128) (group g of 8 takes
// g, g+8, ... in order, then the groups in order) into a level-2 record
// (n, mean, M2); the last CTA of a (lane, channel block) to arrive -- a
// counter, not a reduction, so the result does not depend on arrival order
// -- combines the S records in order and writes the statistics.
__device__ __forceinline__ void chan_combine(float& n, float& mean, float& m2, float nb, float meanb,
                                             float m2b) {
  const float nn = n + nb;
  const float d = meanb - mean;
  mean = mean + d * (nb / nn);
  m2 = m2 + m2b + d * d * (n * nb / nn);
  n = nn;
}
constexpr int STAT_GROUPS = 8;
constexpr int STAT_PER_CTA = 128;  // partials per CTA (16 per group)
constexpr int STAT_MAX_CBLK = 16;  // channel blocks of 32 (C <= 512)
__global__ void __launch_bounds__(256) rn_bn_stats_kernel(const LaneState* __restrict__ lanes,
                                                          const float* __restrict__ part, int64_t part_ls, int P,
                                                          int C, float* __restrict__ l2, int64_t l2_ls,
                                                          unsigned* __restrict__ cnt, float* __restrict__ stats) {
  pdl_begin();
  const int j = blockIdx.z, sblk = blockIdx.y, S = gridDim.y;
  if (!lanes[j].active) return;
  const int cl = threadIdx.x & 31, g = threadIdx.x >> 5, c = blockIdx.x * 32 + cl;
  __shared__ float sh[3][STAT_GROUPS][32];
  __shared__ int last;
  float n = 0.f, mean = 0.f, m2 = 0.f;
  const int p_lo = sblk * STAT_PER_CTA, p_hi = min(P, p_lo + STAT_PER_CTA);
  if (c < C) {
    const float* pp = part + j * part_ls + c;
    for (int p0 = p_lo + g; p0 < p_hi; p0 += 4 * STAT_GROUPS) {
      float mb[4], qb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = p0 + u * STAT_GROUPS;
        mb[u] = q < p_hi ? pp[int64_t(q) * 2 * C] : 0.f;
        qb[u] = q < p_hi ? pp[int64_t(q) * 2 * C + C] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (p0 + u * STAT_GROUPS >= p_hi) break;
        if (n == 0.f) {
          n = 32.f;
          mean = mb[u];
          m2 = qb[u];
        } else {
          chan_combine(n, mean, m2, 32.f, mb[u], qb[u]);
        }
      }
    }
  }
  sh[0][g][cl] = n;
  sh[1][g][cl] = mean;
  sh[2][g][cl] = m2;
  __syncthreads();
  float* rec = l2 + j * l2_ls;  // [S][3][C]
  if (g == 0 && c < C) {
    float N = sh[0][0][cl], M = sh[1][0][cl], Q = sh[2][0][cl];
    for (int k = 1; k < STAT_GROUPS; ++k)
      if (sh[0][k][cl] > 0.f) chan_combine(N, M, Q, sh[0][k][cl], sh[1][k][cl], sh[2][k][cl]);
    rec[(int64_t(sblk) * 3 + 0) * C + c] = N;
    rec[(int64_t(sblk) * 3 + 1) * C + c] = M;
    rec[(int64_t(sblk) * 3 + 2) * C + c] = Q;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* ctr = cnt + j * STAT_MAX_CBLK + blockIdx.x;
    last = atomicAdd(ctr, 1u) == unsigned(S - 1);
    if (last) *ctr = 0u;  // re-armed for the next launch (stream-ordered)
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // groups fold records g, g+8, ... in order; then groups 0..7 in order
  n = 0.f, mean = 0.f, m2 = 0.f;
  if (c < C) {
    for (int r = g; r < S; r += STAT_GROUPS) {
      const float nb = __ldcg(rec + (int64_t(r) * 3 + 0) * C + c);
      const float mb = __ldcg(rec + (int64_t(r) * 3 + 1) * C + c);
      const float qb = __ldcg(rec + (int64_t(r) * 3 + 2) * C + c);
      if (nb <= 0.f) continue;
      if (n == 0.f) {
        n = nb;
        mean = mb;
        m2 = qb;
      } else {
        chan_combine(n, mean, m2, nb, mb, qb);
      }
    }
  }
  sh[0][g][cl] = n;
  sh[1][g][cl] = mean;
  sh[2][g][cl] = m2;
  __syncthreads();
  if (g == 0 && c < C) {
    float N = sh[0][0][cl], M = sh[1][0][cl], Q = sh[2][0][cl];
    for (int k = 1; k < STAT_GROUPS; ++k)
      if (sh[0][k][cl] > 0.f) chan_combine(N, M, Q, sh[0][k][cl], sh[1][k][cl], sh[2][k][cl]);
    stats[(int64_t(j) * 2) * C + c] = M;
    stats[(int64_t(j) * 2 + 1) * C + c] = 1.0f / sqrtf(Q / N + BN_EPS);
  }
}

// ------------------------------------------------------ BN apply (forward) --
// out = bf16(relu((y - mu) rstd g + b  [+ res]))  res: 0 none, 1 bf16 x,
// 2 (yd - mud) rstdd gd + bd.  Per-channel (mu, rstd * g, b) staged in smem;
// 8 channels (16 bytes of bf16) per thread.
__global__ void __launch_bounds__(256) rn_bn_act_kernel(const LaneState* __restrict__ lanes, int64_t n8, int C,
                                                        const uint16_t* __restrict__ y, const float* __restrict__ st,
                                                        const float* __restrict__ params, int64_t pstride,
                                                        int64_t og, int64_t ob, int mode,
                                                        const uint16_t* __restrict__ res,
                                                        const float* __restrict__ std_, int64_t ogd, int64_t obd,
                                                        uint16_t* __restrict__ out) {
  pdl_begin();
  const int j = blockIdx.y;
  if (!lanes[j].active) return;
  __shared__ float cf[6][512];  // mu, rstd*g, b, mud, rstdd*gd, bd
  const float* P = params + j * pstride;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const float rs = st[(int64_t(j) * 2 + 1) * C + c];
    cf[0][c] = st[(int64_t(j) * 2) * C + c];
    cf[1][c] = rs * P[og + c];
    cf[2][c] = P[ob + c];
    if (mode == 2) {
      cf[3][c] = std_[(int64_t(j) * 2) * C + c];
      cf[4][c] = std_[(int64_t(j) * 2 + 1) * C + c] * P[ogd + c];
      cf[5][c] = P[obd + c];
    }
  }
  __syncthreads();
  const int64_t lane_off = int64_t(j) * n8 * 8;
  const int64_t step = int64_t(gridDim.x) * blockDim.x;
  // two 16-byte vectors per thread in flight; C is a power of two
  for (int64_t i0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i0 < n8; i0 += 2 * step) {
    uint4 u[2], rv[2];
    int64_t ii[2] = {i0, i0 + step};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      u[h] = make_uint4(0, 0, 0, 0);
      rv[h] = make_uint4(0, 0, 0, 0);
      if (ii[h] < n8) {
        u[h] = *reinterpret_cast<const uint4*>(y + lane_off + ii[h] * 8);
        if (mode >= 1) rv[h] = *reinterpret_cast<const uint4*>(res + lane_off + ii[h] * 8);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (ii[h] >= n8) break;
      const int c0 = int((ii[h] * 8) & (C - 1));
      const uint32_t uw[4] = {u[h].x, u[h].y, u[h].z, u[h].w};
      const uint32_t rw[4] = {rv[h].x, rv[h].y, rv[h].z, rv[h].w};
      uint32_t ow[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float o2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = c0 + 2 * q + e;
          const float yv = e ? __uint_as_float(uw[q] & 0xffff0000u) : __uint_as_float(uw[q] << 16);
          float v = (yv - cf[0][c]) * cf[1][c] + cf[2][c];
          const float rr = e ? __uint_as_float(rw[q] & 0xffff0000u) : __uint_as_float(rw[q] << 16);
          if (mode == 1) v += rr;
          if (mode == 2) v += (rr - cf[3][c]) * cf[4][c] + cf[5][c];
          o2[e] = fmaxf(v, 0.f);
        }
        ow[q] = pack_bf2(o2[0], o2[1]);
      }
      *reinterpret_cast<uint4*>(out + lane_off + ii[h] * 8) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
    }
  }
}

// ---------------------------------------------------------------- head ------
// grid (lanes, B/8), warp = sample: h = mean_pix o, logits = h W^T + b (fp32),
// CE; G[b][pix][c] = (dl W)[c] / 16; fc partials per CTA (warps in order).
__global__ void __launch_bounds__(256) rn_head_kernel(const LaneState* __restrict__ lanes, int B,
                                                      const uint16_t* __restrict__ o, const int32_t* __restrict__ labels,
                                                      const float* __restrict__ params, int64_t pstride,
                                                      int64_t ow, int64_t ob, float* __restrict__ G,
                                                      float* __restrict__ lossrow, float* __restrict__ fpart,
                                                      int64_t fpart_ls) {
  pdl_begin();
  const int j = blockIdx.x, blk = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (!lanes[j].active) return;
  __shared__ float hs[8][512];
  __shared__ float dls[8][10];
  const int b = blk * 8 + warp;
  const float* W = params + j * pstride + ow;
  const float* bias = params + j * pstride + ob;
  const uint16_t* ob_ = o + (int64_t(j) * B + b) * 16 * 512;
  float h[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int c = lane + 32 * i;
    float s = 0.f;
    for (int p = 0; p < 16; ++p) s += bf2f(ob_[p * 512 + c]);
    h[i] = s / 16.0f;
    hs[warp][c] = h[i];
  }
  float lg[10];
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += h[i] * W[k * 512 + lane + 32 * i];
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    lg[k] = s + bias[k];
  }
  const int y = labels[int64_t(j) * B + b];
  float mx = lg[0];
#pragma unroll
  for (int k = 1; k < 10; ++k) mx = fmaxf(mx, lg[k]);
  float se = 0.f, ly = 0.f;
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    se += expf(lg[k] - mx);
    if (k == y) ly = lg[k];
  }
  if (lane == 0) lossrow[int64_t(j) * B + b] = (mx + logf(se)) - ly;
  float dl[10];
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    dl[k] = (expf(lg[k] - mx) / se - (k == y ? 1.f : 0.f)) / float(B);
    if (lane == 0) dls[warp][k] = dl[k];
  }
  float* Gb = G + (int64_t(j) * B + b) * 16 * 512;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int c = lane + 32 * i;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 10; ++k) s += dl[k] * W[k * 512 + c];
    const float g = s / 16.0f;
    for (int p = 0; p < 16; ++p) Gb[p * 512 + c] = g;
  }
  __syncthreads();
  // fc partials of this CTA's 8 samples: [10][512] weights then [10] bias
  float* fp = fpart + j * fpart_ls + int64_t(blk) * (5120 + 16);
  for (int e = threadIdx.x; e < 5120; e += 256) {
    const int k = e / 512, c = e % 512;
    float s = 0.f;
    for (int w = 0; w < 8; ++w) s += dls[w][k] * hs[w][c];
    fp[e] = s;
  }
  if (threadIdx.x < 10) {
    float s = 0.f;
    for (int w = 0; w < 8; ++w) s += dls[w][threadIdx.x];
    fp[5120 + threadIdx.x] = s;
  }
}

// dst[c] = sum_blk part[lane][blk][c] (fixed order) -> grads
__global__ void rn_reduce_kernel(const LaneState* __restrict__ lanes, const float* __restrict__ part,
                                 int64_t part_ls, int64_t blk_st, int nblk, int C, float* __restrict__ grads,
                                 int64_t pstride, int64_t off0, int split, int64_t off1) {
  pdl_begin();
  const int c = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (!lanes[j].active || c >= C) return;
  const float* p = part + j * part_ls + c;
  float s = 0.f;
  for (int b = 0; b < nblk; ++b) s += p[int64_t(b) * blk_st];
  grads[j * pstride + (c < split ? off0 + c : off1 + (c - split))] = s;
}

__global__ void __launch_bounds__(512) rn_loss_kernel(LaneState* __restrict__ lanes, int B,
                                                      const float* __restrict__ lossrow, float* __restrict__ loss,
                                                      int max_steps, float* __restrict__ last_loss) {
  pdl_begin();
  const int j = blockIdx.x;
  if (!lanes[j].active || threadIdx.x) return;
  float t = 0.f;
  for (int b = 0; b < B; ++b) t += lossrow[int64_t(j) * B + b];
  const float Lm = t / float(B);
  LaneState& ls = lanes[j];
  loss[int64_t(j) * max_steps + ls.steps_done] = Lm;
  last_loss[j] = Lm;
  lane_step_scalars(ls);
}

// ----------------------------------------------------------- BN backward ----
// g = G [mask > 0]; partials per 512-row block: sum g, sum g xh [, sum g xhd].
// CTA = 256 threads = (C/8 channel groups) x (256 / (C/8) row sub-lanes); a
// thread owns 8 channels (16-byte bf16 / 2 x 16-byte fp32 loads), strides
// over the block's rows, and the row sub-lanes are summed in order via smem.
constexpr int BNB_ROWS = 512;
__global__ void __launch_bounds__(256) rn_bn_bwd_reduce_kernel(
    const LaneState* __restrict__ lanes, int64_t M, int C, const float* __restrict__ G,
    const uint16_t* __restrict__ mask, const uint16_t* __restrict__ y, const float* __restrict__ st,
    const uint16_t* __restrict__ yd, const float* __restrict__ std_, float* __restrict__ part, int64_t part_ls) {
  pdl_begin();
  const int blk = blockIdx.x, j = blockIdx.y;
  if (!lanes[j].active) return;
  const int CG = C / 8, R = 256 / CG;
  const int cg = threadIdx.x % CG, sub = threadIdx.x / CG;
  const int c0 = cg * 8;
  const int K = yd ? 3 : 2;
  __shared__ float red[3 * 2048];  // [K][R][C] (R * C = 2048)
  float sg[8], sx[8], sd[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) sg[i] = sx[i] = sd[i] = 0.f;
  if (sub < R) {
    float mu[8], rs[8], mud[8], rsd[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      mu[i] = st[(int64_t(j) * 2) * C + c0 + i];
      rs[i] = st[(int64_t(j) * 2 + 1) * C + c0 + i];
      mud[i] = yd ? std_[(int64_t(j) * 2) * C + c0 + i] : 0.f;
      rsd[i] = yd ? std_[(int64_t(j) * 2 + 1) * C + c0 + i] : 0.f;
    }
    const int64_t base = int64_t(j) * M * C;
    const int64_t r1 = min(M, int64_t(blk + 1) * BNB_ROWS);
#pragma unroll 2
    for (int64_t r = int64_t(blk) * BNB_ROWS + sub; r < r1; r += R) {
      const int64_t e = base + r * C + c0;
      const float4 g0 = *reinterpret_cast<const float4*>(G + e), g1 = *reinterpret_cast<const float4*>(G + e + 4);
      const uint4 mk = *reinterpret_cast<const uint4*>(mask + e), yy = *reinterpret_cast<const uint4*>(y + e);
      uint4 dd = make_uint4(0, 0, 0, 0);
      if (yd) dd = *reinterpret_cast<const uint4*>(yd + e);
      const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      const uint32_t mw[4] = {mk.x, mk.y, mk.z, mk.w}, yw[4] = {yy.x, yy.y, yy.z, yy.w};
      const uint32_t dw[4] = {dd.x, dd.y, dd.z, dd.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t sh = (i & 1) ? 0u : 16u;
        const float mv = __uint_as_float((mw[i >> 1] << sh) & 0xffff0000u);
        const float g = mv > 0.f ? gg[i] : 0.f;
        const float yv = __uint_as_float((yw[i >> 1] << sh) & 0xffff0000u);
        sg[i] += g;
        sx[i] += g * ((yv - mu[i]) * rs[i]);
        if (K == 3) {
          const float dv = __uint_as_float((dw[i >> 1] << sh) & 0xffff0000u);
          sd[i] += g * ((dv - mud[i]) * rsd[i]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      red[(0 * R + sub) * C + c0 + i] = sg[i];
      red[(1 * R + sub) * C + c0 + i] = sx[i];
      if (K == 3) red[(2 * R + sub) * C + c0 + i] = sd[i];
    }
  }
  __syncthreads();
  float* pp = part + j * part_ls + int64_t(blk) * K * C;
  for (int i = threadIdx.x; i < K * C; i += 256) {
    const int k = i / C, c = i % C;
    float s = 0.f;
    for (int r = 0; r < R; ++r) s += red[(k * R + r) * C + c];
    pp[i] = s;
  }
}

// sums[lane][k][C] = sum_blk partials (8 groups of strided blocks, then the
// groups in order); grads: dbeta = sum g, dgamma = sum g xh (and the
// shortcut BN's from k = 2, dbeta_d = sum g)
__global__ void __launch_bounds__(256) rn_bn_bwd_finish_kernel(
    const LaneState* __restrict__ lanes, const float* __restrict__ part, int64_t part_ls, int nblk, int K, int C,
    float* __restrict__ sums, float* __restrict__ grads, int64_t pstride, int64_t og, int64_t ob, int64_t ogd,
    int64_t obd) {
  pdl_begin();
  const int j = blockIdx.y;
  if (!lanes[j].active) return;
  const int cl = threadIdx.x & 31, g = threadIdx.x >> 5, c = blockIdx.x * 32 + cl;
  __shared__ float sh[3][8][32];
  float s[3] = {0.f, 0.f, 0.f};
  if (c < C) {
    const float* p = part + j * part_ls + c;
#pragma unroll 4
    for (int b = g; b < nblk; b += 8)
      for (int k = 0; k < K; ++k) s[k] += p[(int64_t(b) * K + k) * C];
  }
  for (int k = 0; k < 3; ++k) sh[k][g][cl] = s[k];
  __syncthreads();
  if (g == 0 && c < C) {
    float t[3] = {0.f, 0.f, 0.f};
    for (int q = 0; q < 8; ++q)
      for (int k = 0; k < K; ++k) t[k] += sh[k][q][cl];
    for (int k = 0; k < K; ++k) sums[(int64_t(j) * 3 + k) * 512 + c] = t[k];
    float* gr = grads + j * pstride;
    gr[ob + c] = t[0];
    gr[og + c] = t[1];
    if (K == 3) {
      gr[obd + c] = t[0];
      gr[ogd + c] = t[2];
    }
  }
}

// dy = bf16(gamma rstd ((g - sg/M) - xh (sgx/M))) [, dyd likewise] [, gx = g]
// computed as  a g + b (y - mu) + c  with per-channel a = gamma rstd,
// b = -gamma rstd^2 sgx/M, c = -gamma rstd sg/M staged in smem.
__global__ void __launch_bounds__(256) rn_bn_bwd_apply_kernel(
    const LaneState* __restrict__ lanes, int64_t M, int C, const float* __restrict__ G,
    const uint16_t* __restrict__ mask, const uint16_t* __restrict__ y, const float* __restrict__ st,
    const uint16_t* __restrict__ yd, const float* __restrict__ std_, const float* __restrict__ sums,
    const float* __restrict__ params, int64_t pstride, int64_t og, int64_t ogd, uint16_t* __restrict__ dy,
    uint16_t* __restrict__ dyd, float* __restrict__ gx) {
  pdl_begin();
  const int j = blockIdx.y;
  if (!lanes[j].active) return;
  __shared__ float cf[8][512];  // mu, a, b, c, mud, ad, bd, cd
  const float invM = 1.0f / float(M);
  const float* S = sums + int64_t(j) * 3 * 512;
  const float* P = params + j * pstride;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const float mu = st[(int64_t(j) * 2) * C + c], rs = st[(int64_t(j) * 2 + 1) * C + c];
    const float a = P[og + c] * rs;
    cf[0][c] = mu;
    cf[1][c] = a;
    cf[2][c] = -a * rs * (S[512 + c] * invM);
    cf[3][c] = -a * (S[c] * invM);
    if (yd) {
      const float mud = std_[(int64_t(j) * 2) * C + c], rsd = std_[(int64_t(j) * 2 + 1) * C + c];
      const float ad = P[ogd + c] * rsd;
      cf[4][c] = mud;
      cf[5][c] = ad;
      cf[6][c] = -ad * rsd * (S[1024 + c] * invM);
      cf[7][c] = -ad * (S[c] * invM);
    }
  }
  __syncthreads();
  const int64_t n8 = M * C / 8;
  const int64_t step = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i0 < n8; i0 += 2 * step) {
    const int64_t ii[2] = {i0, i0 + step};
    float4 g0[2], g1[2];
    uint4 mk[2], yy[2], dd[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      dd[h] = make_uint4(0, 0, 0, 0);
      if (ii[h] < n8) {
        const int64_t e = int64_t(j) * M * C + ii[h] * 8;
        g0[h] = *reinterpret_cast<const float4*>(G + e);
        g1[h] = *reinterpret_cast<const float4*>(G + e + 4);
        mk[h] = *reinterpret_cast<const uint4*>(mask + e);
        yy[h] = *reinterpret_cast<const uint4*>(y + e);
        if (yd) dd[h] = *reinterpret_cast<const uint4*>(yd + e);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (ii[h] >= n8) break;
      const int64_t e = int64_t(j) * M * C + ii[h] * 8;
      const int c0 = int((ii[h] * 8) & (C - 1));
      const float gg[8] = {g0[h].x, g0[h].y, g0[h].z, g0[h].w, g1[h].x, g1[h].y, g1[h].z, g1[h].w};
      const uint32_t mw[4] = {mk[h].x, mk[h].y, mk[h].z, mk[h].w}, yw[4] = {yy[h].x, yy[h].y, yy[h].z, yy[h].w};
      const uint32_t dw[4] = {dd[h].x, dd[h].y, dd[h].z, dd[h].w};
      float g[8], o1[8], o2[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int c = c0 + k;
        const uint32_t sh = (k & 1) ? 0u : 16u;
        const float mv = __uint_as_float((mw[k >> 1] << sh) & 0xffff0000u);
        g[k] = mv > 0.f ? gg[k] : 0.f;
        const float yv = __uint_as_float((yw[k >> 1] << sh) & 0xffff0000u);
        o1[k] = cf[1][c] * g[k] + cf[2][c] * (yv - cf[0][c]) + cf[3][c];
        if (yd) {
          const float dv = __uint_as_float((dw[k >> 1] << sh) & 0xffff0000u);
          o2[k] = cf[5][c] * g[k] + cf[6][c] * (dv - cf[4][c]) + cf[7][c];
        }
      }
      *reinterpret_cast<uint4*>(dy + e) = make_uint4(pack_bf2(o1[0], o1[1]), pack_bf2(o1[2], o1[3]),
                                                     pack_bf2(o1[4], o1[5]), pack_bf2(o1[6], o1[7]));
      if (yd)
        *reinterpret_cast<uint4*>(dyd + e) = make_uint4(pack_bf2(o2[0], o2[1]), pack_bf2(o2[2], o2[3]),
                                                        pack_bf2(o2[4], o2[5]), pack_bf2(o2[6], o2[7]));
      if (gx) {
        *reinterpret_cast<float4*>(gx + e) = make_float4(g[0], g[1], g[2], g[3]);
        *reinterpret_cast<float4*>(gx + e + 4) = make_float4(g[4], g[5], g[6], g[7]);
      }
    }
  }
}

// ------------------------------------------------------------ stem wgrad ----
// partial[lane][img][co][27] = sum_{pix of image} dy0[pix][co] x[pix + tap][ci]
__global__ void __launch_bounds__(256) rn_stem_wgrad_kernel(const LaneState* __restrict__ lanes, int B,
                                                            const uint16_t* __restrict__ x,
                                                            const uint16_t* __restrict__ dy,
                                                            float* __restrict__ part, int64_t part_ls) {
  pdl_begin();
  const int img = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  if (!lanes[j].active) return;
  __shared__ float xs[34][34][3];
  __shared__ float ds[32][64];
  const uint16_t* xi = x + (int64_t(j) * B + img) * IMG;
  for (int i = tid; i < 34 * 34 * 3; i += 256) {
    const int c = i % 3, xx = (i / 3) % 34, yy = i / 102;
    const int gy = yy - 1, gx = xx - 1;
    xs[yy][xx][c] = (gy >= 0 && gy < 32 && gx >= 0 && gx < 32) ? bf2f(xi[(gy * 32 + gx) * 3 + c]) : 0.f;
  }
  // thread (co, ci) (192 of 256 threads): the 9 taps of its (co, ci) with the
  // 3x3 input window sliding along the row in registers (3 new x values and
  // 9 FMAs per pixel)
  const int co = tid & 63, ci = tid >> 6;
  float acc[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const uint16_t* dyi = dy + (int64_t(j) * B + img) * 1024 * 64;
  // one 16-byte dy vector per thread per row (32 px x 64 ch = 256 x 8 bf16),
  // the next row's vector in flight while this row is consumed
  uint4 nxt = reinterpret_cast<const uint4*>(dyi)[tid];
  for (int row = 0; row < 32; ++row) {
    const uint4 cur = nxt;
    if (row + 1 < 32) nxt = reinterpret_cast<const uint4*>(dyi + (row + 1) * 32 * 64)[tid];
    __syncthreads();
    {
      const uint32_t w4[4] = {cur.x, cur.y, cur.z, cur.w};
      float* dst = &ds[tid >> 3][(tid & 7) * 8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        dst[2 * e] = __uint_as_float(w4[e] << 16);
        dst[2 * e + 1] = __uint_as_float(w4[e] & 0xffff0000u);
      }
    }
    __syncthreads();
    if (ci < 3) {
      float wv[3][3];
#pragma unroll
      for (int kh = 0; kh < 3; ++kh) {
        wv[kh][1] = xs[row + kh][0][ci];
        wv[kh][2] = xs[row + kh][1][ci];
      }
#pragma unroll 4
      for (int px = 0; px < 32; ++px) {
#pragma unroll
        for (int kh = 0; kh < 3; ++kh) {
          wv[kh][0] = wv[kh][1];
          wv[kh][1] = wv[kh][2];
          wv[kh][2] = xs[row + kh][px + 2][ci];
        }
        const float d = ds[px][co];
#pragma unroll
        for (int kh = 0; kh < 3; ++kh)
#pragma unroll
          for (int kw = 0; kw < 3; ++kw) acc[kh * 3 + kw] = fmaf(d, wv[kh][kw], acc[kh * 3 + kw]);
      }
    }
  }
  if (ci < 3) {  // partial[co][tap * 3 + ci] (tap = kh * 3 + kw)
    float* pp = part + j * part_ls + int64_t(img) * 1728 + co * 27;
#pragma unroll
    for (int t = 0; t < 9; ++t) pp[t * 3 + ci] = acc[t];
  }
}

// ------------------------------------------------------------- GEMM glue ----
inline bool getenv_flag(const char* n) {
  const char* v = getenv(n);
  return v && v[0] && v[0] != '0';
}

inline void pix_box(int H, int W, int npix, int& bx, int& by, int& bb) {
  bx = W;
  by = std::min(H, npix / W);
  bb = npix / (bx * by);
}

}  // namespace

// activation map over [lane][B][H][W][C] (stride-1 view) or its (py, px)
// phase (stride-2 view), box (64, bx, by, bb, 1)
static int act_map_l(CUtensorMap* m, const uint16_t* base, int64_t ls, int lanes, int B, int H, int W, int C,
                     int phase, int bx, int by, int bb) {
  uint64_t dims[5], st[4];
  const uint16_t* p = base;
  if (phase < 0) {
    dims[0] = C, dims[1] = W, dims[2] = H, dims[3] = B;
    st[0] = uint64_t(C) * 2, st[1] = uint64_t(W) * C * 2, st[2] = uint64_t(H) * W * C * 2;
  } else {
    const int py = phase >> 1, px = phase & 1;
    p = base + (int64_t(py) * W + px) * C;
    dims[0] = C, dims[1] = W / 2, dims[2] = H / 2, dims[3] = B;
    st[0] = uint64_t(2) * C * 2, st[1] = uint64_t(2) * W * C * 2, st[2] = uint64_t(H) * W * C * 2;
  }
  dims[4] = uint64_t(lanes);
  st[3] = uint64_t(ls) * 2;
  return make_tmap_bf16_5d(m, p, dims, st, 64, uint32_t(bx), uint32_t(by), uint32_t(bb));
}

namespace {

#ifndef TLK_TRY
#define TLK_TRY(x)              \
  do {                          \
    if (int rc_ = (x)) return rc_; \
  } while (0)
#endif

int enqueue_bn_stats(Pack& p, cudaStream_t st, RnBufs& R, int P, int C, float* stats) {
  const int S = (P + STAT_PER_CTA - 1) / STAT_PER_CTA;
  TLK_CHECK(C <= 32 * STAT_MAX_CBLK && int64_t(S) * 3 * C <= R.stat2_ls, TLK_EINVAL, "bn stats: %d x %d", P, C);
  TLK_CUDA(launch(rn_bn_stats_kernel, dim3((C + 31) / 32, S, p.lanes), 256, 0, st, p.lane_dev, R.part, R.part_ls, P, C,
                  R.stat2, R.stat2_ls, R.stat_cnt, stats));
  return TLK_OK;
}

// stride-1 3x3 conv on a grid whose 128-pixel tiles are whole rows of one
// image with 8-row-aligned tap shifts: the halo mode of ConvGemm applies
inline bool halo_ok(const ConvL& L) {
  return L.stride == 1 && L.k == 3 && (L.W == 16 || L.W == 32) && 128 / L.W <= L.H && !getenv_flag("TLK_NO_HALO");
}

template <int BN, bool HALO = false>
int conv_fwd(Pack& p, cudaStream_t st, RnBufs& R, ConvL& L, const uint16_t* x, const char* name) {
  using G = ConvGemm<BN, CONV_FWD, HALO>;
  G g{};
  g.lanes = p.lane_dev;
  g.Hr = L.Ho, g.Wr = L.Wo;
  g.ksz = L.k, g.pad = (L.k - 1) / 2, g.stride = L.stride;
  g.cin_blk = L.cin / 64, g.cout_blk = L.cout / 64;
  int bx, by, bb;
  pix_box(L.Ho, L.Wo, 128, bx, by, bb);
  const int64_t xls = R.act_ls(L.H, L.W, L.cin);
  int rc = 0;
  if (HALO) {
    rc = act_map_l(&g.ta[0], x, xls, p.lanes, R.B, L.H, L.W, L.cin, -1, L.W, 128 / L.W + 2, 1);
  } else if (L.stride == 1) {
    rc = act_map_l(&g.ta[0], x, xls, p.lanes, R.B, L.H, L.W, L.cin, -1, bx, by, bb);
  } else {
    for (int ph = 0; ph < 4 && !rc; ++ph)
      rc = act_map_l(&g.ta[ph], x, xls, p.lanes, R.B, L.H, L.W, L.cin, ph, bx, by, bb);
  }
  if (rc) return rc;
  {
    const int taps = L.k * L.k;
    const uint64_t dims[5] = {uint64_t(taps) * L.cin, uint64_t(L.cout), uint64_t(p.lanes), 1, 1};
    const uint64_t s[4] = {uint64_t(taps) * L.cin * 2, uint64_t(p.stride) * 2, 0, 0};
    rc = make_tmap_bf16_5d(&g.tb[0], p.wbf + p.tinfo[L.t_w].off, dims, s, 64, BN);
    if (rc) return rc;
  }
  const int64_t M = int64_t(R.B) * L.Ho * L.Wo;
  g.mt = int(M / GEMM_BM);
  g.nt = L.cout / BN;
  g.nz = 1;
  g.ntiles = g.mt * g.nt * p.lanes;
  g.kblocks = (HALO ? 3 : L.k * L.k) * g.cin_blk;
  g.out = L.y;
  g.out_ls = M * L.cout;
  g.rows = int(M);
  g.cols = L.cout;
  g.part = R.part;
  g.part_ls = R.part_ls;
  TLK_CUDA(launch_tgemm(g, R.sms, st));
  p.mark(st, name);
  // statistics of this conv's output
  const int P = g.mt * 4;
  TLK_TRY(enqueue_bn_stats(p, st, R, P, L.cout, L.stats));
  TLK_CUDA(cudaGetLastError());
  p.mark(st, "bn_stats");
  return TLK_OK;
}

// dgrad: out[pix(H x W)][cin] (=|+=) sum dY[..][cout] WT ; fp32
template <int BN, bool HALO = false>
int conv_dgrad(Pack& p, cudaStream_t st, RnBufs& R, ConvL& L, const uint16_t* dY, float* out, int accumulate,
               const char* name) {
  using G = ConvGemm<BN, CONV_DGRAD, HALO>;
  G g{};
  g.lanes = p.lane_dev;
  g.ksz = L.k, g.pad = (L.k - 1) / 2, g.stride = L.stride;
  g.cin_blk = L.cin / 64, g.cout_blk = L.cout / 64;
  // GEMM rows: input pixels (stride 1) or one phase grid (stride 2)
  g.Hr = L.stride == 1 ? L.H : L.Ho;
  g.Wr = L.stride == 1 ? L.W : L.Wo;
  int bx, by, bb;
  pix_box(g.Hr, g.Wr, 128, bx, by, bb);
  int rc = HALO ? act_map_l(&g.ta[0], dY, R.act_ls(L.Ho, L.Wo, L.cout), p.lanes, R.B, L.Ho, L.Wo, L.cout, -1, L.Wo,
                            128 / L.Wo + 2, 1)
                : act_map_l(&g.ta[0], dY, R.act_ls(L.Ho, L.Wo, L.cout), p.lanes, R.B, L.Ho, L.Wo, L.cout, -1, bx, by, bb);
  if (rc) return rc;
  {
    const int taps = L.k * L.k;
    const uint64_t dims[5] = {uint64_t(L.cout), uint64_t(L.cin), uint64_t(taps), uint64_t(p.lanes), 1};
    const uint64_t s[4] = {uint64_t(L.cout) * 2, uint64_t(L.cin) * L.cout * 2, uint64_t(p.wt_stride) * 2, 0};
    rc = make_tmap_bf16_5d(&g.tb[0], p.wt + L.wt_off, dims, s, 64, BN);
    if (rc) return rc;
  }
  const int64_t Mr = int64_t(R.B) * g.Hr * g.Wr;
  g.mt = int(Mr / GEMM_BM);
  g.nt = L.cin / BN;
  g.nz = L.stride == 1 ? 1 : (L.k == 1 ? 1 : 4);
  g.ntiles = g.mt * g.nt * g.nz * p.lanes;
  g.kblocks = (HALO ? 3 : L.k * L.k) * g.cout_blk;
  g.out = out;
  g.out_ls = int64_t(R.B) * L.H * L.W * L.cin;
  g.rows = int(Mr);
  g.cols = L.cin;
  g.accumulate = accumulate;
  g.Hf = L.H, g.Wf = L.W;
  TLK_CUDA(launch_tgemm(g, R.sms, st));
  p.mark(st, name);
  return TLK_OK;
}

// wgrad: grads[co][tap][ci] = sum_pix dY[pix][co] X[pix + tap][ci]; split-K
template <int BN, int TG = 1>
int conv_wgrad(Pack& p, cudaStream_t st, RnBufs& R, ConvL& L, const uint16_t* dY, const uint16_t* X,
               const char* name) {
  using G = ConvGemm<BN, CONV_WGRAD, false, TG>;
  G g{};
  g.lanes = p.lane_dev;
  g.ksz = L.k, g.pad = (L.k - 1) / 2, g.stride = L.stride;
  g.cin_blk = L.cin / 64, g.cout_blk = L.cout / 64;
  g.Hr = L.Ho, g.Wr = L.Wo;
  int bx, by, bb;
  pix_box(L.Ho, L.Wo, 64, bx, by, bb);
  int rc = act_map_l(&g.ta[0], dY, R.act_ls(L.Ho, L.Wo, L.cout), p.lanes, R.B, L.Ho, L.Wo, L.cout, -1, bx, by, bb);
  if (rc) return rc;
  const int64_t xls = R.act_ls(L.H, L.W, L.cin);
  if (L.stride == 1) {
    rc = act_map_l(&g.tb[0], X, xls, p.lanes, R.B, L.H, L.W, L.cin, -1, bx, by, bb);
  } else {
    for (int ph = 0; ph < 4 && !rc; ++ph) rc = act_map_l(&g.tb[ph], X, xls, p.lanes, R.B, L.H, L.W, L.cin, ph, bx, by, bb);
  }
  if (rc) return rc;
  const int taps = L.k * L.k;
  g.mt = (L.cout + GEMM_BM - 1) / GEMM_BM;
  g.nt = TG > 1 ? 1 : L.cin / BN;
  g.kb_total = int(int64_t(R.B) * L.Ho * L.Wo / 64);
  // split-K count from the per-lane geometry only (never from the lane
  // count), so a job's summation order -- and its bits -- do not depend on
  // how many jobs share the pack
  const int lane_tiles = g.mt * g.nt * (taps / TG);
  int splits = std::max(1, std::min((64 + lane_tiles - 1) / lane_tiles, g.kb_total / 8));
  const int64_t wsize = int64_t(L.cout) * taps * L.cin;
  if (splits > 1 && int64_t(splits) * wsize > R.wpart_ls) splits = int(std::max<int64_t>(1, R.wpart_ls / wsize));
  g.kb_split = (g.kb_total + splits - 1) / splits;
  splits = (g.kb_total + g.kb_split - 1) / g.kb_split;
  g.splits = splits;
  g.nz = taps / TG * splits;
  g.ntiles = g.mt * g.nt * g.nz * p.lanes;
  g.kblocks = 0;
  g.taps = taps;
  g.rows = L.cout;
  g.cols = L.cin;
  const int64_t goff = p.tinfo[L.t_w].off;
  if (splits == 1) {
    g.out = p.grads + goff;
    g.out_ls = p.stride;
    g.split_st = 0;
  } else {
    g.out = R.wpart;
    g.out_ls = R.wpart_ls;
    g.split_st = wsize;
  }
  TLK_CUDA(launch_tgemm(g, R.sms, st));
  p.mark(st, name);
  if (splits > 1) {
    TLK_CUDA(launch(rn_reduce_kernel, dim3(int((wsize + 255) / 256), p.lanes), 256, 0, st, p.lane_dev, R.wpart, R.wpart_ls, wsize, splits, int(wsize), p.grads, p.stride, goff, int(wsize), goff));
    TLK_CUDA(cudaGetLastError());
    p.mark(st, "wgrad_reduce");
  }
  return TLK_OK;
}

// 256-wide N tiles halve the A-operand (activation) L2 traffic per MMA for
// the 256/512-channel layers (TLK_CONV_BN256=0 restores 128)
inline bool wide_n(int channels) { return channels >= 256 && !(getenv("TLK_CONV_BN256") && getenv("TLK_CONV_BN256")[0] == '0'); }

int conv_fwd_any(Pack& p, cudaStream_t st, RnBufs& R, ConvL& L, const uint16_t* x, const char* name) {
  if (wide_n(L.cout) && !halo_ok(L)) return conv_fwd<256>(p, st, R, L, x, name);
  if (halo_ok(L))
    return L.cout == 64 ? conv_fwd<64, true>(p, st, R, L, x, name) : conv_fwd<128, true>(p, st, R, L, x, name);
  return L.cout == 64 ? conv_fwd<64>(p, st, R, L, x, name) : conv_fwd<128>(p, st, R, L, x, name);
}
int conv_dgrad_any(Pack& p, cudaStream_t st, RnBufs& R, ConvL& L, const uint16_t* dY, float* out, int acc,
                   const char* name) {
  if (wide_n(L.cin) && !halo_ok(L)) return conv_dgrad<256>(p, st, R, L, dY, out, acc, name);
  if (halo_ok(L))
    return L.cin == 64 ? conv_dgrad<64, true>(p, st, R, L, dY, out, acc, name)
                       : conv_dgrad<128, true>(p, st, R, L, dY, out, acc, name);
  return L.cin == 64 ? conv_dgrad<64>(p, st, R, L, dY, out, acc, name)
                     : conv_dgrad<128>(p, st, R, L, dY, out, acc, name);
}
int conv_wgrad_any(Pack& p, cudaStream_t st, RnBufs& R, ConvL& L, const uint16_t* dY, const uint16_t* X,
                   const char* name) {
  if (wide_n(L.cin)) return conv_wgrad<256>(p, st, R, L, dY, X, name);
  if (L.cin == 64 && L.stride == 1 && L.k == 3 && !getenv_flag("TLK_NO_TAPGROUP"))
    return conv_wgrad<192, 3>(p, st, R, L, dY, X, name);
  return L.cin == 64 ? conv_wgrad<64>(p, st, R, L, dY, X, name) : conv_wgrad<128>(p, st, R, L, dY, X, name);
}

}  // namespace

// ------------------------------------------------------------- tensors ------
// oracle/resnet.py::tensors (kind 0 uniform(fan_in), 1 ones, 2 zeros)
void resnet_tensor_list(std::vector<std::pair<int64_t, int>>& cnt_fan, std::vector<int>& kinds) {
  auto add = [&](int64_t n, int fan, int kind) {
    cnt_fan.push_back({n, fan});
    kinds.push_back(kind);
  };
  add(64 * 27, 27, 0), add(64, 27, 1), add(64, 27, 2);
  const int C[4] = {64, 128, 256, 512};
  int cin = 64;
  for (int s = 0; s < 4; ++s)
    for (int b = 0; b < 2; ++b) {
      const int ci = b == 0 ? cin : C[s];
      add(int64_t(C[s]) * 9 * ci, 9 * ci, 0), add(C[s], 9 * ci, 1), add(C[s], 9 * ci, 2);
      add(int64_t(C[s]) * 9 * C[s], 9 * C[s], 0), add(C[s], 9 * C[s], 1), add(C[s], 9 * C[s], 2);
      if (b == 0 && s > 0) add(int64_t(C[s]) * ci, ci, 0), add(C[s], ci, 1), add(C[s], ci, 2);
      if (b == 1) cin = C[s];
    }
  add(5120, 512, 0), add(10, 512, 0);
}

// ------------------------------------------------------------- setup --------
int resnet_setup(Pack& p) {
  const int B = p.batch, L = p.lanes;
  auto* R = new RnBufs{};
  p.scratch = R;
  p.scratch_free = [](void* q) { delete static_cast<RnBufs*>(q); };
  R->B = B;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    R->sms = 148;
    cudaDeviceGetAttribute(&R->sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // conv table (tensor indices follow resnet_tensor_list)
  int t = 0;
  R->conv.push_back(ConvL{3, 64, 3, 1, 32, 32, 32, 32, 0, 1, 2});
  t = 3;
  const int C[4] = {64, 128, 256, 512};
  int cin = 64, res = 32;
  for (int s = 0; s < 4; ++s)
    for (int b = 0; b < 2; ++b) {
      const int stv = (b == 0 && s > 0) ? 2 : 1;
      const int ci = b == 0 ? cin : C[s];
      const int Ho = res / stv;
      Block bk{};
      bk.c1 = int(R->conv.size());
      R->conv.push_back(ConvL{ci, C[s], 3, stv, res, res, Ho, Ho, t, t + 1, t + 2});
      bk.c2 = int(R->conv.size());
      R->conv.push_back(ConvL{C[s], C[s], 3, 1, Ho, Ho, Ho, Ho, t + 3, t + 4, t + 5});
      t += 6;
      bk.cd = -1;
      if (b == 0 && s > 0) {
        bk.cd = int(R->conv.size());
        R->conv.push_back(ConvL{ci, C[s], 1, 2, res, res, Ho, Ho, t, t + 1, t + 2});
        t += 3;
      }
      R->blk.push_back(bk);
      res = Ho;
      if (b == 1) cin = C[s];
    }
  // transposed weight arena (dgrad B operands) for every tensor-core conv
  int64_t wt = 0;
  for (size_t i = 1; i < R->conv.size(); ++i) {
    R->conv[i].wt_off = wt;
    wt = round_up(wt + int64_t(R->conv[i].cout) * R->conv[i].k * R->conv[i].k * R->conv[i].cin, 64);
  }
  p.wt_stride = wt;
  // sizes
  struct Item {
    void** ptr;
    size_t bytes;
  };
  std::vector<Item> items;
  auto add = [&](void** ptr, size_t bytes) { items.push_back({ptr, (bytes + 255) & ~size_t(255)}); };
  add(reinterpret_cast<void**>(&R->xin), size_t(L) * B * IMG * 2);  // first: TLK_BUF_ACTS view
  add(reinterpret_cast<void**>(&p.wt), size_t(L) * wt * 2);
  add(reinterpret_cast<void**>(&R->teacher), 10 * IMG);
  for (auto& c : R->conv) {
    add(reinterpret_cast<void**>(&c.y), size_t(L) * R->act_ls(c.Ho, c.Wo, c.cout) * 2);
    add(reinterpret_cast<void**>(&c.stats), size_t(L) * 2 * c.cout * 4);
  }
  add(reinterpret_cast<void**>(&R->a0), size_t(L) * R->act_ls(32, 32, 64) * 2);
  for (auto& bk : R->blk) {
    const ConvL& c2 = R->conv[bk.c2];
    add(reinterpret_cast<void**>(&bk.a1), size_t(L) * R->act_ls(c2.H, c2.W, c2.cin) * 2);
    add(reinterpret_cast<void**>(&bk.o), size_t(L) * R->act_ls(c2.Ho, c2.Wo, c2.cout) * 2);
  }
  const int64_t big = R->act_ls(32, 32, 64);  // largest activation (elements per lane)
  add(reinterpret_cast<void**>(&R->G0), size_t(L) * big * 4);
  add(reinterpret_cast<void**>(&R->G1), size_t(L) * big * 4);
  add(reinterpret_cast<void**>(&R->da), size_t(L) * big * 4);
  add(reinterpret_cast<void**>(&R->dy), size_t(L) * big * 2);
  add(reinterpret_cast<void**>(&R->dyd), size_t(L) * big * 2);
  // partials: conv stats (M/32 x 2C), BN backward (M/256 x 3C), head, stem wgrad
  int64_t pl = 0;
  for (auto& c : R->conv) {
    const int64_t M = int64_t(B) * c.Ho * c.Wo;
    pl = std::max({pl, M / 32 * 2 * c.cout, (M + BNB_ROWS - 1) / BNB_ROWS * 3 * c.cout});
  }
  pl = std::max({pl, int64_t(B / 8) * (5120 + 16), int64_t(B) * 1728});
  R->part_ls = round_up(pl, 64);
  add(reinterpret_cast<void**>(&R->part), size_t(L) * R->part_ls * 4);
  add(reinterpret_cast<void**>(&R->sums), size_t(L) * 3 * 512 * 4);
  {
    int64_t smax = 1;
    for (auto& c : R->conv) {
      const int64_t P = int64_t(B) * c.Ho * c.Wo / 32;
      smax = std::max(smax, (P + STAT_PER_CTA - 1) / STAT_PER_CTA * 3 * c.cout);
    }
    R->stat2_ls = round_up(smax, 64);
    add(reinterpret_cast<void**>(&R->stat2), size_t(L) * R->stat2_ls * 4);
    add(reinterpret_cast<void**>(&R->stat_cnt), size_t(L) * STAT_MAX_CBLK * 4);
  }
  R->wpart_ls = int64_t(8) * 64 * 9 * 128;  // split-K partials: up to 8 x (128 x 9 x 64) or fewer splits
  add(reinterpret_cast<void**>(&R->wpart), size_t(L) * R->wpart_ls * 4);
  add(reinterpret_cast<void**>(&R->lossrow), size_t(L) * B * 4);
  const bool snaps = (p.flags & TLK_PACK_SNAPSHOTS) != 0;
  if (snaps) {
    for (auto& bk : R->blk) {
      const ConvL& c2 = R->conv[bk.c2];
      add(reinterpret_cast<void**>(&bk.snapG), size_t(L) * R->act_ls(c2.Ho, c2.Wo, c2.cout) * 4);
    }
    add(reinterpret_cast<void**>(&R->snap_stem), size_t(L) * R->act_ls(32, 32, 64) * 4);
  }
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
  // teacher (host restatement of the counter RNG, as oracle/resnet.py::teacher)
  {
    std::vector<int8_t> T(10 * IMG);
    const uint64_t key = rng_key(TEACHER_SEED, STREAM_RTEACHER, 0);
    for (int i = 0; i < 10 * IMG; ++i) T[i] = int8_t(int((rng_bits(key, uint64_t(i)) >> 60) & 15) - 8);
    TLK_CUDA(cudaMemcpy(R->teacher, T.data(), T.size(), cudaMemcpyHostToDevice));
  }
  // block inputs: a0 for block 0, previous block's output after that
  for (size_t i = 0; i < R->blk.size(); ++i) R->blk[i].xin = i == 0 ? R->a0 : R->blk[i - 1].o;
  // named buffers (tlk_pack_named): forward tensors and gradient snapshots
  p.name_buf("xin", R->xin, size_t(L) * B * IMG * 2);
  p.name_buf("a0", R->a0, size_t(L) * R->act_ls(32, 32, 64) * 2);
  for (size_t i = 0; i < R->conv.size(); ++i) {
    const ConvL& c = R->conv[i];
    p.name_buf("conv" + std::to_string(i) + ".y", c.y, size_t(L) * R->act_ls(c.Ho, c.Wo, c.cout) * 2);
    p.name_buf("conv" + std::to_string(i) + ".stats", c.stats, size_t(L) * 2 * c.cout * 4);
  }
  for (size_t i = 0; i < R->blk.size(); ++i) {
    const Block& bk = R->blk[i];
    const ConvL& c2 = R->conv[bk.c2];
    p.name_buf("blk" + std::to_string(i) + ".a1", bk.a1, size_t(L) * R->act_ls(c2.H, c2.W, c2.cin) * 2);
    p.name_buf("blk" + std::to_string(i) + ".o", bk.o, size_t(L) * R->act_ls(c2.Ho, c2.Wo, c2.cout) * 2);
    if (snaps)
      p.name_buf("blk" + std::to_string(i) + ".G", bk.snapG, size_t(L) * R->act_ls(c2.Ho, c2.Wo, c2.cout) * 4);
  }
  if (snaps) p.name_buf("stem.G", R->snap_stem, size_t(L) * R->act_ls(32, 32, 64) * 4);
  p.launches_per_step = 0;
  // bf16 [lanes][batch][32][32][3] images, then int32 [lanes][batch] labels
  p.host_segs = {{R->xin, size_t(L) * B * IMG * 2}, {p.labels, size_t(L) * B * 4}};
  return TLK_OK;
}

// ------------------------------------------------------------- one step -----
int resnet_enqueue_step(Pack& p, cudaStream_t st) {
  RnBufs& R = *static_cast<RnBufs*>(p.scratch);
  const int B = R.B, Lc = p.lanes;
  const LaneState* LS = p.lane_dev;
  const float* PR = p.params;
  const int64_t PS = p.stride;
  auto O = [&](int t) { return p.tinfo[t].off; };
  int count = 0;
  auto marked = [&](const char* name) {
    p.mark(st, name);
    ++count;
  };
  // elementwise BN kernels: ~one full wave over all lanes (8 CTAs of 256 per
  // SM), >= 4 vectors per thread, so the per-CTA channel-coefficient setup
  // is amortised
  auto ew_grid = [&](int64_t n8) {
    const int64_t cap = std::max<int64_t>(1, int64_t(R.sms) * 8 / Lc);
    return dim3(unsigned(std::clamp<int64_t>((n8 + 1023) / 1024, 1, cap)), Lc);
  };

  if (!p.host_input) {  // host-input packs: images and labels came from tlk_step_host_blob
    TLK_CUDA(launch(rn_inputs_kernel, dim3(B, Lc), 256, 0, st, LS, B, R.teacher, R.xin, p.labels));
    TLK_CUDA(cudaGetLastError());
    marked("inputs");
  }
  {  // dgrad weight layouts from this step's bf16 shadow
    WtTable tab{};
    int tiles = 0;
    for (size_t i = 1; i < R.conv.size(); ++i) {
      const ConvL& c = R.conv[i];
      WtEntry& e = tab.e[tab.n++];
      e.src = O(c.t_w);
      e.dst = c.wt_off;
      e.cout = c.cout;
      e.taps = c.k * c.k;
      e.cin = c.cin;
      e.tiles0 = tiles;
      if (c.cin % 64 || c.cout % 64) return fail(TLK_EINVAL, "resnet: conv %zu channels not multiples of 64", i);
      tiles += e.taps * (c.cout / 64) * (c.cin / 64);
    }
    tab.tiles = tiles;
    TLK_CUDA(launch(rn_wt_transpose_kernel, dim3(tiles, Lc), 256, 0, st, LS, tab, p.wbf, PS, p.wt, p.wt_stride));
    TLK_CUDA(cudaGetLastError());
    marked("wt_transpose");
  }
  // ---- forward
  ConvL& S0 = R.conv[0];
  TLK_CUDA(launch(rn_stem_fwd_kernel, dim3(B * 8, Lc), 256, 0, st, LS, B, R.xin, p.wbf, PS, O(S0.t_w), S0.y, R.part, R.part_ls));
  TLK_CUDA(cudaGetLastError());
  marked("stem_fwd");
  TLK_TRY(enqueue_bn_stats(p, st, R, B * 8 * 4, 64, S0.stats));
  TLK_CUDA(cudaGetLastError());
  marked("bn_stats");
  {
    const int64_t n8 = R.act_ls(32, 32, 64) / 8;
    TLK_CUDA(launch(rn_bn_act_kernel, ew_grid(n8), 256, 0, st, LS, n8, 64, S0.y, S0.stats, PR, PS, O(S0.t_g), O(S0.t_b), 0,
                                                  nullptr, nullptr, 0, 0, R.a0));
    TLK_CUDA(cudaGetLastError());
    marked("bn_act");
  }
  for (auto& bk : R.blk) {
    ConvL &c1 = R.conv[bk.c1], &c2 = R.conv[bk.c2];
    int rc = conv_fwd_any(p, st, R, c1, bk.xin, "conv_fwd");
    if (rc) return rc;
    count += 2;
    const int64_t n8a = R.act_ls(c1.Ho, c1.Wo, c1.cout) / 8;
    TLK_CUDA(launch(rn_bn_act_kernel, ew_grid(n8a), 256, 0, st, LS, n8a, c1.cout, c1.y, c1.stats, PR, PS, O(c1.t_g), O(c1.t_b),
                                                   0, nullptr, nullptr, 0, 0, bk.a1));
    TLK_CUDA(cudaGetLastError());
    marked("bn_act");
    rc = conv_fwd_any(p, st, R, c2, bk.a1, "conv_fwd");
    if (rc) return rc;
    count += 2;
    if (bk.cd >= 0) {
      ConvL& cd = R.conv[bk.cd];
      rc = conv_fwd_any(p, st, R, cd, bk.xin, "conv_fwd_ds");
      if (rc) return rc;
      count += 2;
      TLK_CUDA(launch(rn_bn_act_kernel, ew_grid(n8a), 256, 0, st, LS, n8a, c2.cout, c2.y, c2.stats, PR, PS, O(c2.t_g),
                                                     O(c2.t_b), 2, cd.y, cd.stats, O(cd.t_g), O(cd.t_b), bk.o));
    } else {
      TLK_CUDA(launch(rn_bn_act_kernel, ew_grid(n8a), 256, 0, st, LS, n8a, c2.cout, c2.y, c2.stats, PR, PS, O(c2.t_g),
                                                     O(c2.t_b), 1, bk.xin, nullptr, 0, 0, bk.o));
    }
    TLK_CUDA(cudaGetLastError());
    marked("bn_act_res");
  }
  // ---- head
  const int t_fcw = int(p.tinfo.size()) - 2, t_fcb = t_fcw + 1;
  float* G = R.G0;
  float* Gx = R.G1;
  TLK_CUDA(launch(rn_head_kernel, dim3(Lc, B / 8), 256, 0, st, LS, B, R.blk.back().o, p.labels, PR, PS, O(t_fcw), O(t_fcb), G,
                                                  R.lossrow, R.part, R.part_ls));
  TLK_CUDA(cudaGetLastError());
  marked("head");
  TLK_CUDA(launch(rn_reduce_kernel, dim3((5130 + 255) / 256, Lc), 256, 0, st, LS, R.part, R.part_ls, 5136, B / 8, 5130, p.grads,
                                                                  PS, O(t_fcw), 5120, O(t_fcb)));
  TLK_CUDA(cudaGetLastError());
  marked("fc_reduce");
  TLK_CUDA(launch(rn_loss_kernel, Lc, 32, 0, st, p.lane_dev, B, R.lossrow, p.loss, p.max_steps, p.last_loss));
  TLK_CUDA(cudaGetLastError());
  marked("loss");

  // ---- backward
  auto bn_bwd = [&](const float* Gin, const uint16_t* mask, ConvL& c, ConvL* cd, uint16_t* dy, uint16_t* dyd,
                    float* gx) -> int {
    const int64_t M = int64_t(B) * c.Ho * c.Wo;
    const int nblk = int((M + BNB_ROWS - 1) / BNB_ROWS);
    const int K = cd ? 3 : 2;
    TLK_CUDA(launch(rn_bn_bwd_reduce_kernel, dim3(nblk, Lc), 256, 0, st, LS, M, c.cout, Gin, mask, c.y, c.stats,
                                                              cd ? cd->y : nullptr, cd ? cd->stats : nullptr,
                                                              R.part, R.part_ls));
    TLK_CUDA(cudaGetLastError());
    marked("bn_bwd_reduce");
    TLK_CUDA(launch(rn_bn_bwd_finish_kernel, dim3((c.cout + 31) / 32, Lc), 256, 0, st, LS, R.part, R.part_ls, nblk, K, c.cout, R.sums, p.grads, PS, O(c.t_g), O(c.t_b), cd ? O(cd->t_g) : 0,
        cd ? O(cd->t_b) : 0));
    TLK_CUDA(cudaGetLastError());
    marked("bn_bwd_finish");
    const int64_t n8 = M * c.cout / 8;
    TLK_CUDA(launch(rn_bn_bwd_apply_kernel, ew_grid(n8), 256, 0, st, LS, M, c.cout, Gin, mask, c.y, c.stats,
                                                        cd ? cd->y : nullptr, cd ? cd->stats : nullptr, R.sums, PR,
                                                        PS, O(c.t_g), cd ? O(cd->t_g) : 0, dy, dyd, gx));
    TLK_CUDA(cudaGetLastError());
    marked("bn_bwd_apply");
    return TLK_OK;
  };
  for (int i = int(R.blk.size()) - 1; i >= 0; --i) {
    Block& bk = R.blk[i];
    ConvL &c1 = R.conv[bk.c1], &c2 = R.conv[bk.c2];
    ConvL* cd = bk.cd >= 0 ? &R.conv[bk.cd] : nullptr;
    if (bk.snapG)
      TLK_CUDA(cudaMemcpyAsync(bk.snapG, G, size_t(Lc) * R.act_ls(c2.Ho, c2.Wo, c2.cout) * 4,
                               cudaMemcpyDeviceToDevice, st));
    // BN2 (+ shortcut BN) backward; identity blocks pass g straight to Gx
    int rc = bn_bwd(G, bk.o, c2, cd, R.dy, cd ? R.dyd : nullptr, cd ? nullptr : Gx);
    if (rc) return rc;
    rc = conv_wgrad_any(p, st, R, c2, R.dy, bk.a1, "conv_wgrad");
    if (rc) return rc;
    ++count;
    rc = conv_dgrad_any(p, st, R, c2, R.dy, R.da, 0, "conv_dgrad");
    if (rc) return rc;
    ++count;
    rc = bn_bwd(R.da, bk.a1, c1, nullptr, R.dy, nullptr, nullptr);
    if (rc) return rc;
    rc = conv_wgrad_any(p, st, R, c1, R.dy, bk.xin, "conv_wgrad");
    if (rc) return rc;
    ++count;
    // identity blocks: Gx already holds g (the shortcut gradient) -> accumulate;
    // downsample blocks: conv1's stride-2 dgrad covers every input pixel
    // (all four phases) and initialises Gx, the 1x1 shortcut adds its phase
    rc = conv_dgrad_any(p, st, R, c1, R.dy, Gx, cd ? 0 : 1, "conv_dgrad");
    if (rc) return rc;
    ++count;
    if (cd) {
      rc = conv_wgrad_any(p, st, R, *cd, R.dyd, bk.xin, "conv_wgrad_ds");
      if (rc) return rc;
      ++count;
      rc = conv_dgrad_any(p, st, R, *cd, R.dyd, Gx, 1, "conv_dgrad_ds");
      if (rc) return rc;
      ++count;
    }
    std::swap(G, Gx);
  }
  // stem: BN0 backward + SIMT wgrad
  {
    if (R.snap_stem)
      TLK_CUDA(cudaMemcpyAsync(R.snap_stem, G, size_t(Lc) * R.act_ls(32, 32, 64) * 4, cudaMemcpyDeviceToDevice, st));
    int rc = bn_bwd(G, R.a0, S0, nullptr, R.dy, nullptr, nullptr);
    if (rc) return rc;
    TLK_CUDA(launch(rn_stem_wgrad_kernel, dim3(B, Lc), 256, 0, st, LS, B, R.xin, R.dy, R.part, R.part_ls));
    TLK_CUDA(cudaGetLastError());
    marked("stem_wgrad");
    TLK_CUDA(launch(rn_reduce_kernel, dim3((1728 + 255) / 256, Lc), 256, 0, st, LS, R.part, R.part_ls, 1728, B, 1728, p.grads,
                                                                    PS, O(S0.t_w), 1728, O(S0.t_w)));
    TLK_CUDA(cudaGetLastError());
    marked("stem_wgrad_reduce");
  }
  {
    int rc = enqueue_optimizer(p, st);
    if (rc) return rc;
    ++count;
  }
  p.launches_per_step = count;
  return TLK_OK;
}

}  // namespace tlk
