// MNIST CNN pack (pytorch/examples Net without dropout), all lanes per launch.
//
//   x[28,28] -conv1 3x3 (1->32)+ReLU-> h1[26,26,32] -conv2 3x3 (32->64)+ReLU+maxpool2->
//   p2[12,12,64] -flatten (h,w,c)-> fc1 (9216->128)+ReLU -> h3 -> fc2 (128->10) + CE
//
// Launch sequence of one step (10 kernels, graph-captured):
//   inputs + conv1 fwd (CUDA cores, writes h1 in P28 planes) | conv2 fwd
//   (tcgen05, TMA-bulk patch + tap-shifted descriptors; epilogue bias+ReLU+
//   2x2 maxpool+argmax) | fc1 fwd (tcgen05 split-K) | fc1 reduce (+bias+ReLU)
//   + head (fc2+CE+bwd), one 8-CTA cluster per lane | fc1 wgrad (tcgen05) | fc1 dgrad (tcgen05; epilogue
//   = maxpool/ReLU backward scatter into dz2 P28 planes + conv2 bias partials)
//   | conv2 wgrad (tcgen05, 9 tap accumulators in TMEM) | conv2 dgrad
//   (tcgen05; epilogue ReLU mask -> dz1) | conv1 wgrad (CUDA cores) | fc1
//   wgrad + Adam | grad finalize (fixed-order reductions) + optimizer of the
//   remaining parameters + end of step
//
// The P28 layout and the conv2 kernels are described in conv_tc.cuh.
//
// Activation scratch (TLK_BUF_ACTS), each [lanes][...] contiguous, in order:
//   h1 P28 [4][npos][8] | p2 bf16 [B,12,12,64] | idx u8 [B,12,12,64]
//   (argmax | live<<2) | h3 bf16 [B,128] | dz3 bf16 [B,128] |
//   dz2 P28 [8][npos][8] | dz1 P28 [4][npos][8]      (npos = 32 + 784 B + 64)
#include <cstdlib>

#include <cooperative_groups.h>

#include "cnn_common.cuh"
#include "linear.cuh"
#include "inputs.cuh"

namespace tlk {
namespace {


// ------------------------------------------------------- inputs + conv1 -----
#ifndef TLK_C1F_PAIR
#define TLK_C1F_PAIR 1  // conv1 fwd: two positions per iteration
#endif
#ifndef TLK_C1W_UNROLL
#define TLK_C1W_UNROLL 2  // conv1 wgrad position loop unroll (each accumulator keeps its position order; 2: 0.1725 -> 0.1722 ms/step)
#endif
constexpr int C1W_UNROLL = TLK_C1W_UNROLL;
#ifndef TLK_C1F_MINB
#define TLK_C1F_MINB 1  // CTAs per SM the register budget must allow
#endif
// One CTA per (sample, lane): the sample's inputs (inputs.cuh: pixel codes,
// bf16 x for conv1 wgrad, teacher label) straight into shared memory, then
// conv1 in fp32 on the fp32 master weights, writing the 26x26 interior of
// h1's P28 planes (16 B = 8 channels per store).
__global__ void __launch_bounds__(256, TLK_C1F_MINB) conv1_fwd_kernel(const LaneState* __restrict__ lanes,
                                                        const int8_t* __restrict__ teacher,
                                                        uint8_t* __restrict__ px, int32_t* __restrict__ labels,
                                                        uint16_t* __restrict__ x, int host_input,
                                                        const float* __restrict__ params,
                                                        int64_t pstride, int64_t w_off,
                                                        int64_t b_off, CnnBufs buf) {
  TLK_KT(0, lanes[0].steps_done);
  pdl_begin();
  TLK_KT_WAITED();
  const int s = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  if (!lanes[j].active) return;
  __shared__ __align__(16) uint8_t pix[PIXELS];
  __shared__ int part[8][CLASSES];
  __shared__ __align__(16) float xs[784];
  __shared__ float ws[32 * 9];
  __shared__ float bs[32];
  for (int i = tid; i < 288; i += 256) ws[i] = params[j * pstride + w_off + i];
  if (tid < 32) bs[tid] = params[j * pstride + b_off + tid];
  sample_inputs<256>(lanes[j].seed, lanes[j].steps_done, s, size_t(j) * buf.B + s, host_input, teacher, px,
                     labels, x, pix, part);
  __syncthreads();
  for (int i = tid; i < 784; i += 256) xs[i] = float(pix[i]) * (1.0f / 256.0f);  // = bf16 x exactly
  __syncthreads();
  uint16_t* h1 = buf.h1 + int64_t(j) * 4 * buf.npos * 8;
  // thread = (4-channel half h of 8-channel chunk c, position group): its 36
  // weights live in registers (low register count -> more resident warps)
  const int c8 = tid & 7, c = c8 >> 1, h = c8 & 1;
  float w[4][9], bsum[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    bsum[e] = bs[c * 8 + h * 4 + e];
#pragma unroll
    for (int t = 0; t < 9; ++t) w[e][t] = ws[(c * 8 + h * 4 + e) * 9 + t];
  }
  // positions pos = g, g + 32, ...: (oh, ow) and both addresses advance
  // incrementally (32 = 26 + 6: one row and six columns, plus a row on wrap)
  uint2* hout = reinterpret_cast<uint2*>(h1 + (c * buf.npos + p28_pos(s, 1, 1)) * 8 + h * 4);
#if TLK_C1F_PAIR
  // two horizontally adjacent positions per iteration (pairs q = g, g + 32,
  // ... of the 13 x 26 pairs; 32 = 2 rows + 6 pairs): a 3 x 4 input window in
  // six 8-byte loads serves both; every output keeps its tap-ordered FMA chain
  int q = tid >> 3, oh = q / 13, pw = q % 13;
  for (; q < 338; q += 32) {
    const int ow = 2 * pw;
    const float* xp = xs + oh * 28 + ow;
    float xv[3][4];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const float2 a = *reinterpret_cast<const float2*>(xp + r * 28);
      const float2 b = *reinterpret_cast<const float2*>(xp + r * 28 + 2);
      xv[r][0] = a.x, xv[r][1] = a.y, xv[r][2] = b.x, xv[r][3] = b.y;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      float acc[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc[e] = 0.f;
#pragma unroll
        for (int t = 0; t < 9; ++t) acc[e] += xv[t / 3][t % 3 + u] * w[e][t];
      }
      hout[(oh * P28 + ow + u) * 2] =
          make_uint2(pack_bf2(fmaxf(acc[0] + bsum[0], 0.f), fmaxf(acc[1] + bsum[1], 0.f)),
                     pack_bf2(fmaxf(acc[2] + bsum[2], 0.f), fmaxf(acc[3] + bsum[3], 0.f)));
    }
    pw += 6;
    oh += 2;
    if (pw >= 13) {
      pw -= 13;
      oh += 1;
    }
  }
#else
  int pos = tid >> 3, oh = pos / 26, ow = pos % 26;
  for (; pos < 676; pos += 32) {
    const float* xp = xs + oh * 28 + ow;
    float xv[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) xv[t] = xp[(t / 3) * 28 + t % 3];
    float acc[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      acc[e] = 0.f;
#pragma unroll
      for (int t = 0; t < 9; ++t) acc[e] += xv[t] * w[e][t];
    }
    hout[(oh * P28 + ow) * 2] =
        make_uint2(pack_bf2(fmaxf(acc[0] + bsum[0], 0.f), fmaxf(acc[1] + bsum[1], 0.f)),
                   pack_bf2(fmaxf(acc[2] + bsum[2], 0.f), fmaxf(acc[3] + bsum[3], 0.f)));
    {  // next position: one row and six columns on, a row more on wrap (branch-free)
      const int wrap = ow >= 20;
      ow += 6 - 26 * wrap;
      oh += 1 + wrap;
    }
  }
#endif
}

// ------------------------------------------------------ fc1 fwd (TC) --------
// Z^T[o, b] partial sums over a K-split: part[lane][split][o][b].
struct Fc1Fwd {
  static constexpr int KT_ID = 2;  // TLK_KTRACE kernel id
  static constexpr int BN = 64, STAGES = 4;
  static constexpr bool A_MN = false, B_MN = false;
  static constexpr bool TILE_EPILOGUE = false;
  using Work = LaneWork;
  struct Carry {};
  CnnBufs buf;  // first: holds the (64-B aligned) tensor maps
  const LaneState* lanes;

  TLK_DEV bool work(Work& w) const {
    w.j = blockIdx.z / FC1_SPLITS;
    w.split = blockIdx.z % FC1_SPLITS;
    if (!lanes[w.j].active) return false;
    w.m0 = 0;
    w.n0 = 0;
    w.kb_begin = w.split * (144 / FC1_SPLITS);
    w.kb_end = w.kb_begin + 144 / FC1_SPLITS;
    return true;
  }
  TLK_DEV void prefetch() const {
    tma_prefetch_desc(&buf.w1_k);
    tma_prefetch_desc(&buf.p2m);
    tma_prefetch_desc(&buf.p2m_alt);
  }
  TLK_DEV void load_a(const Work& w, int kb, uint32_t dst, uint64_t* bar) const {
    tma_load_3d(dst, &buf.w1_k, kb * GEMM_BK, 0, w.j, bar);
  }
  TLK_DEV void load_b(const Work& w, int kb, uint32_t dst, uint64_t* bar) const {
    // this step's p2 buffer (conv2_tc_kernel<true>: odd steps -> p2_alt)
    tma_load_3d(dst, (lanes[w.j].steps_done & 1) ? &buf.p2m_alt : &buf.p2m, kb * GEMM_BK, 0, w.j, bar);
  }
  TLK_DEV void epilogue(const Work& w, int m, int n0, const float (&v)[32], Carry&) const {
    float* o = buf.part_fc1 + ((int64_t(w.j) * FC1_SPLITS + w.split) * 128 + m) * 64 + n0;
#pragma unroll
    for (int i = 0; i < 32; i += 4)
      *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  }
  TLK_DEV void finish(const Work&, int, Carry&) const {}
};


// -------------------------------------------- fc1 reduce + head (fused) -----
// One cluster of 8 CTAs per lane (16 hidden units each).  CTA r reduces its
// slice of h3 = bf16(relu(sum_s part[s] + b1)) from the split-K partials
// (split order fixed), forms the partial logits of its 16 units, and the
// cluster exchanges them through distributed shared memory: every CTA sums
// the 8 partials in rank order (+ b2), so all hold identical logits.  Then,
// as head_kernel (kernels.cu): softmax-CE, the loss / step scalars / fc2.b
// grad (rank 0), and the backward of its 16 units (dz3, fc2.w, fc1.b grads).
__global__ void __cluster_dims__(HEAD_CL, 1, 1) __launch_bounds__(256)
    cnn_head_kernel(LaneState* __restrict__ lanes, CnnBufs buf, const float* __restrict__ params,
                    float* __restrict__ grads, int64_t stride, int64_t b1_off, int64_t w_off, int64_t b_off,
                    const int32_t* __restrict__ labels, float* __restrict__ loss, int max_steps,
                    float* __restrict__ last_loss) {
  TLK_KT(3, lanes[0].steps_done);
  pdl_begin();
  TLK_KT_WAITED();
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int C = CLASSES, H = 128, HS = HEAD_HS;
  const int j = blockIdx.y, r = int(cluster.block_rank()), tid = threadIdx.x, B = buf.B;
  const int k0 = r * HS;
  const bool active = lanes[j].active;  // uniform over the cluster
  __shared__ float hs[64 * HS], zs[64 * HS], plog[64 * C], logit[64 * C], d[64 * C], lossb[64];
  __shared__ float wsl[C * HS];
  const float* P = params + j * stride;
  if (active) {
    for (int i = tid; i < C * HS; i += 256) wsl[i] = P[w_off + (i / HS) * H + k0 + i % HS];
    // h3 slice: (kk, b) = (i / 64, i % 64), 18 partials in split order
    for (int i = tid; i < HS * 64; i += 256) {
      const int kk = i >> 6, b = i & 63;
      if (b >= B) continue;
      const float* pp = buf.part_fc1 + int64_t(j) * FC1_SPLITS * 128 * 64 + (k0 + kk) * 64 + b;
      float sacc = 0.0f;
#pragma unroll
      for (int k = 0; k < FC1_SPLITS; ++k) sacc += pp[int64_t(k) * 128 * 64];
      const uint16_t hb = f2bf(fmaxf(sacc + P[b1_off + k0 + kk], 0.0f));
      buf.h3[j * buf.h3_st + b * 128 + k0 + kk] = hb;
      hs[b * HS + kk] = bf2f(hb);
    }
  }
  __syncthreads();
  if (active) {
    for (int i = tid; i < B * C; i += 256) {  // partial logits of this slice
      const int b = i / C, c = i % C;
      float sacc = 0.0f;
#pragma unroll
      for (int kk = 0; kk < HS; ++kk) sacc += hs[b * HS + kk] * wsl[c * HS + kk];
      plog[i] = sacc;
    }
  }
  cluster.sync();
  if (active) {
    for (int i = tid; i < B * C; i += 256) {
      float sacc = 0.0f;
#pragma unroll
      for (int q = 0; q < HEAD_CL; ++q) sacc += cluster.map_shared_rank(plog, q)[i];
      logit[i] = sacc + P[b_off + i % C];
    }
  }
  cluster.sync();  // every CTA has read the partials before any may exit
  if (!active) return;
  // this step's fc1.w update (fc1 wgrad + Adam, possibly after the lane's end
  // of step) is due, reading p2 of this step's parity
  if (r == 0 && tid == 0) lanes[j].fc1_due = 1 + (lanes[j].steps_done & 1);
  __syncthreads();
  if (tid < B) {
    const int y = labels[size_t(j) * B + tid];
    const float* l = logit + tid * C;
    float m = l[0];
    for (int c = 1; c < C; ++c) m = fmaxf(m, l[c]);
    float e[C], sacc = 0.0f;
    for (int c = 0; c < C; ++c) {
      e[c] = expf(l[c] - m);
      sacc += e[c];
    }
    lossb[tid] = (m + logf(sacc)) - l[y];
    for (int c = 0; c < C; ++c) d[tid * C + c] = (e[c] / sacc - (c == y ? 1.0f : 0.0f)) / float(B);
  }
  __syncthreads();
  float* G = grads + j * stride;
  if (r == 0) {
    if (tid < C) {
      float sacc = 0.0f;
      for (int b = 0; b < B; ++b) sacc += d[b * C + tid];
      G[b_off + tid] = sacc;
    }
  }
  uint16_t* dzj = buf.dz3 + j * buf.h3_st + k0;
  for (int i = tid; i < B * HS; i += 256) {
    const int b = i / HS, kk = i % HS;
    float dh = 0.0f;
#pragma unroll
    for (int c = 0; c < C; ++c) dh += d[b * C + c] * wsl[c * HS + kk];
    const uint16_t zb = f2bf(hs[i] > 0.0f ? dh : 0.0f);
    dzj[b * H + kk] = zb;
    zs[i] = bf2f(zb);
  }
  __syncthreads();
  for (int i = tid; i < HS * (C + 1); i += 256) {
    const int kk = i % HS, c = i / HS;  // c == C -> fc1.b grad
    float sacc = 0.0f;
    if (c < C) {
      for (int b = 0; b < B; ++b) sacc += d[b * C + c] * hs[b * HS + kk];
      G[w_off + c * H + k0 + kk] = sacc;
    } else {
      for (int b = 0; b < B; ++b) sacc += zs[b * HS + kk];
      G[b1_off + k0 + kk] = sacc;
    }
  }
  // last (off the critical path of this kernel): rank 0's loss and the
  // lane's optimizer scalars for this step (read by the later kernels)
  if (r == 0 && tid == 255) {
    float sacc = 0.0f;
    for (int b = 0; b < B; ++b) sacc += lossb[b];
    const float L = sacc / float(B);
    LaneState& ls = lanes[j];
    loss[size_t(j) * max_steps + ls.steps_done] = L;
    last_loss[j] = L;
    lane_step_scalars(ls);
  }
}

// ---------------------------------------------- fc1 dgrad + unpool (TC) -----
// dp2^T[f, b] = sum_o W[o, f] dz3[b, o]; epilogue scatters through the 2x2
// argmax (live bit = pooled value > 0) into the dz2 P28 planes and
// accumulates the conv2 bias-gradient partial colsum[f] = sum_b dz2 value.
struct Fc1Dgrad {
  static constexpr int KT_ID = 4;  // TLK_KTRACE kernel id
  static constexpr int BN = 64, STAGES = 2, THREADS = 256;
  static constexpr bool A_MN = true, B_MN = false;
  static constexpr bool TILE_EPILOGUE = true;
  using Work = LaneWork;
  struct Carry {};
  CnnBufs buf;
  const LaneState* lanes;

  TLK_DEV bool work(Work& w) const {
    w.j = blockIdx.z;
    if (!lanes[w.j].active) return false;
    w.m0 = blockIdx.x * GEMM_BM;
    w.n0 = 0;
    w.kb_begin = 0;
    w.kb_end = 2;  // K = 128
    w.split = 0;
    return true;
  }
  TLK_DEV void prefetch() const {
    tma_prefetch_desc(&buf.w1_mn);
    tma_prefetch_desc(&buf.dz3m);
  }
  TLK_DEV void load_a(const Work& w, int kb, uint32_t dst, uint64_t* bar) const {
    tma_load_3d(dst, &buf.w1_mn, w.m0, kb * GEMM_BK, w.j, bar);
    tma_load_3d(dst + 8192, &buf.w1_mn, w.m0 + 64, kb * GEMM_BK, w.j, bar);
  }
  TLK_DEV void load_b(const Work& w, int kb, uint32_t dst, uint64_t* bar) const {
    tma_load_3d(dst, &buf.dz3m, kb * GEMM_BK, 0, w.j, bar);
  }
  TLK_DEV void epilogue(const Work&, int, int, const float (&)[32], Carry&) const {}
  TLK_DEV void finish(const Work&, int, Carry&) const {}
  // tile = dp2^T[128 f][64 b] for f = two pooled positions x 64 channels.
  // Phase 1: a group of 8 lanes owns one (image b, 8-channel chunk ch) and
  // lane l writes window position r = l & 3 of pooled position pl = l >> 2:
  // the 16-B store of its dz2 P28 position is bf16(value) on the argmax
  // channels of a live pooled output, zero elsewhere.  A warp's stores are
  // then 64-B runs (two pooled positions' window row) instead of 32
  // scattered 16-B pieces.  The rounded value replaces the tile entry (lane
  // r == 0).  Phase 2: colsum[f] = sum_b (fixed order).
  TLK_DEV void tile_epilogue(const Work& w, float* tile, int ld) const {
    const int tid = threadIdx.x, B = buf.B;
    const int pos0 = w.m0 >> 6;
    const int l8 = tid & 7, pl = l8 >> 2, r = l8 & 3;
    const int pos = pos0 + pl, ph = pos / 12, pw = pos % 12;
    const int dr = r >> 1, dc = r & 1;
#pragma unroll 2
    for (int it = tid >> 3; it < 64 * 8; it += 32) {  // (b, ch) pairs; b is warp-uniform-valid (B % 8 == 0)
      const int b = it & 63, ch = it >> 6;
      const bool ok = b < B;
      const uint2 code2 = ok ? *reinterpret_cast<const uint2*>(buf.idx + w.j * buf.p2_st + int64_t(b) * 9216 +
                                                               pos * 64 + ch * 8)
                             : make_uint2(0u, 0u);
      const uint32_t cw[2] = {code2.x, code2.y};
      float* t0 = tile + (pl * 64 + ch * 8) * ld + b;
      uint16_t z[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t code = (cw[e >> 2] >> (8 * (e & 3))) & 0xFF;
        z[e] = (ok && (code & 4)) ? f2bf(t0[e * ld]) : uint16_t(0);
      }
      __syncwarp();  // every lane has read its tile entries before lane r == 0 rounds them in place
      uint32_t o[4];
#pragma unroll
      for (int e2 = 0; e2 < 4; ++e2) {
        const int e = 2 * e2;
        const int q0 = int((cw[e >> 2] >> (8 * (e & 3))) & 3), q1 = int((cw[(e + 1) >> 2] >> (8 * ((e + 1) & 3))) & 3);
        o[e2] = uint32_t(q0 == r ? z[e] : 0) | (uint32_t(q1 == r ? z[e + 1] : 0) << 16);
      }
      if (ok) {
        if (r == 0) {
#pragma unroll
          for (int e = 0; e < 8; ++e) t0[e * ld] = bf2f(z[e]);
        }
        uint16_t* plane = buf.dz2 + (int64_t(w.j) * 8 + ch) * buf.npos * 8;
        *reinterpret_cast<uint4*>(plane + (p28_pos(b, 2 * ph + 2 + dr, 2 * pw + 2 + dc)) * 8) =
            make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
    __syncthreads();
    if (tid < 128) {
      float s = 0.f;
      for (int b = 0; b < B; ++b) s += tile[tid * ld + b];
      buf.colsum[int64_t(w.j) * 9216 + w.m0 + tid] = s;
    }
  }
};

// ------------------------------------------- fc1 wgrad + optimizer (TC) -----
// dW1^T[f, o] = sum_b p2[b, f] dz3[b, o] (M = 128 input features f, N = all
// 128 outputs o, K = batch; both operands MN-major) with the lane's optimizer
// update applied as the epilogue: fc1.w is 98% of the CNN's parameters, so
// its fp32 gradient never makes the HBM round trip (stored only with
// TLK_PACK_WRITE_ALL_GRADS) and the kernel is an HBM stream of p, m, v (read
// + write) + the bf16 shadow.  Transposed on purpose: TMEM lane = f, so a warp
// holds 32 consecutive f of one output row and every global store is a full
// 128-B line.  Persistent (one CTA per SM), warp-specialised so the stream
// never waits on the GEMM:
//   warp 0   TMA producer: per tile the p2 / dz3 operand boxes, then the
//            tile's p, m, v in four 32-output chunks (3 x 16 KB each,
//            [32 o][128 f] fp32) into a 4-slot ring
//   warp 1   tcgen05.mma issuer, accumulator double-buffered in TMEM
//   warps 2-17  update: thread = (f = its TMEM lane, 8 outputs of the chunk):
//            p, m, v from the slot into registers (the slot is released at
//            once, so 3 slots stay in flight), the update with the optimizer
//            kind resolved once per chunk (IEEE-exact Adam is ~50 issued
//            instructions per element: the kernel is issue-bound), coalesced
//            128-B stores of p, m, v and the bf16 shadow.
// Must run after every reader of this step's fc1 weights (fc1 dgrad).
__global__ void __launch_bounds__(FWA_THREADS, 1) fc1_wgrad_adam_kernel(const __grid_constant__ Fc1WgradAdam p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t gfull, gempty, tfull[2], tempty[2];
  __shared__ __align__(8) uint64_t sfull[FWA_SLOTS], sempty[FWA_SLOTS];
  __shared__ uint32_t tmem_base_s;
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t slot_base = sbase + FWA_STAGE_BYTES;
  const uint8_t* slot_ptr = smem + FWA_STAGE_BYTES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef TLK_KTRACE  // the step being updated: lane 0's due parity vs its (possibly advanced) counter
  const int kt_s = p.lanes[0].steps_done, kt_d = p.lanes[0].fc1_due;
  TLK_KT(8, ((kt_s & 1) == ((kt_d - 1) & 1)) ? kt_s : kt_s - 1);
#endif
  if (tid == 0) {
    mbar_init(&gfull, 1);
    mbar_init(&gempty, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], FWA_UPD_WARPS);
    }
    for (int s = 0; s < FWA_SLOTS; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], FWA_UPD_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<256>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_begin();
  TLK_KT_WAITED();
  const uint32_t tmem = tmem_base_s;
  constexpr uint32_t IDESC = umma_idesc_bf16(GEMM_BM, 128, true, true);

  if (warp == 0) {
    if (lane == 0) {  // producer
      tma_prefetch_desc(&p.dz3m);
      tma_prefetch_desc(&p.p2m);
      tma_prefetch_desc(&p.p2m_alt);
      tma_prefetch_desc(&p.tp);
      tma_prefetch_desc(&p.tm);
      tma_prefetch_desc(&p.tv);
      int it = 0, cs = 0;
      for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const int j = t / FWA_FT, f0 = (t % FWA_FT) * 128;
        const int due = p.lanes[j].fc1_due;
        if (!due) continue;
        const CUtensorMap* p2m = due == 2 ? &p.p2m_alt : &p.p2m;
        for (int kb = 0; kb < p.kblocks; ++kb, ++it) {
          if (it >= 1) mbar_wait(&gempty, (it - 1) & 1);
          mbar_expect_tx(&gfull, FWA_STAGE_BYTES);
          tma_load_3d(sbase, p2m, f0, kb * GEMM_BK, j, &gfull);
          tma_load_3d(sbase + 8192, p2m, f0 + 64, kb * GEMM_BK, j, &gfull);
          tma_load_3d(sbase + 16384, &p.dz3m, 0, kb * GEMM_BK, j, &gfull);
          tma_load_3d(sbase + 24576, &p.dz3m, 64, kb * GEMM_BK, j, &gfull);
        }
        for (int c = 0; c < 4; ++c, ++cs) {
          const int sl = cs % FWA_SLOTS;
          if (cs >= FWA_SLOTS) mbar_wait(&sempty[sl], ((cs / FWA_SLOTS) - 1) & 1);
          const uint32_t d = slot_base + sl * FWA_SLOT_BYTES;
          mbar_expect_tx(&sfull[sl], FWA_SLOT_BYTES);
          tma_load_3d(d, &p.tp, f0, 32 * c, j, &sfull[sl]);
          tma_load_3d(d + FWA_CHUNK, &p.tm, f0, 32 * c, j, &sfull[sl]);
          tma_load_3d(d + 2 * FWA_CHUNK, &p.tv, f0, 32 * c, j, &sfull[sl]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int it = 0, lt = 0;
      for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        if (!p.lanes[t / FWA_FT].fc1_due) continue;
        const int acc = lt & 1;
        if (lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * 128;
        for (int kb = 0; kb < p.kblocks; ++kb, ++it) {
          mbar_wait(&gfull, it & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < GEMM_BK / 16; ++kk)
            mma_bf16(d, stage_desc_tma<GEMM_BM, true>(sbase, kk), stage_desc_tma<128, true>(sbase + 16384, kk),
                     IDESC, (kb > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&gempty);
        }
        mma_commit(&tfull[acc]);
        ++lt;
      }
    }
  } else {  // update warps: TMEM lane quarter q = warp & 3 (hardware rule) -> f; og = 8-output group
    const int q = warp & 3, og = (warp - 2) >> 2, fl = q * 32 + lane;
    int lt = 0, cs = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
      const int j = t / FWA_FT, f0 = (t % FWA_FT) * 128;
      if (!p.lanes[j].fc1_due) continue;
      const LaneState s = p.lanes[j];  // step scalars of the due step (the head writes the next ones)
      const int acc = lt & 1;
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      for (int c = 0; c < 4; ++c, ++cs) {
        const int o0 = 32 * c + 8 * og;  // this thread's outputs o0 .. o0+7
        float g[8];
        tmem_ld8(tmem + acc * 128 + o0 + (uint32_t(q * 32) << 16), g);
        if (c == 3) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        const int sl = cs % FWA_SLOTS;
        mbar_wait(&sfull[sl], (cs / FWA_SLOTS) & 1);
        const float* P = reinterpret_cast<const float*>(slot_ptr + sl * FWA_SLOT_BYTES);
        float pv[8], mv[8], vv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int off = (8 * og + i) * 128 + fl;  // [32 o][128 f]
          pv[i] = P[off];
          mv[i] = P[FWA_CHUNK / 4 + off];
          vv[i] = P[FWA_CHUNK / 2 + off];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[sl]);  // slot refillable as soon as it is read
        if (s.optimizer == TLK_OPT_SGD) {
#pragma unroll
          for (int i = 0; i < 8; ++i) opt_update_k<TLK_OPT_SGD>(s, pv[i], g[i], mv[i], vv[i]);
        } else if (s.optimizer == TLK_OPT_ADAMW) {
#pragma unroll
          for (int i = 0; i < 8; ++i) opt_update_k<TLK_OPT_ADAMW>(s, pv[i], g[i], mv[i], vv[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) opt_update_k<TLK_OPT_ADAM>(s, pv[i], g[i], mv[i], vv[i]);
        }
        const int64_t e = j * p.pstride + p.w_off + int64_t(o0) * 9216 + f0 + fl;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          p.params[e + int64_t(i) * 9216] = pv[i];
          p.m1[e + int64_t(i) * 9216] = mv[i];
          p.m2[e + int64_t(i) * 9216] = vv[i];
          p.wbf[e + int64_t(i) * 9216] = f2bf(pv[i]);
        }
        if (p.write_grads) {
#pragma unroll
          for (int i = 0; i < 8; ++i) p.grads[e + int64_t(i) * 9216] = g[i];
        }
      }
      ++lt;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<256>(tmem);
  if (tid == 0) {  // every CTA has read fc1_due: the last one clears it
    __threadfence();
    if (atomicAdd(p.cnt, 1u) == gridDim.x - 1) {
      __threadfence();
      for (int j = 0; j < p.ntiles / FWA_FT; ++j) p.lanes[j].fc1_due = 0;
      *p.cnt = 0;
    }
  }
}

// ------------------------------------------------ conv1 wgrad (SIMT) --------
// One CTA per (image, lane).  Thread = (8-channel chunk c, position group g):
// acc[e][t] over its positions (t<9: tap products with x, t=9: bias), then a
// fixed-order reduction over the 32 groups -> part1[lane][image][32][10].
__global__ void __launch_bounds__(C1W_THREADS) conv1_wgrad_kernel(const LaneState* __restrict__ lanes,
                                                          CnnBufs buf,
                                                          const uint16_t* __restrict__ x) {
  TLK_KT(7, lanes[0].steps_done);
  pdl_begin();
  TLK_KT_WAITED();
  const int b = blockIdx.x, j = blockIdx.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (!lanes[j].active) return;
  extern __shared__ __align__(16) uint16_t dzs_raw[];  // this image's dz1 planes (50 KB)
  uint16_t(*dzs)[P28_IMG * 8] = reinterpret_cast<uint16_t(*)[P28_IMG * 8]>(dzs_raw);
  __shared__ float xs[784];
  // the per-warp partials reuse the dz1 planes' space once every warp is done
  // with them: 53 KB per CTA -> 4 CTAs per SM, all 512 CTAs of 8 lanes in one wave
  static_assert(C1W_THREADS / 32 * 4 * 80 * 4 <= C1W_SMEM, "conv1 wgrad partials fit the dz1 space");
  float(*red)[4][80] = reinterpret_cast<float(*)[4][80]>(dzs_raw);
  // one barrier for the four chunk planes: every warp holds all four chunks, so
  // a wait per plane would diverge the warp (and turn its shuffles collective)
  __shared__ __align__(8) uint64_t bar;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(&bar, 4 * P28_IMG * 16);
    for (int c = 0; c < 4; ++c)
      tma_bulk_g2s(smem_u32(dzs[c]),
                   buf.dz1 + ((int64_t(j) * 4 + c) * buf.npos + p28_pos(b, 0, 0)) * 8,
                   P28_IMG * 16, &bar);
  }
  const uint4* xr = reinterpret_cast<const uint4*>(x + (size_t(j) * buf.B + b) * 784);
  if (tid < 98) {
    const uint4 v = xr[tid];
    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      xs[tid * 8 + 2 * e] = bf2f(uint16_t(wv[e] & 0xFFFF));
      xs[tid * 8 + 2 * e + 1] = bf2f(uint16_t(wv[e] >> 16));
    }
  }
  __syncthreads();
  // thread = (4-channel half h of chunk c, position group g): 40 accumulators
  // (acc[e][t<9] tap products with x, t = 9: bias), few registers -> 4 CTAs
  // of 8 warps per SM
  const int c8 = tid & 7, c = c8 >> 1, h = c8 & 1, g = tid >> 3;
  float acc[4][10];
#pragma unroll
  for (int e = 0; e < 4; ++e)
#pragma unroll
    for (int t = 0; t < 10; ++t) acc[e][t] = 0.f;
  mbar_wait(&bar, 0);
  static_assert(C1W_THREADS / 8 == 32, "conv1 wgrad walks positions g, g + 32, ...");
  const uint2* dzp = reinterpret_cast<const uint2*>(&dzs[c][(P28 + 1) * 8 + h * 4]);  // position (1, 1)
  int oh = g / 26, ow = g % 26;
#pragma unroll C1W_UNROLL
  for (int q = g; q < 676; q += 32) {
    const uint2 dv = dzp[(oh * P28 + ow) * 2];
    const float d[4] = {__uint_as_float(dv.x << 16), __uint_as_float(dv.x & 0xffff0000u),
                        __uint_as_float(dv.y << 16), __uint_as_float(dv.y & 0xffff0000u)};
    const float* xp = xs + oh * 28 + ow;
    float xv[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) xv[t] = xp[(t / 3) * 28 + t % 3];
    {  // next position: one row and six columns on, a row more on wrap (branch-free)
      const int wrap = ow >= 20;
      ow += 6 - 26 * wrap;
      oh += 1 + wrap;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
#pragma unroll
      for (int t = 0; t < 9; ++t) acc[e][t] += d[e] * xv[t];
      acc[e][9] += d[e];
    }
  }
  // reduce the 4 groups of this warp that share c8 (lanes c8, c8+8, ...), fixed order
#pragma unroll
  for (int e = 0; e < 4; ++e)
#pragma unroll
    for (int t = 0; t < 10; ++t) {
      float v = acc[e][t];
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      acc[e][t] = v;
    }
  __syncthreads();  // every warp is done reading dzs (red aliases it)
  if (lane < 8) {
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int t = 0; t < 10; ++t) red[warp][c][(h * 4 + e) * 10 + t] = acc[e][t];
  }
  __syncthreads();
  for (int o = tid; o < 320; o += C1W_THREADS) {  // o = oc*10 + t; warps summed in order
    const int oc = o / 10, t = o % 10;
    float s = red[0][oc >> 3][(oc & 7) * 10 + t];
#pragma unroll
    for (int w = 1; w < C1W_THREADS / 32; ++w) s += red[w][oc >> 3][(oc & 7) * 10 + t];
    buf.part1[(int64_t(j) * buf.B + b) * 320 + o] = s;
  }
}

// ------------------------------------- grad finalize + optimizer ----------
// Every parameter except fc1.w (updated in its wgrad epilogue), one float4 per
// thread-iteration: the gradient is finalised on the fly with the fixed-order
// reductions of the split partials -- conv2.w (sum over the position splits),
// conv2.b (sum over the 144 pooled positions), conv1.w / conv1.b (sum over
// images) -- or read from the arena (fc1.b, fc2 written by the head), stored
// to the arena, and the lane's optimizer update applied (models.cuh
// opt_update; bf16 shadow + transposed conv2.w copies).  The last CTA of a
// lane ends the lane's step.  Replaces a finalize launch + the batched
// optimizer launch.
__global__ void __launch_bounds__(256) cnn_opt_kernel(const __grid_constant__ CnnOpt a, CnnBufs buf) {
  TLK_KT(a.nheavy == 10 ? 10 : 9, a.lanes[0].steps_done);
  pdl_begin();
  TLK_KT_WAITED();
  const int j = blockIdx.y;
  if (!a.lanes[j].active) return;
  const LaneState s = a.lanes[j];
  const CnnOffs& o = a.o;
  if (a.c2w_done) {  // flag join: the lane's conv2 wgrad partials (side branch) are complete
    if (threadIdx.x == 0) {
      const unsigned long long t0 = gtimer_ns();
      while (ld_acquire_u32(a.c2w_done + j) < unsigned(C2W_SPLITS))
        if (gtimer_ns() - t0 > 2000000000ull) __trap();  // 2 s: a lost producer is an error, not a hang
    }
    __syncthreads();
  }
  if (int(blockIdx.x) < a.nheavy) {
    const int l = threadIdx.x & 31;
    const int h = (a.hb0 + blockIdx.x) * 8 + (threadIdx.x >> 5);  // 0..71 conv1.w, 72..79 conv1.b, 80..95 conv2.b
    {
      float g[4] = {0.f, 0.f, 0.f, 0.f};
      int64_t e;
      if (h < 80) {
        const bool wt = h < 72;
        e = wt ? o.c1w + 4 * h : o.c1b + 4 * (h - 72);
        const float* pp = buf.part1 + int64_t(j) * buf.B * 320;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = wt ? 4 * h + q : 4 * (h - 72) + q;
          const int col = wt ? (r / 9) * 10 + r % 9 : r * 10 + 9;
          for (int k = l; k < buf.B; k += 32) g[q] += pp[int64_t(k) * 320 + col];
        }
      } else {
        const int c = 4 * (h - 80);
        e = o.c2b + c;
        const float* cs = buf.colsum + int64_t(j) * 9216 + c;
        for (int pos = l; pos < 144; pos += 32) {
          const float4 v = *reinterpret_cast<const float4*>(cs + pos * 64);
          g[0] += v.x, g[1] += v.y, g[2] += v.z, g[3] += v.w;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int m = 16; m; m >>= 1) g[q] += __shfl_xor_sync(0xffffffffu, g[q], m);
      if (l == 0) cnn_opt_apply(a, s, j, e / 4, g);
    }
  } else {
    const int64_t s4 = a.stride / 4, work = a.a1 + (s4 - a.b0);
    const int nl = gridDim.x - a.nheavy;
    const int64_t per = (work + nl - 1) / nl;
    const int64_t w0 = (blockIdx.x - a.nheavy) * per, w1 = min(work, w0 + per);
    for (int64_t w = w0 + threadIdx.x; w < w1; w += blockDim.x) {
      const int64_t idx = w < a.a1 ? w : a.b0 + (w - a.a1);
      const int64_t e = idx * 4;
      if ((e >= o.c1w && e < o.c1w + 288) || (e >= o.c1b && e < o.c1b + 32) || (e >= o.c2b && e < o.c2b + 64))
        continue;  // heavy CTAs
      float g[4];
      if (e >= o.c2w && e < o.c2w + CONV2_W) {
        const int r = int(e - o.c2w), oc = r / 288, t = r % 288, tap = t >> 5, ic = t & 31;
        const float* pp = buf.part2 + ((int64_t(j) * C2W_SPLITS * 9 + tap) * 64 + oc) * 32 + ic;
        float4 v[C2W_SPLITS];
#pragma unroll
        for (int k = 0; k < C2W_SPLITS; ++k) v[k] = __ldcg(reinterpret_cast<const float4*>(pp + int64_t(k) * 9 * 64 * 32));
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < C2W_SPLITS; ++k) acc.x += v[k].x, acc.y += v[k].y, acc.z += v[k].z, acc.w += v[k].w;
        g[0] = acc.x, g[1] = acc.y, g[2] = acc.z, g[3] = acc.w;
      } else {
        const float4 v = a.Gr[j * s4 + idx];
        g[0] = v.x, g[1] = v.y, g[2] = v.z, g[3] = v.w;
      }
      cnn_opt_apply(a, s, j, idx, g);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&a.lanes[j].done_ctas, 1u);
    if (prev == (a.total ? unsigned(a.total) : gridDim.x) - 1) {
      __threadfence();
      a.lanes[j].done_ctas = 0;
      if (a.c2w_done) a.c2w_done[j] = 0;  // every CTA of the lane has passed its wait
      lane_end_step(a.lanes[j]);
    }
  }
}

bool cnn_fork() {
  static const bool fork = !(getenv("TLK_CNN_NOFORK") && getenv("TLK_CNN_NOFORK")[0] == '1');
  return fork;
}
int cnn_fwa_side() {
  static const int side = getenv("TLK_CNN_FWA_SIDE") ? atoi(getenv("TLK_CNN_FWA_SIDE")) : 3;
  return side;
}
// CTAs of the fc1 wgrad + Adam stream for placement `mode` (TLK_CNN_FWA_SIDE
// values): all SMs when it runs alone (0); next to other kernels a share of
// them, so that the latency-bound chain keeps SMs of its own -- 96 of 148 on
// the graph's side branch (1, 2), 72 of 148 deferred (3), measured best at
// 8 lanes.  TLK_FWA_CTAS overrides.
int fwa_ctas(const Pack& p, int mode) {
  // read at every capture (bench.py re-profiles the kernel on the full grid)
  const int env = getenv("TLK_FWA_CTAS") ? atoi(getenv("TLK_FWA_CTAS")) : 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ctas = env > 0 ? std::min(env, sms) : mode == 3 ? sms * 72 / 148 : mode ? sms * 96 / 148 : sms;
  // (mode 4: the side branch until the end of the step, 96 of 148)
  return std::min(ctas, p.lanes * FWA_FT);
}
int enqueue_fwa(Pack& p, cudaStream_t s2, int ctas) {
  const CnnBufs& b = *static_cast<CnnBufs*>(p.scratch);
  const int64_t o_f1w = tensor_offset(*p.def, 4);
  Fc1WgradAdam f{b.dz3m, b.p2m, b.fa_p, b.fa_m, b.fa_v, b.p2m_alt, p.lane_dev, p.params, p.mom1, p.mom2,
                 p.grads, p.wbf, p.stride, o_f1w, (p.flags & TLK_PACK_WRITE_ALL_GRADS) ? 1 : 0,
                 (p.batch + GEMM_BK - 1) / GEMM_BK, p.lanes * FWA_FT, b.fwa_cnt};
  TLK_CUDA(launch(fc1_wgrad_adam_kernel, dim3(ctas), FWA_THREADS, FWA_SMEM, s2, f));
  p.mark(s2, "fc1_wgrad_adam");
  return TLK_OK;
}
// the deferred fc1 wgrad + Adam of the step graph just launched (runtime.cu
// launches it on p.defer_st after waiting for the graph's ev_defer_in)
int cnn_defer_fwa(Pack& p, cudaStream_t st) { return enqueue_fwa(p, st, fwa_ctas(p, 3)); }

}  // namespace

int cnn_setup(Pack& p) {
  const int64_t L = p.lanes, B = p.batch;
  TLK_CHECK(B % 8 == 0, TLK_EINVAL, "cnn: batch %d must be a multiple of 8", p.batch);
  auto* b = new CnnBufs{};
  p.scratch = b;
  p.scratch_free = [](void* q) { delete static_cast<CnnBufs*>(q); };
  b->B = int(B);
  b->npos = p28_npos(int(B));
  b->p2_st = B * 9216;
  b->h3_st = B * 128;
  const size_t plane = size_t(b->npos) * 16;  // bytes per chunk plane
  const size_t acts = size_t(L) * (4 * plane + 2 * b->p2_st + b->p2_st + 2 * 2 * b->h3_st +
                                   8 * plane + 4 * plane + 2 * b->p2_st) + 16 * 8;
  const size_t f32s = size_t(L) * (9216 + FC1_SPLITS * 128 * 64 + C2W_SPLITS * 9 * 64 * 32 +
                                   B * 320 + HEAD_CL * 64 * CLASSES + 32) + 32 + 16 + L + 16;
  void* base = nullptr;
  int rc = pack_alloc(p, &base, acts + f32s * 4 + 256);
  if (rc) return rc;
  TLK_CUDA(cudaMemset(base, 0, acts + f32s * 4 + 256));  // P28 borders/pads stay zero
  char* c = static_cast<char*>(base);
  auto take = [&](size_t bytes) {
    char* r = c;
    c += (bytes + 15) & ~size_t(15);
    return r;
  };
  b->h1 = reinterpret_cast<uint16_t*>(take(L * 4 * plane));
  b->p2 = reinterpret_cast<uint16_t*>(take(L * b->p2_st * 2));
  b->idx = reinterpret_cast<uint8_t*>(take(L * b->p2_st));
  b->h3 = reinterpret_cast<uint16_t*>(take(L * b->h3_st * 2));
  b->dz3 = reinterpret_cast<uint16_t*>(take(L * b->h3_st * 2));
  b->dz2 = reinterpret_cast<uint16_t*>(take(L * 8 * plane));
  b->dz1 = reinterpret_cast<uint16_t*>(take(L * 4 * plane));
  b->p2_alt = reinterpret_cast<uint16_t*>(take(L * b->p2_st * 2));  // after the round-1 layout
  p.acts = base;
  p.acts_bytes = size_t(c - static_cast<char*>(base));
  b->colsum = reinterpret_cast<float*>(take(L * 9216 * 4));
  b->part_fc1 = reinterpret_cast<float*>(take(L * FC1_SPLITS * 128 * 64 * 4));
  b->part2 = reinterpret_cast<float*>(take(L * C2W_SPLITS * 9 * 64 * 32 * 4));
  b->part1 = reinterpret_cast<float*>(take(L * B * 320 * 4));
  b->plog = reinterpret_cast<float*>(take(L * HEAD_CL * 64 * CLASSES * 4));
  b->sched = reinterpret_cast<uint32_t*>(take((L + 1) * 32 * 4));
  b->fwa_cnt = reinterpret_cast<uint32_t*>(take(64));
  b->c2w_done = reinterpret_cast<uint32_t*>(take(L * 4));
  {  // TMA maps: lanes stacked as the outermost dimension
    const int64_t o_f1w = tensor_offset(*p.def, 4);
    const uint16_t* w1 = p.wbf + o_f1w;
    if ((rc = make_tmap_bf16_3d(&b->w1_k, w1, 9216, 128, L, 9216 * 2, p.stride * 2, 64, 128)))
      return rc;
    if ((rc = make_tmap_bf16_3d(&b->w1_mn, w1, 9216, 128, L, 9216 * 2, p.stride * 2, 64, 64)))
      return rc;
    if ((rc = make_tmap_bf16_3d(&b->p2m, b->p2, 9216, B, L, 9216 * 2, b->p2_st * 2, 64, 64)) ||
        (rc = make_tmap_bf16_3d(&b->p2m_alt, b->p2_alt, 9216, B, L, 9216 * 2, b->p2_st * 2, 64, 64)))
      return rc;
    if ((rc = make_tmap_bf16_3d(&b->dz3m, b->dz3, 128, B, L, 128 * 2, b->h3_st * 2, 64, 64)))
      return rc;
    const int64_t ws = 9216;  // fc1.w row (one output unit) in floats
    const CUtensorMapDataType F32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    if ((rc = make_tmap_3d(&b->fa_p, F32, p.params + o_f1w, ws, 128, L, ws * 4, p.stride * 4, 128, 32,
                           CU_TENSOR_MAP_SWIZZLE_NONE)) ||
        (rc = make_tmap_3d(&b->fa_m, F32, p.mom1 + o_f1w, ws, 128, L, ws * 4, p.stride * 4, 128, 32,
                           CU_TENSOR_MAP_SWIZZLE_NONE)) ||
        (rc = make_tmap_3d(&b->fa_v, F32, p.mom2 + o_f1w, ws, 128, L, ws * 4, p.stride * 4, 128, 32,
                           CU_TENSOR_MAP_SWIZZLE_NONE)))
      return rc;
    if ((rc = make_tmap_3d(&b->fh_p, F32, p.params + o_f1w, ws, 128, L, ws * 4, p.stride * 4, 128, 16,
                           CU_TENSOR_MAP_SWIZZLE_NONE)) ||
        (rc = make_tmap_3d(&b->fh_m, F32, p.mom1 + o_f1w, ws, 128, L, ws * 4, p.stride * 4, 128, 16,
                           CU_TENSOR_MAP_SWIZZLE_NONE)) ||
        (rc = make_tmap_3d(&b->fh_v, F32, p.mom2 + o_f1w, ws, 128, L, ws * 4, p.stride * 4, 128, 16,
                           CU_TENSOR_MAP_SWIZZLE_NONE)))
      return rc;
  }
  void* wt = nullptr;
  p.wt_stride = 2 * CONV2_W;
  if ((rc = pack_alloc(p, &wt, L * p.wt_stride * 2))) return rc;
  p.wt = static_cast<uint16_t*>(wt);
  TLK_CUDA(cudaFuncSetAttribute(conv2_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                ConvPolicy<true>::SMEM));
  TLK_CUDA(cudaFuncSetAttribute(conv2_tc_kernel<false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, ConvPolicy<false>::SMEM));
  TLK_CUDA(cudaFuncSetAttribute(conv1_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C1W_SMEM));
  TLK_CUDA(cudaFuncSetAttribute(fc1_wgrad_adam_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FWA_SMEM));
  TLK_CUDA(cudaFuncSetAttribute(conv2_wgrad_tc_kernel,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, WG_SMEM));
  p.launches_per_step = cnn_persist_enabled(p) ? 1 : 10;
  if (!cnn_persist_enabled(p) && cnn_fork() && cnn_fwa_side() == 3) {
    p.defer = cnn_defer_fwa;
    TLK_CUDA(cudaStreamCreateWithFlags(&p.defer_st, cudaStreamNonBlocking));
    TLK_CUDA(cudaEventCreateWithFlags(&p.ev_defer_in, cudaEventDisableTiming));
    TLK_CUDA(cudaEventCreateWithFlags(&p.ev_defer_out, cudaEventDisableTiming));
  }
  p.fused_lo = tensor_offset(*p.def, 4);  // fc1.w: updated inside its wgrad epilogue
  p.fused_hi = p.fused_lo + p.def->t[4].count;
  return TLK_OK;
}

int cnn_enqueue_step(Pack& p, cudaStream_t st) {
  if (cnn_persist_enabled(p)) return cnn_persist_enqueue(p, st, 1);
  const CnnBufs& b = *static_cast<CnnBufs*>(p.scratch);
  const ModelDef& d = *p.def;
  const int L = p.lanes, B = p.batch;
  const int64_t o_c1w = tensor_offset(d, 0), o_c1b = tensor_offset(d, 1);
  const int64_t o_c2w = tensor_offset(d, 2), o_c2b = tensor_offset(d, 3);
  const int64_t o_f1w = tensor_offset(d, 4), o_f1b = tensor_offset(d, 5);
  const int64_t o_f2w = tensor_offset(d, 6), o_f2b = tensor_offset(d, 7);
  // TLK_CNN_FLAG_JOIN=1: the optimizer waits for the side branch's
  // conv2 wgrad through a per-lane completion count (conv2 wgrad CTAs
  // release, the optimizer acquires; bounded spin) instead of an event join,
  // so the conv1 wgrad -> optimizer edge keeps its programmatic launch; the
  // side branch rejoins the stream after the optimizer.  The conv2 wgrad is
  // launched ~70 us before the optimizer, so it is resident long before.
  // Bit-identical, measured no faster (0.1732 vs 0.1728 ms/step): off.
  static const bool flag_env = getenv("TLK_CNN_FLAG_JOIN") && getenv("TLK_CNN_FLAG_JOIN")[0] == '1';
  const bool split_req = getenv("TLK_CNN_SPLIT_OPT") && getenv("TLK_CNN_SPLIT_OPT")[0] == '1';
  const bool flag_join = flag_env && cnn_fork() && !p.prof && !split_req;
  ConvArgs ca = conv_args(p, b);
  if (flag_join) ca.c2w_done = b.c2w_done;
  int rc;
  TLK_CUDA(launch(conv1_fwd_kernel, dim3(B, L), 256, 0, st, p.lane_dev, p.teacher, p.pixels, p.labels, p.x,
                  p.host_input, p.params, p.stride, o_c1w, o_c1b, b));
  p.mark(st, "inputs_conv1_fwd");
  TLK_CUDA(cudaGetLastError());
  TLK_CUDA(launch(conv2_tc_kernel<true>, dim3(CONV_CTAS_PER_LANE, L), CONV_FD_THREADS, ConvPolicy<true>::SMEM, st, ca));
  p.mark(st, "conv2_fwd_pool");
  TLK_CUDA(cudaGetLastError());
  // deferred mode: the previous step's fc1 wgrad + Adam (cnn_defer_fwa) has
  // written the fc1 weights this forward reads
  if (p.defer && !p.prof) TLK_CUDA(cudaStreamWaitEvent(st, p.ev_defer_out, cudaEventWaitExternal));
  Fc1Fwd f1{b, p.lane_dev};
  TLK_CUDA(launch_gemm_tma(f1, dim3(1, 1, L * FC1_SPLITS), st));
  p.mark(st, "fc1_fwd_splitk");
TLK_CUDA(launch(cnn_head_kernel, dim3(HEAD_CL, L), 256, 0, st, p.lane_dev, b, p.params, p.grads, p.stride, o_f1b,
                  o_f2w, o_f2b, p.labels, p.loss, p.max_steps, p.last_loss));
  p.mark(st, "fc1_reduce_head");
  Fc1Dgrad f1d{b, p.lane_dev};  // reads this step's fc1 weights
  TLK_CUDA(launch_gemm_tma(f1d, dim3(9216 / GEMM_BM, 1, L), st));
  p.mark(st, "fc1_dgrad_unpool");
  // conv2 wgrad (reads dz2, h1; writes its partials) is independent of the
  // conv2 dgrad -> conv1 wgrad chain: a forked graph branch lets the two
  // latency-bound kernels share the SMs (TLK_CNN_NOFORK=1: serial)
  // where the deferred fc1 wgrad + Adam may start (TLK_FWA_DEFER_AT): 0 right
  // after the fc1 dgrad (beside the conv2 wgrad), 1 after the conv2 wgrad
  // (default), 2 after the conv1 wgrad (beside the optimizer only)
  static const int defer_at = getenv("TLK_FWA_DEFER_AT") ? atoi(getenv("TLK_FWA_DEFER_AT")) : 1;
  const bool deferring = p.defer && !p.prof && cnn_fork() && cnn_fwa_side() == 3;
  if (deferring && defer_at == 0) TLK_CUDA(cudaEventRecordWithFlags(p.ev_defer_in, st, cudaEventRecordExternal));
  // TLK_CNN_FORK_LATE=1: fork the conv2 wgrad branch after the conv2 dgrad
  // (beside the conv1 wgrad) instead of after the fc1 dgrad
  static const bool fork_late = getenv("TLK_CNN_FORK_LATE") && getenv("TLK_CNN_FORK_LATE")[0] == '1';
  const bool dgrad_first = fork_late && cnn_fork() && !p.prof;
  if (dgrad_first) {
    TLK_CUDA(launch(conv2_tc_kernel<false>, dim3(CONV_CTAS_PER_LANE, L), CONV_FD_THREADS, ConvPolicy<false>::SMEM, st, ca));
    p.mark(st, "conv2_dgrad");
    TLK_CUDA(cudaGetLastError());
  }
  cudaStream_t wst = st;
  if (cnn_fork() && !p.prof) {
    TLK_CUDA(cudaEventRecord(p.ev_fork, st));
    TLK_CUDA(cudaStreamWaitEvent(p.side, p.ev_fork, 0));
    wst = p.side;
  }
  // fc1 wgrad + Adam (HBM-bound) needs dz3 / p2 of this step and must follow
  // the fc1 dgrad (which reads this step's fc1 weights).  TLK_CNN_FWA_SIDE:
  //   3 (default) = deferred: launched by the runtime after the step graph on
  //     a stream of its own (cnn_defer_fwa), after this graph's conv2 wgrad
  //     (event recorded below), overlapping this step's conv2 dgrad -> conv1
  //     wgrad -> optimizer tail and the next step's conv1 / conv2 forward; the
  //     next step's fc1 forward waits for it (p2 is double-buffered by step
  //     parity, so the next forward does not overwrite its input);
  //   1 = side branch after conv2 wgrad, 2 = before it, 0 = main stream after
  //     the join.  A profile step (p.prof) serialises every kernel: 0.
  int side_mode = p.prof ? 0 : wst == st ? 0 : cnn_fwa_side();
  if (side_mode == 3 && !p.defer) side_mode = 0;
  if (side_mode == 2 && (rc = enqueue_fwa(p, wst, fwa_ctas(p, 2)))) return rc;
  TLK_CUDA(launch(conv2_wgrad_tc_kernel, dim3(C2W_SPLITS, L), CONV_THREADS, WG_SMEM, wst, ca));
  p.mark(wst, "conv2_wgrad");
  TLK_CUDA(cudaGetLastError());
  if (side_mode == 1 && (rc = enqueue_fwa(p, wst, fwa_ctas(p, 1)))) return rc;
  if (deferring && defer_at == 1) TLK_CUDA(cudaEventRecordWithFlags(p.ev_defer_in, wst, cudaEventRecordExternal));
  if (wst != st) TLK_CUDA(cudaEventRecord(p.ev_join, wst));
  // 4 = on the side branch after conv2 wgrad, joined only at the end of the step
  if (side_mode == 4) {
    if ((rc = enqueue_fwa(p, wst, fwa_ctas(p, 4)))) return rc;
    TLK_CUDA(cudaEventRecord(p.ev_tail, wst));
  }
  if (!dgrad_first) {
    TLK_CUDA(launch(conv2_tc_kernel<false>, dim3(CONV_CTAS_PER_LANE, L), CONV_FD_THREADS, ConvPolicy<false>::SMEM, st, ca));
    p.mark(st, "conv2_dgrad");
    TLK_CUDA(cudaGetLastError());
  }
  // TLK_CNN_SPLIT_OPT=1: the optimizer of every parameter but conv1's runs
  // on the side branch once the conv2 dgrad (which reads this step's conv2
  // weights) is done, beside the conv1 wgrad; the chain then ends with the
  // conv1 update alone (10 CTAs per lane).  The last of the 36 CTAs per lane
  // over both launches ends the lane's step.  Bit-identical, but measured
  // slower at 8 lanes (0.182 vs 0.176 ms/step), so off by default.
  static const bool split_env = getenv("TLK_CNN_SPLIT_OPT") && getenv("TLK_CNN_SPLIT_OPT")[0] == '1';
  const bool split_opt = split_env && wst != st;
  if (split_opt) {
    TLK_CUDA(cudaEventRecord(p.ev_fork, st));
    TLK_CUDA(cudaStreamWaitEvent(wst, p.ev_fork, 0));
    CnnOpt a{p.lane_dev, p.stride, p.fused_lo / 4, p.fused_hi / 4, CnnOffs{o_c1w, o_c1b, o_c2w, o_c2b},
             reinterpret_cast<float4*>(p.params), reinterpret_cast<float4*>(p.grads),
             reinterpret_cast<float4*>(p.mom1), reinterpret_cast<float4*>(p.mom2),
             reinterpret_cast<uint2*>(p.wbf), WtHook{p.wt, p.wt_stride, o_c2w, CONV2_W}};
    a.hb0 = 10;
    a.nheavy = 2;
    a.total = CNN_OPT_HEAVY + CNN_OPT_CTAS;
    TLK_CUDA(launch(cnn_opt_kernel, dim3(2 + CNN_OPT_CTAS, L), 256, 0, wst, a, b));
    p.mark(wst, "grad_finalize_opt");
    TLK_CUDA(cudaEventRecord(p.ev_join, wst));
  }
  // TLK_CNN_JOIN_EARLY=1: join the side branch before the conv1 wgrad (the
  // conv1 wgrad -> optimizer edge stays a programmatic one) instead of after it
  static const bool join_early = getenv("TLK_CNN_JOIN_EARLY") && getenv("TLK_CNN_JOIN_EARLY")[0] == '1';
  if (wst != st && join_early && !flag_join) TLK_CUDA(cudaStreamWaitEvent(st, p.ev_join, 0));
  TLK_CUDA(launch(conv1_wgrad_kernel, dim3(B, L), C1W_THREADS, C1W_SMEM, st, p.lane_dev, b, p.x));
  p.mark(st, "conv1_wgrad");
  TLK_CUDA(cudaGetLastError());
  if (deferring && defer_at == 2) TLK_CUDA(cudaEventRecordWithFlags(p.ev_defer_in, st, cudaEventRecordExternal));
  if (wst != st && !join_early && !flag_join) TLK_CUDA(cudaStreamWaitEvent(st, p.ev_join, 0));
  // (a profile step times the kernel at the grid it has in the step)
  if (side_mode == 0 && (rc = enqueue_fwa(p, st, fwa_ctas(p, p.prof && cnn_fork() ? cnn_fwa_side() : 0))))
    return rc;
  CnnOpt a{p.lane_dev, p.stride, p.fused_lo / 4, p.fused_hi / 4, CnnOffs{o_c1w, o_c1b, o_c2w, o_c2b},
           reinterpret_cast<float4*>(p.params), reinterpret_cast<float4*>(p.grads),
           reinterpret_cast<float4*>(p.mom1), reinterpret_cast<float4*>(p.mom2),
           reinterpret_cast<uint2*>(p.wbf), WtHook{p.wt, p.wt_stride, o_c2w, CONV2_W}};
  if (flag_join && !split_opt) a.c2w_done = b.c2w_done;
  if (split_opt) {  // conv1 parameters only (their gradient is the chain's last one)
    a.hb0 = 0;
    a.nheavy = 10;
    a.total = CNN_OPT_HEAVY + CNN_OPT_CTAS;
    TLK_CUDA(launch(cnn_opt_kernel, dim3(10, L), 256, 0, st, a, b));
    p.mark(st, "conv1_opt");
  } else {
    TLK_CUDA(launch(cnn_opt_kernel, dim3(CNN_OPT_HEAVY + CNN_OPT_CTAS, L), 256, 0, st, a, b));
    p.mark(st, "grad_finalize_opt");
  }
  if (side_mode == 4) TLK_CUDA(cudaStreamWaitEvent(st, p.ev_tail, 0));
  if (flag_join) TLK_CUDA(cudaStreamWaitEvent(st, p.ev_join, 0));  // the side branch rejoins at the end
  return enqueue_end_step(p, st);
}

}  // namespace tlk

// In-graph kernel timeline (-DTLK_KTRACE builds; tools/cnn_timeline.py).
extern "C" int tlk_cnn_ktrace(int32_t reset, uint64_t* out, int32_t n) {
#ifdef TLK_KTRACE
  constexpr int N = 8 * tlk::KT_KERNELS * 3;
  if (reset) {
    static uint64_t init[N];
    for (int i = 0; i < N; ++i) init[i] = (i % 3 == 2) ? 0 : ~0ull;
    TLK_CUDA(cudaMemcpyToSymbol(tlk::g_ktrace, init, sizeof(init)));
    return TLK_OK;
  }
  TLK_CHECK(out && n >= N, TLK_EINVAL, "need %d slots", N);
  TLK_CUDA(cudaMemcpyFromSymbol(out, tlk::g_ktrace, N * sizeof(uint64_t)));
  return TLK_OK;
#else
  (void)reset;
  (void)out;
  (void)n;
  return tlk::fail(TLK_EINVAL, "libtlk was built without TLK_KTRACE");
#endif
}
