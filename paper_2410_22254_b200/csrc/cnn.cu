// MNIST CNN pack (pytorch/examples Net without dropout), all lanes per launch.
//
//   x[28,28] -conv1 3x3 (1->32)+ReLU-> h1[26,26,32] -conv2 3x3 (32->64)+ReLU+maxpool2->
//   p2[12,12,64] -flatten (h,w,c)-> fc1 (9216->128)+ReLU -> h3 -> fc2 (128->10) + CE
//
// Launch sequence of one step (14 kernels, graph-captured):
//   inputs | conv1 fwd (CUDA cores, writes h1 in P28 planes) | conv2 fwd
//   (tcgen05, TMA-bulk patch + tap-shifted descriptors; epilogue bias+ReLU+
//   2x2 maxpool+argmax) | fc1 fwd (tcgen05 split-K) | fc1 reduce (+bias+ReLU)
//   | head (fc2+CE+bwd) | fc1 wgrad (tcgen05) | fc1 dgrad (tcgen05; epilogue
//   = maxpool/ReLU backward scatter into dz2 P28 planes + conv2 bias partials)
//   | conv2 wgrad (tcgen05, 9 tap accumulators in TMEM) | conv2 dgrad
//   (tcgen05; epilogue ReLU mask -> dz1) | conv1 wgrad (CUDA cores) | grad
//   finalize (fixed-order reductions) | optimizer | end_step
//
// The P28 layout and the conv2 kernels are described in conv_tc.cuh.
//
// Activation scratch (TLK_BUF_ACTS), each [lanes][...] contiguous, in order:
//   h1 P28 [4][npos][8] | p2 bf16 [B,12,12,64] | idx u8 [B,12,12,64]
//   (argmax | live<<2) | h3 bf16 [B,128] | dz3 bf16 [B,128] |
//   dz2 P28 [8][npos][8] | dz1 P28 [4][npos][8]      (npos = 32 + 784 B + 64)
#include "conv_tc.cuh"
#include "tma.cuh"
#include "linear.cuh"
#include "pack.cuh"

namespace tlk {
namespace {

constexpr int FC1_SPLITS = 18;     // 144 k-blocks / 8
constexpr int C2W_SPLITS = 18;     // conv2 wgrad position splits per lane
constexpr int C1W_SMEM = 4 * P28_IMG * 16;  // conv1 wgrad: one image's dz1 planes

struct CnnBufs {
  // TMA tensor maps of the plain-layout fc1 operands (lanes = dim 2)
  CUtensorMap w1_k;   // fc1.w bf16 [9216 in][128 out]: box 64 x 128 (K-major A)
  CUtensorMap w1_mn;  // fc1.w bf16: box 64 x 64 (MN-major A of dgrad)
  CUtensorMap p2m;    // p2 [9216][B]: box 64 x 64
  CUtensorMap dz3m;   // dz3 [128][B]: box 64 x 64
  int B;
  int64_t npos;
  uint16_t *h1, *p2, *h3, *dz3, *dz2, *dz1;
  uint8_t* idx;
  float *colsum, *part_fc1, *part2, *part1;
  int64_t p2_st, h3_st;
};

__host__ __device__ inline int64_t p28_pos(int b, int r, int c) {
  return P28_FRONT + int64_t(b) * P28_IMG + r * P28 + c;
}

// ---------------------------------------------------------------- conv1 -----
// One CTA per (sample, lane); fp32 math on fp32 master weights; writes the
// 26x26 interior of h1's P28 planes (16 B = 8 channels per store).
__global__ void __launch_bounds__(256) conv1_fwd_kernel(const LaneState* __restrict__ lanes,
                                                        const uint16_t* __restrict__ x,
                                                        const float* __restrict__ params,
                                                        int64_t pstride, int64_t w_off,
                                                        int64_t b_off, CnnBufs buf) {
  const int s = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  if (!lanes[j].active) return;
  __shared__ float xs[784];
  __shared__ float ws[32 * 9];
  __shared__ float bs[32];
  const uint4* xr = reinterpret_cast<const uint4*>(x + (size_t(j) * buf.B + s) * 784);
  if (tid < 98) {  // 784 bf16 = 98 x 16 B
    const uint4 v = xr[tid];
    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      xs[tid * 8 + 2 * e] = bf2f(uint16_t(wv[e] & 0xFFFF));
      xs[tid * 8 + 2 * e + 1] = bf2f(uint16_t(wv[e] >> 16));
    }
  }
  for (int i = tid; i < 288; i += 256) ws[i] = params[j * pstride + w_off + i];
  if (tid < 32) bs[tid] = params[j * pstride + b_off + tid];
  __syncthreads();
  uint16_t* h1 = buf.h1 + int64_t(j) * 4 * buf.npos * 8;
  const int c = tid & 3;  // this thread's 8-channel chunk: its 72 weights live in registers
  float w[8][9], bsum[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    bsum[e] = bs[c * 8 + e];
#pragma unroll
    for (int t = 0; t < 9; ++t) w[e][t] = ws[(c * 8 + e) * 9 + t];
  }
  for (int pos = tid >> 2; pos < 676; pos += 64) {
    const int oh = pos / 26, ow = pos % 26;
    float xv[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) xv[t] = xs[(oh + t / 3) * 28 + ow + t % 3];
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      acc[e] = 0.f;
#pragma unroll
      for (int t = 0; t < 9; ++t) acc[e] += xv[t] * w[e][t];
    }
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      o[e] = pack_bf2(fmaxf(acc[2 * e] + bsum[2 * e], 0.f), fmaxf(acc[2 * e + 1] + bsum[2 * e + 1], 0.f));
    *reinterpret_cast<uint4*>(h1 + (c * buf.npos + p28_pos(s, oh + 1, ow + 1)) * 8) =
        make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// ------------------------------------------------------ fc1 fwd (TC) --------
// Z^T[o, b] partial sums over a K-split: part[lane][split][o][b].
struct Fc1Fwd {
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
  }
  TLK_DEV void load_a(const Work& w, int kb, uint32_t dst, uint64_t* bar) const {
    tma_load_3d(dst, &buf.w1_k, kb * GEMM_BK, 0, w.j, bar);
  }
  TLK_DEV void load_b(const Work& w, int kb, uint32_t dst, uint64_t* bar) const {
    tma_load_3d(dst, &buf.p2m, kb * GEMM_BK, 0, w.j, bar);
  }
  TLK_DEV void epilogue(const Work& w, int m, int n0, const float (&v)[32], Carry&) const {
    float* o = buf.part_fc1 + ((int64_t(w.j) * FC1_SPLITS + w.split) * 128 + m) * 64 + n0;
#pragma unroll
    for (int i = 0; i < 32; i += 4)
      *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  }
  TLK_DEV void finish(const Work&, int, Carry&) const {}
};

// h3[b][o] = bf16(relu(sum_s part[s][o][b] + bias[o])), fixed split order.
__global__ void fc1_reduce_kernel(const LaneState* __restrict__ lanes, CnnBufs buf,
                                  const float* __restrict__ params, int64_t pstride,
                                  int64_t b_off) {
  const int j = blockIdx.y;
  if (!lanes[j].active) return;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;  // e = o*64 + b
  if (e >= 128 * 64) return;
  const int o = e >> 6, b = e & 63;
  if (b >= buf.B) return;
  const float* pp = buf.part_fc1 + int64_t(j) * FC1_SPLITS * 128 * 64 + e;
  float s = 0.0f;
#pragma unroll
  for (int k = 0; k < FC1_SPLITS; ++k) s += pp[int64_t(k) * 128 * 64];
  buf.h3[j * buf.h3_st + b * 128 + o] = f2bf(fmaxf(s + params[j * pstride + b_off + o], 0.0f));
}

// ---------------------------------------------- fc1 dgrad + unpool (TC) -----
// dp2^T[f, b] = sum_o W[o, f] dz3[b, o]; epilogue scatters through the 2x2
// argmax (live bit = pooled value > 0) into the dz2 P28 planes and
// accumulates the conv2 bias-gradient partial colsum[f] = sum_b dz2 value.
struct Fc1Dgrad {
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
  // Phase 1, item = (b, position, 8-channel chunk): the 2x2 window of the
  // chunk is written as four 16-B stores into the dz2 P28 plane (argmax gets
  // bf16(value) if the pooled output was live, the rest zeros); the rounded
  // value replaces the tile entry.  Phase 2: colsum[f] = sum_b (fixed order).
  TLK_DEV void tile_epilogue(const Work& w, float* tile, int ld) const {
    const int tid = threadIdx.x, B = buf.B;
    const int pos0 = w.m0 >> 6;
    uint2 codes[4];  // all four items' argmax codes in flight before any math
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = tid + 256 * u, b = i & 63, pl = (i >> 6) >> 3, ch = (i >> 6) & 7;
      codes[u] = b < B ? *reinterpret_cast<const uint2*>(buf.idx + w.j * buf.p2_st +
                                                          int64_t(b) * 9216 + (pos0 + pl) * 64 + ch * 8)
                       : make_uint2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = tid + 256 * u;
      const int b = i & 63, pl = (i >> 6) >> 3, ch = (i >> 6) & 7;
      if (b >= B) continue;
      const int pos = pos0 + pl, ph = pos / 12, pw = pos % 12, f = pl * 64 + ch * 8;
      const uint2 code2 = codes[u];
      const uint32_t cw[2] = {code2.x, code2.y};
      uint16_t z[8];
      int q[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t code = (cw[e >> 2] >> (8 * (e & 3))) & 0xFF;
        float* t = tile + (f + e) * ld + b;
        z[e] = (code & 4) ? f2bf(*t) : uint16_t(0);
        q[e] = code & 3;
        *t = bf2f(z[e]);
      }
      uint16_t* plane = buf.dz2 + (int64_t(w.j) * 8 + ch) * buf.npos * 8;
      const int64_t p = p28_pos(b, 2 * ph + 2, 2 * pw + 2);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        uint32_t o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          o[e] = uint32_t(q[2 * e] == r ? z[2 * e] : 0) |
                 (uint32_t(q[2 * e + 1] == r ? z[2 * e + 1] : 0) << 16);
        *reinterpret_cast<uint4*>(plane + (p + (r >> 1) * P28 + (r & 1)) * 8) =
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
// dW1[o, f] = sum_b dz3[b, o] p2[b, f] (M = 128 out, N = 9216 in, K = batch,
// both operands MN-major) with the lane's optimizer update applied in the
// epilogue: fc1.w is 98% of the CNN's parameters, so its fp32 gradient never
// makes the HBM round trip (grads are stored only with
// TLK_PACK_WRITE_ALL_GRADS).  Must run after every reader of this step's fc1
// weights (fc1 dgrad).  (Measured alternative: a separate optimizer pass in a
// forked graph branch concurrent with the conv backward kernels was slower --
// it crowds the SMs the conv kernels need.)
struct Fc1WgradOpt {
  static constexpr int BN = 64, STAGES = 2, THREADS = 256;
  static constexpr bool A_MN = true, B_MN = true;
  static constexpr bool TILE_EPILOGUE = true;
  using Work = LaneWork;
  struct Carry {};
  CnnBufs buf;
  const LaneState* lanes;
  float *params, *grads, *m1, *m2;
  uint16_t* wbf;
  int64_t pstride, w_off;
  int write_grads;

  TLK_DEV bool work(Work& w) const {
    w.j = blockIdx.z;
    if (!lanes[w.j].active) return false;
    w.m0 = 0;
    w.n0 = blockIdx.y * BN;
    w.kb_begin = 0;
    w.kb_end = (buf.B + GEMM_BK - 1) / GEMM_BK;
    w.split = 0;
    return true;
  }
  TLK_DEV void prefetch() const {
    tma_prefetch_desc(&buf.dz3m);
    tma_prefetch_desc(&buf.p2m);
  }
  TLK_DEV void load_a(const Work& w, int kb, uint32_t dst, uint64_t* bar) const {
    tma_load_3d(dst, &buf.dz3m, 0, kb * GEMM_BK, w.j, bar);
    tma_load_3d(dst + 8192, &buf.dz3m, 64, kb * GEMM_BK, w.j, bar);
  }
  TLK_DEV void load_b(const Work& w, int kb, uint32_t dst, uint64_t* bar) const {
    tma_load_3d(dst, &buf.p2m, w.n0, kb * GEMM_BK, w.j, bar);
  }
  TLK_DEV void epilogue(const Work&, int, int, const float (&)[32], Carry&) const {}
  TLK_DEV void finish(const Work&, int, Carry&) const {}
  // tile = dW1[128 o][64 f] in smem.  256 threads: thread -> float4 column
  // c4 = tid % 16 of rows r0 + 16k: a warp covers two 256-B row segments per
  // access; 2 rows (6 float4 loads) in flight per thread before any math.
  TLK_DEV void tile_epilogue(const Work& w, float* tile, int ld) const {
    const LaneState s = lanes[w.j];
    const int tid = threadIdx.x, c4 = tid & 15, r0 = tid >> 4;
    const int64_t base = w.j * pstride + w_off + w.n0 + 4 * c4;
#pragma unroll 1
    for (int k0 = 0; k0 < 8; k0 += 2) {
      float4 p[2], mm[2], vv[2];
      int64_t e[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        e[u] = base + int64_t(r0 + 16 * (k0 + u)) * 9216;
        p[u] = *reinterpret_cast<const float4*>(params + e[u]);
        mm[u] = *reinterpret_cast<const float4*>(m1 + e[u]);
        vv[u] = *reinterpret_cast<const float4*>(m2 + e[u]);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const float4 g = *reinterpret_cast<const float4*>(tile + (r0 + 16 * (k0 + u)) * ld + 4 * c4);
        opt_update(s, p[u].x, g.x, mm[u].x, vv[u].x);
        opt_update(s, p[u].y, g.y, mm[u].y, vv[u].y);
        opt_update(s, p[u].z, g.z, mm[u].z, vv[u].z);
        opt_update(s, p[u].w, g.w, mm[u].w, vv[u].w);
        *reinterpret_cast<float4*>(params + e[u]) = p[u];
        *reinterpret_cast<float4*>(m1 + e[u]) = mm[u];
        *reinterpret_cast<float4*>(m2 + e[u]) = vv[u];
        *reinterpret_cast<uint2*>(wbf + e[u]) =
            make_uint2(pack_bf2(p[u].x, p[u].y), pack_bf2(p[u].z, p[u].w));
        if (write_grads) *reinterpret_cast<float4*>(grads + e[u]) = g;
      }
    }
  }
};

// ------------------------------------------------ conv1 wgrad (SIMT) --------
// One CTA per (image, lane).  Thread = (8-channel chunk c, position group g):
// acc[e][t] over its positions (t<9: tap products with x, t=9: bias), then a
// fixed-order reduction over the 32 groups -> part1[lane][image][32][10].
__global__ void __launch_bounds__(128) conv1_wgrad_kernel(const LaneState* __restrict__ lanes,
                                                          CnnBufs buf,
                                                          const uint16_t* __restrict__ x) {
  const int b = blockIdx.x, j = blockIdx.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (!lanes[j].active) return;
  extern __shared__ __align__(16) uint16_t dzs_raw[];  // this image's dz1 planes (50 KB)
  uint16_t(*dzs)[P28_IMG * 8] = reinterpret_cast<uint16_t(*)[P28_IMG * 8]>(dzs_raw);
  __shared__ float xs[784];
  __shared__ float red[4][4][80];
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
  mbar_wait(&bar, 0);
  const int c = tid & 3, g = tid >> 2;  // chunk, position group (32 groups)
  float acc[8][10];
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int t = 0; t < 10; ++t) acc[e][t] = 0.f;
  for (int q = g; q < 676; q += 32) {
    const int oh = q / 26, ow = q % 26;
    const uint4 dv = *reinterpret_cast<const uint4*>(&dzs[c][((oh + 1) * P28 + ow + 1) * 8]);
    const uint32_t dw[4] = {dv.x, dv.y, dv.z, dv.w};
    float d[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      d[2 * e] = bf2f(uint16_t(dw[e] & 0xFFFF));
      d[2 * e + 1] = bf2f(uint16_t(dw[e] >> 16));
    }
    float xv[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) xv[t] = xs[(oh + t / 3) * 28 + ow + t % 3];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
#pragma unroll
      for (int t = 0; t < 9; ++t) acc[e][t] += d[e] * xv[t];
      acc[e][9] += d[e];
    }
  }
  // reduce the 8 groups of this warp that share chunk c (lanes c, c+4, ...), fixed order
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int t = 0; t < 10; ++t) {
      float v = acc[e][t];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      acc[e][t] = v;
    }
  if (lane < 4) {
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int t = 0; t < 10; ++t) red[warp][c][e * 10 + t] = acc[e][t];
  }
  __syncthreads();
  for (int o = tid; o < 320; o += 128) {  // o = oc*10 + t
    const int oc = o / 10, t = o % 10;
    const float s = red[0][oc >> 3][(oc & 7) * 10 + t] + red[1][oc >> 3][(oc & 7) * 10 + t] +
                    red[2][oc >> 3][(oc & 7) * 10 + t] + red[3][oc >> 3][(oc & 7) * 10 + t];
    buf.part1[(int64_t(j) * buf.B + b) * 320 + o] = s;
  }
}

// ------------------------------------------------ grad finalize -------------
// Deterministic fixed-order reductions of the split partials into grads:
// conv2.w (sum over position splits), conv2.b (sum over 144 pooled
// positions), conv1.w / conv1.b (sum over images).
__global__ void __launch_bounds__(256) cnn_finalize_kernel(const LaneState* __restrict__ lanes,
                                                           CnnBufs buf, float* __restrict__ grads,
                                                           int64_t pstride, int64_t o_c1w,
                                                           int64_t o_c1b, int64_t o_c2w,
                                                           int64_t o_c2b) {
  const int j = blockIdx.y;
  if (!lanes[j].active) return;
  float* G = grads + j * pstride;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < 18432) {  // e = oc*288 + tap*32 + ic
    const int oc = e / 288, r = e % 288, tap = r >> 5, ic = r & 31;
    const float* pp = buf.part2 + ((int64_t(j) * C2W_SPLITS * 9 + tap) * 64 + oc) * 32 + ic;
    float s = 0.f;
#pragma unroll 6
    for (int k = 0; k < C2W_SPLITS; ++k) s += pp[int64_t(k) * 9 * 64 * 32];
    G[o_c2w + e] = s;
  } else if (e < 18432 + 64) {
    const int c = e - 18432;
    const float* cs = buf.colsum + int64_t(j) * 9216 + c;
    float s = 0.f;
    for (int pos = 0; pos < 144; ++pos) s += cs[pos * 64];
    G[o_c2b + c] = s;
  } else if (e < 18432 + 64 + 320) {
    const int r = e - 18432 - 64, o = r / 10, t = r % 10;
    const float* pp = buf.part1 + int64_t(j) * buf.B * 320 + r;
    float s = 0.f;
    for (int k = 0; k < buf.B; ++k) s += pp[int64_t(k) * 320];
    if (t < 9)
      G[o_c1w + o * 9 + t] = s;
    else
      G[o_c1b + o] = s;
  }
}

ConvArgs conv_args(const Pack& p, const CnnBufs& b) {
  ConvArgs a{};
  a.lanes = p.lane_dev;
  a.B = b.B;
  a.npos = b.npos;
  a.h1 = b.h1;
  a.dz2 = b.dz2;
  a.dz1 = b.dz1;
  a.p2 = b.p2;
  a.idx = b.idx;
  a.wt = p.wt;
  a.wt_stride = p.wt_stride;
  a.params = p.params;
  a.pstride = p.stride;
  a.b2_off = tensor_offset(*p.def, 3);
  a.part2 = b.part2;
  a.wgrad_splits = C2W_SPLITS;
  return a;
}

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
                                   8 * plane + 4 * plane);
  const size_t f32s = size_t(L) * (9216 + FC1_SPLITS * 128 * 64 + C2W_SPLITS * 9 * 64 * 32 +
                                   B * 320);
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
  p.acts = base;
  p.acts_bytes = size_t(c - static_cast<char*>(base));
  b->colsum = reinterpret_cast<float*>(take(L * 9216 * 4));
  b->part_fc1 = reinterpret_cast<float*>(take(L * FC1_SPLITS * 128 * 64 * 4));
  b->part2 = reinterpret_cast<float*>(take(L * C2W_SPLITS * 9 * 64 * 32 * 4));
  b->part1 = reinterpret_cast<float*>(take(L * B * 320 * 4));
  {  // TMA maps: lanes stacked as the outermost dimension
    const int64_t o_f1w = tensor_offset(*p.def, 4);
    const uint16_t* w1 = p.wbf + o_f1w;
    if ((rc = make_tmap_bf16_3d(&b->w1_k, w1, 9216, 128, L, 9216 * 2, p.stride * 2, 64, 128)))
      return rc;
    if ((rc = make_tmap_bf16_3d(&b->w1_mn, w1, 9216, 128, L, 9216 * 2, p.stride * 2, 64, 64)))
      return rc;
    if ((rc = make_tmap_bf16_3d(&b->p2m, b->p2, 9216, B, L, 9216 * 2, b->p2_st * 2, 64, 64)))
      return rc;
    if ((rc = make_tmap_bf16_3d(&b->dz3m, b->dz3, 128, B, L, 128 * 2, b->h3_st * 2, 64, 64)))
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
  TLK_CUDA(cudaFuncSetAttribute(conv2_wgrad_tc_kernel,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, WG_SMEM));
  p.launches_per_step = 13;
  p.fused_lo = tensor_offset(*p.def, 4);  // fc1.w: updated inside its wgrad epilogue
  p.fused_hi = p.fused_lo + p.def->t[4].count;
  return TLK_OK;
}

int cnn_enqueue_step(Pack& p, cudaStream_t st) {
  const CnnBufs& b = *static_cast<CnnBufs*>(p.scratch);
  const ModelDef& d = *p.def;
  const int L = p.lanes, B = p.batch;
  const int64_t o_c1w = tensor_offset(d, 0), o_c1b = tensor_offset(d, 1);
  const int64_t o_c2w = tensor_offset(d, 2), o_c2b = tensor_offset(d, 3);
  const int64_t o_f1w = tensor_offset(d, 4), o_f1b = tensor_offset(d, 5);
  const int64_t o_f2w = tensor_offset(d, 6), o_f2b = tensor_offset(d, 7);
  const ConvArgs ca = conv_args(p, b);
  int rc;
  if ((rc = enqueue_inputs(p, st))) return rc;
  conv1_fwd_kernel<<<dim3(B, L), 256, 0, st>>>(p.lane_dev, p.x, p.params, p.stride, o_c1w, o_c1b, b);
  p.mark(st, "conv1_fwd");
  TLK_CUDA(cudaGetLastError());
  conv2_tc_kernel<true><<<dim3(CONV_CTAS_PER_LANE, L), CONV_THREADS, ConvPolicy<true>::SMEM, st>>>(ca);
  p.mark(st, "conv2_fwd_pool");
  TLK_CUDA(cudaGetLastError());
  Fc1Fwd f1{b, p.lane_dev};
  TLK_CUDA(launch_gemm_tma(f1, dim3(1, 1, L * FC1_SPLITS), st));
  p.mark(st, "fc1_fwd_splitk");
  fc1_reduce_kernel<<<dim3(128 * 64 / 256, L), 256, 0, st>>>(p.lane_dev, b, p.params, p.stride,
                                                              o_f1b);
  p.mark(st, "fc1_reduce");
  TLK_CUDA(cudaGetLastError());
  if ((rc = enqueue_head(p, st, b.h3, 128, o_f2w, o_f2b, b.dz3, o_f1b))) return rc;
  Fc1Dgrad f1d{b, p.lane_dev};  // reads this step's fc1 weights
  TLK_CUDA(launch_gemm_tma(f1d, dim3(9216 / GEMM_BM, 1, L), st));
  p.mark(st, "fc1_dgrad_unpool");
  conv2_wgrad_tc_kernel<<<dim3(C2W_SPLITS, L), CONV_THREADS, WG_SMEM, st>>>(ca);
  p.mark(st, "conv2_wgrad");
  TLK_CUDA(cudaGetLastError());
  conv2_tc_kernel<false><<<dim3(CONV_CTAS_PER_LANE, L), CONV_THREADS, ConvPolicy<false>::SMEM, st>>>(ca);
  p.mark(st, "conv2_dgrad");
  TLK_CUDA(cudaGetLastError());
  conv1_wgrad_kernel<<<dim3(B, L), 128, C1W_SMEM, st>>>(p.lane_dev, b, p.x);
  p.mark(st, "conv1_wgrad");
  TLK_CUDA(cudaGetLastError());
  Fc1WgradOpt f1w{b, p.lane_dev, p.params, p.grads, p.mom1, p.mom2, p.wbf, p.stride, o_f1w,
                  (p.flags & TLK_PACK_WRITE_ALL_GRADS) ? 1 : 0};
  TLK_CUDA(launch_gemm_tma(f1w, dim3(1, 9216 / Fc1WgradOpt::BN, L), st));
  p.mark(st, "fc1_wgrad_adam");
  cnn_finalize_kernel<<<dim3((18432 + 64 + 320 + 255) / 256, L), 256, 0, st>>>(
      p.lane_dev, b, p.grads, p.stride, o_c1w, o_c1b, o_c2w, o_c2b);
  p.mark(st, "grad_finalize");
  TLK_CUDA(cudaGetLastError());
  if ((rc = enqueue_optimizer(p, st))) return rc;
  return enqueue_end_step(p, st);
}

}  // namespace tlk
