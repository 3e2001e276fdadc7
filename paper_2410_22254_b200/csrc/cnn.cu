// MNIST CNN pack (pytorch/examples Net without dropout), NHWC, all lanes per launch.
//
//   x[28,28] -conv1 3x3 (1->32)+ReLU-> h1[26,26,32] -conv2 3x3 (32->64)+ReLU+maxpool2->
//   p2[12,12,64] -flatten (h,w,c)-> fc1 (9216->128)+ReLU -> h3 -> fc2 (128->10) + CE
//
// Launch sequence of one step (14 kernels, graph-captured):
//   inputs | conv1 fwd (SIMT) | conv2 fwd (tcgen05, im2col gather; epilogue
//   bias+ReLU+2x2 maxpool+argmax) | fc1 fwd (tcgen05 split-K) | fc1 reduce
//   (+bias+ReLU) | head (fc2+CE+bwd) | fc1 wgrad (tcgen05) | fc1 dgrad
//   (tcgen05; epilogue = maxpool/ReLU backward scatter into dz2 + conv2 bias
//   partial sums) | conv2 wgrad (tcgen05 split-K, im2col as MN-major A) |
//   conv2 dgrad (tcgen05, flipped-tap gather of dz2; epilogue ReLU mask) |
//   conv1 wgrad (SIMT split) | grad finalize (deterministic fixed-order
//   reductions) | optimizer | end_step
//
// conv2's output rows are ordered "window-major": m = ((b*12+ph)*12+pw)*4 + q,
// q = dy*2+dx, (oh, ow) = (2ph+dy, 2pw+dx), so every 2x2 pooling window is 4
// consecutive TMEM lanes of one warp and pools with 3 shuffles.
//
// Activation scratch (TLK_BUF_ACTS), each [lanes][...] contiguous, in order:
//   h1 bf16 [B,26,26,32] | p2 bf16 [B,12,12,64] | idx u8 [B,12,12,64] |
//   h3 bf16 [B,128] | dz3 bf16 [B,128] | dz2 bf16 [B*576 window-major, 64] |
//   dz1 bf16 [B,26,26,32]
#include "linear.cuh"
#include "pack.cuh"

namespace tlk {
namespace {

constexpr int FC1_SPLITS = 18;     // 144 k-blocks / 8
constexpr int C2W_SPLITS = 24;     // conv2 wgrad: 576 k-blocks (B=64) / 24
constexpr int C1W_SPLITS = 32;     // conv1 wgrad position splits

struct CnnBufs {
  int B;
  uint16_t *h1, *p2, *h3, *dz3, *dz2, *dz1;
  uint8_t* idx;
  float *colsum, *part_fc1, *part2, *part1;
  int64_t h1_st, p2_st, h3_st, dz2_st, c2w_kb;  // per-lane strides (elements), conv2-wgrad k-blocks
};

// ---------------------------------------------------------------- conv1 -----
// One CTA per (sample, lane).  fp32 math on fp32 master weights.
__global__ void __launch_bounds__(256) conv1_fwd_kernel(const LaneState* __restrict__ lanes,
                                                        const uint16_t* __restrict__ x,
                                                        const float* __restrict__ params,
                                                        int64_t pstride, int64_t w_off,
                                                        int64_t b_off, uint16_t* __restrict__ h1,
                                                        int B) {
  const int s = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  if (!lanes[j].active) return;
  __shared__ float xs[784];
  __shared__ float ws[32 * 9];
  __shared__ float bs[32];
  const uint16_t* xr = x + (size_t(j) * B + s) * 784;
  for (int i = tid; i < 784; i += 256) xs[i] = bf2f(xr[i]);
  for (int i = tid; i < 288; i += 256) ws[i] = params[j * pstride + w_off + i];
  if (tid < 32) bs[tid] = params[j * pstride + b_off + tid];
  __syncthreads();
  uint32_t* out = reinterpret_cast<uint32_t*>(h1 + (size_t(j) * B + s) * 676 * 32);
  for (int i = tid; i < 676 * 16; i += 256) {
    const int pos = i >> 4, oc = (i & 15) * 2;
    const int oh = pos / 26, ow = pos % 26;
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int kh = 0; kh < 3; ++kh)
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) {
        const float xv = xs[(oh + kh) * 28 + ow + kw];
        a0 += xv * ws[oc * 9 + kh * 3 + kw];
        a1 += xv * ws[(oc + 1) * 9 + kh * 3 + kw];
      }
    out[i] = pack_bf2(fmaxf(a0 + bs[oc], 0.f), fmaxf(a1 + bs[oc + 1], 0.f));
  }
}

// ------------------------------------------------------ conv2 fwd (TC) ------
struct Conv2Fwd {
  static constexpr int BN = 64, STAGES = 4;
  static constexpr bool A_MN = false, B_MN = false;
  using Work = LaneWork;
  struct Carry {};
  const LaneState* lanes;
  CnnBufs buf;
  const uint16_t* wbf;
  const float* params;
  int64_t pstride, w_off, b_off;

  TLK_DEV bool work(Work& w) const {
    w.j = blockIdx.z;
    if (!lanes[w.j].active) return false;
    w.m0 = blockIdx.x * GEMM_BM;
    w.n0 = 0;
    w.kb_begin = 0;
    w.kb_end = 5;  // K = 288 -> 4.5 k-blocks
    w.split = 0;
    return true;
  }
  TLK_DEV const void* zero_src() const { return wbf; }
  TLK_DEV const void* a_src(const Work& w, int m, int k) const {
    if (k >= 288) return nullptr;
    const int tap = k >> 5, ic = k & 31, kh = tap / 3, kw = tap % 3;
    const int q = m & 3, win = m >> 2, pw = win % 12, t2 = win / 12, ph = t2 % 12, b = t2 / 12;
    const int oh = 2 * ph + (q >> 1), ow = 2 * pw + (q & 1);
    return buf.h1 + w.j * buf.h1_st + ((int64_t(b) * 26 + oh + kh) * 26 + ow + kw) * 32 + ic;
  }
  TLK_DEV const void* b_src(const Work& w, int n, int k) const {
    return k < 288 ? wbf + w.j * pstride + w_off + n * 288 + k : nullptr;
  }
  TLK_DEV void epilogue(const Work& w, int m, int n0, const float (&v)[32], Carry&) const {
    const int lane = threadIdx.x & 31, base = lane & ~3, q = lane & 3;
    const float* bias = params + w.j * pstride + b_off + n0;
    const int win = m >> 2;  // (b*12+ph)*12+pw
    uint16_t* pout = buf.p2 + w.j * buf.p2_st + int64_t(win) * 64 + n0;
    uint8_t* iout = buf.idx + w.j * buf.p2_st + int64_t(win) * 64 + n0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float a = fmaxf(v[i] + bias[i], 0.0f);
      const float a0 = __shfl_sync(0xffffffffu, a, base + 0);
      const float a1 = __shfl_sync(0xffffffffu, a, base + 1);
      const float a2 = __shfl_sync(0xffffffffu, a, base + 2);
      const float a3 = __shfl_sync(0xffffffffu, a, base + 3);
      if ((i & 3) == q) {  // spread the window's 32 outputs over its 4 lanes
        float mx = a0;
        int arg = 0;
        if (a1 > mx) { mx = a1; arg = 1; }
        if (a2 > mx) { mx = a2; arg = 2; }
        if (a3 > mx) { mx = a3; arg = 3; }
        pout[i] = f2bf(mx);
        iout[i] = uint8_t(arg);
      }
    }
  }
  TLK_DEV void finish(const Work&, int, Carry&) const {}
};

// ------------------------------------------------------ fc1 fwd (TC) --------
// Z^T[o, b] partial sums over a K-split: part[lane][split][o][b].
struct Fc1Fwd {
  static constexpr int BN = 64, STAGES = 4;
  static constexpr bool A_MN = false, B_MN = false;
  using Work = LaneWork;
  struct Carry {};
  const LaneState* lanes;
  CnnBufs buf;
  const uint16_t* wbf;
  int64_t pstride, w_off;

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
  TLK_DEV const void* zero_src() const { return wbf; }
  TLK_DEV const void* a_src(const Work& w, int m, int k) const {
    return wbf + w.j * pstride + w_off + int64_t(m) * 9216 + k;
  }
  TLK_DEV const void* b_src(const Work& w, int n, int k) const {
    return n < buf.B ? buf.p2 + w.j * buf.p2_st + int64_t(n) * 9216 + k : nullptr;
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
// argmax (ReLU mask = pooled value > 0) into dz2 (window-major) and
// accumulates the conv2 bias-gradient partial colsum[f] = sum_b dz2 value.
struct Fc1Dgrad {
  static constexpr int BN = 64, STAGES = 4;
  static constexpr bool A_MN = true, B_MN = false;
  using Work = LaneWork;
  struct Carry {
    float s;
  };
  const LaneState* lanes;
  CnnBufs buf;
  const uint16_t* wbf;
  int64_t pstride, w_off;

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
  TLK_DEV const void* zero_src() const { return wbf; }
  TLK_DEV const void* a_src(const Work& w, int m, int k) const {
    return wbf + w.j * pstride + w_off + int64_t(k) * 9216 + m;
  }
  TLK_DEV const void* b_src(const Work& w, int n, int k) const {
    return n < buf.B ? buf.dz3 + w.j * buf.h3_st + n * 128 + k : nullptr;
  }
  TLK_DEV void epilogue(const Work& w, int f, int n0, const float (&v)[32], Carry& c) const {
    const int pos = f >> 6, ch = f & 63;
    const uint16_t* p2 = buf.p2 + w.j * buf.p2_st + f;
    const uint8_t* ix = buf.idx + w.j * buf.p2_st + f;
    uint16_t* dz = buf.dz2 + w.j * buf.dz2_st + ch;
#pragma unroll 4
    for (int i = 0; i < 32; ++i) {
      const int b = n0 + i;
      if (b >= buf.B) break;
      const int64_t pf = int64_t(b) * 9216;
      const bool live = bf2f(p2[pf]) > 0.0f;
      const uint16_t z = live ? f2bf(v[i]) : uint16_t(0);
      const int q = ix[pf];
      const int64_t row = (int64_t(b) * 144 + pos) * 4;
#pragma unroll
      for (int r = 0; r < 4; ++r) dz[(row + r) * 64] = (r == q) ? z : uint16_t(0);
      c.s += bf2f(z);
    }
  }
  TLK_DEV void finish(const Work& w, int f, Carry& c) const {
    buf.colsum[int64_t(w.j) * 9216 + f] = c.s;
  }
};

// ------------------------------------------------ conv2 wgrad (TC) ----------
// dW2^T[(tap,ic), oc] = sum_m im2col(h1)[m, (tap,ic)] dz2[m, oc] over a K-split
// of m; A = im2col read MN-major (8 channels of one tap per chunk).
struct Conv2Wgrad {
  static constexpr int BN = 64, STAGES = 4;
  static constexpr bool A_MN = true, B_MN = true;
  using Work = LaneWork;
  struct Carry {};
  const LaneState* lanes;
  CnnBufs buf;

  TLK_DEV bool work(Work& w) const {
    w.j = blockIdx.z / C2W_SPLITS;
    w.split = blockIdx.z % C2W_SPLITS;
    if (!lanes[w.j].active) return false;
    w.m0 = blockIdx.x * GEMM_BM;
    w.n0 = 0;
    const int per = int(buf.c2w_kb / C2W_SPLITS);
    w.kb_begin = w.split * per;
    w.kb_end = w.kb_begin + per;
    return true;
  }
  TLK_DEV const void* zero_src() const { return buf.h1; }
  TLK_DEV const void* a_src(const Work& w, int mr, int m) const {
    if (mr >= 288) return nullptr;
    const int tap = mr >> 5, ic = mr & 31, kh = tap / 3, kw = tap % 3;
    const int q = m & 3, win = m >> 2, pw = win % 12, t2 = win / 12, ph = t2 % 12, b = t2 / 12;
    const int oh = 2 * ph + (q >> 1), ow = 2 * pw + (q & 1);
    return buf.h1 + w.j * buf.h1_st + ((int64_t(b) * 26 + oh + kh) * 26 + ow + kw) * 32 + ic;
  }
  TLK_DEV const void* b_src(const Work& w, int n, int m) const {
    return buf.dz2 + w.j * buf.dz2_st + int64_t(m) * 64 + n;
  }
  TLK_DEV void epilogue(const Work& w, int mr, int n0, const float (&v)[32], Carry&) const {
    if (mr >= 288) return;
    float* o = buf.part2 + ((int64_t(w.j) * C2W_SPLITS + w.split) * 288 + mr) * 64 + n0;
#pragma unroll
    for (int i = 0; i < 32; i += 4)
      *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  }
  TLK_DEV void finish(const Work&, int, Carry&) const {}
};

// ------------------------------------------------ conv2 dgrad (TC) ----------
// dh1[(b,ih,iw), ic] = sum_{tap,oc} dz2[(b, ih-kh, iw-kw), oc] W2[oc, tap, ic];
// A gathers the shifted dz2 rows (zero outside 24x24), B = transposed bf16
// shadow W2t[ic][tap][oc] (K-major).  Epilogue: dz1 = bf16(dh1 * [h1 > 0]).
struct Conv2Dgrad {
  static constexpr int BN = 32, STAGES = 4;
  static constexpr bool A_MN = false, B_MN = false;
  using Work = LaneWork;
  struct Carry {};
  const LaneState* lanes;
  CnnBufs buf;
  const uint16_t* wt;
  int64_t wt_st;

  TLK_DEV bool work(Work& w) const {
    w.j = blockIdx.z;
    if (!lanes[w.j].active) return false;
    w.m0 = blockIdx.x * GEMM_BM;
    w.n0 = 0;
    w.kb_begin = 0;
    w.kb_end = 9;
    w.split = 0;
    return true;
  }
  TLK_DEV const void* zero_src() const { return wt; }
  TLK_DEV const void* a_src(const Work& w, int m, int k) const {
    if (m >= buf.B * 676) return nullptr;
    const int tap = k >> 6, oc = k & 63, kh = tap / 3, kw = tap % 3;
    const int iw = m % 26, t = m / 26, ih = t % 26, b = t / 26;
    const int oh = ih - kh, ow = iw - kw;
    if (oh < 0 || oh >= 24 || ow < 0 || ow >= 24) return nullptr;
    const int row = ((b * 12 + (oh >> 1)) * 12 + (ow >> 1)) * 4 + (oh & 1) * 2 + (ow & 1);
    return buf.dz2 + w.j * buf.dz2_st + int64_t(row) * 64 + oc;
  }
  TLK_DEV const void* b_src(const Work& w, int n, int k) const {
    return wt + w.j * wt_st + n * 576 + k;
  }
  TLK_DEV void epilogue(const Work& w, int m, int n0, const float (&v)[32], Carry&) const {
    if (m >= buf.B * 676) return;
    const int64_t base = w.j * buf.h1_st + int64_t(m) * 32;
    const uint4* h = reinterpret_cast<const uint4*>(buf.h1 + base);
    uint4* o = reinterpret_cast<uint4*>(buf.dz1 + base);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 hv = h[c];
      const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
      uint32_t ow[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float lo = bf2f(uint16_t(hw[e] & 0xFFFF)) > 0.f ? v[c * 8 + 2 * e] : 0.f;
        const float hi = bf2f(uint16_t(hw[e] >> 16)) > 0.f ? v[c * 8 + 2 * e + 1] : 0.f;
        ow[e] = pack_bf2(lo, hi);
      }
      o[c] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
    }
  }
  TLK_DEV void finish(const Work&, int, Carry&) const {}
};

// ------------------------------------------------ conv1 wgrad (SIMT) --------
// part1[lane][split][oc][0..8] = tap sums, [9] = bias sum, over a slice of the
// B*676 output positions; thread = (oc, position group), fixed-order reduce.
__global__ void __launch_bounds__(256) conv1_wgrad_kernel(const LaneState* __restrict__ lanes,
                                                          CnnBufs buf,
                                                          const uint16_t* __restrict__ x) {
  const int split = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  if (!lanes[j].active) return;
  const int oc = tid & 31, grp = tid >> 5;
  const int total = buf.B * 676, per = (total + C1W_SPLITS - 1) / C1W_SPLITS;
  const int p0 = split * per, p1 = min(total, p0 + per);
  float acc[10];
#pragma unroll
  for (int t = 0; t < 10; ++t) acc[t] = 0.f;
  const uint16_t* xj = x + int64_t(j) * buf.B * 784;
  const uint16_t* dz = buf.dz1 + j * buf.h1_st;
  for (int p = p0 + grp; p < p1; p += 8) {
    const float g = bf2f(dz[int64_t(p) * 32 + oc]);
    const int ow = p % 26, t = p / 26, oh = t % 26, b = t / 26;
    const uint16_t* xb = xj + b * 784 + oh * 28 + ow;
#pragma unroll
    for (int kh = 0; kh < 3; ++kh)
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) acc[kh * 3 + kw] += g * bf2f(xb[kh * 28 + kw]);
    acc[9] += g;
  }
  __shared__ float red[8][32][10];
#pragma unroll
  for (int t = 0; t < 10; ++t) red[grp][oc][t] = acc[t];
  __syncthreads();
  for (int e = tid; e < 320; e += 256) {
    const int o = e / 10, t = e % 10;
    float s = 0.f;
#pragma unroll
    for (int g = 0; g < 8; ++g) s += red[g][o][t];
    buf.part1[((int64_t(j) * C1W_SPLITS + split) * 32 + o) * 10 + t] = s;
  }
}

// ------------------------------------------------ grad finalize -------------
// Deterministic fixed-order reductions of the split partials into grads:
// conv2.w (transpose back to (oc, tap, ic)), conv2.b (sum over 144 window
// positions), conv1.w / conv1.b (sum over splits).
__global__ void __launch_bounds__(256) cnn_finalize_kernel(const LaneState* __restrict__ lanes,
                                                           CnnBufs buf, float* __restrict__ grads,
                                                           int64_t pstride, int64_t o_c1w,
                                                           int64_t o_c1b, int64_t o_c2w,
                                                           int64_t o_c2b) {
  const int j = blockIdx.y;
  if (!lanes[j].active) return;
  float* G = grads + j * pstride;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < 18432) {  // e = oc*288 + (tap*32+ic)
    const int oc = e / 288, r = e % 288;
    const float* pp = buf.part2 + int64_t(j) * C2W_SPLITS * 288 * 64 + r * 64 + oc;
    float s = 0.f;
#pragma unroll 4
    for (int k = 0; k < C2W_SPLITS; ++k) s += pp[int64_t(k) * 288 * 64];
    G[o_c2w + e] = s;
  } else if (e < 18432 + 64) {
    const int c = e - 18432;
    const float* cs = buf.colsum + int64_t(j) * 9216 + c;
    float s = 0.f;
    for (int pos = 0; pos < 144; ++pos) s += cs[pos * 64];
    G[o_c2b + c] = s;
  } else if (e < 18432 + 64 + 320) {
    const int r = e - 18432 - 64, o = r / 10, t = r % 10;
    const float* pp = buf.part1 + (int64_t(j) * C1W_SPLITS * 32 + o) * 10 + t;
    float s = 0.f;
    for (int k = 0; k < C1W_SPLITS; ++k) s += pp[int64_t(k) * 320];
    if (t < 9)
      G[o_c1w + o * 9 + t] = s;
    else
      G[o_c1b + o] = s;
  }
}

}  // namespace

int cnn_setup(Pack& p) {
  const int64_t L = p.lanes, B = p.batch;
  TLK_CHECK((B * 9) % C2W_SPLITS == 0 && (B * 576) % GEMM_BM == 0, TLK_EINVAL,
            "cnn: batch %d must be a multiple of 8", p.batch);
  auto* b = new CnnBufs{};
  p.scratch = b;
  p.scratch_free = [](void* q) { delete static_cast<CnnBufs*>(q); };
  b->B = int(B);
  b->h1_st = B * 676 * 32;
  b->p2_st = B * 9216;
  b->h3_st = B * 128;
  b->dz2_st = B * 576 * 64;
  b->c2w_kb = B * 576 / 64;
  const size_t acts = size_t(L) * (2 * b->h1_st + 2 * b->p2_st + b->p2_st + 2 * 2 * b->h3_st +
                                   2 * b->dz2_st + 2 * b->h1_st);
  const size_t f32s = size_t(L) * (9216 + FC1_SPLITS * 128 * 64 + C2W_SPLITS * 288 * 64 +
                                   C1W_SPLITS * 320);
  void* base = nullptr;
  int rc = pack_alloc(p, &base, acts + f32s * 4 + 256);
  if (rc) return rc;
  char* c = static_cast<char*>(base);
  auto take = [&](size_t bytes) {
    char* r = c;
    c += (bytes + 15) & ~size_t(15);
    return r;
  };
  b->h1 = reinterpret_cast<uint16_t*>(take(L * b->h1_st * 2));
  b->p2 = reinterpret_cast<uint16_t*>(take(L * b->p2_st * 2));
  b->idx = reinterpret_cast<uint8_t*>(take(L * b->p2_st));
  b->h3 = reinterpret_cast<uint16_t*>(take(L * b->h3_st * 2));
  b->dz3 = reinterpret_cast<uint16_t*>(take(L * b->h3_st * 2));
  b->dz2 = reinterpret_cast<uint16_t*>(take(L * b->dz2_st * 2));
  b->dz1 = reinterpret_cast<uint16_t*>(take(L * b->h1_st * 2));
  p.acts = base;
  p.acts_bytes = size_t(c - static_cast<char*>(base));
  b->colsum = reinterpret_cast<float*>(take(L * 9216 * 4));
  b->part_fc1 = reinterpret_cast<float*>(take(L * FC1_SPLITS * 128 * 64 * 4));
  b->part2 = reinterpret_cast<float*>(take(L * C2W_SPLITS * 288 * 64 * 4));
  b->part1 = reinterpret_cast<float*>(take(L * C1W_SPLITS * 320 * 4));
  void* wt = nullptr;
  p.wt_stride = 576 * 32;
  if ((rc = pack_alloc(p, &wt, L * p.wt_stride * 2))) return rc;
  p.wt = static_cast<uint16_t*>(wt);
  p.launches_per_step = 14;
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
  int rc;
  if ((rc = enqueue_inputs(p, st))) return rc;
  conv1_fwd_kernel<<<dim3(B, L), 256, 0, st>>>(p.lane_dev, p.x, p.params, p.stride, o_c1w, o_c1b,
                                                b.h1, B);
  p.mark(st, "conv1_fwd");
  TLK_CUDA(cudaGetLastError());
  Conv2Fwd c2f{p.lane_dev, b, p.wbf, p.params, p.stride, o_c2w, o_c2b};
  TLK_CUDA(launch_gemm(c2f, dim3(B * 576 / GEMM_BM, 1, L), st));
  p.mark(st, "conv2_fwd_pool");
  Fc1Fwd f1{p.lane_dev, b, p.wbf, p.stride, o_f1w};
  TLK_CUDA(launch_gemm(f1, dim3(1, 1, L * FC1_SPLITS), st));
  p.mark(st, "fc1_fwd_splitk");
  fc1_reduce_kernel<<<dim3(128 * 64 / 256, L), 256, 0, st>>>(p.lane_dev, b, p.params, p.stride,
                                                              o_f1b);
  p.mark(st, "fc1_reduce");
  TLK_CUDA(cudaGetLastError());
  if ((rc = enqueue_head(p, st, b.h3, 128, o_f2w, o_f2b, b.dz3, o_f1b))) return rc;
  LinWgrad f1w{p.lane_dev, b.dz3, b.h3_st, b.p2, b.p2_st, p.grads, p.stride, o_f1w, 128, 9216, B};
  TLK_CUDA(launch_gemm(f1w, dim3(1, 9216 / LinWgrad::BN, L), st));
  p.mark(st, "fc1_wgrad");
  Fc1Dgrad f1d{p.lane_dev, b, p.wbf, p.stride, o_f1w};
  TLK_CUDA(launch_gemm(f1d, dim3(9216 / GEMM_BM, 1, L), st));
  p.mark(st, "fc1_dgrad_unpool");
  Conv2Wgrad c2w{p.lane_dev, b};
  TLK_CUDA(launch_gemm(c2w, dim3(3, 1, L * C2W_SPLITS), st));
  p.mark(st, "conv2_wgrad_splitk");
  Conv2Dgrad c2d{p.lane_dev, b, p.wt, p.wt_stride};
  TLK_CUDA(launch_gemm(c2d, dim3((B * 676 + GEMM_BM - 1) / GEMM_BM, 1, L), st));
  p.mark(st, "conv2_dgrad");
  conv1_wgrad_kernel<<<dim3(C1W_SPLITS, L), 256, 0, st>>>(p.lane_dev, b, p.x);
  p.mark(st, "conv1_wgrad");
  TLK_CUDA(cudaGetLastError());
  cnn_finalize_kernel<<<dim3((18432 + 64 + 320 + 255) / 256, L), 256, 0, st>>>(
      p.lane_dev, b, p.grads, p.stride, o_c1w, o_c1b, o_c2w, o_c2b);
  p.mark(st, "grad_finalize");
  TLK_CUDA(cudaGetLastError());
  if ((rc = enqueue_optimizer(p, st))) return rc;
  return enqueue_end_step(p, st);
}

}  // namespace tlk
