// Shared definitions of the MNIST CNN pack: buffer table, split counts,
// optimizer-kernel arguments.  Used by the per-phase kernels of the step
// graph (cnn.cu) and by the persistent per-GPU scheduler kernel
// (cnn_persist.cu), which run the same arithmetic.
#pragma once
#include "conv_tc.cuh"
#include "tma.cuh"
#include "pack.cuh"

namespace tlk {

#ifndef TLK_FC1_SPLITS
#define TLK_FC1_SPLITS 18
#endif
constexpr int FC1_SPLITS = TLK_FC1_SPLITS;  // split-K of the fc1 forward (144 k-blocks / 8)
static_assert(144 % FC1_SPLITS == 0, "fc1 split-K must divide the 144 k-blocks");
#ifndef TLK_C2W_SPLITS
#define TLK_C2W_SPLITS 18
#endif
constexpr int C2W_SPLITS = TLK_C2W_SPLITS;  // conv2 wgrad position splits per lane
// every split needs >= 1 of the B * 784 / 128 position chunks (49 at the
// smallest batch, 8): an empty split would commit no MMA and write stale TMEM
static_assert(C2W_SPLITS >= 1 && C2W_SPLITS <= 49, "conv2 wgrad splits must be in [1, 49]");
constexpr int C1W_SMEM = 4 * P28_IMG * 16;  // conv1 wgrad: one image's dz1 planes
#ifndef TLK_C1W_THREADS
#define TLK_C1W_THREADS 256
#endif
constexpr int C1W_THREADS = TLK_C1W_THREADS;  // 8 warps per image: the per-SM warp count hides latency
constexpr int CNN_OPT_CTAS = 24;  // per lane: ~5.4k float4 of non-fc1.w parameters (~1 per thread)

struct CnnBufs {
  // TMA tensor maps of the plain-layout fc1 operands (lanes = dim 2)
  CUtensorMap w1_k;   // fc1.w bf16 [9216 in][128 out]: box 64 x 128 (K-major A)
  CUtensorMap w1_mn;  // fc1.w bf16: box 64 x 64 (MN-major A of dgrad)
  CUtensorMap p2m;    // p2 [9216][B]: box 64 x 64
  CUtensorMap p2m_alt;  // the second p2 buffer (odd steps of a lane; graph path)
  CUtensorMap dz3m;   // dz3 [128][B]: box 64 x 64
  CUtensorMap fa_p, fa_m, fa_v;  // fc1.w optimizer state tiles (fc1 wgrad + Adam), box 128 f x 32 o
  CUtensorMap fh_p, fh_m, fh_v;  // the same, box 128 f x 16 o (persistent path)
  int B;
  int64_t npos;
  uint16_t *h1, *p2, *h3, *dz3, *dz2, *dz1;
  // graph path: conv2 fwd of a lane's odd steps writes p2_alt, so the fc1
  // wgrad + Adam of step k can still read p2(k) while step k+1's forward runs
  uint16_t* p2_alt;
  uint32_t* fwa_cnt;  // fc1 wgrad + Adam: finished CTAs (the last one clears fc1_due)
  uint32_t* c2w_done;  // [L] finished conv2 wgrad CTAs of the step (flag join; reset by the optimizer)
  uint8_t* idx;
  float *colsum, *part_fc1, *part2, *part1;
  float* plog;      // [L][HEAD_CL][64][10] partial logits of the 16-unit slices (persistent path)
  uint32_t* sched;  // persistent path: queue head (u64) + [L][phases] completion counters
  int64_t p2_st, h3_st;
};

__host__ __device__ inline int64_t p28_pos(int b, int r, int c) {
  return P28_FRONT + int64_t(b) * P28_IMG + r * P28 + c;
}

constexpr int HEAD_CL = 8, HEAD_HS = 16;  // fc1 reduce + head: 8 slices of 16 hidden units

constexpr int FWA_SLOTS = 4, FWA_UPD_WARPS = 16;
constexpr int FWA_STAGE_BYTES = 2 * 128 * 64 * 2;  // p2^T and dz3^T tiles (two 64-wide boxes each)
constexpr int FWA_CHUNK = 32 * 128 * 4;            // one tensor's [32 o][128 f] chunk
constexpr int FWA_SLOT_BYTES = 3 * FWA_CHUNK;
constexpr int FWA_SMEM = FWA_STAGE_BYTES + FWA_SLOTS * FWA_SLOT_BYTES + 1024;
constexpr int FWA_THREADS = (2 + FWA_UPD_WARPS) * 32;
constexpr int FWA_FT = 9216 / 128;  // f tiles per lane
struct Fc1WgradAdam {
  CUtensorMap dz3m, p2m;      // operands (bf16, SWIZZLE_128B boxes 64 x 64)
  CUtensorMap tp, tm, tv;     // fc1.w params / m / v: fp32 [lane][128 o][9216 f], box 128 f x 32 o
  CUtensorMap p2m_alt;        // p2 of the lane's odd steps
  LaneState* lanes;           // fc1_due selects the lanes (and their p2 buffer)
  float *params, *m1, *m2, *grads;
  uint16_t* wbf;
  int64_t pstride, w_off;
  int write_grads, kblocks, ntiles;
  uint32_t* cnt;              // finished-CTA counter (last CTA clears fc1_due)
};


constexpr int CNN_OPT_HEAVY_N = 12;
struct CnnOffs {
  int64_t c1w, c1b, c2w, c2b;
};
struct CnnOpt {
  LaneState* lanes;
  int64_t stride, a1, b0;  // float4 units: [0, a1) u [b0, stride/4) of every lane
  CnnOffs o;
  float4 *P, *Gr, *M, *V;
  uint2* Wb;
  WtHook hook;
  uint32_t* c2w_done = nullptr;  // flag join: wait for C2W_SPLITS finished conv2 wgrad CTAs per lane
  // graph-path launch split (cnn.cu): heavy CTAs cover warps h = (hb0 + blockIdx.x) * 8 + w
  // for blockIdx.x < nheavy (h < 80: conv1, 80..95: conv2.b), the rest are light
  // CTAs; `total` CTAs per lane over every launch of the step end it (0: gridDim.x)
  int hb0 = 0, nheavy = CNN_OPT_HEAVY_N, total = 0;
};
__device__ __forceinline__ void cnn_opt_apply(const CnnOpt& a, const LaneState& s, int j, int64_t idx,
                                              const float (&g)[4]) {
  const int64_t i = j * (a.stride / 4) + idx, e = idx * 4;
  a.Gr[i] = make_float4(g[0], g[1], g[2], g[3]);
  float4 pa = a.P[i], ma = a.M[i], va = a.V[i];
  opt_update(s, pa.x, g[0], ma.x, va.x);
  opt_update(s, pa.y, g[1], ma.y, va.y);
  opt_update(s, pa.z, g[2], ma.z, va.z);
  opt_update(s, pa.w, g[3], ma.w, va.w);
  a.P[i] = pa;
  a.M[i] = ma;
  a.V[i] = va;
  const uint32_t lo = pack_bf2(pa.x, pa.y), hi = pack_bf2(pa.z, pa.w);
  a.Wb[i] = make_uint2(lo, hi);
  if (e >= a.hook.off && e < a.hook.off + a.hook.count) {
    wt_write(a.hook, j, e + 0, uint16_t(lo & 0xFFFF));
    wt_write(a.hook, j, e + 1, uint16_t(lo >> 16));
    wt_write(a.hook, j, e + 2, uint16_t(hi & 0xFFFF));
    wt_write(a.hook, j, e + 3, uint16_t(hi >> 16));
  }
}
// CTAs 0..11 of a lane: the 96 float4 whose gradients are long reductions
// (conv1.w / conv1.b over the batch's images, conv2.b over the 144 pooled
// positions), one warp per float4: lane l sums terms l, l+32, ... in order,
// then a fixed xor-shuffle tree.  CTAs 12..: everything else, one float4 per
// thread.
constexpr int CNN_OPT_HEAVY = CNN_OPT_HEAVY_N;

inline ConvArgs conv_args(const Pack& p, const CnnBufs& b) {
  ConvArgs a{};
  a.lanes = p.lane_dev;
  a.B = b.B;
  a.npos = b.npos;
  a.h1 = b.h1;
  a.dz2 = b.dz2;
  a.dz1 = b.dz1;
  a.p2 = b.p2;
  a.p2_alt = b.p2_alt;
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


}  // namespace tlk
