// tcgen05 conv2 kernels (fwd / dgrad / wgrad) -- see conv_layout.cuh for the
// P28 layout and why every tap is a descriptor offset.
#pragma once
#include "conv_layout.cuh"
#include "models.cuh"
#include "tlk_ptx.cuh"

namespace tlk {

struct ConvArgs {
  const LaneState* lanes;
  int B;
  int64_t npos;          // positions per plane
  const uint16_t* h1;    // [L][4][npos][8]
  uint16_t* dz2;         // [L][8][npos][8]
  uint16_t* dz1;         // [L][4][npos][8]
  uint16_t* p2;          // [L][B][144][64]
  uint8_t* idx;          // [L][B][144][64]: argmax (bits 0-1) | live (bit 2)
  const uint16_t* wt;    // [L][wt_stride] (wf | wd)
  int64_t wt_stride;
  const float* params;   // fp32 master (bias)
  int64_t pstride, b2_off;
  float* part2;          // conv2 wgrad partials [L][splits][9][64][32]
  int wgrad_splits;
};

// ------------------------------------------------------------ conv2 fwd ----
// CTA = (4 output rows of one image, lane): M = 128 P28 positions starting at
// row 2+4i (112 real + 16 spill), N = 64 oc, K = 9 taps x 32 ic = 18 MMAs.
// Epilogue: bias + ReLU + 2x2 maxpool + argmax through a shared-memory tile.
constexpr int FWD_SMEM_A = 4 * PATCH_BYTES;           // 11904
constexpr int FWD_SMEM_B = 9 * 4 * 1024;              // 36864
constexpr int FWD_SMEM = FWD_SMEM_A + FWD_SMEM_B + 128;
constexpr int FWD_TILE_LD = 68;                       // floats per staged row

__global__ void __launch_bounds__(128) conv2_fwd_tc_kernel(ConvArgs a) {
  const int tile = blockIdx.x, j = blockIdx.y;
  if (!a.lanes[j].active) return;
  const int b = tile / 6, ti = tile % 6;
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full_bar, done_bar;
  __shared__ uint32_t tmem_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sA = smem_u32(sm), sB = sA + FWD_SMEM_A;
  const int64_t p0 = P28_FRONT + int64_t(b) * P28_IMG + (2 + 4 * ti) * P28;

  if (tid == 0) {
    mbar_init(&full_bar, 1);
    mbar_init(&done_bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<64>(&tmem_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;

  if (tid == 0) {
    mbar_expect_tx(&full_bar, FWD_SMEM_A + FWD_SMEM_B);
    const uint16_t* h1 = a.h1 + int64_t(j) * 4 * a.npos * 8;
    for (int c = 0; c < 4; ++c)
      tma_bulk_g2s(sA + c * PATCH_BYTES, h1 + (c * a.npos + p0 - HALO) * 8, PATCH_BYTES, &full_bar);
    const uint16_t* wf = a.wt + int64_t(j) * a.wt_stride;
    for (int t = 0; t < 9; ++t)
      tma_bulk_g2s(sB + t * 4096, wf + t * 2048, 4096, &full_bar);
    mbar_wait(&full_bar, 0);
    tc_fence_after();
    constexpr uint32_t IDESC = umma_idesc_bf16(128, 64, false, false);
#pragma unroll 1
    for (int t = 0; t < 9; ++t)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint64_t ad = umma_desc_interleave(
            sA + 2 * h * PATCH_BYTES + (HALO + tap_off_fwd(t)) * 16, PATCH_BYTES, 128);
        const uint64_t bd = umma_desc_interleave(sB + (t * 4 + 2 * h) * 1024, 1024, 128);
        mma_bf16(tmem, ad, bd, IDESC, (t | h) ? 1u : 0u);
      }
    mma_commit(&done_bar);
  }
  mbar_wait(&done_bar, 0);
  tc_fence_after();
  // TMEM -> shared tile [128][68] fp32 (the operand area is free now)
  float* tileS = reinterpret_cast<float*>(sm);
  const int row = warp * 32 + lane;
#pragma unroll 1
  for (int cc = 0; cc < 2; ++cc) {
    float v[32];
    tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + cc * 32, v);
#pragma unroll
    for (int i = 0; i < 32; i += 4)
      *reinterpret_cast<float4*>(tileS + row * FWD_TILE_LD + cc * 32 + i) =
          make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  }
  tc_fence_before();
  __syncthreads();
  // 2 pooled rows x 12 pooled cols x 8 channel chunks = 192 items
  const float* bias = a.params + j * a.pstride + a.b2_off;
  for (int it = tid; it < 192; it += 128) {
    const int ch = it & 7, pw = (it >> 3) % 12, phl = (it >> 3) / 12;
    float mx[8], bb[8];
    int arg[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) bb[e] = bias[ch * 8 + e];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int m = (2 * phl + (q >> 1)) * P28 + 2 + 2 * pw + (q & 1);
      const float4 lo = *reinterpret_cast<const float4*>(tileS + m * FWD_TILE_LD + ch * 8);
      const float4 hi = *reinterpret_cast<const float4*>(tileS + m * FWD_TILE_LD + ch * 8 + 4);
      const float z[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float r = fmaxf(z[e] + bb[e], 0.0f);
        if (q == 0 || r > mx[e]) {
          mx[e] = r;
          arg[e] = q;
        }
      }
    }
    const int ph = 2 * ti + phl;
    const int64_t o = ((int64_t(j) * a.B + b) * 144 + ph * 12 + pw) * 64 + ch * 8;
    uint32_t w[4];
    uint32_t i0 = 0, i1 = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) w[e] = pack_bf2(mx[2 * e], mx[2 * e + 1]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      i0 |= uint32_t(arg[e] | (mx[e] > 0.0f ? 4 : 0)) << (8 * e);
      i1 |= uint32_t(arg[e + 4] | (mx[e + 4] > 0.0f ? 4 : 0)) << (8 * e);
    }
    *reinterpret_cast<uint4*>(a.p2 + o) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint2*>(a.idx + o) = make_uint2(i0, i1);
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc<64>(tmem);
}

// ------------------------------------------------------------ conv2 dgrad --
// CTA = 128 consecutive P28 positions (rows 1..26 of one image, 6 tiles),
// N = 32 ic, K = 9 taps x 64 oc (36 MMAs).  Epilogue: ReLU mask with h1,
// write dz1 (valid 26x26 positions only; the border stays zero).
constexpr int DG_SMEM_A = 8 * PATCH_BYTES;       // 23808
constexpr int DG_SMEM_B = 9 * 8 * 512;           // 36864
constexpr int DG_SMEM = DG_SMEM_A + DG_SMEM_B + 128;

__global__ void __launch_bounds__(128) conv2_dgrad_tc_kernel(ConvArgs a) {
  const int tile = blockIdx.x, j = blockIdx.y;
  if (!a.lanes[j].active) return;
  const int b = tile / 6, tk = tile % 6;
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full_bar, done_bar;
  __shared__ uint32_t tmem_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sA = smem_u32(sm), sB = sA + DG_SMEM_A;
  const int64_t p0 = P28_FRONT + int64_t(b) * P28_IMG + P28 + 128 * tk;

  if (tid == 0) {
    mbar_init(&full_bar, 1);
    mbar_init(&done_bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<32>(&tmem_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;

  if (tid == 0) {
    mbar_expect_tx(&full_bar, DG_SMEM_A + DG_SMEM_B);
    const uint16_t* dz2 = a.dz2 + int64_t(j) * 8 * a.npos * 8;
    for (int c = 0; c < 8; ++c)
      tma_bulk_g2s(sA + c * PATCH_BYTES, dz2 + (c * a.npos + p0 - HALO) * 8, PATCH_BYTES, &full_bar);
    const uint16_t* wd = a.wt + int64_t(j) * a.wt_stride + CONV2_W;
    for (int t = 0; t < 9; ++t)
      tma_bulk_g2s(sB + t * 4096, wd + t * 2048, 4096, &full_bar);
    mbar_wait(&full_bar, 0);
    tc_fence_after();
    constexpr uint32_t IDESC = umma_idesc_bf16(128, 32, false, false);
#pragma unroll 1
    for (int t = 0; t < 9; ++t)
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const uint64_t ad = umma_desc_interleave(
            sA + 2 * s * PATCH_BYTES + (HALO + tap_off_dgrad(t)) * 16, PATCH_BYTES, 128);
        const uint64_t bd = umma_desc_interleave(sB + (t * 8 + 2 * s) * 512, 512, 128);
        mma_bf16(tmem, ad, bd, IDESC, (t | s) ? 1u : 0u);
      }
    mma_commit(&done_bar);
  }
  mbar_wait(&done_bar, 0);
  tc_fence_after();
  float v[32];
  tmem_ld32(tmem + (uint32_t(warp * 32) << 16), v);
  const int r = (P28 + 128 * tk + warp * 32 + lane);  // position within image
  const int pr = r / P28, pc = r % P28;
  if (pr >= 1 && pr <= 26 && pc >= 1 && pc <= 26) {
    const int64_t pos = p0 + warp * 32 + lane;
    const int64_t base = int64_t(j) * 4 * a.npos * 8;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 hv = *reinterpret_cast<const uint4*>(a.h1 + base + (c * a.npos + pos) * 8);
      const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
      uint32_t ow[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float lo = bf2f(uint16_t(hw[e] & 0xFFFF)) > 0.f ? v[c * 8 + 2 * e] : 0.f;
        const float hi = bf2f(uint16_t(hw[e] >> 16)) > 0.f ? v[c * 8 + 2 * e + 1] : 0.f;
        ow[e] = pack_bf2(lo, hi);
      }
      *reinterpret_cast<uint4*>(a.dz1 + base + (c * a.npos + pos) * 8) =
          make_uint4(ow[0], ow[1], ow[2], ow[3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<32>(tmem);
}

// ------------------------------------------------------------ conv2 wgrad --
// dW2[oc][tap][ic] = sum_p dz2[p][oc] * h1[p + off(tap)][ic] over all P28
// positions p (dz2's zero border kills invalid ones).  K = positions, both
// operands MN-major.  M = 64 oc + 64 zero rows (UMMA M = 128), N = 32 ic per
// tap, 9 accumulators in TMEM columns [32t, 32t+32).  CTA = (position range,
// lane); 3-stage TMA-bulk ring of 128-position chunks.
constexpr int WG_KC = 128;                        // positions per stage
constexpr int WG_A_PLANE = WG_KC * 16;            // 2048
constexpr int WG_A_BYTES = 16 * WG_A_PLANE;       // 8 real + 8 zero planes
constexpr int WG_B_PLANE = 192 * 16;              // 186 used, padded to 192
constexpr int WG_B_BYTES = 4 * WG_B_PLANE;
constexpr int WG_STAGE = WG_A_BYTES + WG_B_BYTES; // 45056
constexpr int WG_STAGES = 3;
constexpr int WG_SMEM = WG_STAGES * WG_STAGE + 128;
constexpr uint32_t WG_TX = 8 * WG_A_PLANE + 4 * PATCH_BYTES;

__global__ void __launch_bounds__(128) conv2_wgrad_tc_kernel(ConvArgs a) {
  const int split = blockIdx.x, j = blockIdx.y;
  if (!a.lanes[j].active) return;
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full_bar[WG_STAGES], empty_bar[WG_STAGES], done_bar;
  __shared__ uint32_t tmem_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t s0 = smem_u32(sm);
  const int nch = a.B * P28_IMG / WG_KC;
  const int c_begin = split * nch / a.wgrad_splits, c_end = (split + 1) * nch / a.wgrad_splits;

  // zero the padding planes (A rows 64..127) of every stage once
  for (int s = 0; s < WG_STAGES; ++s) {
    uint4* z = reinterpret_cast<uint4*>(sm + s * WG_STAGE + 8 * WG_A_PLANE);
    for (int i = tid; i < 8 * WG_A_PLANE / 16; i += 128) z[i] = make_uint4(0, 0, 0, 0);
  }
  fence_proxy_async_smem();
  if (tid == 0) {
    for (int s = 0; s < WG_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;

  if (tid == 0) {
    const uint16_t* dz2 = a.dz2 + int64_t(j) * 8 * a.npos * 8;
    const uint16_t* h1 = a.h1 + int64_t(j) * 4 * a.npos * 8;
    auto load = [&](int c, int s) {
      const int64_t q0 = P28_FRONT + int64_t(c) * WG_KC;
      const uint32_t st = s0 + s * WG_STAGE;
      mbar_expect_tx(&full_bar[s], WG_TX);
      for (int k = 0; k < 8; ++k)
        tma_bulk_g2s(st + k * WG_A_PLANE, dz2 + (k * a.npos + q0) * 8, WG_A_PLANE, &full_bar[s]);
      for (int k = 0; k < 4; ++k)
        tma_bulk_g2s(st + WG_A_BYTES + k * WG_B_PLANE, h1 + (k * a.npos + q0 - HALO) * 8,
                     PATCH_BYTES, &full_bar[s]);
    };
    const int n = c_end - c_begin;
    for (int i = 0; i < WG_STAGES - 1 && i < n; ++i) load(c_begin + i, i);
    constexpr uint32_t IDESC = umma_idesc_bf16(128, 32, true, true);
    for (int i = 0; i < n; ++i) {
      const int s = i % WG_STAGES;
      mbar_wait(&full_bar[s], (i / WG_STAGES) & 1);
      tc_fence_after();
      const uint32_t st = s0 + s * WG_STAGE;
#pragma unroll 1
      for (int k = 0; k < WG_KC / 16; ++k)
#pragma unroll
        for (int t = 0; t < 9; ++t) {
          const uint64_t ad = umma_desc_interleave(st + k * 256, 128, WG_A_PLANE);
          const uint64_t bd = umma_desc_interleave(
              st + WG_A_BYTES + (HALO + tap_off_fwd(t) + 16 * k) * 16, 128, WG_B_PLANE);
          mma_bf16(tmem + 32 * t, ad, bd, IDESC, (i | k) ? 1u : 0u);
        }
      mma_commit(&empty_bar[s]);
      const int nxt = i + WG_STAGES - 1;
      if (nxt < n) {
        const int sn = nxt % WG_STAGES;
        if (nxt >= WG_STAGES) mbar_wait(&empty_bar[sn], ((nxt / WG_STAGES) - 1) & 1);
        load(c_begin + nxt, sn);
      }
    }
    mma_commit(&done_bar);
  }
  mbar_wait(&done_bar, 0);
  tc_fence_after();
  if (warp < 2) {  // rows 0..63 = oc
    const int oc = warp * 32 + lane;
    float* out = a.part2 + ((int64_t(j) * a.wgrad_splits + split) * 9 * 64 + oc) * 32;
#pragma unroll 1
    for (int t = 0; t < 9; ++t) {
      float v[32];
      tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + 32 * t, v);
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        *reinterpret_cast<float4*>(out + t * 64 * 32 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

}  // namespace tlk
