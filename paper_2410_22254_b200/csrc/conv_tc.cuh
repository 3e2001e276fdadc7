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
  uint16_t* p2_alt;      // p2 of a lane's odd steps (graph path; null: one buffer)
  uint8_t* idx;          // [L][B][144][64]: argmax (bits 0-1) | live (bit 2)
  const uint16_t* wt;    // [L][wt_stride] (wf | wd)
  int64_t wt_stride;
  const float* params;   // fp32 master (bias)
  int64_t pstride, b2_off;
  float* part2;          // conv2 wgrad partials [L][splits][9][64][32]
  int wgrad_splits;
  // graph path, TLK_CNN_FLAG_JOIN: per-lane count of finished conv2 wgrad
  // CTAs (release); the optimizer waits for it instead of an event join
  uint32_t* c2w_done;
};


// ------------------------------------------- persistent conv2 fwd / dgrad --
// Grid = (CTAS_PER_LANE, lanes); a CTA keeps its lane's weight operand
// resident in shared memory (one TMA bulk load) and loops over that lane's
// 128-position tiles.  Warp roles: warp 4 = TMA producer (double-buffered
// patches), warp 5 = MMA issuer (double-buffered TMEM accumulators), warps
// 0-3 = epilogue (TMEM lane quarters).  Tile i's epilogue overlaps tile i+1's
// patch load and MMAs.
//
//   fwd   : A = h1 patch (4 planes), B = wf, N = 64, 9 taps x 2 K-steps,
//           tiles = 4 output rows of an image (6 per image), epilogue =
//           bias + ReLU + 2x2 maxpool + argmax via a shared fp32 tile.
//   dgrad : A = dz2 patch (8 planes), B = wd, N = 32, 9 taps x 4 K-steps,
//           tiles = 128 positions from row 1 of an image (6 per image),
//           epilogue = ReLU mask with h1 -> dz1 (valid positions only).
#ifndef TLK_CONV_EPW
#define TLK_CONV_EPW 8
#endif
#ifndef TLK_CONV_DBG
#define TLK_CONV_DBG 0  // bits: 1 no MMAs, 2 no epilogue work, 4 no patch loads (timing experiments only)
#endif
#ifndef TLK_CONV_TS
#define TLK_CONV_TS 2
#endif
#ifndef TLK_CONV_AS
#define TLK_CONV_AS 2
#endif
template <bool FWD>
struct ConvPolicy {
  static constexpr int PLANES = FWD ? 4 : 8;
  static constexpr int N = FWD ? 64 : 32;
  static constexpr int KSTEPS = FWD ? 2 : 4;   // K16 steps per tap
  static constexpr int BCHUNK = N * 16;        // bytes per 8-wide K chunk of B
  static constexpr int A_BYTES = PLANES * PATCH_BYTES;
  static constexpr int B_BYTES = 9 * 2 * KSTEPS * BCHUNK;  // 36864 for both
  static constexpr int TILE_BYTES = FWD ? 128 * 68 * 4 : 0;
  static constexpr int AS = TLK_CONV_AS;         // patch stages
  static constexpr int SMEM = B_BYTES + AS * A_BYTES + TILE_BYTES + 128;
  static constexpr int TS = TLK_CONV_TS;         // TMEM accumulators
  static constexpr uint32_t TCOLS = TS * N;
  TLK_DEV static int tap_off(int t) { return FWD ? tap_off_fwd(t) : tap_off_dgrad(t); }
  TLK_DEV static int64_t tile_p0(int tile) {   // first position of the tile
    const int b = tile / 6, k = tile % 6;
    return P28_FRONT + int64_t(b) * P28_IMG + (FWD ? (2 + 4 * k) * P28 : P28 + 128 * k);
  }
};
#ifndef TLK_CONV_CTAS
#define TLK_CONV_CTAS 36
#endif
constexpr int CONV_CTAS_PER_LANE = TLK_CONV_CTAS;
constexpr int CONV_THREADS = 192;  // conv2 wgrad: 4 epilogue + producer + MMA warps
// conv2 fwd / dgrad: EPW epilogue warps (two per TMEM lane quarter when 8,
// each owning half of the accumulator columns), then producer and MMA warps

constexpr int CONV_EPW = TLK_CONV_EPW;
constexpr int CONV_FD_THREADS = 32 * (CONV_EPW + 2);
static_assert(CONV_EPW == 4 || CONV_EPW == 8, "conv2 epilogue warps");

template <bool FWD>
__global__ void __launch_bounds__(CONV_FD_THREADS) conv2_tc_kernel(ConvArgs a) {
  using P = ConvPolicy<FWD>;
  const int j = blockIdx.y;
  if (!a.lanes[j].active) return;
  TLK_KT(FWD ? 1 : 6, a.lanes[0].steps_done);
  const int ntiles = a.B * 6;
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t wfull, afull[P::AS], aempty[P::AS], tfull[P::TS], tempty[P::TS];
  __shared__ uint32_t tmem_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sB = smem_u32(sm), sA0 = sB + P::B_BYTES;
  float* tileS = reinterpret_cast<float*>(sm + P::B_BYTES + P::AS * P::A_BYTES);

  if (tid == 0) {
    mbar_init(&wfull, 1);
    for (int s = 0; s < P::AS; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < P::TS; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], CONV_EPW);  // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<P::TCOLS>(&tmem_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_begin();  // barrier init / TMEM allocation overlap the previous kernel's flush
  TLK_KT_WAITED();
  const uint32_t tmem = tmem_s;
  const uint16_t* src = FWD ? a.h1 + int64_t(j) * 4 * a.npos * 8 : a.dz2 + int64_t(j) * 8 * a.npos * 8;

  constexpr int CH = CONV_EPW / 4;  // column halves per lane quarter
  if (warp == CONV_EPW) {  // ---------------- TMA producer
    if (lane == 0) {
      const uint16_t* w = a.wt + int64_t(j) * a.wt_stride + (FWD ? 0 : CONV2_W);
      mbar_expect_tx(&wfull, P::B_BYTES);
      tma_bulk_g2s(sB, w, P::B_BYTES, &wfull);  // the 9 taps are contiguous
      int i = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
        const int s = i % P::AS;
        if (i >= P::AS) mbar_wait(&aempty[s], ((i / P::AS) - 1) & 1);
        const int64_t p0 = P::tile_p0(tile);
#if TLK_CONV_DBG & 4
        mbar_arrive(&afull[s]);
        (void)p0;
#else
        mbar_expect_tx(&afull[s], P::A_BYTES);
        for (int c = 0; c < P::PLANES; ++c)
          tma_bulk_g2s(sA0 + s * P::A_BYTES + c * PATCH_BYTES, src + (c * a.npos + p0 - HALO) * 8,
                       PATCH_BYTES, &afull[s]);
#endif
      }
    }
  } else if (warp == CONV_EPW + 1) {  // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC = umma_idesc_bf16(128, P::N, false, false);
      const uint64_t bd0 = umma_desc_interleave(sB, P::BCHUNK, 128);
      mbar_wait(&wfull, 0);
      int i = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
        const int s = i % P::AS, ts = i % P::TS;
        mbar_wait(&afull[s], (i / P::AS) & 1);
        if (i >= P::TS) mbar_wait(&tempty[ts], ((i / P::TS) - 1) & 1);
        tc_fence_after();
        const uint64_t ad0 = umma_desc_interleave(sA0 + s * P::A_BYTES + HALO * 16, PATCH_BYTES, 128);
        const uint32_t d = tmem + ts * P::N;
#pragma unroll 1
        for (int t = 0; t < 9; ++t) {
          const int toff = P::tap_off(t);
#pragma unroll
          for (int k = 0; k < P::KSTEPS; ++k) {
            // descriptor start field is address >> 4: offsets add directly
            const uint64_t ad = ad0 + uint64_t((2 * k * PATCH_BYTES + toff * 16) >> 4);
            const uint64_t bd = bd0 + uint64_t(((t * 2 * P::KSTEPS + 2 * k) * P::BCHUNK) >> 4);
#if !(TLK_CONV_DBG & 1)
            mma_bf16(d, ad, bd, IDESC, (t | k) ? 1u : 0u);
#endif
          }
        }
        mma_commit(&aempty[s]);
        mma_commit(&tfull[ts]);
      }
    }
  } else {  // ---------------- epilogue warps (TMEM lanes 32q..32q+31, column half hh)
    const int q4 = warp & 3, hh = warp >> 2;
    const int row = q4 * 32 + lane;
    // dgrad: the h1 ReLU-mask rows of a tile are fetched one tile ahead
    constexpr int NPL = 4 / CH;  // h1 / dz1 planes (8 channels each) of a dgrad warp
    const int c0 = hh * NPL;
    const int64_t hbase = int64_t(j) * 4 * a.npos * 8;
    auto h1_valid = [&](int64_t p0) {
      const int r = int(p0 - P28_FRONT) % P28_IMG + row;  // position within the image
      const int pr = r / P28, pc = r % P28;
      return pr >= 1 && pr <= 26 && pc >= 1 && pc <= 26;
    };
    auto h1_fetch = [&](int tile, uint4 (&hv)[NPL]) {
      const int64_t p0 = P::tile_p0(tile);
      const bool ok = tile < ntiles && h1_valid(p0);
#pragma unroll
      for (int c = 0; c < NPL; ++c)
        hv[c] = ok ? *reinterpret_cast<const uint4*>(a.h1 + hbase + ((c0 + c) * a.npos + p0 + row) * 8)
                   : make_uint4(0, 0, 0, 0);
    };
    uint4 hnext[NPL];
    if constexpr (!FWD) h1_fetch(blockIdx.x, hnext);
    // fwd: a thread's pooled items all have channel chunk tid & 7 (stride 32 * EPW)
    float bb[8];
    // p2 buffer of this step: a lane's odd steps write the second one (graph path)
    uint16_t* const p2 = (a.p2_alt && (a.lanes[j].steps_done & 1)) ? a.p2_alt : a.p2;
    if constexpr (FWD) {
      const float* bias = a.params + j * a.pstride + a.b2_off + (tid & 7) * 8;
#pragma unroll
      for (int e = 0; e < 8; ++e) bb[e] = bias[e];
    }
    int i = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
      const int s = i % P::TS;
      const uint32_t taddr = tmem + s * P::N + (uint32_t(q4 * 32) << 16);
      const int64_t p0 = P::tile_p0(tile);
      if constexpr (FWD) {
        mbar_wait(&tfull[s], (i / P::TS) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int cc = hh; cc < 2; cc += CH) {
          float v[32];
          tmem_ld32(taddr + cc * 32, v);
#pragma unroll
          for (int q = 0; q < 32; q += 4)
            *reinterpret_cast<float4*>(tileS + row * 68 + cc * 32 + q) =
                make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[s]);
        named_bar_sync(1, 32 * CONV_EPW);
        const int b = tile / 6, ti = tile % 6;
        for (int it = tid; it < ((TLK_CONV_DBG & 2) ? 0 : 192); it += 32 * CONV_EPW) {
          const int ch = it & 7, pw = (it >> 3) % 12, phl = (it >> 3) / 12;
          float mx[8];
          int arg[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int m = (2 * phl + (q >> 1)) * P28 + 2 + 2 * pw + (q & 1);
            const float4 lo = *reinterpret_cast<const float4*>(tileS + m * 68 + ch * 8);
            const float4 hi = *reinterpret_cast<const float4*>(tileS + m * 68 + ch * 8 + 4);
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
          uint32_t w4[4], i0 = 0, i1 = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) w4[e] = pack_bf2(mx[2 * e], mx[2 * e + 1]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            i0 |= uint32_t(arg[e] | (mx[e] > 0.0f ? 4 : 0)) << (8 * e);
            i1 |= uint32_t(arg[e + 4] | (mx[e + 4] > 0.0f ? 4 : 0)) << (8 * e);
          }
          *reinterpret_cast<uint4*>(p2 + o) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
          *reinterpret_cast<uint2*>(a.idx + o) = make_uint2(i0, i1);
        }
        named_bar_sync(1, 32 * CONV_EPW);  // tile buffer free for the next tile
      } else {
        const bool valid = h1_valid(p0);
        const int64_t pos = p0 + row;
        const int64_t base = hbase;
        uint4 hv[NPL];
#pragma unroll
        for (int c = 0; c < NPL; ++c) hv[c] = hnext[c];
        h1_fetch(tile + gridDim.x, hnext);  // in flight during this tile's wait and stores
        mbar_wait(&tfull[s], (i / P::TS) & 1);
        tc_fence_after();
        float v[8 * NPL];
        if constexpr (NPL == 4) tmem_ld32(taddr, *reinterpret_cast<float(*)[32]>(v));
        else tmem_ld16(taddr + 8 * c0, *reinterpret_cast<float(*)[16]>(v));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[s]);
        if (!(TLK_CONV_DBG & 2) && valid) {
#pragma unroll
          for (int c = 0; c < NPL; ++c) {
            const uint32_t hw[4] = {hv[c].x, hv[c].y, hv[c].z, hv[c].w};
            uint32_t ow[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float lo = bf2f(uint16_t(hw[e] & 0xFFFF)) > 0.f ? v[c * 8 + 2 * e] : 0.f;
              const float hi = bf2f(uint16_t(hw[e] >> 16)) > 0.f ? v[c * 8 + 2 * e + 1] : 0.f;
              ow[e] = pack_bf2(lo, hi);
            }
            *reinterpret_cast<uint4*>(a.dz1 + base + ((c0 + c) * a.npos + pos) * 8) =
                make_uint4(ow[0], ow[1], ow[2], ow[3]);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<P::TCOLS>(tmem);
}

// ------------------------------------------------------------ conv2 wgrad --
// dW2[oc][tap][ic] = sum_p dz2[p][oc] * h1[p + off(tap)][ic] over all P28
// positions p (dz2's zero border kills invalid ones).  K = positions, both
// operands MN-major (SWIZZLE_NONE).
//   A = h1: for each ic chunk c, FOUR copies of the plane shifted by
//       k = 0..3 positions are staged side by side (MN group g = 4c + k), so
//       A's 128 rows = (ic chunk, kw shift) and ONE M=128 MMA computes the
//       three kw taps of a kernel row (rows with k = 3 are spare).
//   B = dz2 planes: N = 64 oc.
//   D[kh] (TMEM cols 64kh..64kh+63) = rows (k, ic) x cols oc.
// Per 16 positions: 3 MMAs (one per kh) instead of 9, and no zero padding.
// Warp 4 = TMA producer (3-stage ring), warp 5 = MMA issuer, warps 0-2
// write the partials (warp k holds tap kw = k).
constexpr int WG_KC = 128;                        // positions per stage
constexpr int WG_ACOPY = 184 * 16;                // one shifted copy: 184 positions
constexpr int WG_ASTRIDE = 192 * 16;              // copy stride in smem (SBO)
constexpr int WG_A_BYTES = 16 * WG_ASTRIDE;       // 49152
constexpr int WG_B_PLANE = WG_KC * 16;            // 2048
constexpr int WG_B_BYTES = 8 * WG_B_PLANE;        // 16384
constexpr int WG_STAGE = WG_A_BYTES + WG_B_BYTES; // 65536
constexpr int WG_STAGES = 3;
constexpr int WG_SMEM = WG_STAGES * WG_STAGE + 128;
// the k' = 3 copies (spare MMA rows, never read back) are not loaded
constexpr uint32_t WG_TX = 12 * WG_ACOPY + WG_B_BYTES;

static __global__ void __launch_bounds__(CONV_THREADS) conv2_wgrad_tc_kernel(ConvArgs a) {
  const int split = blockIdx.x, j = blockIdx.y;
  if (!a.lanes[j].active) return;
  TLK_KT(5, a.lanes[0].steps_done);
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full_bar[WG_STAGES], empty_bar[WG_STAGES], done_bar;
  __shared__ uint32_t tmem_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t s0 = smem_u32(sm);
  const int nch = a.B * P28_IMG / WG_KC;
  const int c_begin = split * nch / a.wgrad_splits, c_end = (split + 1) * nch / a.wgrad_splits;
  const int n = c_end - c_begin;

  if (tid == 0) {
    for (int s = 0; s < WG_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(&tmem_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_begin();
  TLK_KT_WAITED();
  const uint32_t tmem = tmem_s;

  if (warp == 4) {  // ---------------- TMA producer
    if (lane == 0) {
      const uint16_t* dz2 = a.dz2 + int64_t(j) * 8 * a.npos * 8;
      const uint16_t* h1 = a.h1 + int64_t(j) * 4 * a.npos * 8;
      for (int i = 0; i < n; ++i) {
        const int s = i % WG_STAGES;
        if (i >= WG_STAGES) mbar_wait(&empty_bar[s], ((i / WG_STAGES) - 1) & 1);
        const int64_t q0 = P28_FRONT + int64_t(c_begin + i) * WG_KC;
        const uint32_t st = s0 + s * WG_STAGE;
        mbar_expect_tx(&full_bar[s], WG_TX);
        for (int c = 0; c < 4; ++c)
          for (int k = 0; k < 3; ++k)
            tma_bulk_g2s(st + (c * 4 + k) * WG_ASTRIDE, h1 + (c * a.npos + q0 - HALO + k) * 8,
                         WG_ACOPY, &full_bar[s]);
        for (int c = 0; c < 8; ++c)
          tma_bulk_g2s(st + WG_A_BYTES + c * WG_B_PLANE, dz2 + (c * a.npos + q0) * 8, WG_B_PLANE,
                       &full_bar[s]);
      }
    }
  } else if (warp == 5) {  // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC = umma_idesc_bf16(128, 64, true, true);
      for (int i = 0; i < n; ++i) {
        const int s = i % WG_STAGES;
        mbar_wait(&full_bar[s], (i / WG_STAGES) & 1);
        tc_fence_after();
        const uint32_t st = s0 + s * WG_STAGE;
        const uint64_t ad0 = umma_desc_interleave(st, 128, WG_ASTRIDE);
        const uint64_t bd0 = umma_desc_interleave(st + WG_A_BYTES, 128, WG_B_PLANE);
#pragma unroll
        for (int k = 0; k < WG_KC / 16; ++k)
#pragma unroll
          for (int kh = 0; kh < 3; ++kh) {
            // copy k' of plane c starts at position q0-29+k', so tap (kh, kw=k')
            // of position q0+16k+r sits at index 16k + 28kh + r in every copy
            const uint64_t ad = ad0 + uint64_t(((16 * k + 28 * kh) * 16) >> 4);
            const uint64_t bd = bd0 + uint64_t((k * 256) >> 4);
            mma_bf16(tmem + 64 * kh, ad, bd, IDESC, (i | k) ? 1u : 0u);
          }
        mma_commit(&empty_bar[s]);
      }
      mma_commit(&done_bar);
    }
  }
  if (warp < 4) mbar_wait(&done_bar, 0);
  __syncthreads();
  tc_fence_after();
  if (warp < 4) {
    // TMEM row r = 8g + e with MN group g = 4c + k': warp w holds ic chunk
    // c = w, shift k' = lane >> 3 (k' = 3 is the spare copy), ic = 8c + e.
    const int kp = lane >> 3, ic = warp * 8 + (lane & 7);
    float* out = a.part2 + (int64_t(j) * a.wgrad_splits + split) * 9 * 64 * 32;
#pragma unroll 1
    for (int kh = 0; kh < 3; ++kh)
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        float v[32];
        tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + 64 * kh + 32 * h, v);
        if (kp < 3) {
          float* o = out + ((kh * 3 + kp) * 64 + 32 * h) * 32 + ic;
#pragma unroll
          for (int q = 0; q < 32; ++q) o[q * 32] = v[q];
        }
      }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
  if (a.c2w_done && tid == 0) {  // this CTA's partials are written (release to the optimizer)
    __threadfence();
    atomicAdd(a.c2w_done + j, 1u);
  }
}

}  // namespace tlk
