// Fused causal attention for the transformer packs: one persistent launch
// for the forward, one for the backward, per layer.  S, P, dP and dS never
// leave the SM; only Q/K/V/dY are read and Y, dQ/dK/dV plus two floats of row
// statistics per query are written.  Replaces the scores / PV / dP / dQ / dK /
// dV launches of the unfused path (gpt.cu, TLK_ATTN_FUSED=0), which
// materialise P and dS in HBM ([T][T] bf16 per sequence and head).
//
// Work item = one (lane, sequence, head).  T = NB x 128 (NB = 1, 2); dh = 64.
// Every 128-row block of Q / K / V / dY is one 16 KB TMA box (64 bf16 x 128
// rows, 128-byte swizzle) in a ring of smem slots.  A box is a K-major UMMA
// operand (K = head dim) AND, read with the MN-major descriptor, the
// MN-major operand of the products whose K runs over sequence positions --
// the same bytes, two descriptors.  The P / dS tiles the softmax warps write
// are laid out the same way, so P serves as the K-major A of P V and as the
// MN-major A of P^T dY.
//
// Numerics are the unfused path's, operation for operation (bit-identical
// outputs are the contract, tests/test_gpu_attn.py):
//   forward  row max / sum over the same column halves (two warps per TMEM
//            lane quarter), p = ex2(s k2 - m k2) / sum on the SFU, P stored
//            bf16, Y = bf16(P V) with the keys in ascending order;
//   backward P recomputed from S with the forward's (m k2, 1/sum) row stats
//            (identical bits), dS = bf16(bf16(P) (dP - D) scale) with
//            D = rowsum(dY o Y) (attn_rowdot_kernel), dQ / dK / dV = bf16 of
//            the causal k-range products, their qkv.b column partials from the
//            shared bf16 epilogue (EpiOps::tile4).
#pragma once
#include "sgemm.cuh"
#include "tma.cuh"

namespace tlk {

constexpr int ATT_ROWS = 128;                  // rows per block (queries or keys)
constexpr uint32_t ATT_BOX = 128 * 64 * 2;     // one block: 128 rows x 64 bf16 (16 KB)
constexpr int ATT_EW = 8;                      // softmax / epilogue warps
constexpr int ATT_THREADS = (ATT_EW + 2) * 32;  // + TMA producer + MMA issuer
constexpr int ATT_STAGING = ATT_EW * 32 * 33 * 4;

struct AttnArgs {
  CUtensorMap tq, tk, tv, tdy;  // 5-D {dh, T, head, sequence, lane} views, box {64, 128}
  const LaneState* lanes;
  int nb, nh, items;            // sequences per lane, heads, lanes * nb * nh
  float scale;
  float* stats;                 // [lane][b][h][T] x (m k2, 1 / sum), written fwd, read bwd
  const float* D;               // bwd: rowsum(dY o Y), same indexing as stats
  EpiOps ey;                    // fwd: Y (EPI_BF16)
  EpiOps edq, edk, edv;         // bwd: dQ / dK / dV (EPI_BF16 + qkv.b column partials)
};

// K-major SW128 operand: 128-byte rows, 8-row atoms 1 KB apart; K step of 16
// elements = +32 B.  MN-major: K rows of 64 MN elements; 16 K rows = +2 KB;
// 64-wide MN blocks `lbo` bytes apart.
TLK_DEV uint64_t att_kdesc(uint32_t base, int kk) { return umma_desc_sw128(base + kk * 32, 16, 1024); }
TLK_DEV uint64_t att_mdesc(uint32_t base, int kk, uint32_t lbo) {
  return umma_desc_sw128(base + kk * 2048, lbo, 1024);
}

TLK_DEV bool att_item(const AttnArgs& a, int it, ZWork& w) {
  const int per = a.nb * a.nh;
  w.j = it / per;
  const int r = it % per;
  w.zb = r / a.nh;
  w.zh = r % a.nh;
  w.n0 = 0;
  return a.lanes[w.j].active != 0;
}

TLK_DEV int64_t att_row(const AttnArgs& a, const ZWork& w, int T, int m) {
  return ((int64_t(w.j) * a.nb + w.zb) * a.nh + w.zh) * T + m;
}

// Write 32 values (columns c0 .. c0+31 of row r) as bf16 into a SW128 tile
// whose 64-column blocks are 16 KB apart.
TLK_DEV void att_put32(uint8_t* tile, int r, int c0, const uint32_t (&pk)[16]) {
  uint8_t* blk = tile + (c0 >> 6) * ATT_BOX;
  const int ch0 = (c0 & 63) >> 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    *reinterpret_cast<uint4*>(blk + sw128(r, ch0 + i)) = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
}

// ============================================================== forward ====
// Tiles t = (item, qb) in order; S(t) goes to TMEM buffer t & 1 (NB x 128
// columns), O(t) = P(t) V into the first 64 columns of the same buffer once
// the softmax warps have consumed S(t).  Ring order per item: Q0 K0 V0 Q1 K1 V1.
template <int NB>
struct AttnFwdCfg {
  static constexpr int T = NB * ATT_ROWS;
  static constexpr int NSLOT = 6;
  static constexpr uint32_t BW = NB * 128;  // TMEM columns per S buffer
  static constexpr uint32_t TCOLS = NB == 1 ? 256 : 512;
  static constexpr uint32_t P_BYTES = NB * 2 * ATT_BOX;  // 128 rows x T keys
  static constexpr int SMEM = NSLOT * ATT_BOX + P_BYTES + ATT_STAGING + 1024;
};

template <int NB>
__global__ void __launch_bounds__(ATT_THREADS, 1) attn_fwd_kernel(const __grid_constant__ AttnArgs a) {
  using C = AttnFwdCfg<NB>;
  constexpr int T = C::T, NSLOT = C::NSLOT;
  constexpr uint32_t IDESC_S = umma_idesc_bf16(128, 128, false, false);
  constexpr uint32_t IDESC_O = umma_idesc_bf16(128, 64, false, true);
  pdl_begin();
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[NSLOT], empty[NSLOT], sfull[2], tempty[2], pfull, ofull;
  __shared__ uint32_t tmem_s;
  __shared__ float xchg[2][2][128];  // [max, sum][part][row]
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t ring = smem_u32(smem);
  uint8_t* Pt = smem + NSLOT * ATT_BOX;
  const uint32_t psm = smem_u32(Pt);
  float* staging = reinterpret_cast<float*>(Pt + C::P_BYTES);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sfull[b], 1);
      mbar_init(&tempty[b], ATT_EW);
    }
    mbar_init(&pfull, 1);
    mbar_init(&ofull, 1);
    fence_mbar_init();
  }
  if (warp == ATT_EW + 1) tmem_alloc<C::TCOLS>(&tmem_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;

  if (warp == ATT_EW) {  // ------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&a.tq);
      tma_prefetch_desc(&a.tk);
      tma_prefetch_desc(&a.tv);
      int bc = 0;
      for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
        ZWork w;
        if (!att_item(a, it, w)) continue;
        for (int qb = 0; qb < NB; ++qb)
          for (int k = 0; k < 3; ++k, ++bc) {
            const int s = bc % NSLOT;
            if (bc >= NSLOT) mbar_wait(&empty[s], ((bc / NSLOT) - 1) & 1);
            mbar_expect_tx(&full[s], ATT_BOX);
            const CUtensorMap* m = k == 0 ? &a.tq : k == 1 ? &a.tk : &a.tv;
            tma_load_5d(ring + s * ATT_BOX, m, 0, qb * ATT_ROWS, w.zh, w.zb, w.j, &full[s]);
          }
      }
    }
  } else if (warp == ATT_EW + 1) {  // ------------------------- MMA issuer
    if (lane == 0) {
      // block (qb, kind) of the item starting at ring counter `base`
      auto slot = [&](int base, int qb, int k) { return (base + 3 * qb + k) % NSLOT; };
      auto par = [&](int base, int qb, int k) { return uint32_t(((base + 3 * qb + k) / NSLOT) & 1); };
      int bc = 0, t = 0;
      int pbase = -1, pqb = 0, pt = 0;  // the tile whose O product is pending
      auto issue_o = [&]() {
        const uint32_t d = tmem + (pt & 1) * C::BW;
        mbar_wait(&pfull, pt & 1);
        tc_fence_after();
        for (int kb = 0; kb <= pqb; ++kb) {
          mbar_wait(&full[slot(pbase, kb, 2)], par(pbase, kb, 2));
          tc_fence_after();
          const uint32_t vs = ring + slot(pbase, kb, 2) * ATT_BOX;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int key = kb * 128 + kk * 16;
            mma_bf16(d, att_kdesc(psm + (key >> 6) * ATT_BOX, (key & 63) >> 4), att_mdesc(vs, kk, 8192), IDESC_O,
                     (kb > 0 || kk > 0) ? 1u : 0u);
          }
        }
        mma_commit(&ofull);
        if (pqb == NB - 1)
          for (int kb = 0; kb < NB; ++kb) mma_commit(&empty[slot(pbase, kb, 2)]);
      };
      for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
        ZWork w;
        if (!att_item(a, it, w)) continue;
        const int base = bc;
        bc += 3 * NB;
        for (int qb = 0; qb < NB; ++qb, ++t) {
          const int b = t & 1;
          if (t >= 2) mbar_wait(&tempty[b], ((t >> 1) - 1) & 1);
          mbar_wait(&full[slot(base, qb, 0)], par(base, qb, 0));
          tc_fence_after();
          const uint32_t qs = ring + slot(base, qb, 0) * ATT_BOX, d = tmem + b * C::BW;
          for (int kb = 0; kb <= qb; ++kb) {
            mbar_wait(&full[slot(base, kb, 1)], par(base, kb, 1));
            tc_fence_after();
            const uint32_t ks = ring + slot(base, kb, 1) * ATT_BOX;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16(d + kb * 128, att_kdesc(qs, kk), att_kdesc(ks, kk), IDESC_S, kk > 0 ? 1u : 0u);
          }
          mma_commit(&sfull[b]);
          mma_commit(&empty[slot(base, qb, 0)]);
          if (qb == NB - 1)
            for (int kb = 0; kb < NB; ++kb) mma_commit(&empty[slot(base, kb, 1)]);
          if (pbase >= 0) issue_o();
          pbase = base;
          pqb = qb;
          pt = t;
        }
      }
      if (pbase >= 0) issue_o();
    }
  } else {  // -------------------------------- softmax + Y epilogue warps
    const int q = warp & 3, part = warp >> 2;
    float* buf = staging + warp * (32 * 33);
    const float k2 = a.scale * 1.4426950408889634f;
    constexpr int HALF = T / 2;  // the unfused row epilogue's column parts
    int t = 0;
    for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
      ZWork w;
      if (!att_item(a, it, w)) continue;
      for (int qb = 0; qb < NB; ++qb, ++t) {
        const int b = t & 1;
        const int row0 = qb * ATT_ROWS + q * 32, m = row0 + lane, r = q * 32 + lane;
        const int ncols = (qb + 1) * ATT_ROWS;     // keys this query block sees
        const int wlim = min(T, row0 + 32);        // warp-uniform causal chunk bound
        const int lim = m + 1;
        const int cbeg = part * HALF, cend = min(cbeg + HALF, wlim);
        const uint32_t ts = tmem + b * C::BW + (uint32_t(q * 32) << 16);
        mbar_wait(&sfull[b], (t >> 1) & 1);
        tc_fence_after();
        float v[32];
        float mx = -INFINITY;
        for (int c0 = cbeg; c0 < cend; c0 += 32) {
          tmem_ld32(ts + c0, v);
          if (c0 < row0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) mx = fmaxf(mx, v[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c0 + i < lim) mx = fmaxf(mx, v[i]);
          }
        }
        xchg[0][part][r] = mx;
        named_bar_sync(1, ATT_EW * 32);
        mx = fmaxf(xchg[0][0][r], xchg[0][1][r]);
        const float mk = mx * k2;
        float s = 0.f;
        for (int c0 = cbeg; c0 < cend; c0 += 32) {
          tmem_ld32(ts + c0, v);
          if (c0 < row0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) s += ex2_approx(fmaf(v[i], k2, -mk));
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c0 + i < lim) s += ex2_approx(fmaf(v[i], k2, -mk));
          }
        }
        xchg[1][part][r] = s;
        named_bar_sync(1, ATT_EW * 32);
        s = xchg[1][0][r] + xchg[1][1][r];
        const float inv = 1.f / s;
        if (part == 0) {
          float2* st = reinterpret_cast<float2*>(a.stats) + att_row(a, w, T, m);
          *st = make_float2(mk, inv);
        }
        // P (bf16) for keys [0, ncols): the two parts split the valid range
        const int pw = ncols / 2, pb0 = part * pw, pb1 = pb0 + pw;
        for (int c0 = pb0; c0 < pb1; c0 += 32) {
          uint32_t pk[16];
          if (c0 < wlim) {
            tmem_ld32(ts + c0, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float p0 = (c0 + 2 * i < lim) ? ex2_approx(fmaf(v[2 * i], k2, -mk)) * inv : 0.f;
              const float p1 = (c0 + 2 * i + 1 < lim) ? ex2_approx(fmaf(v[2 * i + 1], k2, -mk)) * inv : 0.f;
              pk[i] = pack_bf2(p0, p1);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = 0u;
          }
          att_put32(Pt, r, c0, pk);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        named_bar_sync(1, ATT_EW * 32);
        if (warp == 0 && lane == 0) mbar_arrive(&pfull);
        // Y = P V (TMEM buffer b, columns 0..63) -> bf16 rows
        mbar_wait(&ofull, t & 1);
        tc_fence_after();
        w.m0 = qb * ATT_ROWS;
        a.ey.template tile4<EPI_BF16, 64, 2>(w, tmem + b * C::BW + (uint32_t(q * 32) << 16), row0, buf, lane, part);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == ATT_EW + 1) tmem_dealloc<C::TCOLS>(tmem);
}

// ============================================================= backward ====
// Tiles t = (item, kb, qb >= kb), key block outermost: dK[kb] and dV[kb]
// accumulate over the query blocks in TMEM, dQ[qb] over the key blocks.
// TMEM: S [0,128), dP [128,256), dV [256,320), dK [320,384), dQ[qb] at
// 384 + 64 qb.  Ring order per item: K0 V0 Q0 dY0 Q1 dY1 .. K1 V1 ..
template <int NB>
struct AttnBwdCfg {
  static constexpr int T = NB * ATT_ROWS;
  static constexpr int NSLOT = 7;
  static constexpr uint32_t TCOLS = 512;
  static constexpr int SMEM = NSLOT * ATT_BOX + 4 * ATT_BOX + ATT_STAGING + 1024;  // + P and dS tiles
  static constexpr int BLOCKS = 4 * NB;
  // ring position of a block within the item
  static __device__ __forceinline__ int kpos(int kb) { return kb == 0 ? 0 : 2 + 2 * NB + 2 * (kb - 1); }
  static __device__ __forceinline__ int qpos(int qb) { return 2 + 2 * qb; }
};

template <int NB>
__global__ void __launch_bounds__(ATT_THREADS, 1) attn_bwd_kernel(const __grid_constant__ AttnArgs a) {
  using C = AttnBwdCfg<NB>;
  constexpr int T = C::T, NSLOT = C::NSLOT;
  constexpr uint32_t IDESC_SP = umma_idesc_bf16(128, 128, false, false);
  constexpr uint32_t IDESC_T = umma_idesc_bf16(128, 64, true, true);   // P^T dY, dS^T Q
  constexpr uint32_t IDESC_Q = umma_idesc_bf16(128, 64, false, true);  // dS K
  constexpr uint32_t T_S = 0, T_DP = 128, T_DV = 256, T_DK = 320, T_DQ = 384;
  pdl_begin();
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[NSLOT], empty[NSLOT];
  __shared__ __align__(8) uint64_t sdp_full, sdp_empty, pds_full, mma_done, acc_full, acc_empty, dq_full, dq_empty;
  __shared__ uint32_t tmem_s;
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t ring = smem_u32(smem);
  uint8_t* Pt = smem + NSLOT * ATT_BOX;
  uint8_t* dSt = Pt + 2 * ATT_BOX;
  const uint32_t psm = smem_u32(Pt), dssm = smem_u32(dSt);
  float* staging = reinterpret_cast<float*>(dSt + 2 * ATT_BOX);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&sdp_full, 1);
    mbar_init(&sdp_empty, 1);
    mbar_init(&pds_full, 1);
    mbar_init(&mma_done, 1);
    mbar_init(&acc_full, 1);
    mbar_init(&acc_empty, ATT_EW);
    mbar_init(&dq_full, 1);
    mbar_init(&dq_empty, ATT_EW);
    fence_mbar_init();
  }
  if (warp == ATT_EW + 1) tmem_alloc<C::TCOLS>(&tmem_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;

  if (warp == ATT_EW) {  // ------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&a.tq);
      tma_prefetch_desc(&a.tk);
      tma_prefetch_desc(&a.tv);
      tma_prefetch_desc(&a.tdy);
      int bc = 0;
      for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
        ZWork w;
        if (!att_item(a, it, w)) continue;
        for (int i = 0; i < C::BLOCKS; ++i, ++bc) {
          // position -> (tensor, block): K0 V0 | Q0 dY0 .. | K1 V1 ..
          const CUtensorMap* m;
          int blk;
          if (i < 2) {
            m = i == 0 ? &a.tk : &a.tv;
            blk = 0;
          } else if (i < 2 + 2 * NB) {
            m = ((i - 2) & 1) ? &a.tdy : &a.tq;
            blk = (i - 2) >> 1;
          } else {
            m = ((i - 2 - 2 * NB) & 1) ? &a.tv : &a.tk;
            blk = 1 + ((i - 2 - 2 * NB) >> 1);
          }
          const int s = bc % NSLOT;
          if (bc >= NSLOT) mbar_wait(&empty[s], ((bc / NSLOT) - 1) & 1);
          mbar_expect_tx(&full[s], ATT_BOX);
          tma_load_5d(ring + s * ATT_BOX, m, 0, blk * ATT_ROWS, w.zh, w.zb, w.j, &full[s]);
        }
      }
    }
  } else if (warp == ATT_EW + 1) {  // ------------------------- MMA issuer
    if (lane == 0) {
      int bc = 0, t = 0, g = 0, item = 0;
      auto sl = [&](int base, int pos) { return (base + pos) % NSLOT; };
      auto ready = [&](int base, int pos) {
        mbar_wait(&full[sl(base, pos)], uint32_t(((base + pos) / NSLOT) & 1));
      };
      for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
        ZWork w;
        if (!att_item(a, it, w)) continue;
        const int base = bc;
        bc += C::BLOCKS;
        for (int kb = 0; kb < NB; ++kb, ++g) {
          for (int qb = kb; qb < NB; ++qb, ++t) {
            const int kp = C::kpos(kb), qp = C::qpos(qb);
            const uint32_t ks = ring + sl(base, kp) * ATT_BOX, vs = ring + sl(base, kp + 1) * ATT_BOX;
            const uint32_t qs = ring + sl(base, qp) * ATT_BOX, ys = ring + sl(base, qp + 1) * ATT_BOX;
            if (t > 0) mbar_wait(&sdp_empty, (t - 1) & 1);
            ready(base, kp);
            ready(base, kp + 1);
            ready(base, qp);
            ready(base, qp + 1);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16(tmem + T_S, att_kdesc(qs, kk), att_kdesc(ks, kk), IDESC_SP, kk > 0 ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16(tmem + T_DP, att_kdesc(ys, kk), att_kdesc(vs, kk), IDESC_SP, kk > 0 ? 1u : 0u);
            mma_commit(&sdp_full);
            mbar_wait(&pds_full, t & 1);
            tc_fence_after();
            if (qb == kb && g > 0) mbar_wait(&acc_empty, (g - 1) & 1);
            if (kb == 0 && qb == 0 && item > 0) mbar_wait(&dq_empty, (item - 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)  // dV[kb] += P^T dY[qb]   (K = queries)
              mma_bf16(tmem + T_DV, att_mdesc(psm, kk, ATT_BOX), att_mdesc(ys, kk, 8192), IDESC_T,
                       (qb > kb || kk > 0) ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)  // dK[kb] += dS^T Q[qb]
              mma_bf16(tmem + T_DK, att_mdesc(dssm, kk, ATT_BOX), att_mdesc(qs, kk, 8192), IDESC_T,
                       (qb > kb || kk > 0) ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)  // dQ[qb] += dS K[kb]     (K = keys)
              mma_bf16(tmem + T_DQ + 64 * qb, att_kdesc(dssm + (kk >> 2) * ATT_BOX, kk & 3),
                       att_mdesc(ks, kk, 8192), IDESC_Q, (kb > 0 || kk > 0) ? 1u : 0u);
            mma_commit(&mma_done);
            if (qb == kb) {
              mma_commit(&empty[sl(base, qp)]);
              mma_commit(&empty[sl(base, qp + 1)]);
              mma_commit(&dq_full);
            }
            if (qb == NB - 1) {
              mma_commit(&empty[sl(base, kp)]);
              mma_commit(&empty[sl(base, kp + 1)]);
              mma_commit(&acc_full);
            }
          }
        }
        ++item;
      }
    }
  } else {  // ---------------------------------- P / dS + epilogue warps
    const int q = warp & 3, part = warp >> 2;
    float* buf = staging + warp * (32 * 33);
    const float k2 = a.scale * 1.4426950408889634f;
    int t = 0, g = 0, dqc = 0;
    for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
      ZWork w;
      if (!att_item(a, it, w)) continue;
      for (int kb = 0; kb < NB; ++kb, ++g) {
        for (int qb = kb; qb < NB; ++qb, ++t) {
          const int r = q * 32 + lane, m = qb * ATT_ROWS + r;
          const float2 st = reinterpret_cast<const float2*>(a.stats)[att_row(a, w, T, m)];
          const float D = a.D[att_row(a, w, T, m)];
          const bool diag = kb == qb;
          mbar_wait(&sdp_full, t & 1);
          tc_fence_after();
          if (t > 0) mbar_wait(&mma_done, (t - 1) & 1);  // P / dS tiles free
          const uint32_t tq = tmem + (uint32_t(q * 32) << 16);
#pragma unroll 1
          for (int c0 = part * 64; c0 < part * 64 + 64; c0 += 32) {
            uint32_t pk[16], dk[16];
            if (diag && c0 >= q * 32 + 32) {  // the whole warp's rows see none of these keys
#pragma unroll
              for (int i = 0; i < 16; ++i) pk[i] = dk[i] = 0u;
            } else {
              float v[32];
              tmem_ld32(tq + T_S + c0, v);
              const int lim = diag ? r + 1 : 128;  // keys (tile-local) this row sees
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float p0 = (c0 + 2 * i < lim) ? ex2_approx(fmaf(v[2 * i], k2, -st.x)) * st.y : 0.f;
                const float p1 = (c0 + 2 * i + 1 < lim) ? ex2_approx(fmaf(v[2 * i + 1], k2, -st.x)) * st.y : 0.f;
                pk[i] = pack_bf2(p0, p1);
              }
              tmem_ld32(tq + T_DP + c0, v);
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float p0 = __uint_as_float(pk[i] << 16), p1 = __uint_as_float(pk[i] & 0xffff0000u);
                dk[i] = pack_bf2(p0 * (v[2 * i] - D) * a.scale, p1 * (v[2 * i + 1] - D) * a.scale);
              }
            }
            att_put32(Pt, r, c0, pk);
            att_put32(dSt, r, c0, dk);
          }
          fence_proxy_async_smem();
          tc_fence_before();
          named_bar_sync(1, ATT_EW * 32);
          if (warp == 0 && lane == 0) {
            mbar_arrive(&pds_full);
            mbar_arrive(&sdp_empty);
          }
          if (diag) {  // dQ[qb] complete
            mbar_wait(&dq_full, dqc & 1);
            ++dqc;
            tc_fence_after();
            w.m0 = qb * ATT_ROWS;
            a.edq.template tile4<EPI_BF16, 64, 2>(w, tq + T_DQ + 64 * qb, w.m0 + q * 32, buf, lane, part);
            if (qb == NB - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&dq_empty);
            }
          }
          if (qb == NB - 1) {  // dV[kb], dK[kb] complete
            mbar_wait(&acc_full, g & 1);
            tc_fence_after();
            w.m0 = kb * ATT_ROWS;
            a.edv.template tile4<EPI_BF16, 64, 2>(w, tq + T_DV, w.m0 + q * 32, buf, lane, part);
            a.edk.template tile4<EPI_BF16, 64, 2>(w, tq + T_DK, w.m0 + q * 32, buf, lane, part);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == ATT_EW + 1) tmem_dealloc<C::TCOLS>(tmem);
}

template <int NB>
inline cudaError_t launch_attn_fwd(const AttnArgs& a, int sms, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         AttnFwdCfg<NB>::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int grid = std::max(1, std::min(a.items, sms));
  if (cudaError_t e = launch(attn_fwd_kernel<NB>, grid, ATT_THREADS, AttnFwdCfg<NB>::SMEM, st, a); e != cudaSuccess)
    return e;
  return cudaGetLastError();
}

template <int NB>
inline cudaError_t launch_attn_bwd(const AttnArgs& a, int sms, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         AttnBwdCfg<NB>::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int grid = std::max(1, std::min(a.items, sms));
  if (cudaError_t e = launch(attn_bwd_kernel<NB>, grid, ATT_THREADS, AttnBwdCfg<NB>::SMEM, st, a); e != cudaSuccess)
    return e;
  return cudaGetLastError();
}

}  // namespace tlk
