// Persistent, warp-specialised grouped GEMM (transformer packs; the ResNet
// implicit-GEMM convolutions in conv.cuh reuse the kernel with their own
// tile / load / epilogue hooks).
//
//   D[z][m, n] = sum_k A[z][m, k] * B[z][n, k]      z = (lane, b, h)
//
// Every operand of the transformer step is a strided 5-D view of a pack
// buffer (k or mn contiguous, then mn/k, head, sequence, lane), so one TMA
// tensor map per operand covers all z of a launch.  The launch is persistent
// (one CTA per SM) and walks the flattened (z, m-tile, n-tile) list:
//
//   warp EW     lane 0: TMA producer -> STAGES-deep smem ring (full/empty)
//   warp EW+1   lane 0: tcgen05.mma issuer, accumulator double-buffered in
//                       TMEM (2 x BN columns): tile i+1's mainloop runs while
//                       the epilogue warps drain tile i
//   warps 0..EW-1     : epilogue in two groups of 4 (one per TMEM buffer):
//                       TMEM -> registers -> smem transpose -> coalesced
//                       stores, or whole-row softmax / CE epilogues.
//
// The epilogues (bias / GELU / residual / softmax / softmax-backward / CE)
// are EpiOps (sgemm.cuh), resolved once per tile from the launch's Epi kind.
#pragma once
#include "sgemm.cuh"
#include "tma.cuh"

namespace tlk {

// One 64-deep k-block of a stage: four K=16 tcgen05.mma into accumulator d.
template <int BN, bool AMN, bool BMN, uint32_t IDESC>
TLK_DEV void gemm_stage_mma(uint32_t d, uint32_t a_s, uint32_t b_s, bool acc) {
#pragma unroll
  for (int kk = 0; kk < GEMM_BK / 16; ++kk)
    mma_bf16(d, stage_desc_tma<GEMM_BM, AMN>(a_s, kk), stage_desc_tma<BN, BMN>(b_s, kk), IDESC,
             (acc || kk > 0) ? 1u : 0u);
}

template <int BN_, bool AMN, bool BMN, bool ROW, bool LIGHT = false, bool COMPACT = false>
struct TGemm {
  static constexpr int BN = BN_;
  // epilogue warps: two groups (one per TMEM accumulator) of 4 lane-quarter
  // warps, x2 for 64-aligned tiles: two warps per lane quarter, each taking
  // half of the tile's columns (row epilogues exchange the row max / sum
  // through smem).  The epilogues (GELU / GELU', softmax, bf16 packing) are
  // issue-bound: twice the warps hide the TMEM / SFU / store latency.  Weight
  // gradients (both operands MN-major, K = tokens) have a small fp32 output
  // and a long DRAM-streaming mainloop, and LIGHT tiles (plain fp32 output:
  // the dgrads, K = d or 4d) a cheap epilogue: one warp per lane quarter,
  // and the freed staging smem becomes pipeline stages.
#ifndef TLK_ROW_PARTS
#define TLK_ROW_PARTS 2
#endif
#ifndef TLK_DENSE_PARTS
#define TLK_DENSE_PARTS 2
#endif
#ifndef TLK_WGRAD_PARTS
#define TLK_WGRAD_PARTS 1
#endif
  static constexpr int PARTS = BN_ % 64 != 0 ? 1
                               : ROW         ? TLK_ROW_PARTS
                               : (AMN && BMN) || LIGHT ? TLK_WGRAD_PARTS
                                              : TLK_DENSE_PARTS;
  static constexpr int EW = 8 * PARTS;
  static constexpr int THREADS = (EW + 2) * 32;
  static constexpr bool A_MN = AMN, B_MN = BMN, ROW_EPI = ROW;
  using Work = ZWork;
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr int B_BYTES = BN_ * GEMM_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // COMPACT (bf16-output kinds on the TMA epilogue only): 2 x 1 KB staging
  // tiles per warp instead of the 32 x 33 fp32 transpose buffer -> one more
  // pipeline stage for the wide tiles
  // TMA_NB tiles per warp: the aux operand is prefetched TMA_NB - 1 chunks
  // ahead (two chunks hide the load latency behind the chunk math)
  static constexpr int TMA_TB = COMPACT ? 1024 : 2048;
  static constexpr int TMA_NB = COMPACT || BN_ <= 192 ? 3 : 2;
  static constexpr int TILE4_BYTES = EW * 32 * 33 * 4;
  static constexpr int STAGING_BYTES = COMPACT                                ? EW * TMA_NB * TMA_TB
                                       : TILE4_BYTES > EW * TMA_NB * TMA_TB ? TILE4_BYTES
                                                                            : EW * TMA_NB * TMA_TB;
  static constexpr int XCHG_BYTES = ROW ? 2 * 3 * 2 * 128 * 4 : 0;  // [group][max, sum, aux][part][row]
  // row-epilogue GEMMs (attention scores / dP, LM head) have K = head dim or
  // d (1-6 k-blocks per tile): two stages suffice, and the freed smem is L1
  // for the epilogue's global P loads.  Dense tiles take as many stages as
  // the 227 KB (less 1 KB of static barriers) hold, up to 8.
  static constexpr int DYN_LIMIT = 232448 - 1024;
  static constexpr int FIT = (DYN_LIMIT - STAGING_BYTES - XCHG_BYTES - 1024) / STAGE_BYTES;
  static constexpr int STAGES = ROW ? 2 : (FIT < 8 ? FIT : 8);
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + STAGING_BYTES + XCHG_BYTES + 1024;
  static constexpr uint32_t TCOLS = BN_ <= 64 ? 128 : BN_ <= 128 ? 256 : 512;  // 2 accumulators
  static_assert(STAGES >= 2, "at least two pipeline stages");
  static_assert(ROW || STAGING_BYTES >= EW * TMA_NB * TMA_TB, "TMA epilogue staging tiles");
  static_assert(!COMPACT || !ROW, "compact staging is for dense epilogues");
  static_assert(2 * BN_ <= 512, "two accumulators must fit TMEM");
  static_assert(!BMN || BN_ % 64 == 0, "MN-major B is loaded in 64-wide boxes");

  CUtensorMap ta, tb;
  CUtensorMap to, to2, tx;  // TMA-staged dense epilogue: out, out2 (GELU z), aux
  EpiOps g;                 // epilogue state (g.e, g.lanes, z decomposition)
  int mt, nt, ntiles;
  int tma_epi;  // dense epilogue through EpiOps::tile_tma (host-checked layout)
  static constexpr bool TMA_EPI = !ROW;

  TLK_DEV bool tile(int t, ZWork& w) const {
    const int n_t = t % nt;
    const int r = t / nt;
    const int m_t = r % mt;
    const int z = r / mt, per = g.nb * g.nh;
    w.j = z / per;
    const int rr = z % per;
    w.zb = rr / g.nh;
    w.zh = rr % g.nh;
    if (!g.lanes[w.j].active) return false;
    w.m0 = m_t * GEMM_BM;
    w.n0 = n_t * BN_;
    w.kb_begin = 0;
    w.kb_end = g.kblocks;
    if (g.e.causal_k == 1)
      w.kb_end = min(w.kb_end, (w.m0 + GEMM_BM + GEMM_BK - 1) / GEMM_BK);
    else if (g.e.causal_k == 2)
      w.kb_begin = w.m0 / GEMM_BK;
    w.split = 0;
    return true;
  }
  TLK_DEV void prefetch() const {
    tma_prefetch_desc(&ta);
    tma_prefetch_desc(&tb);
  }
  TLK_DEV uint32_t tx_bytes() const { return STAGE_BYTES; }
  template <uint32_t IDESC>
  TLK_DEV void issue_mma(uint32_t d, uint32_t a_s, bool acc) const {
    gemm_stage_mma<BN_, AMN, BMN, IDESC>(d, a_s, a_s + A_BYTES, acc);
  }
  TLK_DEV void epilogue(const ZWork& w, uint32_t tq, int row0, float* buf, int lane, int part, float* xchg,
                        int bar) const {
    if constexpr (ROW)
      g.template row_tile<BN_, PARTS>(w, tq, row0, buf, lane, part, xchg, bar);
    else if constexpr (!COMPACT)
      g.template tile<BN_, PARTS>(w, tq, row0, buf, lane, false, part);
    else
      __trap();  // compact tiles exist only on the TMA epilogue path (host-checked)
  }
  TLK_DEV void epi_pre(const ZWork& w, int row0, int lane, int part, uint32_t stg, uint64_t* abar,
                       uint32_t cnt) const {
    g.template tma_pre_any<BN_, PARTS, TMA_TB, TMA_NB>(w, row0, lane, part, stg, abar, cnt, &tx);
  }
  TLK_DEV void epi_tma(const ZWork& w, uint32_t tq, int row0, int lane, int part, uint8_t* stg, uint64_t* abar,
                       uint32_t& cnt) const {
    g.template tile_tma_any<BN_, PARTS, TMA_TB, TMA_NB>(w, tq, row0, lane, part, stg, abar, cnt, &to, &to2, &tx);
  }
  // L2 prefetch of a tile's A boxes (the activation operand streams from
  // DRAM; B, the weights, stays L2-resident)
  TLK_DEV void prefetch_tile(const ZWork& w) const {
    for (int kb = w.kb_begin; kb < w.kb_end; ++kb) {
      const int k0 = kb * GEMM_BK;
      if (!AMN) {
        tma_prefetch_l2_5d(&ta, k0, w.m0, w.zh, w.zb, w.j);
      } else {
        tma_prefetch_l2_5d(&ta, w.m0, k0, w.zh, w.zb, w.j);
        tma_prefetch_l2_5d(&ta, w.m0 + 64, k0, w.zh, w.zb, w.j);
      }
    }
  }
  TLK_DEV void load(const ZWork& w, int kb, uint32_t a_s, uint64_t* bar) const {
    const int k0 = kb * GEMM_BK;
    if (!AMN) {
      tma_load_5d(a_s, &ta, k0, w.m0, w.zh, w.zb, w.j, bar);
    } else {
      tma_load_5d(a_s, &ta, w.m0, k0, w.zh, w.zb, w.j, bar);
      tma_load_5d(a_s + 8192, &ta, w.m0 + 64, k0, w.zh, w.zb, w.j, bar);
    }
    const uint32_t b_s = a_s + A_BYTES;
    if (!BMN) {
      tma_load_5d(b_s, &tb, k0, w.n0, w.zh, w.zb, w.j, bar);
    } else {
#pragma unroll
      for (int i = 0; i < BN_ / 64; ++i) tma_load_5d(b_s + i * 8192, &tb, w.n0 + 64 * i, k0, w.zh, w.zb, w.j, bar);
    }
  }
};

#ifndef TLK_GEMM_L2PF
#define TLK_GEMM_L2PF 0
#endif
// (18 warps: 5 on some SM sub-partitions, so at most 96 registers per thread)
template <class P>
__global__ void __launch_bounds__(P::THREADS, 1) tgemm_kernel(const __grid_constant__ P p) {
  pdl_begin();
  constexpr int BN = P::BN, STAGES = P::STAGES, EW = P::EW;
  constexpr uint32_t IDESC = umma_idesc_bf16(GEMM_BM, BN, P::A_MN, P::B_MN);
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], tfull[2], tempty[2];
  __shared__ __align__(8) uint64_t abar_s[P::TMA_EPI ? EW : 1][3];  // TMA epilogue aux loads, per warp
  __shared__ uint32_t tmem_base_s;
  // align by offsetting smem_raw (not via an integer cast) so that pointers
  // derived from it stay in the shared window (STS/LDS, not generic ST/LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  float* staging = reinterpret_cast<float*>(smem + STAGES * P::STAGE_BYTES);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], EW / 2);
    }
    if constexpr (P::TMA_EPI)
      for (int w = 0; w < EW; ++w)
        for (int k = 0; k < 3; ++k) mbar_init(&abar_s[w][k], 1);
    fence_mbar_init();
  }
  if (warp == EW) tmem_alloc<P::TCOLS>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  if (warp == EW) {
    if (lane == 0) {  // TMA producer
      p.prefetch();
      int it = 0;
      for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        typename P::Work w;
        if (!p.tile(t, w)) continue;
#if TLK_GEMM_L2PF
        if constexpr (P::TMA_EPI) {  // this CTA's tile after next: its A into L2 now
          typename P::Work wn;
          const int tn = t + TLK_GEMM_L2PF * gridDim.x;
          if (tn < p.ntiles && p.tile(tn, wn) && wn.kb_end - wn.kb_begin <= 8) p.prefetch_tile(wn);
        }
#endif
        for (int kb = w.kb_begin; kb < w.kb_end; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty_bar[s], ((it / STAGES) - 1) & 1);
          mbar_expect_tx(&full_bar[s], p.tx_bytes());
          p.load(w, kb, sbase + s * P::STAGE_BYTES, &full_bar[s]);
        }
      }
    }
  } else if (warp == EW + 1) {
    if (lane == 0) {  // MMA issuer
      int it = 0, lt = 0;
      for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        typename P::Work w;
        if (!p.tile(t, w)) continue;
        const int buf = lt & 1;
        if (lt >= 2) mbar_wait(&tempty[buf], ((lt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * BN;
        for (int kb = w.kb_begin; kb < w.kb_end; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full_bar[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t a_s = sbase + s * P::STAGE_BYTES;
          p.template issue_mma<IDESC>(d, a_s, kb > w.kb_begin);
          mma_commit(&empty_bar[s]);
        }
        mma_commit(&tfull[buf]);
        ++lt;
      }
    }
  } else {  // epilogue warps: group ((warp >> 2) & 1) drains TMEM buffer
           // `group`, i.e. the CTA's even / odd local tiles, so two tiles'
           // epilogues run concurrently (4 warps = the 4 TMEM lane quarters
           // each, x PARTS column parts)
    const int q = warp & 3, group = (warp >> 2) & 1, part = warp >> 3;
    float* buf = staging + warp * (32 * 33);
    float* xchg = staging + EW * (32 * 33) + group * (3 * 2 * 128);  // row epilogues only
    // TMA epilogue: 2 x 2 KB staging tiles per warp (1 KB aligned) in the same area
    uint8_t* stg = nullptr;
    if constexpr (P::TMA_EPI) stg = reinterpret_cast<uint8_t*>(staging) + warp * (P::TMA_NB * P::TMA_TB);
    uint32_t ecnt = 0;
    bool tma_epi = false;
    if constexpr (P::TMA_EPI) tma_epi = p.tma_epi != 0;
    int lt = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
      typename P::Work w;
      if (!p.tile(t, w)) continue;
      const int b = lt & 1;
      if (b != group) {
        ++lt;
        continue;
      }
      if constexpr (P::TMA_EPI)
        if (tma_epi) p.epi_pre(w, w.m0 + q * 32, lane, part, smem_u32(stg), abar_s[warp], ecnt);
      // one warp of the group polls the accumulator barrier; the others
      // block on a named barrier (no issue slots spent spinning)
      if (q == 0 && part == 0) mbar_wait(&tfull[b], (lt >> 1) & 1);
      named_bar_sync(3 + group, EW * 16);
      tc_fence_after();
      const uint32_t tq = tmem + b * BN + (uint32_t(q * 32) << 16);
      if constexpr (P::TMA_EPI) {
        if (tma_epi)
          p.epi_tma(w, tq, w.m0 + q * 32, lane, part, stg, abar_s[warp], ecnt);
        else
          p.epilogue(w, tq, w.m0 + q * 32, buf, lane, part, xchg, 1 + group);
      } else {
        p.epilogue(w, tq, w.m0 + q * 32, buf, lane, part, xchg, 1 + group);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
      ++lt;
    }
    if constexpr (P::TMA_EPI)
      if (tma_epi && lane == 0) bulk_wait<0>();  // stores complete before the grid ends
  }
  tc_fence_before();
  __syncthreads();
  if (warp == EW) tmem_dealloc<P::TCOLS>(tmem);
}

// Host: 5-D tensor map of a strided operand.  K-major: dims {K, MN, h, b,
// lane}, box {64, rows}; MN-major: dims {MN, K, h, b, lane}, box {64, 64}.
inline int make_operand_map(CUtensorMap* m, const Operand& o, bool mn_major, int box_rows, int lanes,
                            int nb, int nh) {
  uint64_t dims[5], st[4];
  if (!mn_major) {
    TLK_CHECK(o.k_st == 1, TLK_EINVAL, "K-major operand must have unit k stride");
    dims[0] = uint64_t(o.K);
    dims[1] = uint64_t(o.MN);
    st[0] = uint64_t(o.mn_st) * 2;
  } else {
    TLK_CHECK(o.mn_st == 1, TLK_EINVAL, "MN-major operand must have unit mn stride");
    dims[0] = uint64_t(o.MN);
    dims[1] = uint64_t(o.K);
    st[0] = uint64_t(o.k_st) * 2;
    box_rows = 64;
  }
  dims[2] = uint64_t(nh);
  dims[3] = uint64_t(nb);
  dims[4] = uint64_t(lanes);
  st[1] = uint64_t(o.hs) * 2;
  st[2] = uint64_t(o.bs) * 2;
  st[3] = uint64_t(o.ls) * 2;
  return make_tmap_bf16_5d(m, o.base, dims, st, 64, uint32_t(box_rows));
}

template <class P>
inline cudaError_t launch_tgemm(const P& p, int sms, cudaStream_t stream) {
  static bool configured = false;  // per instantiation
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(tgemm_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         P::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int grid = std::max(1, std::min(p.ntiles, sms));
  if (cudaError_t le = launch(tgemm_kernel<P>, grid, P::THREADS, P::SMEM_BYTES, stream, p); le != cudaSuccess) return le;
  return cudaGetLastError();
}

}  // namespace tlk
