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
// the same bytes, two descriptors.  The P / dS tiles the compute warps write
// are laid out the same way, so P serves as the K-major A of P V and as the
// MN-major A of P^T dY.
//
// Warp roles: compute warps (16 forward / 8 backward: four / two per TMEM
// lane quarter, each owning a slice of the tile's columns), one TMA producer,
// one MMA issuer.  The compute warps read their S / dP columns from TMEM into
// registers and release the TMEM at once, so the MMA warp computes the next
// tile's S (and dP) while they do the exponentials; the MMA warp issues the
// products that consume P / dS one tile behind.  Synchronisation is per TMEM
// lane quarter (named barriers of the quarter's warps, per-warp mbarrier
// arrivals) -- no CTA-wide barrier inside the tile loop; each quarter stores
// its 32 output rows with its own TMA store.  The CTA's active work items
// are listed in shared memory once at launch.
//
// Numerics (the oracle's bf16 mode, oracle/gpt.py): p = ex2(s k2 - m k2) / sum
// on the SFU with k2 = log2(e) / sqrt(dh), P stored bf16, Y = bf16(P V);
// backward recomputes P from S with the forward's (m k2, 1 / sum) row stats
// (identical bits), dS = bf16(bf16(P) (dP - D) scale) with D = rowsum(dY o Y)
// (attn_rowdot_kernel), dQ / dK / dV = bf16 of the causal k-range products,
// the qkv.b gradient from fixed-order column partials of the stored bf16
// values.  Against the unfused path only the order of the row-sum additions
// differs (tests/test_gpu_attn.py).
#pragma once
#include "sgemm.cuh"
#include "tma.cuh"

#include <type_traits>

namespace tlk {

constexpr int ATT_ROWS = 128;               // rows per block (queries or keys)
constexpr uint32_t ATT_BOX = 128 * 64 * 2;  // one block: 128 rows x 64 bf16 (16 KB)
constexpr int ATT_MAX_ITEMS = 512;          // work items per CTA (host-checked)

struct AttnArgs {
  CUtensorMap tq, tk, tv, tdy;  // 5-D {dh, T, head, sequence, lane} views, box {64, 128}
  CUtensorMap to[3];            // outputs, box {64, 32} (one lane quarter): fwd Y; bwd dQ, dK, dV
  const LaneState* lanes;
  int nb, nh, items;            // sequences per lane, heads, lanes * nb * nh
  float scale;
  float* stats;                 // [lane][b][h][T] x (m k2, 1 / sum), written fwd, read bwd
  const float* D;               // bwd: rowsum(dY o Y), same indexing as stats
  Epi ey;                       // fwd: Y (bf16)
  Epi edq, edk, edv;            // bwd: dQ / dK / dV (bf16 + qkv.b column partials)
  unsigned long long* trace;    // debug (TLK_ATTN_TRACE=1): CTA 0's event clocks [tile < 64][32]
};

// debug timeline: CTA 0, first 64 tiles, 32 event slots per tile (clock64)
#define ATT_TR(tile, slot)                                                                    \
  do {                                                                                        \
    if (a.trace && blockIdx.x == 0 && (tile) < 64) a.trace[(tile) * 32 + (slot)] = clock64(); \
  } while (0)

// K-major SW128 operand: 128-byte rows, 8-row atoms 1 KB apart; K step of 16
// elements = +32 B.  MN-major: K rows of 64 MN elements; 16 K rows = +2 KB;
// 64-wide MN blocks `lbo` bytes apart.
TLK_DEV uint64_t att_kdesc(uint32_t base, int kk) { return umma_desc_sw128(base + kk * 32, 16, 1024); }
TLK_DEV uint64_t att_mdesc(uint32_t base, int kk, uint32_t lbo) {
  return umma_desc_sw128(base + kk * 2048, lbo, 1024);
}

TLK_DEV void att_decode(const AttnArgs& a, int k, ZWork& w) {
  const int per = a.nb * a.nh, it = blockIdx.x + k * gridDim.x;
  w.j = it / per;
  const int r = it % per;
  w.zb = r / a.nh;
  w.zh = r % a.nh;
  w.n0 = 0;
}

TLK_DEV int64_t att_row(const AttnArgs& a, const ZWork& w, int T, int m) {
  return ((int64_t(w.j) * a.nb + w.zb) * a.nh + w.zh) * T + m;
}

// The CTA's work items (it = blockIdx.x + k gridDim.x) whose lane is active:
// their k, compacted into `list` by one warp (lane 0 writes *count).
TLK_DEV void att_list_items(const AttnArgs& a, uint16_t* list, int* count, int lane) {
  const int per = a.nb * a.nh;
  int n = 0;
  for (int k0 = 0; blockIdx.x + k0 * gridDim.x < a.items; k0 += 32) {
    const int it = blockIdx.x + (k0 + lane) * gridDim.x;
    const bool ok = it < a.items && a.lanes[it / per].active != 0;
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if (ok) list[n + __popc(m & ((1u << lane) - 1u))] = uint16_t(k0 + lane);
    n += __popc(m);
  }
  if (lane == 0) *count = n;
}

// Write 32 values (columns c0 .. c0+31 of row r) as bf16 into a SW128 tile
// whose 64-column blocks are 16 KB apart.
TLK_DEV void att_put32(uint8_t* tile, int r, int c0, const uint32_t* pk) {
  uint8_t* blk = tile + (c0 >> 6) * ATT_BOX;
  const int ch0 = (c0 & 63) >> 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    *reinterpret_cast<uint4*>(blk + sw128(r, ch0 + i)) = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
}

// Drain 16 accumulator columns (TMEM `taddr`, this warp's lane quarter) of a
// 128 x 64 output tile into the SW128 staging tile `stg` (row r = tile row,
// the layout of a TMA box), and, with e.colpart, the fixed-order column sums
// of the warp's 32 rows of the stored bf16 values (a 16-shuffle
// reduce-scatter: lane l ends with column (l >> 1) & 15).
TLK_DEV void att_drain16(const Epi& e, const ZWork& w, uint32_t taddr, uint8_t* stg, int r, int row0, int col0,
                         int lane) {
  float v[16];
  tmem_ld16(taddr, v);
  uint32_t pk[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) pk[i] = pack_bf2(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(stg + sw128(r, col0 >> 3)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  *reinterpret_cast<uint4*>(stg + sw128(r, (col0 >> 3) + 1)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
  if (!e.colpart) return;
  float c[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    c[2 * i] = __uint_as_float(pk[i] << 16);
    c[2 * i + 1] = __uint_as_float(pk[i] & 0xffff0000u);
  }
  {  // xor 16: keep half b4 (8 values)
    const bool hi = lane & 16;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float keep = hi ? c[8 + i] : c[i], give = hi ? c[i] : c[8 + i];
      c[i] = keep + __shfl_xor_sync(0xffffffffu, give, 16);
    }
  }
  {  // xor 8: quarter b3
    const bool hi = lane & 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float keep = hi ? c[4 + i] : c[i], give = hi ? c[i] : c[4 + i];
      c[i] = keep + __shfl_xor_sync(0xffffffffu, give, 8);
    }
  }
  {
    const bool hi = lane & 4;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float keep = hi ? c[2 + i] : c[i], give = hi ? c[i] : c[2 + i];
      c[i] = keep + __shfl_xor_sync(0xffffffffu, give, 4);
    }
  }
  {
    const bool hi = lane & 2;
    const float keep = hi ? c[1] : c[0], give = hi ? c[0] : c[1];
    c[0] = keep + __shfl_xor_sync(0xffffffffu, give, 2);
  }
  c[0] += __shfl_xor_sync(0xffffffffu, c[0], 1);
  if ((lane & 1) == 0) {
    const int col = col0 + ((lane >> 1) & 15);
    const int64_t frow = int64_t(w.zb) * (e.bs / e.ld) + row0;  // token index within the lane
    e.colpart[w.j * e.cp_ls + (frow >> 5) * e.cp_cols + e.cp_col0 + w.zh * e.hs + col] = c[0];
  }
}

// Stage 32 packed bf16 columns (col0 .. col0+31 of row r) of a 128 x 64
// output tile and, with e.colpart, write the fixed-order column sums of the
// warp's 32 rows (a 31-shuffle reduce-scatter: lane l ends with column l).
TLK_DEV void att_emit32(const Epi& e, const ZWork& w, const uint32_t (&pk)[16], uint8_t* stg, int r, int row0,
                        int col0, int lane) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    *reinterpret_cast<uint4*>(stg + sw128(r, (col0 >> 3) + i)) =
        make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
  if (!e.colpart) return;
  float c[32];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    c[2 * i] = __uint_as_float(pk[i] << 16);
    c[2 * i + 1] = __uint_as_float(pk[i] & 0xffff0000u);
  }
#pragma unroll
  for (int st = 16; st >= 1; st >>= 1) {  // keep the half selected by lane bit `st`
    const bool hi = lane & st;
#pragma unroll
    for (int i = 0; i < st; ++i) {
      const float keep = hi ? c[st + i] : c[i], give = hi ? c[i] : c[st + i];
      c[i] = keep + __shfl_xor_sync(0xffffffffu, give, st);
    }
  }
  const int64_t frow = int64_t(w.zb) * (e.bs / e.ld) + row0;  // token index within the lane
  e.colpart[w.j * e.cp_ls + (frow >> 5) * e.cp_cols + e.cp_col0 + w.zh * e.hs + col0 + lane] = c[0];
}

// 32 accumulator columns (this warp's lane quarter) -> packed bf16 pairs
TLK_DEV void att_load32(uint32_t taddr, uint32_t (&pk)[16]) {
  float v[32];
  tmem_ld32(taddr, v);
#pragma unroll
  for (int i = 0; i < 16; ++i) pk[i] = pack_bf2(v[2 * i], v[2 * i + 1]);
}

// A lane quarter's 32 staged rows (rows q*32 .. of the staging tile) -> one
// TMA store.  The quarter's warps made their writes visible to the async
// proxy and meet at the quarter barrier; before it the quarter leader waits
// until all but its latest store have read their staging rows: with two
// staging tiles used alternately, the tile written next is free again.
TLK_DEV void att_qstore(const CUtensorMap* m, uint8_t* stg, int q, const ZWork& w, int row0, bool qleader,
                        int qthreads) {
  fence_proxy_async_smem();
  if (qleader) bulk_wait_read<1>();  // the store two back (same staging tile) has read it
  named_bar_sync(1 + q, qthreads);
  if (qleader) {
    tma_store_5d(m, smem_u32(stg + q * 32 * 128), 0, row0, w.zh, w.zb, w.j);
    bulk_commit();
  }
}

// ============================================================== forward ====
// Tiles t = (item, qb) in order.  TMEM: S(t) in S buffer t & 1, O(t) = P(t) V
// in O buffer t & 1 (NB = 2: S buffers [0,128) for qb 0 and [128,384) for
// qb 1 tiles, O at 384 / 448; NB = 1: S at 0 / 128, O at 256 / 320).  The
// softmax warps walk their columns in 32-column chunks (max; exp + sum, the
// exponentials written back over S; P), so S(t + 1) is computed while they
// work on S(t).  P is double-buffered in smem (NB = 2:
// a 128-key buffer for qb 0 tiles and a 256-key one for qb 1 tiles); once
// O(t) is complete, the first 16 KB of P(t)'s buffer stage Y(t) (a quarter's
// Y rows overlay only that quarter's P rows).  Ring order per item: Q0 Q1 ..
// K0 K1 .. V0 V1 .. (the next item's Q / K blocks load as soon as this item's
// S products are done).
constexpr int ATT_FCW = 16;                       // forward compute warps
constexpr int ATT_FTHREADS = (ATT_FCW + 2) * 32;  // + TMA producer + MMA issuer

template <int NB>
struct AttnFwdCfg {
  static constexpr int T = NB * ATT_ROWS;
  static constexpr int NSLOT = 6;
  static constexpr uint32_t TCOLS = 512;
  static constexpr uint32_t S_OFF1 = 128;  // S buffer 1 (buffer 0 at column 0)
  static constexpr uint32_t O_OFF = NB == 2 ? 384 : 256;
  static constexpr uint32_t P0_BYTES = 2 * ATT_BOX;       // 128 keys
  static constexpr uint32_t P1_BYTES = NB * 2 * ATT_BOX;  // T keys
  static constexpr int SMEM = NSLOT * ATT_BOX + P0_BYTES + P1_BYTES + 1024;
};

template <int NB>
__global__ void __launch_bounds__(ATT_FTHREADS, 1) attn_fwd_kernel(const __grid_constant__ AttnArgs a) {
  using C = AttnFwdCfg<NB>;
  constexpr int T = C::T, NSLOT = C::NSLOT, PROD = ATT_FCW, MMA = ATT_FCW + 1;
  constexpr uint32_t IDESC_S = umma_idesc_bf16(128, 128, false, false);
  constexpr uint32_t IDESC_S256 = umma_idesc_bf16(128, 256, false, false);
  constexpr uint32_t IDESC_O = umma_idesc_bf16(128, 64, false, true);
  static_assert(NB != 2 || C::NSLOT == 3 * NB, "an item must start at slot 0 (adjacent K blocks)");
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[NSLOT], empty[NSLOT], sfull[2], sfree[2], pfull, ofull[2], oempty[2];
  __shared__ uint32_t tmem_s;
  __shared__ uint16_t ilist[ATT_MAX_ITEMS];
  __shared__ int icount;
  __shared__ float xchg[2][4][128];  // [max, sum][column quarter][row]
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t ring = smem_u32(smem);
  uint8_t* Pbuf[2] = {smem + NSLOT * ATT_BOX, smem + NSLOT * ATT_BOX + C::P0_BYTES};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&pfull, ATT_FCW);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sfull[b], 1);
      mbar_init(&sfree[b], ATT_FCW);
      mbar_init(&ofull[b], 1);
      mbar_init(&oempty[b], ATT_FCW);
    }
    fence_mbar_init();
  }
  if (warp == MMA) tmem_alloc<C::TCOLS>(&tmem_s);
  pdl_begin();  // the lane flags and Q/K/V come from upstream kernels
  if (warp == PROD) att_list_items(a, ilist, &icount, lane);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;
  const int nitems = icount;

  if (warp == PROD) {  // -------------------------------------- TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&a.tq);
      tma_prefetch_desc(&a.tk);
      tma_prefetch_desc(&a.tv);
      int bc = 0;
      for (int k = 0; k < nitems; ++k) {
        ZWork w;
        att_decode(a, ilist[k], w);
        for (int i = 0; i < 3 * NB; ++i, ++bc) {  // Q0 Q1 .. K0 K1 .. V0 V1 ..
          const int s = bc % NSLOT;
          if (bc >= NSLOT) mbar_wait(&empty[s], ((bc / NSLOT) - 1) & 1);
          ATT_TR(k * NB, 16 + i);
          mbar_expect_tx(&full[s], ATT_BOX);
          const CUtensorMap* m = i < NB ? &a.tq : i < 2 * NB ? &a.tk : &a.tv;
          const int blk = i % NB;
          tma_load_5d(ring + s * ATT_BOX, m, 0, blk * ATT_ROWS, w.zh, w.zb, w.j, &full[s]);
        }
      }
    }
  } else if (warp == MMA) {  // ---------------------------------- MMA issuer
    if (lane == 0) {
      // ring position of block qb of tensor k (0 Q, 1 K, 2 V); with NSLOT = 3 NB
      // (NB = 2) every item starts at slot 0, so K0 K1 are adjacent slots: the
      // 256-key S of a qb 1 tile is ONE N = 256 MMA per k step
      auto pos = [](int qb, int k) { return k * NB + qb; };
      auto slot = [&](int base, int qb, int k) { return (base + pos(qb, k)) % NSLOT; };
      auto par = [&](int base, int qb, int k) { return uint32_t(((base + pos(qb, k)) / NSLOT) & 1); };
      const uint32_t pa[2] = {smem_u32(Pbuf[0]), smem_u32(Pbuf[1])};
      int t = 0;
      int pbase = -1, pqb = 0, pt = 0;  // the tile whose O product is pending
      auto issue_o = [&]() {
        const int ob = pt & 1;
        mbar_wait(&pfull, pt & 1);
        if (pt >= 2) mbar_wait(&oempty[ob], ((pt >> 1) - 1) & 1);
        ATT_TR(pt, 11);
        tc_fence_after();
        const uint32_t d = tmem + C::O_OFF + 64 * ob, ps = pa[NB == 2 ? pqb : ob];
        for (int kb = 0; kb <= pqb; ++kb) {
          mbar_wait(&full[slot(pbase, kb, 2)], par(pbase, kb, 2));
          tc_fence_after();
          const uint32_t vs = ring + slot(pbase, kb, 2) * ATT_BOX;
          const uint64_t pd0 = att_kdesc(ps, 0), vd0 = att_mdesc(vs, 0, 8192);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {  // descriptors advance by (bytes >> 4) in the address field
            const int key = kb * 128 + kk * 16;
            mma_bf16(d, pd0 + uint64_t(((key >> 6) * ATT_BOX + ((key & 63) >> 4) * 32) >> 4),
                     vd0 + uint64_t(kk * (2048 >> 4)), IDESC_O, (kb > 0 || kk > 0) ? 1u : 0u);
          }
        }
        mma_commit(&ofull[ob]);
        ATT_TR(pt, 12);
        if (pqb == NB - 1)
          for (int kb = 0; kb < NB; ++kb) mma_commit(&empty[slot(pbase, kb, 2)]);
      };
      for (int k = 0; k < nitems; ++k) {
        const int base = k * 3 * NB;
        for (int qb = 0; qb < NB; ++qb, ++t) {
          const int sb = t & 1;
          if (t >= 2) mbar_wait(&sfree[sb], ((t >> 1) - 1) & 1);
          ATT_TR(t, 8);
          mbar_wait(&full[slot(base, qb, 0)], par(base, qb, 0));
          tc_fence_after();
          const uint32_t qs = ring + slot(base, qb, 0) * ATT_BOX;
          const uint64_t qd0 = att_kdesc(qs, 0);
          for (int kb = 0; kb <= qb; ++kb) {
            mbar_wait(&full[slot(base, kb, 1)], par(base, kb, 1));
            tc_fence_after();
          }
          const uint32_t dS = tmem + (sb ? C::S_OFF1 : 0u);
          if (NB == 2 && qb == 1) {  // keys 0..255: K0, K1 adjacent -> N = 256
            const uint64_t kd0 = att_kdesc(ring + slot(base, 0, 1) * ATT_BOX, 0);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16(dS, qd0 + uint64_t(kk * 2), kd0 + uint64_t(kk * 2), IDESC_S256, kk > 0 ? 1u : 0u);
          } else {
            for (int kb = 0; kb <= qb; ++kb) {
              const uint64_t kd0 = att_kdesc(ring + slot(base, kb, 1) * ATT_BOX, 0);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma_bf16(dS + kb * 128, qd0 + uint64_t(kk * 2), kd0 + uint64_t(kk * 2), IDESC_S, kk > 0 ? 1u : 0u);
            }
          }
          mma_commit(&sfull[sb]);
          ATT_TR(t, 10);
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
  } else {  // ----------------------------------- softmax + Y epilogue warps
    const int q = warp & 3, part = warp >> 2;
    const float k2 = a.scale * 1.4426950408889634f;
    const int r = q * 32 + lane;
    const bool qleader = part == 0 && lane == 0;  // issues this quarter's Y stores
    ZWork pw{};                                   // the tile whose Y is drained next
    int pqb = 0;
    auto drain = [&](int pt) {  // Y(pt) = O(pt) -> bf16, staged in P(pt)'s buffer
      const int ob = pt & 1;
      uint8_t* stg = Pbuf[NB == 2 ? pqb : ob];
      mbar_wait(&ofull[ob], (pt >> 1) & 1);
      tc_fence_after();
      att_drain16(a.ey, pw, tmem + C::O_OFF + 64 * ob + (uint32_t(q * 32) << 16) + part * 16, stg, r,
                  pqb * ATT_ROWS + q * 32, part * 16, lane);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&oempty[ob]);
      att_qstore(&a.to[0], stg, q, pw, pqb * ATT_ROWS + q * 32, qleader, 128);
    };
    int t = 0;
    for (int k = 0; k < nitems; ++k) {
      ZWork w;
      att_decode(a, ilist[k], w);
      for (int qb = 0; qb < NB; ++qb, ++t) {
        const int row0 = qb * ATT_ROWS + q * 32, m = row0 + lane;  // query index in the sequence
        const int cw = (qb + 1) * 32;                              // columns per warp: ncols / 4
        const int c0 = part * cw;
        const bool any = c0 <= row0 + 31;  // some row of the warp sees a key here
        // NV = this warp's columns (32, or 64 for the 256-key tile), handled
        // as NV / 32 chunks: compile-time, so the per-element loops are
        // straight-line code (selects, no branches) on 32 live values
        float xv[32];  // softmax3: one chunk of exponentials
        auto softmax3 = [&](auto nvc) {  // NV = 64: three 32-column passes over TMEM (register budget)
          constexpr int NV = decltype(nvc)::value, NC = NV / 32;
          const int sb = t & 1;
          mbar_wait(&sfull[sb], (t >> 1) & 1);
          if (warp == 0 && lane == 0) ATT_TR(t, 0);
          tc_fence_after();
          const uint32_t ts = tmem + (sb ? C::S_OFF1 : 0u) + (uint32_t(q * 32) << 16) + c0;
          float mx = -INFINITY;
          if (any) {
#pragma unroll
            for (int h = 0; h < NC; ++h) {
              float v[32];
              tmem_ld32(ts + h * 32, v);
              if (c0 + h * 32 + 31 > row0) {  // the causal diagonal crosses this chunk
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = (c0 + h * 32 + i > m) ? -INFINITY : v[i];
              }
#pragma unroll
              for (int i = 0; i < 32; ++i) mx = fmaxf(mx, v[i]);
            }
          }
          if (warp == 0 && lane == 0) ATT_TR(t, 1);
          xchg[0][part][r] = mx;
          named_bar_sync(1 + q, 128);
          if (warp == 0 && lane == 0) ATT_TR(t, 2);
          mx = fmaxf(fmaxf(xchg[0][0][r], xchg[0][1][r]), fmaxf(xchg[0][2][r], xchg[0][3][r]));
          const float mk = mx * k2;
          float s4[4] = {0.f, 0.f, 0.f, 0.f};
          if (any) {
#pragma unroll
            for (int h = 0; h < NC; ++h) {
              float v[32];
              tmem_ld32(ts + h * 32, v);
              const bool msk = c0 + h * 32 + 31 > row0;
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const float e = ex2_approx(fmaf(v[i], k2, -mk));
                v[i] = (msk && c0 + h * 32 + i > m) ? 0.f : e;
                s4[i & 3] += v[i];
              }
              if (NC > 1) tmem_st32(ts + h * 32, v);  // the exponentials replace S
              if (NC == 1) {                          // single chunk: keep them in registers
#pragma unroll
                for (int i = 0; i < 32; ++i) xv[i] = v[i];
              }
            }
          }
          xchg[1][part][r] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
          if (qleader) bulk_wait_read<0>();  // Y(t - 2)'s store has read this quarter's rows of P(t)'s buffer
          named_bar_sync(1 + q, 128);
          const float s = (xchg[1][0][r] + xchg[1][1][r]) + (xchg[1][2][r] + xchg[1][3][r]);
          const float inv = 1.f / s;
          if (part == 0) reinterpret_cast<float2*>(a.stats)[att_row(a, w, T, m)] = make_float2(mk, inv);
          // P(t) -> smem buffer t & 1 (free: O(t - 2) completed before Y(t - 2) was drained)
          uint8_t* P = Pbuf[NB == 2 ? qb : (t & 1)];
#pragma unroll
          for (int h = 0; h < NC; ++h) {
            uint32_t pk[16];
            if (any) {
              if (NC > 1) tmem_ld32(ts + h * 32, xv);
#pragma unroll
              for (int i = 0; i < 16; ++i) pk[i] = pack_bf2(xv[2 * i] * inv, xv[2 * i + 1] * inv);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) pk[i] = 0u;
            }
            att_put32(P, r, c0 + h * 32, pk);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sfree[sb]);  // S(t)'s buffer may take S(t + 2)
        };
        auto softmax1 = [&](auto nvc) {  // NV = 32: S read once into registers
          constexpr int NV = decltype(nvc)::value, NC = NV / 32;
          const int sb = t & 1;
          mbar_wait(&sfull[sb], (t >> 1) & 1);
          if (warp == 0 && lane == 0) ATT_TR(t, 0);
          tc_fence_after();
          const uint32_t ts = tmem + (sb ? C::S_OFF1 : 0u) + (uint32_t(q * 32) << 16) + c0;
          // ONE pass over TMEM (its read bandwidth, 64 B/clk/SM, is the
          // scarce resource here): S -> registers, mask, max; exponentials in
          // place; P from the registers
          float v[NV];
          float mx = -INFINITY;
          if (any) {
            if constexpr (NV == 64)
              tmem_ld64(ts, v);
            else
              tmem_ld32(ts, v);
#pragma unroll
            for (int h = 0; h < NC; ++h)
              if (c0 + h * 32 + 31 > row0) {  // the causal diagonal crosses this chunk
#pragma unroll
                for (int i = 0; i < 32; ++i) v[h * 32 + i] = (c0 + h * 32 + i > m) ? -INFINITY : v[h * 32 + i];
              }
#pragma unroll
            for (int i = 0; i < NV; ++i) mx = fmaxf(mx, v[i]);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sfree[sb]);  // S(t) consumed: its buffer may take S(t + 2)
          if (warp == 0 && lane == 0) ATT_TR(t, 1);
          xchg[0][part][r] = mx;
          named_bar_sync(1 + q, 128);
          if (warp == 0 && lane == 0) ATT_TR(t, 2);
          mx = fmaxf(fmaxf(xchg[0][0][r], xchg[0][1][r]), fmaxf(xchg[0][2][r], xchg[0][3][r]));
          const float mk = mx * k2;
          float s4[4] = {0.f, 0.f, 0.f, 0.f};
          if (any) {
#pragma unroll
            for (int i = 0; i < NV; ++i) {
              v[i] = ex2_approx(fmaf(v[i], k2, -mk));  // masked: ex2(-inf) = 0
              s4[i & 3] += v[i];
            }
          }
          xchg[1][part][r] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
          if (qleader) bulk_wait_read<0>();  // Y(t - 2)'s store has read this quarter's rows of P(t)'s buffer
          named_bar_sync(1 + q, 128);
          const float s = (xchg[1][0][r] + xchg[1][1][r]) + (xchg[1][2][r] + xchg[1][3][r]);
          const float inv = 1.f / s;
          if (part == 0) reinterpret_cast<float2*>(a.stats)[att_row(a, w, T, m)] = make_float2(mk, inv);
          // P(t) -> smem buffer t & 1 (free: O(t - 2) completed before Y(t - 2) was drained)
          uint8_t* P = Pbuf[NB == 2 ? qb : (t & 1)];
#pragma unroll
          for (int h = 0; h < NC; ++h) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
              pk[i] = any ? pack_bf2(v[h * 32 + 2 * i] * inv, v[h * 32 + 2 * i + 1] * inv) : 0u;
            att_put32(P, r, c0 + h * 32, pk);
          }
        };
        if (NB == 2 && qb == 1)
          softmax3(std::integral_constant<int, 64>{});
        else
          softmax1(std::integral_constant<int, 32>{});
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull);
        if (warp == 0 && lane == 0) ATT_TR(t, 4);
        if (t >= 1) drain(t - 1);
        if (warp == 0 && lane == 0) ATT_TR(t, 5);
        pw = w;
        pqb = qb;
      }
    }
    if (t >= 1) drain(t - 1);
    if (qleader) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMA) tmem_dealloc<C::TCOLS>(tmem);
}

// ============================================================= backward ====
// Tiles t = (item, kb, qb >= kb), key block outermost: dK[kb] and dV[kb]
// accumulate over the query blocks in TMEM, dQ[qb] over the key blocks.
// TMEM: S [0,128), dP [128,256), dV [256,320), dK [320,384), dQ[qb] at
// 384 + 64 qb.  MMA order: S/dP(t), then the dV / dK / dQ products of t - 1.
// Ring order per item: Q0 dY0 K0 V0 Q1 dY1 K1 V1 (a whole item fits the
// ring: the next item's first S/dP is issued before this item's last dV/dK/dQ).
// Eight compute warps (two per lane quarter, 64 key columns each, processed
// as two 32-column chunks): up to 168 registers, no spills.
constexpr int ATT_BCW = 8;
constexpr int ATT_BTHREADS = (ATT_BCW + 2) * 32;

template <int NB>
struct AttnBwdCfg {
  static constexpr int T = NB * ATT_ROWS;
  static constexpr int BLOCKS = 4 * NB;
  static constexpr int NSLOT = 8;
  static constexpr uint32_t TCOLS = 512;
  static constexpr int SMEM = NSLOT * ATT_BOX + 6 * ATT_BOX + 1024;  // + P, dS tiles, 2 staging tiles
};

template <int NB>
__global__ void __launch_bounds__(ATT_BTHREADS, 1) attn_bwd_kernel(const __grid_constant__ AttnArgs a) {
  using C = AttnBwdCfg<NB>;
  constexpr int T = C::T, NSLOT = C::NSLOT, PROD = ATT_BCW, MMA = ATT_BCW + 1;
  constexpr uint32_t IDESC_SP = umma_idesc_bf16(128, 128, false, false);
  constexpr uint32_t IDESC_T = umma_idesc_bf16(128, 64, true, true);   // P^T dY, dS^T Q
  constexpr uint32_t IDESC_Q = umma_idesc_bf16(128, 64, false, true);  // dS K
  constexpr uint32_t T_S = 0, T_DP = 128, T_DV = 256, T_DK = 320, T_DQ = 384;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[NSLOT], empty[NSLOT];
  __shared__ __align__(8) uint64_t sdp_full, sdp_free, pds_full, mma_done, acc_full, acc_empty, dq_full, dq_empty[2];
  __shared__ uint32_t tmem_s;
  __shared__ uint16_t ilist[ATT_MAX_ITEMS];
  __shared__ int icount;
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t ring = smem_u32(smem);
  uint8_t* Pt = smem + NSLOT * ATT_BOX;
  uint8_t* dSt = Pt + 2 * ATT_BOX;
  uint8_t* stg0 = dSt + 2 * ATT_BOX;  // two 16 KB output staging tiles
  const uint32_t psm = smem_u32(Pt), dssm = smem_u32(dSt);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&sdp_full, 1);
    mbar_init(&sdp_free, ATT_BCW);
    mbar_init(&pds_full, ATT_BCW);
    mbar_init(&mma_done, 1);
    mbar_init(&acc_full, 1);
    mbar_init(&acc_empty, ATT_BCW);
    mbar_init(&dq_full, 1);
    mbar_init(&dq_empty[0], ATT_BCW);
    mbar_init(&dq_empty[1], ATT_BCW);
    fence_mbar_init();
  }
  if (warp == MMA) tmem_alloc<C::TCOLS>(&tmem_s);
  pdl_begin();
  if (warp == PROD) att_list_items(a, ilist, &icount, lane);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;
  const int nitems = icount;
  // ring position of a block within the item: Q0 dY0 K0 V0 | Q1 dY1 K1 V1
  auto qpos = [](int qb) { return 4 * qb; };
  auto kpos = [](int kb) { return 4 * kb + 2; };

  if (warp == PROD) {  // -------------------------------------- TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&a.tq);
      tma_prefetch_desc(&a.tk);
      tma_prefetch_desc(&a.tv);
      tma_prefetch_desc(&a.tdy);
      int bc = 0;
      for (int k = 0; k < nitems; ++k) {
        ZWork w;
        att_decode(a, ilist[k], w);
        for (int i = 0; i < C::BLOCKS; ++i, ++bc) {
          const CUtensorMap* m = (i & 3) == 0 ? &a.tq : (i & 3) == 1 ? &a.tdy : (i & 3) == 2 ? &a.tk : &a.tv;
          const int s = bc % NSLOT;
          if (bc >= NSLOT) mbar_wait(&empty[s], ((bc / NSLOT) - 1) & 1);
          ATT_TR(k * (NB * (NB + 1) / 2), 16 + i);
          mbar_expect_tx(&full[s], ATT_BOX);
          tma_load_5d(ring + s * ATT_BOX, m, 0, (i >> 2) * ATT_ROWS, w.zh, w.zb, w.j, &full[s]);
        }
      }
    }
  } else if (warp == MMA) {  // ---------------------------------- MMA issuer
    if (lane == 0) {
      auto sl = [&](int base, int pos) { return (base + pos) % NSLOT; };
      auto ready = [&](int base, int pos) {
        mbar_wait(&full[sl(base, pos)], uint32_t(((base + pos) / NSLOT) & 1));
      };
      struct Tile {
        int base, kb, qb, g, item;
      };
      Tile pend{-1, 0, 0, 0, 0};
      int tc = 0;  // tiles whose dV/dK/dQ were issued
      auto issue_vkq = [&](const Tile& p) {
        const uint32_t ks = ring + sl(p.base, kpos(p.kb)) * ATT_BOX;
        const uint32_t qs = ring + sl(p.base, qpos(p.qb)) * ATT_BOX, ys = ring + sl(p.base, qpos(p.qb) + 1) * ATT_BOX;
        mbar_wait(&pds_full, tc & 1);
        ATT_TR(tc, 11);
        if (p.qb == p.kb && p.g > 0) mbar_wait(&acc_empty, (p.g - 1) & 1);
        if (p.kb == 0 && p.item > 0) mbar_wait(&dq_empty[p.qb], (p.item - 1) & 1);
        ATT_TR(tc, 12);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dV[kb] += P^T dY[qb]   (K = queries)
          mma_bf16(tmem + T_DV, att_mdesc(psm, kk, ATT_BOX), att_mdesc(ys, kk, 8192), IDESC_T,
                   (p.qb > p.kb || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dK[kb] += dS^T Q[qb]
          mma_bf16(tmem + T_DK, att_mdesc(dssm, kk, ATT_BOX), att_mdesc(qs, kk, 8192), IDESC_T,
                   (p.qb > p.kb || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dQ[qb] += dS K[kb]     (K = keys)
          mma_bf16(tmem + T_DQ + 64 * p.qb, att_kdesc(dssm + (kk >> 2) * ATT_BOX, kk & 3), att_mdesc(ks, kk, 8192),
                   IDESC_Q, (p.kb > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&mma_done);
        ATT_TR(tc, 13);
        if (p.qb == p.kb) {
          mma_commit(&empty[sl(p.base, qpos(p.qb))]);
          mma_commit(&empty[sl(p.base, qpos(p.qb) + 1)]);
          mma_commit(&dq_full);
        }
        if (p.qb == NB - 1) {
          mma_commit(&empty[sl(p.base, kpos(p.kb))]);
          mma_commit(&empty[sl(p.base, kpos(p.kb) + 1)]);
          mma_commit(&acc_full);
        }
        ++tc;
      };
      int t = 0, g = 0;
      for (int item = 0; item < nitems; ++item) {
        const int base = item * C::BLOCKS;
        for (int kb = 0; kb < NB; ++kb, ++g) {
          for (int qb = kb; qb < NB; ++qb, ++t) {
            const int kp = kpos(kb), qp = qpos(qb);
            if (t > 0) mbar_wait(&sdp_free, (t - 1) & 1);
            ATT_TR(t, 8);
            ready(base, kp);
            ready(base, kp + 1);
            ready(base, qp);
            ready(base, qp + 1);
            ATT_TR(t, 9);
            tc_fence_after();
            const uint32_t ks = ring + sl(base, kp) * ATT_BOX, vs = ring + sl(base, kp + 1) * ATT_BOX;
            const uint32_t qs = ring + sl(base, qp) * ATT_BOX, ys = ring + sl(base, qp + 1) * ATT_BOX;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16(tmem + T_S, att_kdesc(qs, kk), att_kdesc(ks, kk), IDESC_SP, kk > 0 ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16(tmem + T_DP, att_kdesc(ys, kk), att_kdesc(vs, kk), IDESC_SP, kk > 0 ? 1u : 0u);
            mma_commit(&sdp_full);
            ATT_TR(t, 10);
            if (pend.base >= 0) issue_vkq(pend);
            pend = Tile{base, kb, qb, g, item};
          }
        }
      }
      if (pend.base >= 0) issue_vkq(pend);
    }
  } else {  // -------------------------------------- P / dS + drain warps
    const int q = warp & 3, part = warp >> 2;  // part: key columns [64 part, 64 part + 64)
    const float k2 = a.scale * 1.4426950408889634f;
    const int r = q * 32 + lane;
    const bool qleader = part == 0 && lane == 0;
    int t = 0, dqc = 0, gdone = 0, nst = 0;
    ZWork pw{};
    int pkb = -1, pqb = 0;
    // accumulators completed by the dV / dK / dQ products of the previous
    // tile: read them (this warp's 32 columns), release the TMEM, then stage
    // and store (two staging tiles used alternately)
    auto emit = [&](const Epi& e, const CUtensorMap* m, const uint32_t (&pk)[16], int row_base) {
      uint8_t* sg = stg0 + (nst & 1) * ATT_BOX;
      att_emit32(e, pw, pk, sg, r, row_base + q * 32, part * 32, lane);
      att_qstore(m, sg, q, pw, row_base + q * 32, qleader, 64);
      ++nst;
    };
    auto drains = [&]() {
      if (pkb < 0) return;
      const uint32_t tq = tmem + (uint32_t(q * 32) << 16) + part * 32;
      if (pkb == pqb) {  // dQ[pqb]
        uint32_t pq[16];
        mbar_wait(&dq_full, dqc & 1);
        ++dqc;
        tc_fence_after();
        att_load32(tq + T_DQ + 64 * pqb, pq);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dq_empty[pqb]);
        emit(a.edq, &a.to[0], pq, pqb * ATT_ROWS);
      }
      if (pqb == NB - 1) {  // dV[pkb], dK[pkb]
        uint32_t pv[16], pk2[16];
        mbar_wait(&acc_full, gdone & 1);
        ++gdone;
        tc_fence_after();
        att_load32(tq + T_DV, pv);
        att_load32(tq + T_DK, pk2);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty);
        emit(a.edv, &a.to[2], pv, pkb * ATT_ROWS);
        emit(a.edk, &a.to[1], pk2, pkb * ATT_ROWS);
      }
    };
    for (int k = 0; k < nitems; ++k) {
      ZWork w;
      att_decode(a, ilist[k], w);
      for (int kb = 0; kb < NB; ++kb) {
        for (int qb = kb; qb < NB; ++qb, ++t) {
          const int m = qb * ATT_ROWS + r;  // query index
          const float2 st = reinterpret_cast<const float2*>(a.stats)[att_row(a, w, T, m)];
          const float D = a.D[att_row(a, w, T, m)];
          const bool diag = kb == qb;
          mbar_wait(&sdp_full, t & 1);
          if (warp == 0 && lane == 0) ATT_TR(t, 0);
          tc_fence_after();
          const uint32_t tq = tmem + (uint32_t(q * 32) << 16);
          uint32_t pk[2][16], dk[2][16];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c0 = part * 64 + h * 32;  // tile-local key columns of this chunk
            const bool any = !diag || c0 <= q * 32 + 31;
            const bool masked = diag && c0 + 31 > q * 32;
            if (any) {
              float sd[64];  // S in [0, 32), dP in [32, 64)
              tmem_ld32x2(tq + T_S + c0, tq + T_DP + c0, sd);
#pragma unroll
              for (int i = 0; i < 32; ++i) sd[i] = ex2_approx(fmaf(sd[i], k2, -st.x)) * st.y;
              if (masked) {
#pragma unroll
                for (int i = 0; i < 32; ++i) sd[i] = (c0 + i <= r) ? sd[i] : 0.f;
              }
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                pk[h][i] = pack_bf2(sd[2 * i], sd[2 * i + 1]);
                const float b0 = __uint_as_float(pk[h][i] << 16), b1 = __uint_as_float(pk[h][i] & 0xffff0000u);
                dk[h][i] = pack_bf2(b0 * (sd[32 + 2 * i] - D) * a.scale, b1 * (sd[32 + 2 * i + 1] - D) * a.scale);
              }
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) pk[h][i] = dk[h][i] = 0u;
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sdp_free);
          if (warp == 0 && lane == 0) ATT_TR(t, 2);
          if (t > 0) mbar_wait(&mma_done, (t - 1) & 1);  // the P / dS tiles are free
          if (warp == 0 && lane == 0) ATT_TR(t, 3);
          att_put32(Pt, r, part * 64, pk[0]);
          att_put32(Pt, r, part * 64 + 32, pk[1]);
          att_put32(dSt, r, part * 64, dk[0]);
          att_put32(dSt, r, part * 64 + 32, dk[1]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&pds_full);
          if (warp == 0 && lane == 0) ATT_TR(t, 4);
          drains();
          if (warp == 0 && lane == 0) ATT_TR(t, 5);
          pw = w;
          pkb = kb;
          pqb = qb;
        }
      }
    }
    drains();
    if (qleader) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMA) tmem_dealloc<C::TCOLS>(tmem);
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
  if (cudaError_t e = launch(attn_fwd_kernel<NB>, grid, ATT_FTHREADS, AttnFwdCfg<NB>::SMEM, st, a);
      e != cudaSuccess)
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
  if (cudaError_t e = launch(attn_bwd_kernel<NB>, grid, ATT_BTHREADS, AttnBwdCfg<NB>::SMEM, st, a);
      e != cudaSuccess)
    return e;
  return cudaGetLastError();
}

}  // namespace tlk
