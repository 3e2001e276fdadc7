// Implicit-GEMM convolutions for the ResNet pack on the persistent tcgen05
// kernel of tgemm.cuh.  Activations are NHWC bf16 [lane][B][H][W][C] with NO
// padding in memory: TMA coordinates are signed and out-of-range elements are
// zero-filled, so a 3x3 tap is a coordinate shift of a 5-D box
//     (64 channels, bx pixels along W, by rows, bb images, 1 lane)
// whose smem image is exactly the SW128 K-major (or MN-major) UMMA tile.
// Stride-2 layers read the input through four parity "phase" tensor maps
// (base + (py*W + px)*C, pixel strides doubled): input row 2y + d is phase
// (d & 1) at coordinate y + (d - (d & 1)) / 2.
//
//   FWD   D[pix][co]  = sum_{tap, ci} X[pix + tap][ci] W[co][tap][ci]
//         epilogue: y = bf16(D), per-32-row (mean, M2) of y (BN statistics)
//   DGRAD D[pix][ci]  = sum_{tap, co} dY[pix - tap][co] WT[tap][ci][co]
//         stride 2: one GEMM per input phase over the taps of that parity;
//         epilogue: fp32 store or in-place accumulate (residual branches)
//   WGRAD D[co][ci]   = sum_pix dY[pix][co] X[pix + tap][ci]   (one z per tap,
//         split-K over pixel blocks; fp32 partials per split)
#pragma once
#include <algorithm>

#include "tgemm.cuh"

namespace tlk {

enum ConvMode { CONV_FWD = 0, CONV_DGRAD = 1, CONV_WGRAD = 2 };

struct ConvWork {
  int j, m0, n0, kb_begin, kb_end;
  int z;      // DGRAD stride 2: phase; WGRAD: tap
  int split;  // WGRAD
  int mt;     // m-tile index (FWD stats partials)
};

// HALO (stride-1 3x3 FWD / DGRAD on 16- or 32-wide grids, 128 % W == 0):
// a 128-pixel tile is 128/W whole image rows, so one TMA box of those rows
// plus a one-row halo above and below -- (64 ch, W px, 128/W + 2 rows) at x
// shift dx -- holds the A operand of all three taps (dh = -1, 0, 1) of that
// dx: tap dh is the same smem image with the UMMA start moved by (1 + dh) * W
// rows (a multiple of the 8-row SW128 atom for W = 16, 32).  A stage = that
// box + the three taps' B tiles, 12 MMAs; A traffic drops from 9 to 3 boxes
// per 64 channels (L2 -> SM bytes per MMA from 96 to ~60 B/clk at BN 64).
// TG = 3 (WGRAD, 64 input channels): one tile computes the three taps of a
// kernel row at once, N = 3 x 64 -- the dY operand (A) is loaded once for
// three taps and each MMA does 3x the work of a single-tap tile.
template <int BN_, int MODE, bool HALO = false, int TG = 1>
struct ConvGemm {
  static constexpr int BN = BN_;
  static_assert(TG == 1 || (MODE == CONV_WGRAD && BN_ == 64 * TG), "tap groups: WGRAD, 64 channels per tap");
  static constexpr int A_BYTES = HALO ? 6 * 32 * 128 : GEMM_BM * GEMM_BK * 2;  // halo: <= (128/W + 2) W rows
  static constexpr int B_BYTES = (HALO ? 3 : 1) * BN_ * GEMM_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
#ifndef TLK_CONV_PARTS
#define TLK_CONV_PARTS 2
#endif
  // epilogue: two groups (TMEM accumulators) x 4 lane quarters x PARTS
  // column halves (the bf16 / BN-partial / fp32-accumulate epilogues are
  // issue- and latency-bound; 64-aligned tiles split their chunks in two)
  static constexpr int PARTS = BN_ % 64 == 0 ? TLK_CONV_PARTS : 1;
  static constexpr int EW = 8 * PARTS;
  static constexpr int STAGES = HALO ? (BN_ <= 64 ? 3 : 2)
                                     : (BN_ <= 64 ? 6 : BN_ <= 128 ? 4 : BN_ <= 192 ? 4 - (PARTS - 1) : 3);
  static constexpr int THREADS = (EW + 2) * 32;
  static constexpr bool A_MN = MODE == CONV_WGRAD, B_MN = MODE == CONV_WGRAD, ROW_EPI = false, TMA_EPI = false;
  static_assert(!HALO || MODE != CONV_WGRAD, "halo mode is FWD / DGRAD only");
  static constexpr int STAGING_BYTES = EW * 32 * 33 * 4;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + STAGING_BYTES + 1024;
  static constexpr uint32_t TCOLS = BN_ <= 64 ? 128 : BN_ <= 128 ? 256 : 512;
  using Work = ConvWork;

  CUtensorMap ta[4], tb[4];
  const LaneState* lanes;
  // GEMM-row pixel grid (FWD: output grid, DGRAD: input grid or phase grid)
  int Hr, Wr;
  int ksz, pad, stride;      // kernel size (3 or 1), padding, stride
  int cin_blk, cout_blk;     // channels / 64
  int mt, nt, nz, ntiles;
  int kblocks;               // FWD / DGRAD stride 1
  int splits, kb_split, kb_total;  // WGRAD
  int bx, by, bb;            // pixel box of one k-block (WGRAD, 64 px) / m-tile (128 px)
  // epilogue
  void* out;
  int64_t out_ls;            // per-lane stride (elements)
  int rows, cols;            // valid extent of D
  int accumulate;            // DGRAD: out += D
  int Hf, Wf;                // DGRAD stride 2: full-resolution output grid
  float* part;               // FWD: [lane][mtile][4 quarters][2][Cout]
  int64_t part_ls;
  int64_t split_st;          // WGRAD: partial stride between splits (elements)
  int taps;                  // WGRAD: taps per output channel row (ld = taps * Cin)

  TLK_DEV void prefetch() const {
    tma_prefetch_desc(&ta[0]);
    tma_prefetch_desc(&tb[0]);
  }
  TLK_DEV uint32_t tx_bytes() const {
    return HALO ? uint32_t((GEMM_BM / Wr + 2) * Wr * 128 + B_BYTES) : uint32_t(STAGE_BYTES);
  }
  // halo k-block kb = (dx index, channel block): taps kh = 0..2 at kw = dx
  template <uint32_t IDESC>
  TLK_DEV void issue_mma(uint32_t d, uint32_t a_s, bool acc) const {
    if constexpr (!HALO) {
      gemm_stage_mma<BN_, A_MN, B_MN, IDESC>(d, a_s, a_s + A_BYTES, acc);
    } else {
#pragma unroll
      for (int kh = 0; kh < 3; ++kh) {
        const int r = MODE == CONV_FWD ? kh : 2 - kh;  // 1 + dh (fwd) or 1 - dh (dgrad)
        gemm_stage_mma<BN_, false, false, IDESC>(d, a_s + uint32_t(r * Wr * 128),
                                                 a_s + A_BYTES + uint32_t(kh * BN_ * 128), acc || kh > 0);
      }
    }
  }
  // taps of stride-2 dgrad phase p (parity of d = k - pad must equal p)
  TLK_DEV int ntap1(int parity) const {
    int n = 0;
    for (int k = 0; k < ksz; ++k) n += (((k - pad) - parity) & 1) == 0;
    return n;
  }
  TLK_DEV int tap1(int parity, int i) const {
    for (int k = 0; k < ksz; ++k)
      if ((((k - pad) - parity) & 1) == 0 && i-- == 0) return k;
    return 0;
  }

  TLK_DEV bool tile(int t, ConvWork& w) const {
    const int n_t = t % nt;
    int r = t / nt;
    const int m_t = r % mt;
    r /= mt;
    const int z = r % nz;
    w.j = r / nz;
    if (!lanes[w.j].active) return false;
    w.m0 = m_t * GEMM_BM;
    w.n0 = n_t * BN_;
    w.mt = m_t;
    w.z = z;
    w.split = 0;
    w.kb_begin = 0;
    w.kb_end = kblocks;
    if (MODE == CONV_DGRAD && stride == 2) {
      w.kb_end = ntap1(z >> 1) * ntap1(z & 1) * cout_blk;
      if (w.kb_end == 0) return false;
    } else if (MODE == CONV_WGRAD) {
      w.z = z / splits;
      w.split = z % splits;
      w.kb_begin = w.split * kb_split;
      w.kb_end = min(kb_total, w.kb_begin + kb_split);
      if (w.kb_begin >= w.kb_end) return false;
    }
    return true;
  }

  // pixel block -> (b0, y0) for a box of npix pixels at a (H, W) grid
  TLK_DEV void pix_origin(int base, int H, int W, int& b0, int& y0) const {
    b0 = base / (H * W);
    y0 = (base % (H * W)) / W;
  }

  TLK_DEV void load(const ConvWork& w, int kb, uint32_t a_s, uint64_t* bar) const {
    const uint32_t b_s = a_s + A_BYTES;
    if constexpr (HALO) {
      int b0, y0;
      pix_origin(w.m0, Hr, Wr, b0, y0);
      const int cblk = MODE == CONV_FWD ? cin_blk : cout_blk;
      const int kw = kb / cblk, c0 = (kb % cblk) * 64, dw = kw - 1;
      tma_load_5d(a_s, &ta[0], c0, MODE == CONV_FWD ? dw : -dw, y0 - 1, b0, w.j, bar);
#pragma unroll
      for (int kh = 0; kh < 3; ++kh) {
        const int tap = kh * 3 + kw;
        if (MODE == CONV_FWD)
          tma_load_5d(b_s + kh * BN_ * 128, &tb[0], tap * cin_blk * 64 + c0, w.n0, w.j, 0, 0, bar);
        else
          tma_load_5d(b_s + kh * BN_ * 128, &tb[0], c0, w.n0, tap, w.j, 0, bar);
      }
      return;
    }
    if (MODE == CONV_FWD) {
      const int tap = kb / cin_blk, c0 = (kb % cin_blk) * 64;
      const int dh = tap / ksz - pad, dw = tap % ksz - pad;
      int b0, y0;
      pix_origin(w.m0, Hr, Wr, b0, y0);
      if (stride == 1) {
        tma_load_5d(a_s, &ta[0], c0, dw, y0 + dh, b0, w.j, bar);
      } else {
        const int py = dh & 1, px = dw & 1;
        tma_load_5d(a_s, &ta[py * 2 + px], c0, (dw - px) / 2, y0 + (dh - py) / 2, b0, w.j, bar);
      }
      tma_load_5d(b_s, &tb[0], tap * cin_blk * 64 + c0, w.n0, w.j, 0, 0, bar);
    } else if (MODE == CONV_DGRAD) {
      int b0, y0;
      pix_origin(w.m0, Hr, Wr, b0, y0);
      int tap, co0, oy, ox;
      if (stride == 1) {
        tap = kb / cout_blk;
        co0 = (kb % cout_blk) * 64;
        oy = -(tap / ksz - pad);
        ox = -(tap % ksz - pad);
      } else {
        const int py = w.z >> 1, px = w.z & 1, nw = ntap1(px);
        const int ti = kb / cout_blk;
        co0 = (kb % cout_blk) * 64;
        const int kh = tap1(py, ti / nw), kw = tap1(px, ti % nw);
        tap = kh * ksz + kw;
        oy = (py - (kh - pad)) / 2;  // input row 2u+py <- output row u + oy
        ox = (px - (kw - pad)) / 2;
      }
      tma_load_5d(a_s, &ta[0], co0, ox, y0 + oy, b0, w.j, bar);
      tma_load_5d(b_s, &tb[0], co0, w.n0, tap, w.j, 0, bar);
    } else {  // WGRAD: K = 64-pixel blocks of the output grid (Hr x Wr)
      int b0, y0;
      pix_origin(kb * 64, Hr, Wr, b0, y0);
      const int dh = w.z / ksz - pad, dw = w.z % ksz - pad;
      tma_load_5d(a_s, &ta[0], w.m0, 0, y0, b0, w.j, bar);
      tma_load_5d(a_s + 8192, &ta[0], w.m0 + 64, 0, y0, b0, w.j, bar);
      if constexpr (TG > 1) {  // stride 1, taps TG*z .. TG*z+TG-1 (one kernel row)
#pragma unroll
        for (int i = 0; i < TG; ++i) {
          const int tap = w.z * TG + i;
          tma_load_5d(b_s + i * 8192, &tb[0], 0, tap % ksz - pad, y0 + tap / ksz - pad, b0, w.j, bar);
        }
        return;
      }
#pragma unroll
      for (int i = 0; i < BN_ / 64; ++i) {
        if (stride == 1) {
          tma_load_5d(b_s + i * 8192, &tb[0], w.n0 + 64 * i, dw, y0 + dh, b0, w.j, bar);
        } else {
          const int py = dh & 1, px = dw & 1;
          tma_load_5d(b_s + i * 8192, &tb[py * 2 + px], w.n0 + 64 * i, (dw - px) / 2, y0 + (dh - py) / 2,
                      b0, w.j, bar);
        }
      }
    }
  }

  // element offset of D row m (within lane w.j), column 0
  TLK_DEV int64_t row_off(const ConvWork& w, int m) const {
    if (MODE == CONV_FWD) return int64_t(m) * cols;
    if (MODE == CONV_WGRAD)  // (tap group z, column n) -> tap TG z + n / cols, channel n % cols
      return int64_t(w.split) * split_st + int64_t(m) * taps * cols + int64_t(w.z) * TG * cols;
    if (stride == 1) return int64_t(m) * cols;
    const int py = w.z >> 1, px = w.z & 1;
    const int v = m % Wr, u = (m / Wr) % Hr, b = m / (Wr * Hr);
    return ((int64_t(b) * Hf + 2 * u + py) * Wf + 2 * v + px) * cols;
  }

  TLK_DEV void epilogue(const ConvWork& w, uint32_t tq, int row0, float* buf, int lane, int cpart, float*,
                        int) const {
    const int rsub = lane >> 3, c4 = (lane & 7) * 4;
    constexpr int NC = BN_ / 32;
#pragma unroll 1
    for (int cc = cpart * (NC / PARTS); cc < (cpart + 1) * (NC / PARTS); ++cc) {
      const int n = w.n0 + cc * 32 + c4;
      float v[32];
      tmem_ld32(tq + cc * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) buf[lane * 33 + i] = v[i];
      __syncwarp();
      const bool col_ok = n < cols * TG;
      if (MODE == CONV_FWD) {
        // y = bf16(D); BN statistics of the stored values as (mean, M2) of
        // this warp's 32 rows (centred: combined with Chan's formula later)
        uint16_t* y = static_cast<uint16_t*>(out) + w.j * out_ls;
        float r[8][4];
        float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int m = row0 + 4 * k + rsub;
          const float* x = buf + (4 * k + rsub) * 33 + c4;
          const uint32_t lo = pack_bf2(x[0], x[1]), hi = pack_bf2(x[2], x[3]);
          r[k][0] = __uint_as_float(lo << 16);
          r[k][1] = __uint_as_float(lo & 0xffff0000u);
          r[k][2] = __uint_as_float(hi << 16);
          r[k][3] = __uint_as_float(hi & 0xffff0000u);
#pragma unroll
          for (int i = 0; i < 4; ++i) s[i] += r[k][i];
          if (col_ok && m < rows) *reinterpret_cast<uint2*>(y + row_off(w, m) + n) = make_uint2(lo, hi);
        }
        float mean[4], q[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          s[i] += __shfl_xor_sync(0xffffffffu, s[i], 8);
          s[i] += __shfl_xor_sync(0xffffffffu, s[i], 16);
          mean[i] = s[i] * (1.0f / 32.0f);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
          for (int i = 0; i < 4; ++i) q[i] += (r[k][i] - mean[i]) * (r[k][i] - mean[i]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          q[i] += __shfl_xor_sync(0xffffffffu, q[i], 8);
          q[i] += __shfl_xor_sync(0xffffffffu, q[i], 16);
        }
        if (rsub == 0 && col_ok) {
          const int quarter = (row0 - w.m0) >> 5;
          float* pp = part + w.j * part_ls + (int64_t(w.mt) * 4 + quarter) * 2 * cols + n;
          *reinterpret_cast<float4*>(pp) = make_float4(mean[0], mean[1], mean[2], mean[3]);
          *reinterpret_cast<float4*>(pp + cols) = make_float4(q[0], q[1], q[2], q[3]);
        }
      } else {
        float* o = static_cast<float*>(out) + w.j * out_ls;
        float4 prev[8];  // accumulate: all eight row loads in flight before any add
        if (MODE == CONV_DGRAD && accumulate) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int m = row0 + 4 * k + rsub;
            prev[k] = (col_ok && m < rows) ? *reinterpret_cast<const float4*>(o + row_off(w, m) + n)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int m = row0 + 4 * k + rsub;
          if (!col_ok || m >= rows) continue;
          const float* x = buf + (4 * k + rsub) * 33 + c4;
          float4 val = make_float4(x[0], x[1], x[2], x[3]);
          if (MODE == CONV_DGRAD && accumulate)
            val = make_float4(prev[k].x + val.x, prev[k].y + val.y, prev[k].z + val.z, prev[k].w + val.w);
          *reinterpret_cast<float4*>(o + row_off(w, m) + n) = val;
        }
      }
      __syncwarp();
    }
  }
};

}  // namespace tlk
