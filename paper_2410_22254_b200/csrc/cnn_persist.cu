// Persistent per-GPU scheduler kernel for the MNIST CNN pack.
//
// ONE launch runs `nsteps` training steps of every lane of the pack.  One CTA
// per SM holding TWO independent worker groups ("virtual CTAs": 10 warps,
// half the shared memory, 256 TMEM columns, barriers and ring counters of
// their own) and one scheduler warp whose lanes 0 / 1 feed group 0 / 1 --
// two items in flight per SM, so one item's memory latency overlaps the
// other's work (a single item per SM left the SM idle on every DRAM round
// trip: measured 0.31 ms/step vs 0.18 for the kernel graph at 8 lanes).
// The work of a step is cut into
// items = (step, phase, lane, index); the items of all lanes and all steps
// form one queue, ordered step-major then phase-major (every item's
// dependencies come earlier in the queue, so the queue order is a topological
// order and the kernel cannot deadlock: the lowest unfinished item always
// has its inputs ready).
//
//   scheduler warp (lane g for group g): takes the next queue index (one global atomic),
//     decodes it, spins (ld.acquire.gpu) until the per-(lane, phase)
//     completion counters its phase depends on reach the target, and hands
//     the item to the workers through a double-buffered shared-memory slot
//     (mbarrier ready/freed) -- so the queue fetch and dependency wait of
//     item k+1 overlap item k.
//   workers (10 warps per group): run the item's phase function with the
//     group's resources (104 KB shared memory, 256 TMEM columns),
//     then one thread publishes completion: __threadfence + atomicAdd on the
//     (lane, phase) counter (generic-proxy writes are made visible to the
//     async proxy -- TMA reads of the consumer -- with fence.proxy.async on
//     both sides).
//
// Lanes progress independently: lane 3 can be in its conv2 backward while
// lane 5 is still in its fc1 forward and lane 0 already in the next step's
// inputs, so the latency-bound phases of different lanes overlap instead of
// forming one launch chain per step.  Every phase runs the same arithmetic,
// in the same order, as the per-phase kernels of the graph path (cnn.cu), so
// the two paths are bit-identical (tests/test_gpu_persistent.py).
//
// Phases (items per lane; dependencies within the step):
//   C1F  inputs + conv1 fwd      B (one sample)   <- prev step OPT, FWA
//   C2F  conv2 fwd+bias+ReLU+pool 36 CTA slices   <- C1F
//   F1F  fc1 fwd split-K          18 splits       <- C2F
//   HR   fc1 reduce+ReLU, partial logits  8 x 16 hidden units  <- F1F
//   HD   head: logits, CE, loss, step scalars, dz3, fc2 / fc1.b grads  1  <- HR
//   F1D  fc1 dgrad + unpool       72 M tiles      <- HD
//   C2D  conv2 dgrad + ReLU mask  36              <- F1D
//   C2W  conv2 wgrad              18 splits       <- F1D
//   FWA  fc1 wgrad + optimizer    72 f tiles      <- F1D
//   C1W  conv1 wgrad              B (one image)   <- C2D
//   OPT  grad finalize + optimizer 36             <- C2W, C1W
// The last of a lane-step's FWA + OPT items ends the lane's step
// (lane_end_step), before it publishes its own completion.
//
// Barrier phases: every mbarrier belongs to one phase type and every ring
// index (tiles, k-blocks, chunks) is a running per-CTA count across all items
// of that type (shared memory), exactly like the tile loop of a persistent
// kernel -- no barrier is ever re-initialised.
#include <cstdlib>
#include <utility>
#include <vector>

#include "cnn_common.cuh"
#include "inputs.cuh"
#include "tc_gemm.cuh"

namespace tlk {

int cnn_persist_enqueue(Pack& p, cudaStream_t st, int nsteps);
bool cnn_persist_enabled(const Pack& p);

namespace {

constexpr int NG = 2;                      // worker groups per CTA
constexpr int PW = 10;                     // worker warps per group
constexpr int PWT = PW * 32;               // worker threads per group
constexpr int P_THREADS = NG * PWT + 32;   // + scheduler warp
constexpr int SCHED_WARP = NG * PW;
constexpr int GSMEM = 104 * 1024;          // shared memory per group
constexpr int GTMEM = 256;                 // TMEM columns per group
constexpr int CEPW = 4;                    // conv epilogue warps (one per TMEM lane quarter)
enum : int { C1F, C2F, F1F, HR, HD, F1D, C2D, C2W, FWA, C1W, OPT, NPH };
constexpr int CNT_STRIDE = 32;  // a lane's completion counters fill one 128-B line

// A worker group's view of the CTA: local thread / warp index, the hardware
// TMEM lane quarter of its warp (warp id mod 4 -- group 1 starts at warp 10),
// its shared memory, TMEM columns and named barriers (3 per group:
// all workers, conv epilogue, 256-thread sub-group).
struct Grp {
  int g, t, lw, q;
  long long item;
  unsigned long long* probe;
  uint8_t* sm;
  uint32_t tmem;
  TLK_DEV void wsync() const { named_bar_sync(1 + 3 * g, PWT); }
  TLK_DEV void conv_sync() const { named_bar_sync(2 + 3 * g, 32 * CEPW); }
  TLK_DEV void sync256() const { named_bar_sync(3 + 3 * g, 256); }
  TLK_DEV GroupSync s256() const { return GroupSync{3 + 3 * g, 256}; }
};
TLK_DEV uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
TLK_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
TLK_DEV uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
TLK_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

struct PArgs {
  CnnBufs buf;  // first: its tensor maps need 64-B alignment
  ConvArgs ca;
  CnnOpt opt;
  LaneState* lanes;
  const int8_t* teacher;
  uint8_t* px;
  int32_t* labels;
  uint16_t* x;
  float *params, *grads, *m1, *m2;
  uint16_t* wbf;
  float *loss, *last_loss;
  uint32_t* cnt;                  // [L][NPH] completion counters (zeroed per launch)
  unsigned long long* next;       // queue head (zeroed per launch)
  int64_t pstride, o_c1w, o_c1b, o_f1w, o_f1b, o_f2w, o_f2b;
  long long total, per_step;
  unsigned long long* probe;      // optional [total][16] timestamps inside items (TLK_PERSIST_PROBE)
  unsigned long long* trace;      // optional [total][5]: fetched, deps ready, started, ended (ns), sm*NG+group
  int host_input, max_steps, write_grads, L, B, nsteps, kblocks;
  int n[NPH];                     // items per lane per step
};

// one set per worker group
#define PROBE(k)                                  \
  do {                                            \
    if (G.probe) G.probe[G.item * 16 + (k)] = gtimer(); \
  } while (0)
struct PBars {
  uint64_t cw_full[2], ca_full[2][2], ca_empty[2][2], ct_full[2][2], ct_empty[2][2];  // conv fwd / dgrad
  uint64_t g_full[2][4], g_empty[2][4], g_done[2];                                      // fc1 fwd / dgrad
  uint64_t w_full[3], w_empty[3], w_done;                                                // conv2 wgrad
  uint64_t f_gfull, f_gempty, f_tfull[2], f_tempty[2], f_sfull[3], f_sempty[3];         // fc1 wgrad + opt
  uint64_t c1w;
  uint64_t ready[2], freed[2];                                                           // dispatcher slots
};
// running per-group counts (ring positions / phase parities of every barrier)
struct PCount {
  uint32_t items[NPH];
  uint32_t conv_tiles[2], gemm_kb[2], wg_stages, fwa_kb, fwa_tiles, fwa_chunks;
};

// ------------------------------------------------------------------ C1F ----
// conv1_fwd_kernel for one sample (threads 0-255 of the group).
__device__ __noinline__ void ph_c1f(const PArgs& a, const Grp& G, int j, int s) {
  const int t = G.t;
  if (t >= 256) return;
  uint8_t* pix = G.sm;
  int(*part)[CLASSES] = reinterpret_cast<int(*)[CLASSES]>(G.sm + 800);
  float* xs = reinterpret_cast<float*>(G.sm + 1120);
  float* ws = reinterpret_cast<float*>(G.sm + 4256);
  float* bs = reinterpret_cast<float*>(G.sm + 5408);
  const GroupSync sync = G.s256();
  const float* params = a.params;
  const LaneState* lanes = a.lanes;
  for (int i = t; i < 288; i += 256) ws[i] = params[j * a.pstride + a.o_c1w + i];
  if (t < 32) bs[t] = params[j * a.pstride + a.o_c1b + t];
  sample_inputs_g<256>(t, sync, lanes[j].seed, lanes[j].steps_done, s, size_t(j) * a.B + s, a.host_input,
                       a.teacher, a.px, a.labels, a.x, pix, part);
  sync();
  for (int i = t; i < 784; i += 256) xs[i] = float(pix[i]) * (1.0f / 256.0f);
  sync();
  const CnnBufs& buf = a.buf;
  uint16_t* h1 = buf.h1 + int64_t(j) * 4 * buf.npos * 8;
  const int c8 = t & 7, c = c8 >> 1, hh = c8 & 1;
  float w[4][9], bsum[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    bsum[e] = bs[c * 8 + hh * 4 + e];
#pragma unroll
    for (int q = 0; q < 9; ++q) w[e][q] = ws[(c * 8 + hh * 4 + e) * 9 + q];
  }
  for (int pos = t >> 3; pos < 676; pos += 32) {
    const int oh = pos / 26, ow = pos % 26;
    float xv[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) xv[q] = xs[(oh + q / 3) * 28 + ow + q % 3];
    float acc[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      acc[e] = 0.f;
#pragma unroll
      for (int q = 0; q < 9; ++q) acc[e] += xv[q] * w[e][q];
    }
    *reinterpret_cast<uint2*>(h1 + (c * buf.npos + p28_pos(s, oh + 1, ow + 1)) * 8 + hh * 4) =
        make_uint2(pack_bf2(fmaxf(acc[0] + bsum[0], 0.f), fmaxf(acc[1] + bsum[1], 0.f)),
                   pack_bf2(fmaxf(acc[2] + bsum[2], 0.f), fmaxf(acc[3] + bsum[3], 0.f)));
  }
}

// ------------------------------------------------------------ C2F / C2D ----
// conv2_tc_kernel (conv_tc.cuh) as a phase: item = the tile slice `cta` of
// lane j (tiles cta, cta + 36, ...); warps 0-3 epilogue (one per TMEM lane
// quarter), 4 TMA, 5 MMA.
template <bool FWD>
__device__ __noinline__ void ph_conv(const ConvArgs& a, const Grp& G, PBars& bars, uint32_t tiles0, uint32_t items0,
                                     int j, int cta) {
  using P = ConvPolicy<FWD>;
  constexpr int NCTA = CONV_CTAS_PER_LANE;
  constexpr int F = FWD ? 0 : 1;
  uint64_t& wfull = bars.cw_full[F];
  uint64_t* afull = bars.ca_full[F];
  uint64_t* aempty = bars.ca_empty[F];
  uint64_t* tfull = bars.ct_full[F];
  uint64_t* tempty = bars.ct_empty[F];
  const int ntiles = a.B * 6;
  const int lw = G.lw, lane = G.t & 31;
  const uint32_t sB = smem_u32(G.sm), sA0 = sB + P::B_BYTES;
  float* tileS = reinterpret_cast<float*>(G.sm + P::B_BYTES + P::AS * P::A_BYTES);
  const uint16_t* src = FWD ? a.h1 + int64_t(j) * 4 * a.npos * 8 : a.dz2 + int64_t(j) * 8 * a.npos * 8;
  if (lw == CEPW) {  // TMA producer
    if (lane == 0) {
      const uint16_t* w = a.wt + int64_t(j) * a.wt_stride + (FWD ? 0 : CONV2_W);
      mbar_expect_tx(&wfull, P::B_BYTES);
      tma_bulk_g2s(sB, w, P::B_BYTES, &wfull);  // the 9 taps are contiguous
      uint32_t i = tiles0;
      for (int tile = cta; tile < ntiles; tile += NCTA, ++i) {
        const int s = i % P::AS;
        if (i >= uint32_t(P::AS)) mbar_wait(&aempty[s], ((i / P::AS) - 1) & 1);
        const int64_t p0 = P::tile_p0(tile);
        mbar_expect_tx(&afull[s], P::A_BYTES);
        for (int c = 0; c < P::PLANES; ++c)
          tma_bulk_g2s(sA0 + s * P::A_BYTES + c * PATCH_BYTES, src + (c * a.npos + p0 - HALO) * 8, PATCH_BYTES,
                       &afull[s]);
      }
    }
  } else if (lw == CEPW + 1) {  // MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC = umma_idesc_bf16(128, P::N, false, false);
      const uint64_t bd0 = umma_desc_interleave(sB, P::BCHUNK, 128);
      mbar_wait(&wfull, items0 & 1);
      uint32_t i = tiles0;
      for (int tile = cta; tile < ntiles; tile += NCTA, ++i) {
        const int s = i % P::AS, ts = i % P::TS;
        mbar_wait(&afull[s], (i / P::AS) & 1);
        if (i >= uint32_t(P::TS)) mbar_wait(&tempty[ts], ((i / P::TS) - 1) & 1);
        tc_fence_after();
        const uint64_t ad0 = umma_desc_interleave(sA0 + s * P::A_BYTES + HALO * 16, PATCH_BYTES, 128);
        const uint32_t d = G.tmem + ts * P::N;
#pragma unroll 1
        for (int t = 0; t < 9; ++t) {
          const int toff = P::tap_off(t);
#pragma unroll
          for (int k = 0; k < P::KSTEPS; ++k) {
            const uint64_t ad = ad0 + uint64_t((2 * k * PATCH_BYTES + toff * 16) >> 4);
            const uint64_t bd = bd0 + uint64_t(((t * 2 * P::KSTEPS + 2 * k) * P::BCHUNK) >> 4);
            mma_bf16(d, ad, bd, IDESC, (t | k) ? 1u : 0u);
          }
        }
        mma_commit(&aempty[s]);
        mma_commit(&tfull[ts]);
      }
    }
  } else if (lw < CEPW) {  // epilogue warps: TMEM lane quarter G.q
    const int row = G.q * 32 + lane;
    const int64_t hbase = int64_t(j) * 4 * a.npos * 8;
    auto h1_valid = [&](int64_t p0) {
      const int r = int(p0 - P28_FRONT) % P28_IMG + row;
      const int pr = r / P28, pc = r % P28;
      return pr >= 1 && pr <= 26 && pc >= 1 && pc <= 26;
    };
    auto h1_fetch = [&](int tile, uint4(&hv)[4]) {
      const int64_t p0 = P::tile_p0(tile);
      const bool ok = tile < ntiles && h1_valid(p0);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        hv[c] = ok ? *reinterpret_cast<const uint4*>(a.h1 + hbase + (c * a.npos + p0 + row) * 8) : make_uint4(0, 0, 0, 0);
    };
    uint4 hnext[4];
    if constexpr (!FWD) h1_fetch(cta, hnext);
    float bb[8];
    if constexpr (FWD) {
      const float* bias = a.params + j * a.pstride + a.b2_off + (G.t & 7) * 8;
#pragma unroll
      for (int e = 0; e < 8; ++e) bb[e] = bias[e];
    }
    uint32_t i = tiles0;
    for (int tile = cta; tile < ntiles; tile += NCTA, ++i) {
      const int s = i % P::TS;
      const uint32_t taddr = G.tmem + s * P::N + (uint32_t(G.q * 32) << 16);
      const int64_t p0 = P::tile_p0(tile);
      if constexpr (FWD) {
        mbar_wait(&tfull[s], (i / P::TS) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int cc = 0; cc < 2; ++cc) {
          float v[32];
          tmem_ld32(taddr + cc * 32, v);
#pragma unroll
          for (int q = 0; q < 32; q += 4)
            *reinterpret_cast<float4*>(tileS + row * 68 + cc * 32 + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[s]);
        G.conv_sync();
        const int b = tile / 6, ti = tile % 6;
        for (int it = G.t; it < 192; it += 32 * CEPW) {
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
          *reinterpret_cast<uint4*>(a.p2 + o) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
          *reinterpret_cast<uint2*>(a.idx + o) = make_uint2(i0, i1);
        }
        G.conv_sync();
      } else {
        const bool valid = h1_valid(p0);
        const int64_t pos = p0 + row;
        uint4 hv[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) hv[c] = hnext[c];
        h1_fetch(tile + NCTA, hnext);
        mbar_wait(&tfull[s], (i / P::TS) & 1);
        tc_fence_after();
        float v[32];
        tmem_ld32(taddr, v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[s]);
        if (valid) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t hw[4] = {hv[c].x, hv[c].y, hv[c].z, hv[c].w};
            uint32_t ow[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float lo = bf2f(uint16_t(hw[e] & 0xFFFF)) > 0.f ? v[c * 8 + 2 * e] : 0.f;
              const float hi = bf2f(uint16_t(hw[e] >> 16)) > 0.f ? v[c * 8 + 2 * e + 1] : 0.f;
              ow[e] = pack_bf2(lo, hi);
            }
            *reinterpret_cast<uint4*>(a.dz1 + hbase + (c * a.npos + pos) * 8) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
          }
        }
      }
    }
  }
}
__host__ __device__ constexpr int conv_tiles_of(int B, int cta) {
  return cta < B * 6 ? (B * 6 - cta + CONV_CTAS_PER_LANE - 1) / CONV_CTAS_PER_LANE : 0;
}

// ------------------------------------------------------------- F1F / F1D ----
// tc_gemm_tma_kernel (tc_gemm.cuh) with the Fc1Fwd / Fc1Dgrad problems of
// cnn.cu: warp 0 lane 0 TMA, warp 1 lane 0 MMA, k-block ring positions are
// running counts.  F1F: 128 threads (split-K partials); F1D: 256 threads,
// tile epilogue (unpool scatter + conv2 bias partials).
constexpr int F1F_STAGES = 4, F1D_STAGES = 2;
constexpr int GEMM_A_BYTES = GEMM_BM * GEMM_BK * 2;  // 16 KB
constexpr int GEMM_STAGE = GEMM_A_BYTES + 64 * GEMM_BK * 2;

template <bool DGRAD>
__device__ __noinline__ void ph_fc1(const PArgs& a, const Grp& G, PBars& bars, uint32_t kb0, uint32_t items0, int j,
                                    int idx) {
  constexpr int STAGES = DGRAD ? F1D_STAGES : F1F_STAGES;
  constexpr int GI = DGRAD ? 1 : 0;
  const CnnBufs& buf = a.buf;
  const int lw = G.lw, lane = G.t & 31, tid = G.t;
  const uint32_t sbase = smem_u32(G.sm);
  const int nk = DGRAD ? 2 : 144 / FC1_SPLITS;
  const int kbb = DGRAD ? 0 : idx * (144 / FC1_SPLITS);
  const int m0 = DGRAD ? idx * GEMM_BM : 0;
  uint64_t* full = bars.g_full[GI];
  uint64_t* empty = bars.g_empty[GI];
  constexpr uint32_t IDESC = umma_idesc_bf16(GEMM_BM, 64, DGRAD, false);
  if (lw == 0 && lane == 0) {
    for (int it = 0; it < nk; ++it) {
      const uint32_t ia = kb0 + it;
      const int s = ia % STAGES;
      if (ia >= uint32_t(STAGES)) mbar_wait(&empty[s], ((ia / STAGES) - 1) & 1);
      const uint32_t a_s = sbase + s * GEMM_STAGE;
      mbar_expect_tx(&full[s], GEMM_STAGE);
      const int kb = kbb + it;
      if (DGRAD) {
        tma_load_3d(a_s, &buf.w1_mn, m0, kb * GEMM_BK, j, &full[s]);
        tma_load_3d(a_s + 8192, &buf.w1_mn, m0 + 64, kb * GEMM_BK, j, &full[s]);
        tma_load_3d(a_s + GEMM_A_BYTES, &buf.dz3m, kb * GEMM_BK, 0, j, &full[s]);
      } else {
        tma_load_3d(a_s, &buf.w1_k, kb * GEMM_BK, 0, j, &full[s]);
        tma_load_3d(a_s + GEMM_A_BYTES, &buf.p2m, kb * GEMM_BK, 0, j, &full[s]);
      }
    }
  } else if (lw == 1 && lane == 0) {
    for (int it = 0; it < nk; ++it) {
      const uint32_t ia = kb0 + it;
      const int s = ia % STAGES;
      mbar_wait(&full[s], (ia / STAGES) & 1);
      tc_fence_after();
      const uint32_t a_s = sbase + s * GEMM_STAGE;
      const uint32_t b_s = a_s + GEMM_A_BYTES;
#pragma unroll
      for (int kk = 0; kk < GEMM_BK / 16; ++kk)
        mma_bf16(G.tmem, stage_desc_tma<GEMM_BM, DGRAD>(a_s, kk), stage_desc_tma<64, false>(b_s, kk), IDESC,
                 (it > 0 || kk > 0) ? 1u : 0u);
      mma_commit(&empty[s]);
      if (it == nk - 1) mma_commit(&bars.g_done[GI]);
    }
  }
  if (tid >= (DGRAD ? 256 : 128)) return;
  mbar_wait(&bars.g_done[GI], items0 & 1);
  tc_fence_after();
  const int row = G.q * 32 + lane;
  const uint32_t tl = G.tmem + (uint32_t(G.q * 32) << 16);
  if constexpr (!DGRAD) {  // Fc1Fwd::epilogue: split-K partial of Z^T
#pragma unroll 1
    for (int cc = 0; cc < 2; ++cc) {
      float v[32];
      tmem_ld32(tl + cc * 32, v);
      float* o = buf.part_fc1 + ((int64_t(j) * FC1_SPLITS + idx) * 128 + row) * 64 + cc * 32;
#pragma unroll
      for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    }
  } else {  // Fc1Dgrad::tile_epilogue
    constexpr int LD = 64 + 4;
    float* tile = reinterpret_cast<float*>(G.sm);
    if (lw < 4) {
#pragma unroll 1
      for (int cc = 0; cc < 2; ++cc) {
        float v[32];
        tmem_ld32(tl + cc * 32, v);
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(tile + row * LD + cc * 32 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
    }
    G.sync256();
    const int B = buf.B;
    const int pos0 = m0 >> 6;
    const int l8 = tid & 7, pl = l8 >> 2, r = l8 & 3;
    const int pos = pos0 + pl, ph = pos / 12, pw = pos % 12;
    const int dr = r >> 1, dc = r & 1;
#pragma unroll 2
    for (int it = tid >> 3; it < 64 * 8; it += 32) {
      const int b = it & 63, ch = it >> 6;
      const bool ok = b < B;
      const uint2 code2 = ok ? *reinterpret_cast<const uint2*>(buf.idx + j * buf.p2_st + int64_t(b) * 9216 + pos * 64 +
                                                               ch * 8)
                             : make_uint2(0u, 0u);
      const uint32_t cw[2] = {code2.x, code2.y};
      float* t0 = tile + (pl * 64 + ch * 8) * LD + b;
      uint16_t z[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t code = (cw[e >> 2] >> (8 * (e & 3))) & 0xFF;
        z[e] = (ok && (code & 4)) ? f2bf(t0[e * LD]) : uint16_t(0);
      }
      __syncwarp();
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
          for (int e = 0; e < 8; ++e) t0[e * LD] = bf2f(z[e]);
        }
        uint16_t* plane = buf.dz2 + (int64_t(j) * 8 + ch) * buf.npos * 8;
        *reinterpret_cast<uint4*>(plane + (p28_pos(b, 2 * ph + 2 + dr, 2 * pw + 2 + dc)) * 8) =
            make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
    G.sync256();
    if (tid < 128) {
      float s = 0.f;
      for (int b = 0; b < B; ++b) s += tile[tid * LD + b];
      buf.colsum[int64_t(j) * 9216 + m0 + tid] = s;
    }
  }
}

// ------------------------------------------------------------- HR / HD -----
// cnn_head_kernel split in two phases: HR (8 items per lane) = what each CTA
// of the 8-CTA cluster computes before the DSMEM exchange (its h3 slice and
// partial logits, written to buf.plog); HD (1 item) = the rest, for all 128
// hidden units (same per-element formulas and summation orders).
__device__ __noinline__ void ph_hr(const PArgs& a, const Grp& G, int j, int r) {
  const int tid = G.t;
  if (tid >= 256) return;
  constexpr int C = CLASSES, H = 128, HS = HEAD_HS;
  const CnnBufs& buf = a.buf;
  const int B = buf.B, k0 = r * HS;
  float* hs = reinterpret_cast<float*>(G.sm);  // [64][HS]
  float* wsl = hs + 64 * HS;                   // [C][HS]
  const float* P = a.params + j * a.pstride;
  for (int i = tid; i < C * HS; i += 256) wsl[i] = P[a.o_f2w + (i / HS) * H + k0 + i % HS];
  for (int i = tid; i < HS * 64; i += 256) {
    const int kk = i >> 6, b = i & 63;
    if (b >= B) continue;
    const float* pp = buf.part_fc1 + int64_t(j) * FC1_SPLITS * 128 * 64 + (k0 + kk) * 64 + b;
    float sacc = 0.0f;
#pragma unroll
    for (int k = 0; k < FC1_SPLITS; ++k) sacc += pp[int64_t(k) * 128 * 64];
    const uint16_t hb = f2bf(fmaxf(sacc + P[a.o_f1b + k0 + kk], 0.0f));
    buf.h3[j * buf.h3_st + b * 128 + k0 + kk] = hb;
    hs[b * HS + kk] = bf2f(hb);
  }
  G.sync256();
  float* plog = buf.plog + (int64_t(j) * HEAD_CL + r) * 64 * C;
  for (int i = tid; i < B * C; i += 256) {
    const int b = i / C, c = i % C;
    float sacc = 0.0f;
#pragma unroll
    for (int kk = 0; kk < HS; ++kk) sacc += hs[b * HS + kk] * wsl[c * HS + kk];
    plog[i] = sacc;
  }
}

__device__ __noinline__ void ph_hd(const PArgs& a, const Grp& G, int j) {
  const int tid = G.t;
  if (tid >= 256) return;
  constexpr int C = CLASSES, H = 128;
  const CnnBufs& buf = a.buf;
  const int B = buf.B;
  float* logit = reinterpret_cast<float*>(G.sm);  // [64][C]
  float* d = logit + 64 * C;                       // [64][C]
  float* lossb = d + 64 * C;                       // [64]
  float* hs = lossb + 64;                          // [64][128]
  float* zs = hs + 64 * H;                         // [64][128]
  float* w2 = zs + 64 * H;                         // [C][128]
  const float* P = a.params + j * a.pstride;
  float* Gr = a.grads + j * a.pstride;
  {  // every global load of this prologue is issued before the first use
    float pv[3][HEAD_CL];
    const float* pl0 = buf.plog + int64_t(j) * HEAD_CL * 64 * C;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int i = tid + r * 256;
#pragma unroll
      for (int q = 0; q < HEAD_CL; ++q) pv[r][q] = i < B * C ? pl0[q * 64 * C + i] : 0.0f;
    }
    uint4 hv[4];
    const uint4* h3v = reinterpret_cast<const uint4*>(buf.h3 + j * buf.h3_st);
#pragma unroll
    for (int r = 0; r < 4; ++r) hv[r] = (tid + r * 256) * 8 < B * H ? h3v[tid + r * 256] : make_uint4(0, 0, 0, 0);
    float wv[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) wv[r] = P[a.o_f2w + tid + r * 256];
    float bv[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) bv[r] = P[a.o_f2b + (tid + r * 256) % C];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int i = tid + r * 256;
      float sacc = 0.0f;
#pragma unroll
      for (int q = 0; q < HEAD_CL; ++q) sacc += pv[r][q];
      if (i < B * C) logit[i] = sacc + bv[r];
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = (tid + r * 256) * 8;
      if (i < B * H) {
        const uint32_t w[4] = {hv[r].x, hv[r].y, hv[r].z, hv[r].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          hs[i + 2 * e] = bf2f(uint16_t(w[e] & 0xFFFF));
          hs[i + 2 * e + 1] = bf2f(uint16_t(w[e] >> 16));
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 5; ++r) w2[tid + r * 256] = wv[r];
  }

  G.sync256();
  if (tid == 0) PROBE(3);
  if (tid < B) {
    const int y = a.labels[size_t(j) * B + tid];
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
  G.sync256();
  if (tid == 0) {
    float sacc = 0.0f;
    for (int b = 0; b < B; ++b) sacc += lossb[b];
    const float L = sacc / float(B);
    LaneState& ls = a.lanes[j];
    a.loss[size_t(j) * a.max_steps + ls.steps_done] = L;
    a.last_loss[j] = L;
    lane_step_scalars(ls);
    PROBE(4);
  }
  if (tid >= 64 && tid < 64 + C) {
    const int c = tid - 64;
    float sacc = 0.0f;
    for (int b = 0; b < B; ++b) sacc += d[b * C + c];
    Gr[a.o_f2b + c] = sacc;
  }
  uint16_t* dzj = buf.dz3 + j * buf.h3_st;
  for (int i = tid; i < B * H; i += 256) {
    const int b = i / H, k = i % H;
    float dh = 0.0f;
#pragma unroll
    for (int c = 0; c < C; ++c) dh += d[b * C + c] * w2[c * H + k];
    const uint16_t zb = f2bf(hs[i] > 0.0f ? dh : 0.0f);
    dzj[b * H + k] = zb;
    zs[i] = bf2f(zb);
  }
  G.sync256();
  for (int i = tid; i < H * (C + 1); i += 256) {
    const int k = i % H, c = i / H;
    float sacc = 0.0f;
    if (c < C) {
      for (int b = 0; b < B; ++b) sacc += d[b * C + c] * hs[b * H + k];
      Gr[a.o_f2w + c * H + k] = sacc;
    } else {
      for (int b = 0; b < B; ++b) sacc += zs[b * H + k];
      Gr[a.o_f1b + k] = sacc;
    }
  }
}

// ------------------------------------------------------------------ C2W ----
// conv2_wgrad_tc_kernel as a phase (warps 0-3 epilogue, 4 TMA, 5 MMA).  The
// split boundaries are the graph path's 128-position chunks; each chunk is
// staged as two 64-position halves, and the A rows are ordered (shift k',
// ic chunk c) -- group g = 4k' + c -- so the 4 spare k' = 3 groups are the
// LAST 32 rows: they read whatever follows the 12 loaded copies and take no
// shared memory (3 stages fit a group).  TMEM row = 32 k' + ic: warp quarter
// q holds tap kw = q and ic = lane.  The MMA sequence and the products per
// accumulator element are the graph kernel's.
constexpr int WGH_KC = 64;
constexpr int WGH_ACOPY = (WGH_KC + 56) * 16;   // 120 positions
constexpr int WGH_ASTRIDE = WGH_ACOPY;
constexpr int WGH_A_BYTES = 12 * WGH_ASTRIDE;   // 22.5 KB
constexpr int WGH_B_PLANE = WGH_KC * 16;        // 1 KB
constexpr int WGH_STAGE = WGH_A_BYTES + 8 * WGH_B_PLANE;
constexpr int WGH_STAGES = 3;  // = the size of PBars::w_full / w_empty
static_assert(16 * WGH_ASTRIDE <= WGH_STAGE, "spare rows stay inside the stage");
constexpr uint32_t WGH_TX = 12 * WGH_ACOPY + 8 * WGH_B_PLANE;

__device__ __noinline__ void ph_c2w(const ConvArgs& a, const Grp& G, PBars& bars, uint32_t st0, uint32_t items0,
                                    int j, int split) {
  const int lw = G.lw, lane = G.t & 31;
  const uint32_t s0 = smem_u32(G.sm);
  const int nch = a.B * P28_IMG / WG_KC;
  const int c_begin = split * nch / a.wgrad_splits, c_end = (split + 1) * nch / a.wgrad_splits;
  const int n = 2 * (c_end - c_begin);  // half-chunk stages
  if (lw == 4) {
    if (lane == 0) {
      const uint16_t* dz2 = a.dz2 + int64_t(j) * 8 * a.npos * 8;
      const uint16_t* h1 = a.h1 + int64_t(j) * 4 * a.npos * 8;
      for (int i = 0; i < n; ++i) {
        const uint32_t ia = st0 + i;
        const int s = ia % WGH_STAGES;
        if (ia >= uint32_t(WGH_STAGES)) mbar_wait(&bars.w_empty[s], ((ia / WGH_STAGES) - 1) & 1);
        if (i < 6) PROBE(i);
        const int64_t q0 = P28_FRONT + int64_t(c_begin) * WG_KC + int64_t(i) * WGH_KC;
        const uint32_t st = s0 + s * WGH_STAGE;
        mbar_expect_tx(&bars.w_full[s], WGH_TX);
        for (int c = 0; c < 4; ++c)
          for (int k = 0; k < 3; ++k)
            tma_bulk_g2s(st + (k * 4 + c) * WGH_ASTRIDE, h1 + (c * a.npos + q0 - HALO + k) * 8, WGH_ACOPY,
                         &bars.w_full[s]);
        for (int c = 0; c < 8; ++c)
          tma_bulk_g2s(st + WGH_A_BYTES + c * WGH_B_PLANE, dz2 + (c * a.npos + q0) * 8, WGH_B_PLANE, &bars.w_full[s]);
      }
    }
  } else if (lw == 5) {
    if (lane == 0) {
      constexpr uint32_t IDESC = umma_idesc_bf16(128, 64, true, true);
      for (int i = 0; i < n; ++i) {
        const uint32_t ia = st0 + i;
        const int s = ia % WGH_STAGES;
        mbar_wait(&bars.w_full[s], (ia / WGH_STAGES) & 1);
        if (i < 6) PROBE(6 + i);
        tc_fence_after();
        const uint32_t st = s0 + s * WGH_STAGE;
        const uint64_t ad0 = umma_desc_interleave(st, 128, WGH_ASTRIDE);
        const uint64_t bd0 = umma_desc_interleave(st + WGH_A_BYTES, 128, WGH_B_PLANE);
#pragma unroll
        for (int k = 0; k < WGH_KC / 16; ++k)
#pragma unroll
          for (int kh = 0; kh < 3; ++kh) {
            const uint64_t ad = ad0 + uint64_t(((16 * k + 28 * kh) * 16) >> 4);
            const uint64_t bd = bd0 + uint64_t((k * 256) >> 4);
            mma_bf16(G.tmem + 64 * kh, ad, bd, IDESC, (i | k) ? 1u : 0u);
          }
        mma_commit(&bars.w_empty[s]);
      }
      mma_commit(&bars.w_done);
    }
  } else if (lw < 4) {
    mbar_wait(&bars.w_done, items0 & 1);
    if (G.t == 0) PROBE(12);
    tc_fence_after();
    const int kp = G.q, ic = lane;
    float* out = a.part2 + (int64_t(j) * a.wgrad_splits + split) * 9 * 64 * 32;
#pragma unroll 1
    for (int kh = 0; kh < 3; ++kh)
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        float v[32];
        tmem_ld32(G.tmem + (uint32_t(G.q * 32) << 16) + 64 * kh + 32 * h, v);
        if (kp < 3) {
          float* o = out + ((kh * 3 + kp) * 64 + 32 * h) * 32 + ic;
#pragma unroll
          for (int q = 0; q < 32; ++q) o[q * 32] = v[q];
        }
      }
  }
}
__host__ __device__ constexpr int c2w_stages_of(int B, int split) {
  return 2 * ((split + 1) * (B * P28_IMG / WG_KC) / C2W_SPLITS - split * (B * P28_IMG / WG_KC) / C2W_SPLITS);
}

// ------------------------------------------------------------------ FWA ----
// fc1_wgrad_adam_kernel as a phase: item = one 128-feature tile of lane j;
// warp 0 TMA, warp 1 MMA, warps 2-9 update (two per TMEM lane quarter);
// the tile's p / m / v stream in 16-output chunks through a 3-slot ring.
constexpr int FH_SLOTS = 3;
constexpr int FH_CHUNK = 16 * 128 * 4;           // one tensor's [16 o][128 f] chunk
constexpr int FH_SLOT_BYTES = 3 * FH_CHUNK;      // 24 KB
constexpr int FH_CHUNKS = 8;                     // per tile
constexpr int FH_UPD = 8;                        // update warps
static_assert(FWA_STAGE_BYTES + FH_SLOTS * FH_SLOT_BYTES <= GSMEM, "fc1 wgrad+opt fits a group");

__device__ __noinline__ void ph_fwa(const PArgs& a, const Grp& G, PBars& bars, uint32_t kb0, uint32_t lt, uint32_t cs0,
                                    int j, int ft) {
  const CnnBufs& p = a.buf;  // tensor maps (param space)
  const int lw = G.lw, lane = G.t & 31;
  const uint32_t sbase = smem_u32(G.sm);
  const uint32_t slot_base = sbase + FWA_STAGE_BYTES;
  const uint8_t* slot_ptr = G.sm + FWA_STAGE_BYTES;
  const int f0 = ft * 128;
  constexpr uint32_t IDESC = umma_idesc_bf16(GEMM_BM, 128, true, true);
  const int acc = lt & 1;
  if (lw == 0) {
    if (lane == 0) {
      PROBE(6);
      for (int kb = 0; kb < a.kblocks; ++kb) {
        const uint32_t ia = kb0 + kb;
        if (ia >= 1) mbar_wait(&bars.f_gempty, (ia - 1) & 1);
        mbar_expect_tx(&bars.f_gfull, FWA_STAGE_BYTES);
        tma_load_3d(sbase, &p.p2m, f0, kb * GEMM_BK, j, &bars.f_gfull);
        tma_load_3d(sbase + 8192, &p.p2m, f0 + 64, kb * GEMM_BK, j, &bars.f_gfull);
        tma_load_3d(sbase + 16384, &p.dz3m, 0, kb * GEMM_BK, j, &bars.f_gfull);
        tma_load_3d(sbase + 24576, &p.dz3m, 64, kb * GEMM_BK, j, &bars.f_gfull);
      }
      for (int c = 0; c < FH_CHUNKS; ++c) {
        const uint32_t cs = cs0 + c;
        const int sl = cs % FH_SLOTS;
        if (cs >= uint32_t(FH_SLOTS)) mbar_wait(&bars.f_sempty[sl], ((cs / FH_SLOTS) - 1) & 1);
        const uint32_t d = slot_base + sl * FH_SLOT_BYTES;
        mbar_expect_tx(&bars.f_sfull[sl], FH_SLOT_BYTES);
        tma_load_3d(d, &p.fh_p, f0, 16 * c, j, &bars.f_sfull[sl]);
        tma_load_3d(d + FH_CHUNK, &p.fh_m, f0, 16 * c, j, &bars.f_sfull[sl]);
        tma_load_3d(d + 2 * FH_CHUNK, &p.fh_v, f0, 16 * c, j, &bars.f_sfull[sl]);
      }
    }
  } else if (lw == 1) {
    if (lane == 0) {
      if (lt >= 2) mbar_wait(&bars.f_tempty[acc], ((lt >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t d = G.tmem + acc * 128;
      for (int kb = 0; kb < a.kblocks; ++kb) {
        const uint32_t ia = kb0 + kb;
        mbar_wait(&bars.f_gfull, ia & 1);
        PROBE(8);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < GEMM_BK / 16; ++kk)
          mma_bf16(d, stage_desc_tma<GEMM_BM, true>(sbase, kk), stage_desc_tma<128, true>(sbase + 16384, kk), IDESC,
                   (kb > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&bars.f_gempty);
      }
      mma_commit(&bars.f_tfull[acc]);
    }
  } else {
    const int og = (lw - 2) >> 2, fl = G.q * 32 + lane;
    const LaneState s = a.lanes[j];
    mbar_wait(&bars.f_tfull[acc], (lt >> 1) & 1);
    if (G.t == 64) PROBE(10);
    tc_fence_after();
    for (int c = 0; c < FH_CHUNKS; ++c) {
      const uint32_t cs = cs0 + c;
      const int o0 = 16 * c + 8 * og;
      float g[8];
      tmem_ld8(G.tmem + acc * 128 + o0 + (uint32_t(G.q * 32) << 16), g);
      if (c == FH_CHUNKS - 1) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.f_tempty[acc]);
      }
      const int sl = cs % FH_SLOTS;
      mbar_wait(&bars.f_sfull[sl], (cs / FH_SLOTS) & 1);
      if (G.t == 64 && c == 0) PROBE(11);
      if (G.t == 64 && c == FH_CHUNKS - 1) PROBE(12);
      const float* P = reinterpret_cast<const float*>(slot_ptr + sl * FH_SLOT_BYTES);
      float pv[8], mv[8], vv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int off = (8 * og + i) * 128 + fl;
        pv[i] = P[off];
        mv[i] = P[FH_CHUNK / 4 + off];
        vv[i] = P[FH_CHUNK / 2 + off];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.f_sempty[sl]);
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
      const int64_t e = j * a.pstride + a.o_f1w + int64_t(o0) * 9216 + f0 + fl;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        a.params[e + int64_t(i) * 9216] = pv[i];
        a.m1[e + int64_t(i) * 9216] = mv[i];
        a.m2[e + int64_t(i) * 9216] = vv[i];
        a.wbf[e + int64_t(i) * 9216] = f2bf(pv[i]);
      }
      if (a.write_grads) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a.grads[e + int64_t(i) * 9216] = g[i];
      }
    }
  }
}

// ------------------------------------------------------------------ C1W ----
// conv1_wgrad_kernel for one image (threads 0-255 of the group).
__device__ __noinline__ void ph_c1w(const PArgs& a, const Grp& G, PBars& bars, uint32_t items0, int j, int b) {
  const int t = G.t;
  if (t >= 256) return;
  const int warp = t >> 5, lane = t & 31;
  const CnnBufs& buf = a.buf;
  uint16_t(*dzs)[P28_IMG * 8] = reinterpret_cast<uint16_t(*)[P28_IMG * 8]>(G.sm);
  float* xs = reinterpret_cast<float*>(G.sm + C1W_SMEM);
  float(*red)[4][80] = reinterpret_cast<float(*)[4][80]>(G.sm + C1W_SMEM + 784 * 4);
  const GroupSync sync = G.s256();
  uint64_t* bar = &bars.c1w;
  if (t == 0) {
    mbar_expect_tx(bar, 4 * P28_IMG * 16);
    for (int c = 0; c < 4; ++c)
      tma_bulk_g2s(smem_u32(dzs[c]), buf.dz1 + ((int64_t(j) * 4 + c) * buf.npos + p28_pos(b, 0, 0)) * 8, P28_IMG * 16,
                   bar);
  }
  const uint4* xr = reinterpret_cast<const uint4*>(a.x + (size_t(j) * buf.B + b) * 784);
  if (t < 98) {
    const uint4 v = xr[t];
    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      xs[t * 8 + 2 * e] = bf2f(uint16_t(wv[e] & 0xFFFF));
      xs[t * 8 + 2 * e + 1] = bf2f(uint16_t(wv[e] >> 16));
    }
  }
  sync();
  mbar_wait(bar, items0 & 1);
  const int c8 = t & 7, c = c8 >> 1, hh = c8 & 1, g = t >> 3;
  float acc[4][10];
#pragma unroll
  for (int e = 0; e < 4; ++e)
#pragma unroll
    for (int q = 0; q < 10; ++q) acc[e][q] = 0.f;
  for (int q = g; q < 676; q += C1W_THREADS / 8) {
    const int oh = q / 26, ow = q % 26;
    const uint2 dv = *reinterpret_cast<const uint2*>(&dzs[c][((oh + 1) * P28 + ow + 1) * 8 + hh * 4]);
    const float d[4] = {__uint_as_float(dv.x << 16), __uint_as_float(dv.x & 0xffff0000u),
                        __uint_as_float(dv.y << 16), __uint_as_float(dv.y & 0xffff0000u)};
    float xv[9];
#pragma unroll
    for (int tt = 0; tt < 9; ++tt) xv[tt] = xs[(oh + tt / 3) * 28 + ow + tt % 3];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
#pragma unroll
      for (int tt = 0; tt < 9; ++tt) acc[e][tt] += d[e] * xv[tt];
      acc[e][9] += d[e];
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e)
#pragma unroll
    for (int tt = 0; tt < 10; ++tt) {
      float v = acc[e][tt];
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      acc[e][tt] = v;
    }
  if (lane < 8) {
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int tt = 0; tt < 10; ++tt) red[warp][c][(hh * 4 + e) * 10 + tt] = acc[e][tt];
  }
  sync();
  for (int o = t; o < 320; o += C1W_THREADS) {
    const int oc = o / 10, tt = o % 10;
    float s = red[0][oc >> 3][(oc & 7) * 10 + tt];
#pragma unroll
    for (int w = 1; w < C1W_THREADS / 32; ++w) s += red[w][oc >> 3][(oc & 7) * 10 + tt];
    buf.part1[(int64_t(j) * buf.B + b) * 320 + o] = s;
  }
}

// ------------------------------------------------------------------ OPT ----
// cnn_opt_kernel as a phase (item = its CTA index; 256 threads); the end of
// the lane's step moved to the completion bookkeeping (FWA + OPT items).
__device__ __noinline__ void ph_opt(const PArgs& a0, const Grp& G, int j, int bx) {
  const int tid = G.t;
  if (tid >= 256) return;
  const CnnOpt& a = a0.opt;
  const CnnBufs& buf = a0.buf;
  const LaneState s = a.lanes[j];
  const CnnOffs& o = a.o;
  if (bx < CNN_OPT_HEAVY) {
    const int l = tid & 31;
    const int h = bx * 8 + (tid >> 5);
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
  } else {
    const int64_t s4 = a.stride / 4, work = a.a1 + (s4 - a.b0);
    const int nl = a0.n[OPT] - CNN_OPT_HEAVY;
    const int64_t per = (work + nl - 1) / nl;
    const int64_t w0 = (bx - CNN_OPT_HEAVY) * per, w1 = min(work, w0 + per);
    for (int64_t w = w0 + tid; w < w1; w += 256) {
      const int64_t idx = w < a.a1 ? w : a.b0 + (w - a.a1);
      const int64_t e = idx * 4;
      if ((e >= o.c1w && e < o.c1w + 288) || (e >= o.c1b && e < o.c1b + 32) || (e >= o.c2b && e < o.c2b + 64))
        continue;
      float g[4];
      if (e >= o.c2w && e < o.c2w + CONV2_W) {
        const int r = int(e - o.c2w), oc = r / 288, t = r % 288, tap = t >> 5, ic = t & 31;
        const float* pp = buf.part2 + ((int64_t(j) * C2W_SPLITS * 9 + tap) * 64 + oc) * 32 + ic;
        float4 v[C2W_SPLITS];
#pragma unroll
        for (int k = 0; k < C2W_SPLITS; ++k) v[k] = *reinterpret_cast<const float4*>(pp + int64_t(k) * 9 * 64 * 32);
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
}

// --------------------------------------------------------------- kernel ----
constexpr int P_SMEM = NG * GSMEM + 1024;
static_assert(ConvPolicy<true>::B_BYTES + 2 * ConvPolicy<true>::A_BYTES + ConvPolicy<true>::TILE_BYTES <= GSMEM, "");
static_assert(ConvPolicy<false>::B_BYTES + 2 * ConvPolicy<false>::A_BYTES <= GSMEM, "");
static_assert(F1F_STAGES * GEMM_STAGE <= GSMEM && WGH_STAGES * WGH_STAGE <= GSMEM, "");
static_assert(C1W_SMEM + 784 * 4 + 8 * 4 * 80 * 4 <= GSMEM, "");

struct Item {
  int s, ph, j, idx;
};
TLK_DEV Item decode(const PArgs& a, long long it) {
  Item d;
  d.s = int(it / a.per_step);
  long long r = it % a.per_step;
  d.ph = 0;
  for (int ph = 0; ph < NPH; ++ph) {
    const long long n = (long long)a.L * a.n[ph];
    if (r < n) {
      d.ph = ph;
      d.j = int(r / a.n[ph]);
      d.idx = int(r % a.n[ph]);
      return d;
    }
    r -= n;
  }
  d.j = d.idx = 0;
  return d;
}

TLK_DEV uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spin with relaxed loads (an acquire load invalidates the SM's L1 -- on
// every poll that would evict the worker groups' cached data), back off, and
// acquire once when the target is reached (the caller's fence).
TLK_DEV void wait_count(const uint32_t* c, uint32_t target) {
  uint32_t ns = 32;
  while (ld_relaxed(c) < target) {
    __nanosleep(ns);
    ns = ns < 256 ? ns * 2 : 256;
  }
}

// dependencies of an item: completion counts (same lane) it must see
TLK_DEV void wait_deps(const PArgs& a, const Item& d) {
  const uint32_t* c = a.cnt + d.j * CNT_STRIDE;
  const uint32_t s1 = uint32_t(d.s + 1);
  switch (d.ph) {
    case C1F:
      if (d.s > 0) {
        wait_count(c + OPT, uint32_t(a.n[OPT]) * d.s);
        wait_count(c + FWA, uint32_t(a.n[FWA]) * d.s);
      }
      break;
    case C2F: wait_count(c + C1F, a.n[C1F] * s1); break;
    case F1F: wait_count(c + C2F, a.n[C2F] * s1); break;
    case HR: wait_count(c + F1F, a.n[F1F] * s1); break;
    case HD: wait_count(c + HR, a.n[HR] * s1); break;
    case F1D: wait_count(c + HD, a.n[HD] * s1); break;
    case C2D:
    case C2W:
    case FWA: wait_count(c + F1D, a.n[F1D] * s1); break;
    case C1W: wait_count(c + C2D, a.n[C2D] * s1); break;
    case OPT:
      wait_count(c + C2W, a.n[C2W] * s1);
      wait_count(c + C1W, a.n[C1W] * s1);
      break;
  }
}

TLK_DEV void init_bars(PBars& b) {
  for (int f = 0; f < 2; ++f) {
    mbar_init(&b.cw_full[f], 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&b.ca_full[f][s], 1);
      mbar_init(&b.ca_empty[f][s], 1);
      mbar_init(&b.ct_full[f][s], 1);
      mbar_init(&b.ct_empty[f][s], CEPW);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&b.g_full[f][s], 1);
      mbar_init(&b.g_empty[f][s], 1);
    }
    mbar_init(&b.g_done[f], 1);
    mbar_init(&b.f_tfull[f], 1);
    mbar_init(&b.f_tempty[f], FH_UPD);
    mbar_init(&b.ready[f], 1);
    mbar_init(&b.freed[f], 1);
  }
  for (int s = 0; s < 3; ++s) {
    mbar_init(&b.w_full[s], 1);
    mbar_init(&b.w_empty[s], 1);
  }
  mbar_init(&b.w_done, 1);
  mbar_init(&b.f_gfull, 1);
  mbar_init(&b.f_gempty, 1);
  for (int s = 0; s < FH_SLOTS; ++s) {
    mbar_init(&b.f_sfull[s], 1);
    mbar_init(&b.f_sempty[s], FH_UPD);
  }
  mbar_init(&b.c1w, 1);
}

__global__ void __launch_bounds__(P_THREADS, 1) cnn_persist_kernel(const __grid_constant__ PArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) PBars bars_all[NG];
  __shared__ PCount pc_all[NG];
  __shared__ int4 slot_item[NG][2];
  __shared__ long long slot_id[NG][2];
  __shared__ uint32_t tmem_s;
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int g = 0; g < NG; ++g) init_bars(bars_all[g]);
    fence_mbar_init();
    uint32_t* z = reinterpret_cast<uint32_t*>(pc_all);
    for (int i = 0; i < int(sizeof(pc_all) / 4); ++i) z[i] = 0;
  }
  if (warp == 0) tmem_alloc<NG * GTMEM>(&tmem_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == SCHED_WARP) {  // ------------------- scheduler: lane g feeds group g
    if (lane < NG) {
      PBars& bars = bars_all[lane];
      for (uint32_t k = 0;; ++k) {
        const int sl = k & 1;
        if (k >= 2) mbar_wait(&bars.freed[sl], ((k >> 1) - 1) & 1);
        const long long it = (long long)atomicAdd(a.next, 1ull);
        int4 v = make_int4(-1, 0, 0, 0);
        if (it < a.total) {
          const unsigned long long t0 = a.trace ? gtimer() : 0;
          const Item d = decode(a, it);
          wait_deps(a, d);
          asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire what the counters published
          v = make_int4(d.s, d.ph, d.j, d.idx);
          if (a.trace) {
            a.trace[it * 5 + 0] = t0;
            a.trace[it * 5 + 1] = gtimer();
          }
        }
        slot_item[lane][sl] = v;
        slot_id[lane][sl] = it;
        mbar_arrive(&bars.ready[sl]);
        if (v.x < 0) break;
      }
    }
  } else {  // ------------------------------------- worker group
    const int g = warp / PW;
    Grp G;
    G.g = g;
    G.t = tid - g * PWT;
    G.lw = warp - g * PW;
    G.q = warp & 3;
    G.sm = sm + g * GSMEM;
    G.tmem = tmem_s + g * GTMEM;
    G.item = 0;
    G.probe = nullptr;
    PBars& bars = bars_all[g];
    PCount& pc = pc_all[g];
    for (uint32_t k = 0;; ++k) {
      const int sl = k & 1;
      mbar_wait(&bars.ready[sl], (k >> 1) & 1);
      const int4 v = slot_item[g][sl];
      if (v.x < 0) break;
      const int ph = v.y, j = v.z, idx = v.w;
      const long long item_id = slot_id[g][sl];
      G.item = item_id;
      G.probe = a.probe;
      if (G.t == 0) PROBE(13);
      if (a.trace && G.t == 0) {
        a.trace[item_id * 5 + 2] = gtimer();
        a.trace[item_id * 5 + 4] = smid() * NG + g;
      }
      const bool active = a.lanes[j].active != 0;
      fence_proxy_async_global();  // TMA reads below see the generic writes this item depends on
      uint32_t d_tiles = 0, d_kb = 0, d_st = 0;
      if (active) {
        switch (ph) {
          case C1F: ph_c1f(a, G, j, idx); break;
          case C2F:
            ph_conv<true>(a.ca, G, bars, pc.conv_tiles[0], pc.items[C2F], j, idx);
            d_tiles = conv_tiles_of(a.B, idx);
            break;
          case C2D:
            ph_conv<false>(a.ca, G, bars, pc.conv_tiles[1], pc.items[C2D], j, idx);
            d_tiles = conv_tiles_of(a.B, idx);
            break;
          case F1F:
            ph_fc1<false>(a, G, bars, pc.gemm_kb[0], pc.items[F1F], j, idx);
            d_kb = 144 / FC1_SPLITS;
            break;
          case F1D:
            ph_fc1<true>(a, G, bars, pc.gemm_kb[1], pc.items[F1D], j, idx);
            d_kb = 2;
            break;
          case HR: ph_hr(a, G, j, idx); break;
          case HD: ph_hd(a, G, j); break;
          case C2W:
            ph_c2w(a.ca, G, bars, pc.wg_stages, pc.items[C2W], j, idx);
            d_st = c2w_stages_of(a.B, idx);
            break;
          case FWA:
            ph_fwa(a, G, bars, pc.fwa_kb, pc.fwa_tiles, pc.fwa_chunks, j, idx);
            d_kb = a.kblocks;
            break;
          case C1W: ph_c1w(a, G, bars, pc.items[C1W], j, idx); break;
          case OPT: ph_opt(a, G, j, idx); break;
        }
      }
      fence_proxy_async_global();  // this item's generic writes -> later TMA reads (other CTAs)
      tc_fence_before();
      G.wsync();
      tc_fence_after();
      if (G.t == 0) PROBE(14);
      if (G.t == 0) {
        if (active) {
          pc.items[ph] += 1;
          if (ph == C2F) pc.conv_tiles[0] += d_tiles;
          if (ph == C2D) pc.conv_tiles[1] += d_tiles;
          if (ph == F1F) pc.gemm_kb[0] += d_kb;
          if (ph == F1D) pc.gemm_kb[1] += d_kb;
          if (ph == C2W) pc.wg_stages += d_st;
          if (ph == FWA) {
            pc.fwa_kb += d_kb;
            pc.fwa_tiles += 1;
            pc.fwa_chunks += FH_CHUNKS;
          }
        }
        __threadfence();
        if (active && (ph == FWA || ph == OPT)) {
          const unsigned prev = atomicAdd(&a.lanes[j].done_ctas, 1u);
          if (prev == unsigned(a.n[FWA] + a.n[OPT] - 1)) {  // the lane-step's last FWA / OPT item
            a.lanes[j].done_ctas = 0;
            lane_end_step(a.lanes[j]);
            __threadfence();
          }
        }
        atomicAdd(a.cnt + j * CNT_STRIDE + ph, 1u);
        if (a.trace) a.trace[item_id * 5 + 3] = gtimer();
        mbar_arrive(&bars.freed[sl]);
      }
      G.wsync();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<NG * GTMEM>(tmem_s);
}

}  // namespace

bool cnn_persist_enabled(const Pack& p) {
  static const char* e = getenv("TLK_CNN_PERSIST");  // 1: every CNN pack, 0: none
  if (e && e[0] == '1') return true;
  if (e && e[0] == '0') return false;
  return (p.flags & TLK_PACK_PERSISTENT) != 0;
}

int cnn_persist_enqueue(Pack& p, cudaStream_t st, int nsteps) {
  const CnnBufs& b = *static_cast<CnnBufs*>(p.scratch);
  const ModelDef& d = *p.def;
  static bool configured = false;
  if (!configured) {
    TLK_CUDA(cudaFuncSetAttribute(cnn_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM));
    configured = true;
  }
  PArgs a{};
  a.buf = b;
  a.ca = conv_args(p, b);
  const int64_t o_c1w = tensor_offset(d, 0), o_c1b = tensor_offset(d, 1);
  const int64_t o_c2w = tensor_offset(d, 2), o_c2b = tensor_offset(d, 3);
  a.opt = CnnOpt{p.lane_dev, p.stride, p.fused_lo / 4, p.fused_hi / 4, CnnOffs{o_c1w, o_c1b, o_c2w, o_c2b},
                 reinterpret_cast<float4*>(p.params), reinterpret_cast<float4*>(p.grads),
                 reinterpret_cast<float4*>(p.mom1), reinterpret_cast<float4*>(p.mom2),
                 reinterpret_cast<uint2*>(p.wbf), WtHook{p.wt, p.wt_stride, o_c2w, CONV2_W}};
  a.lanes = p.lane_dev;
  a.teacher = p.teacher;
  a.px = p.pixels;
  a.labels = p.labels;
  a.x = p.x;
  a.params = p.params;
  a.grads = p.grads;
  a.m1 = p.mom1;
  a.m2 = p.mom2;
  a.wbf = p.wbf;
  a.loss = p.loss;
  a.last_loss = p.last_loss;
  a.next = reinterpret_cast<unsigned long long*>(b.sched);  // queue head (own line), then the counters
  a.cnt = b.sched + CNT_STRIDE;
  a.pstride = p.stride;
  a.o_c1w = o_c1w;
  a.o_c1b = o_c1b;
  a.o_f1w = tensor_offset(d, 4);
  a.o_f1b = tensor_offset(d, 5);
  a.o_f2w = tensor_offset(d, 6);
  a.o_f2b = tensor_offset(d, 7);
  a.host_input = p.host_input;
  a.max_steps = p.max_steps;
  a.write_grads = (p.flags & TLK_PACK_WRITE_ALL_GRADS) ? 1 : 0;
  a.L = p.lanes;
  a.B = p.batch;
  a.nsteps = nsteps;
  a.kblocks = (p.batch + GEMM_BK - 1) / GEMM_BK;
  const int n[NPH] = {p.batch, CONV_CTAS_PER_LANE, FC1_SPLITS, HEAD_CL, 1, 9216 / GEMM_BM,
                      CONV_CTAS_PER_LANE, C2W_SPLITS, FWA_FT, p.batch, CNN_OPT_HEAVY + CNN_OPT_CTAS};
  long long per = 0;
  for (int i = 0; i < NPH; ++i) {
    a.n[i] = n[i];
    per += (long long)n[i] * p.lanes;
  }
  a.per_step = per;
  a.total = per * nsteps;
  static const bool trace = getenv("TLK_PERSIST_TRACE") && getenv("TLK_PERSIST_TRACE")[0] == '1';
  a.trace = nullptr;
  if (trace && !p.prof) {  // debug: per-item timeline of the latest launch (tlk_pack_named "persist.trace")
    static std::vector<std::pair<Pack*, void*>> bufs;
    const size_t cap = size_t(per) * 64 * 5 * 8, need = size_t(a.total) * 5 * 8;
    void* tb = nullptr;
    for (auto& pb : bufs)
      if (pb.first == &p) tb = pb.second;
    if (!tb) {
      int rc = pack_alloc(p, &tb, cap);
      if (rc) return rc;
      bufs.push_back({&p, tb});
      p.name_buf("persist.trace", tb, cap);
    }
    TLK_CHECK(need <= cap, TLK_EINVAL, "trace: at most 64 steps per launch");
    TLK_CUDA(cudaMemsetAsync(tb, 0, need, st));
    a.trace = static_cast<unsigned long long*>(tb);
  }
  static const bool probe = getenv("TLK_PERSIST_PROBE") && getenv("TLK_PERSIST_PROBE")[0] == '1';
  a.probe = nullptr;
  if (probe && !p.prof) {  // debug: timestamps inside items (tlk_pack_named "persist.probe")
    static std::vector<std::pair<Pack*, void*>> pbufs;
    const size_t cap = size_t(per) * 64 * 16 * 8;
    void* tb = nullptr;
    for (auto& pb : pbufs)
      if (pb.first == &p) tb = pb.second;
    if (!tb) {
      int rc = pack_alloc(p, &tb, cap);
      if (rc) return rc;
      pbufs.push_back({&p, tb});
      p.name_buf("persist.probe", tb, cap);
    }
    TLK_CUDA(cudaMemsetAsync(tb, 0, size_t(a.total) * 16 * 8, st));
    a.probe = static_cast<unsigned long long*>(tb);
  }
  TLK_CUDA(cudaMemsetAsync(b.sched, 0, (size_t(p.lanes) + 1) * CNT_STRIDE * 4, st));
  int dev = 0, sms = 148;
  TLK_CUDA(cudaGetDevice(&dev));
  TLK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(P_THREADS);
  cfg.dynamicSmemBytes = P_SMEM;
  cfg.stream = st;
  TLK_CUDA(cudaLaunchKernelEx(&cfg, cnn_persist_kernel, a));
  p.mark(st, "cnn_step_persistent");
  return TLK_OK;
}

}  // namespace tlk
