// MNIST MLP 784-512-512-10 pack, batch 64: one training step in TWO launches.
//
//   mlp_step_kernel   one 4-CTA cluster per lane, CTA c owning the 128-wide
//                     slice c of every hidden layer:
//                       inputs (counter RNG / host bytes, teacher labels) ->
//                       fc1 = W1[c] x^T (tcgen05, K = 784) -> h1 slice ->
//                       h1 slices exchanged by bulk copies into every CTA's
//                       shared memory -> fc2 = W2[c] h1^T -> h2 slice ->
//                       partial logits exchanged (st.async) -> CE, dz3 (every
//                       CTA, identical) -> dz2 slice, fc3 / fc2.b / fc3.b
//                       grads, loss, step scalars -> dz2 slices exchanged ->
//                       fc2 dgrad = W2[:, c]^T dz2^T -> dz1 slice, fc1.b grad.
//                     W1 / W2 / W2^T tiles stream through one TMA ring; the
//                     exchanges complete on mbarriers (no cluster barrier
//                     between the phases).
//   mlp_wgrad_adam_kernel  dW^T tiles (M = 128 input features, N = 128
//                     outputs, K = batch, both operands MN-major TMA boxes)
//                     with the optimizer update fused into the epilogue
//                     (TMEM lane = input feature: a warp's accesses of one
//                     output row are one 128-B line); one extra CTA per lane
//                     updates the small tensors (fc1.b, fc2.b, fc3.w, fc3.b);
//                     the last CTA of a lane ends its step.
//
// Numerics are the oracle's (oracle/models.py::mlp_step, bf16 mode) and the
// 8-kernel path's (mlp.cu) except for fp32 summation order: bf16 GEMM
// operands, fp32 accumulation, h / dz stored bf16, the classifier head on the
// fp32 master fc3 weights, the IEEE-exact optimizer (models.cuh opt_update_k).
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "linear.cuh"
#include "pack.cuh"
#include "rng.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace tlk {
namespace {

constexpr int MB = 64;         // batch (UMMA N)
constexpr int MC = 4;          // CTAs per lane (cluster)
constexpr int MH = 512;        // hidden width
constexpr int MIN = 784;       // input width
constexpr int MKB1 = 13;       // fc1 k-blocks (784 -> 832, zero padded)
constexpr uint32_t KBLK = MB * 128;   // one 64-deep k-block of a 64-row operand (8 KB)
constexpr uint32_t ABLK = 128 * 128;  // one 64-deep k-block of a 128-row operand (16 KB)
constexpr int MSTAGES = 3;
constexpr int M_THREADS = 256;  // warps 0-3: TMEM quarters, 4: TMA, 5: MMA, 6-7: labels
// dynamic shared memory: X (fc1 B operand, 13 k-blocks) | H1 (8 k-blocks) | W ring
constexpr uint32_t SM_X = 0, SM_H1 = MKB1 * KBLK, SM_RING = SM_H1 + 8 * KBLK;
constexpr uint32_t M_SMEM = SM_RING + MSTAGES * ABLK + 1024;
// X is dead once fc1 has completed; it then holds DZ2 (8 k-blocks), the
// partial-logit exchange, dz3, h2^T and the fc3 weight slice
constexpr uint32_t SM_DZ2 = 0, SM_PLOG = 8 * KBLK, SM_DZ3 = SM_PLOG + MC * 640 * 4,
                   SM_HS = SM_DZ3 + MB * CLASSES * 4, SM_W3 = SM_HS + MB * 136 * 2;
static_assert(SM_W3 + 128 * 12 * 4 <= MKB1 * KBLK, "head scratch fits in X");

struct MlpArgs {
  CUtensorMap h1m, dz2m;    // h1 / dz2 [lane][64][512] bf16, box {64 units, 64 samples}: stores of
                            // this CTA's two k-blocks straight from shared memory
  CUtensorMap w1, w2, w2t;  // bf16 shadows: W1 {784, 512, lane} box {64,128}; W2 {512, 512, lane}
                            // box {64,128}; W2 as MN-major A of the dgrad, box {64, 64}
  LaneState* lanes;
  const int8_t* teacher;
  uint8_t* px;
  int32_t* labels;
  uint16_t* x;
  float* params;
  float *grads, *m1, *m2;
  uint16_t* wbf;
  int64_t stride, o_b1, o_b2, o_w3, o_b3;
  uint16_t *h1, *h2, *dz1, *dz2;  // [lane][64][512]
  float *loss, *last_loss;
  int max_steps, host_input;
  unsigned long long* trace;  // debug (TLK_MLP_TRACE=1): cluster (0, lane 0) event clocks [CTA][32]
};
#define MLP_TR(slot)                                                                     \
  do {                                                                                   \
    if (a.trace && j == 0) a.trace[c * 32 + (slot)] = clock64();                         \
  } while (0)

TLK_DEV uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// shared::cta -> shared::cluster bulk copy completing on the destination CTA's mbarrier
TLK_DEV void bulk_s2cluster(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst),
               "r"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
TLK_DEV void st_async_f32(uint32_t dst, float v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(dst),
               "r"(__float_as_uint(v)), "r"(mbar)
               : "memory");
}
TLK_DEV void fence_proxy_async_cluster() { asm volatile("fence.proxy.async.shared::cluster;" ::: "memory"); }

// mbarrier wait; -DTLK_HANG_DEBUG: bounded, reports the waiting site and traps
#ifdef TLK_HANG_DEBUG
TLK_DEV void mwait(uint64_t* bar, uint32_t parity, int tag) {
  const uint32_t addr = smem_u32(bar);
  for (long long i = 0;; ++i) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) return;
    if (i == (1ll << 24)) {
      printf("mlp2 hang: tag %d block (%d,%d) thread %d parity %u\n", tag, blockIdx.x, blockIdx.y, threadIdx.x, parity);
      return;  // debug build: give up (wrong numbers) so the kernel ends and printf flushes
    }
  }
}
#else
TLK_DEV void mwait(uint64_t* bar, uint32_t parity, int) { mbar_wait(bar, parity); }
#endif

// element (row s, k) of a 64-row K-major SW128 operand built from 8 KB k-blocks
TLK_DEV uint32_t kmaj_off(int s, int k) {
  return uint32_t(k >> 6) * KBLK + sw128(uint32_t(s), uint32_t((k & 63) >> 3)) + uint32_t(k & 7) * 2;
}

__global__ void __cluster_dims__(MC, 1, 1) __launch_bounds__(M_THREADS, 1)
    mlp_step_kernel(const __grid_constant__ MlpArgs a) {
  constexpr uint32_t IDESC = umma_idesc_bf16(128, MB, false, false);
  constexpr uint32_t IDESC_T = umma_idesc_bf16(128, MB, true, false);
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[MSTAGES], empty[MSTAGES], acc[3], x_rem, lbl_rem, h1_loc, h1_rem, dz2_loc,
      dz2_rem, plog_rem;
  __shared__ uint32_t tmem_s;
  __shared__ int32_t lbl[MB];
  __shared__ float lossb[MB];
  __shared__ float b3s[CLASSES];  // fc3.b as read before CTA 0 updates it
  cg::cluster_group cluster = cg::this_cluster();
  const int c = int(cluster.block_rank()), j = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sb = smem_u32(smem);
  pdl_begin();  // lane state and weights come from the previous step
  const bool active = a.lanes[j].active;  // uniform over the cluster
  if (!active) return;
  if (tid == 0) {
    for (int s = 0; s < MSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 3; ++i) mbar_init(&acc[i], 1);
    mbar_init(&x_rem, 1);
    mbar_init(&lbl_rem, 1);
    mbar_init(&h1_loc, 1);
    mbar_init(&h1_rem, 1);
    mbar_init(&dz2_loc, 1);
    mbar_init(&dz2_rem, 1);
    mbar_init(&plog_rem, 1);
    fence_mbar_init();
    // the bytes the three peers will deliver into this CTA
    mbar_expect_tx(&x_rem, (MC - 1) * MKB1 * 16 * 128);  // 16 sample rows of every X k-block
    mbar_expect_tx(&lbl_rem, (MC - 1) * 16 * 4);
    mbar_expect_tx(&h1_rem, (MC - 1) * 2 * KBLK);
    mbar_expect_tx(&dz2_rem, (MC - 1) * 2 * KBLK);
    mbar_expect_tx(&plog_rem, (MC - 1) * 640 * 4);
  }
  if (warp == 5) tmem_alloc<256>(&tmem_s);
  if (tid == 0) MLP_TR(0);
  const LaneState ls = a.lanes[j];
  const uint64_t key = rng_key(ls.seed, STREAM_DATA, uint64_t(ls.steps_done));
  // ---- inputs of samples [16c, 16c + 16): x (bf16 k/256) rows of fc1's
  // K-major B operand, px / x to global, teacher labels (16 threads per
  // sample, integer dp4a partials summed by shuffles: exact); then the 16
  // rows of every k-block and the labels go to the three peers
  cluster.sync();  // every CTA's mbarriers are initialised before any remote arrival
  if (tid == 0) MLP_TR(17);
  // the producer thread starts the W1 stream now (the weights do not depend on
  // the inputs): the first MSTAGES tiles land while the inputs are generated
  auto produce = [&](int it) {
    const int s = it % MSTAGES;
    if (it >= MSTAGES) mwait(&empty[s], ((it / MSTAGES) - 1) & 1, 2);
    mbar_expect_tx(&full[s], ABLK);
    const uint32_t dst = sb + SM_RING + s * ABLK;
    if (it < MKB1) {
      tma_load_3d(dst, &a.w1, it * 64, c * 128, j, &full[s]);
    } else if (it < MKB1 + 8) {
      tma_load_3d(dst, &a.w2, (it - MKB1) * 64, c * 128, j, &full[s]);
    } else {
      const int kb = it - MKB1 - 8;  // W2[kb*64 .. +64 o2][c*128 .. +128 o1], o1 contiguous
      tma_load_3d(dst, &a.w2t, c * 128, kb * 64, j, &full[s]);
      tma_load_3d(dst + 8192, &a.w2t, c * 128 + 64, kb * 64, j, &full[s]);
    }
  };
  if (tid == 128) {
    tma_prefetch_desc(&a.w1);
    tma_prefetch_desc(&a.w2);
    tma_prefetch_desc(&a.w2t);
    for (int it = 0; it < MSTAGES; ++it) produce(it);
  }
  {
    // teacher [10][784] in H1, idle until this CTA's fc1 epilogue (no peer
    // sends h1 before it has this CTA's x rows, i.e. before this phase ends)
    int8_t* tch = reinterpret_cast<int8_t*>(smem + SM_H1);
    __shared__ int tsum[CLASSES];  // sum_i t[c][i]: label score = 2 sum t p - 255 sum t (exact)
    for (int i = tid; i < CLASSES * PIXELS / 16; i += M_THREADS)
      reinterpret_cast<uint4*>(tch)[i] = reinterpret_cast<const uint4*>(a.teacher)[i];
    for (int cl = warp; cl < CLASSES; cl += M_THREADS / 32) {  // the class's teacher byte sum
      int t = 0;
      for (int i = lane; i < PIXELS / 4; i += 32) {
        int ts;
        asm("dp4a.s32.u32 %0, %1, %2, %3;" : "=r"(ts)
            : "r"(reinterpret_cast<const int*>(a.teacher + cl * PIXELS)[i]), "r"(0x01010101u), "r"(0));
        t += ts;
      }
#pragma unroll
      for (int m = 16; m; m >>= 1) t += __shfl_xor_sync(0xffffffffu, t, m);
      if (lane == 0) tsum[cl] = t;
    }
    __syncthreads();
    if (tid == 0) MLP_TR(18);
    const int sl = tid >> 4, s = c * 16 + sl, part = tid & 15;  // sample, word phase
    int accv[CLASSES];
#pragma unroll
    for (int cl = 0; cl < CLASSES; ++cl) accv[cl] = 0;
    for (int q = part; q < MKB1 * 8; q += 16) {  // 8-pixel words (>= 98: zero padding)
      uint64_t wv = 0;
      const size_t g = (size_t(j) * MB + s) * WORDS_PER_SAMPLE + q;
      if (q < WORDS_PER_SAMPLE)
        wv = a.host_input ? reinterpret_cast<const uint64_t*>(a.px)[g] : rng_bits(key, uint64_t(s) * WORDS_PER_SAMPLE + q);
      uint32_t w4[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        w4[e] = pack_bf2(float((wv >> (16 * e)) & 0xFF) * (1.0f / 256.0f),
                         float((wv >> (16 * e + 8)) & 0xFF) * (1.0f / 256.0f));
      const uint4 v4 = make_uint4(w4[0], w4[1], w4[2], w4[3]);
      *reinterpret_cast<uint4*>(smem + SM_X + (q >> 3) * KBLK + sw128(s, q & 7)) = v4;
      if (q < WORDS_PER_SAMPLE) {
        if (!a.host_input) reinterpret_cast<uint64_t*>(a.px)[g] = wv;
        reinterpret_cast<uint4*>(a.x)[g] = v4;
        if (!a.host_input) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t pw = uint32_t(wv >> (32 * h));
#pragma unroll
            for (int cl = 0; cl < CLASSES; ++cl) {
              const int tw = reinterpret_cast<const int*>(tch + cl * PIXELS)[2 * q + h];
              asm("dp4a.s32.u32 %0, %1, %2, %0;" : "+r"(accv[cl]) : "r"(tw), "r"(pw));
            }
          }
        }
      }
    }
    if (tid == 0) MLP_TR(19);
    if (!a.host_input) {
#pragma unroll
      for (int cl = 0; cl < CLASSES; ++cl)
#pragma unroll
        for (int o = 8; o; o >>= 1) accv[cl] += __shfl_xor_sync(0xffffffffu, accv[cl], o);
    }
    if (part == 0) {
      int best = 0;
      if (a.host_input) {
        best = a.labels[size_t(j) * MB + s];
      } else {
        int bestv = 0;
#pragma unroll
        for (int cl = 0; cl < CLASSES; ++cl) {
          const int v = 2 * accv[cl] - 255 * tsum[cl];
          if (cl == 0 || v > bestv) {
            best = cl;
            bestv = v;
          }
        }
        a.labels[size_t(j) * MB + s] = best;
      }
      lbl[s] = best;
      const uint32_t la = smem_u32(&lbl[s]);
      for (int pr = 1; pr < MC; ++pr) {
        const uint32_t peer = uint32_t((c + pr) % MC);
        st_async_f32(mapa(la, peer), __int_as_float(best), mapa(smem_u32(&lbl_rem), peer));
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid < MKB1) {  // k-block tid: this CTA's 16 rows (2 KB) -> every peer
      const uint32_t src = sb + SM_X + tid * KBLK + c * 16 * 128;
      for (int pr = 1; pr < MC; ++pr) {
        const uint32_t peer = uint32_t((c + pr) % MC);
        bulk_s2cluster(mapa(src, peer), src, 16 * 128, mapa(smem_u32(&x_rem), peer));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) MLP_TR(1);
  const uint32_t tmem = tmem_s;
  const float* P = a.params + j * a.stride;
  float* G = a.grads + j * a.stride;
  // the small tensors (fc1.b, fc2.b, fc3.w, fc3.b) are updated here, right
  // after their gradients (each CTA its slice) -- the step's optimizer scalars
  // computed from the lane state exactly as the head does for the lane table
  LaneState ost = ls;
  lane_step_scalars(ost);
  // N updates with every load issued before the first update (one latency)
  auto upd_n = [&](auto nc, const int64_t* e, const float* g) {  // e: offsets within the lane
    constexpr int N = decltype(nc)::value;
    float pv[N], mv[N], vv[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int64_t i = j * a.stride + e[k];
      pv[k] = a.params[i];
      mv[k] = a.m1[i];
      vv[k] = a.m2[i];
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int64_t i = j * a.stride + e[k];
      opt_update(ost, pv[k], g[k], mv[k], vv[k]);
      a.params[i] = pv[k];
      a.m1[i] = mv[k];
      a.m2[i] = vv[k];
      a.wbf[i] = f2bf(pv[k]);
    }
  };

  if (warp == 4) {  // ------------------------------------------ TMA producer
    if (lane == 0)
      for (int it = MSTAGES; it < MKB1 + 16; ++it) produce(it);
  } else if (warp == 5) {  // -------------------------------------- MMA issuer
    if (lane == 0) {
      int it = 0;
      mwait(&x_rem, 0, 14);  // the peers' sample rows of X
      auto gemm = [&](uint32_t d, uint32_t bbase, int nkb, bool amn, int ai) {
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % MSTAGES;
          mwait(&full[s], (it / MSTAGES) & 1, 3);
          if (it < 12) MLP_TR(20 + it);
          tc_fence_after();
          const uint32_t as = sb + SM_RING + s * ABLK;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = amn ? umma_desc_sw128(as + kk * 2048, 8192, 1024) : umma_desc_sw128(as + kk * 32, 16, 1024);
            mma_bf16(d, ad, umma_desc_sw128(bbase + kb * KBLK + kk * 32, 16, 1024), amn ? IDESC_T : IDESC,
                     (kb > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&acc[ai]);
      };
      gemm(tmem, sb + SM_X, MKB1, false, 0);  // fc1
      MLP_TR(2);
      mwait(&h1_loc, 0, 4);
      mwait(&h1_rem, 0, 5);
      MLP_TR(3);
      tc_fence_after();
      gemm(tmem + 64, sb + SM_H1, 8, false, 1);  // fc2
      MLP_TR(4);
      mwait(&dz2_loc, 0, 6);
      mwait(&dz2_rem, 0, 7);
      MLP_TR(5);
      tc_fence_after();
      gemm(tmem + 128, sb + SM_DZ2, 8, true, 2);  // fc2 dgrad
      MLP_TR(6);
    }
  } else if (warp >= 6) {  // (idle after the inputs phase)
  } else {  // ------------------------------- TMEM-quarter warps 0..3 (row o)
    const int q = warp, r = q * 32 + lane, o = c * 128 + r;  // r: row of the slice, o: unit
    const uint32_t tq = tmem + (uint32_t(q * 32) << 16);
    float v[MB];
    int64_t ue[CLASSES + 1];  // deferred small-tensor updates of unit o (fc3.w column, fc2.b)
    float ug[CLASSES + 1];
    // this unit's biases and fc3.w column, loaded while fc1 runs
    const float b1o = P[a.o_b1 + o], b2o = P[a.o_b2 + o];
    float w3c[CLASSES];
#pragma unroll
    for (int cl = 0; cl < CLASSES; ++cl) w3c[cl] = P[a.o_w3 + cl * MH + o];
    const float b3r = r < CLASSES ? P[a.o_b3 + r] : 0.f;
    // fc1 -> h1 = bf16(relu(acc + b1)): own H1 k-blocks (2c, 2c+1) + global
    mwait(&acc[0], 0, 8);
    if (tid == 0) MLP_TR(8);
    tc_fence_after();
    tmem_ld64(tq, v);
    {
      const float bb = b1o;
#pragma unroll
      for (int s = 0; s < MB; ++s)
        *reinterpret_cast<uint16_t*>(smem + SM_H1 + kmaj_off(s, o)) = f2bf(fmaxf(v[s] + bb, 0.0f));
    }
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (tid == 0) {  // this CTA's 16 KB of H1 -> every peer's H1 (same offset)
      MLP_TR(9);
      mbar_arrive(&h1_loc);
      const uint32_t src = sb + SM_H1 + 2 * c * KBLK;
      tma_store_3d(&a.h1m, src, 2 * c * 64, 0, j);
      tma_store_3d(&a.h1m, src + KBLK, 2 * c * 64 + 64, 0, j);
      bulk_commit();
      for (int pr = 1; pr < MC; ++pr) {
        const uint32_t peer = uint32_t((c + pr) % MC);
        bulk_s2cluster(mapa(src, peer), src, 2 * KBLK, mapa(smem_u32(&h1_rem), peer));
      }
    }
    // fc2 -> h2 = bf16(relu(acc + b2)) (registers, global, h2^T in smem)
    mwait(&acc[1], 0, 9);
    if (tid == 0) MLP_TR(10);
    tc_fence_after();
    tmem_ld64(tq + 64, v);
    {
      const float bb = b2o;

      uint16_t* hs = reinterpret_cast<uint16_t*>(smem + SM_HS);
#pragma unroll
      for (int s = 0; s < MB; ++s) {
        const uint16_t h = f2bf(fmaxf(v[s] + bb, 0.0f));
        v[s] = bf2f(h);
        hs[s * 136 + r] = h;

      }
      float* w3t = reinterpret_cast<float*>(smem + SM_W3);  // fc3.w[:, slice]^T (fp32 master), [unit][12]
      for (int cl = 0; cl < CLASSES; ++cl) w3t[r * 12 + cl] = w3c[cl];
      if (r < CLASSES) b3s[r] = b3r;
    }
    named_bar_sync(1, 128);
    // partial logits of this slice, plog[c][s * 10 + cl], in every CTA of the
    // cluster: thread (s, half) sums 64 of the 128 units for all 10 classes
    // (ten independent accumulators), the halves meet by one shuffle
    {
      const uint16_t* hs = reinterpret_cast<const uint16_t*>(smem + SM_HS);
      const float* w3t = reinterpret_cast<const float*>(smem + SM_W3);  // [unit][12]
      float* plog = reinterpret_cast<float*>(smem + SM_PLOG);
      const int s = r >> 1, half = r & 1;
      {  // h2[s][slice units half*64 .. +64] -> global: eight 16-B stores per thread
        const uint4* src = reinterpret_cast<const uint4*>(hs + s * 136 + half * 64);
        uint4* dst = reinterpret_cast<uint4*>(a.h2 + (size_t(j) * MB + s) * MH + c * 128 + half * 64);
#pragma unroll
        for (int i = 0; i < 8; ++i) dst[i] = src[i];
      }
      float acc10[CLASSES];
#pragma unroll
      for (int cl = 0; cl < CLASSES; ++cl) acc10[cl] = 0.f;
#pragma unroll 4
      for (int u = half * 64; u < half * 64 + 64; ++u) {
        const float h = bf2f(hs[s * 136 + u]);
        const float4 w0 = *reinterpret_cast<const float4*>(w3t + u * 12);
        const float4 w1 = *reinterpret_cast<const float4*>(w3t + u * 12 + 4);
        const float2 w2 = *reinterpret_cast<const float2*>(w3t + u * 12 + 8);
        acc10[0] += h * w0.x;
        acc10[1] += h * w0.y;
        acc10[2] += h * w0.z;
        acc10[3] += h * w0.w;
        acc10[4] += h * w1.x;
        acc10[5] += h * w1.y;
        acc10[6] += h * w1.z;
        acc10[7] += h * w1.w;
        acc10[8] += h * w2.x;
        acc10[9] += h * w2.y;
      }
#pragma unroll
      for (int cl = 0; cl < CLASSES; ++cl) acc10[cl] += __shfl_xor_sync(0xffffffffu, acc10[cl], 1);
      if (half == 0) {
#pragma unroll
        for (int cl = 0; cl < CLASSES; ++cl) {
          const int i = s * CLASSES + cl;
          plog[c * 640 + i] = acc10[cl];
          const uint32_t la = smem_u32(&plog[c * 640 + i]);
          for (int pr = 1; pr < MC; ++pr) {
            const uint32_t peer = uint32_t((c + pr) % MC);
            st_async_f32(mapa(la, peer), acc10[cl], mapa(smem_u32(&plog_rem), peer));
          }
        }
      }
    }
    if (tid == 0) MLP_TR(11);
    mwait(&plog_rem, 0, 10);
    mwait(&lbl_rem, 0, 15);
    if (tid == 0) MLP_TR(12);
    named_bar_sync(1, 128);  // the local partials
    // logits (ranks summed in order, + fc3.b), cross entropy, dz3 = (softmax - onehot) / B
    float* dz3 = reinterpret_cast<float*>(smem + SM_DZ3);
    if (r < MB) {
      const float* plog = reinterpret_cast<const float*>(smem + SM_PLOG);
      float l[CLASSES];
#pragma unroll
      for (int cl = 0; cl < CLASSES; ++cl) {
        float sacc = 0.f;
#pragma unroll
        for (int k = 0; k < MC; ++k) sacc += plog[k * 640 + r * CLASSES + cl];
        l[cl] = sacc + b3s[cl];
      }
      const int y = lbl[r];
      float m = l[0];
#pragma unroll
      for (int cl = 1; cl < CLASSES; ++cl) m = fmaxf(m, l[cl]);
      float e[CLASSES], ssum = 0.f;
#pragma unroll
      for (int cl = 0; cl < CLASSES; ++cl) {
        e[cl] = __expf(l[cl] - m);
        ssum += e[cl];
      }
      lossb[r] = (m + logf(ssum)) - l[y];
      const float inv = 1.0f / ssum;
#pragma unroll
      for (int cl = 0; cl < CLASSES; ++cl)
        dz3[r * CLASSES + cl] = (e[cl] * inv - (cl == y ? 1.0f : 0.0f)) * (1.0f / float(MB));
    }
    named_bar_sync(1, 128);
    // dz2 = bf16(dz3 W3[:, o] * [h2 > 0]), fc2.b / fc3.w grads of unit o: one
    // pass over the samples (dz3 rows are broadcast loads)
    {
      const float* w3t = reinterpret_cast<const float*>(smem + SM_W3);
      float w3o[CLASSES], gw[CLASSES];
#pragma unroll
      for (int cl = 0; cl < CLASSES; ++cl) {
        w3o[cl] = w3t[r * 12 + cl];
        gw[cl] = 0.f;
      }
      float db = 0.f;
#pragma unroll
      for (int s = 0; s < MB; ++s) {  // fully unrolled: v[] stays in registers
        float d[CLASSES];
#pragma unroll
        for (int cl = 0; cl < CLASSES; cl += 2) {
          const float2 t2 = *reinterpret_cast<const float2*>(dz3 + s * CLASSES + cl);
          d[cl] = t2.x;
          d[cl + 1] = t2.y;
        }
        float dh = 0.f;
#pragma unroll
        for (int cl = 0; cl < CLASSES; ++cl) {
          dh += d[cl] * w3o[cl];
          gw[cl] += d[cl] * v[s];
        }
        const uint16_t z = f2bf(v[s] > 0.0f ? dh : 0.0f);
        *reinterpret_cast<uint16_t*>(smem + SM_DZ2 + kmaj_off(s, o)) = z;
        db += bf2f(z);
      }
      G[a.o_b2 + o] = db;
#pragma unroll
      for (int cl = 0; cl < CLASSES; ++cl) G[a.o_w3 + cl * MH + o] = gw[cl];
      // fc2.b / fc3.w have been read for the last time this step (h2, logits,
      // dz2); updated below, once dz2 is on its way
#pragma unroll
      for (int cl = 0; cl < CLASSES; ++cl) {
        ue[cl] = a.o_w3 + cl * MH + o;
        ug[cl] = gw[cl];
      }
      ue[CLASSES] = a.o_b2 + o;
      ug[CLASSES] = db;
    }
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (tid == 0) {  // this CTA's 16 KB of DZ2 -> every peer
      MLP_TR(13);
      mbar_arrive(&dz2_loc);
      const uint32_t src = sb + SM_DZ2 + 2 * c * KBLK;
      tma_store_3d(&a.dz2m, src, 2 * c * 64, 0, j);
      tma_store_3d(&a.dz2m, src + KBLK, 2 * c * 64 + 64, 0, j);
      bulk_commit();
      for (int pr = 1; pr < MC; ++pr) {
        const uint32_t peer = uint32_t((c + pr) % MC);
        bulk_s2cluster(mapa(src, peer), src, 2 * KBLK, mapa(smem_u32(&dz2_rem), peer));
      }
    }
    upd_n(std::integral_constant<int, CLASSES + 1>{}, ue, ug);  // overlaps the exchange and the dgrad
    // off the critical path (dz2 is on its way): CTA 0's loss, fc3.b grad and
    // update, and this step's optimizer scalars in the lane table
    if (c == 0 && r == 0) {  // loss, fc3.b grad, this step's optimizer scalars
      float sl = 0.f;
      for (int s = 0; s < MB; ++s) sl += lossb[s];
      const float L = sl / float(MB);
      LaneState& st = a.lanes[j];
      a.loss[size_t(j) * a.max_steps + st.steps_done] = L;
      a.last_loss[j] = L;
      lane_step_scalars(st);
    }
    if (c == 0 && r >= 32 && r < 32 + CLASSES) {
      const int cl = r - 32;
      float sacc = 0.f;
      for (int s = 0; s < MB; ++s) sacc += dz3[s * CLASSES + cl];
      G[a.o_b3 + cl] = sacc;
      const int64_t e1[1] = {a.o_b3 + cl};
      const float g1[1] = {sacc};
      upd_n(std::integral_constant<int, 1>{}, e1, g1);
    }

    // fc2 dgrad -> dz1 = bf16(acc * [h1 > 0]) of input unit o, fc1.b grad
    mwait(&acc[2], 0, 11);
    if (tid == 0) MLP_TR(14);
    tc_fence_after();
    tmem_ld64(tq + 128, v);
    {
      uint16_t* zg = a.dz1 + size_t(j) * MB * MH + o;
      float db = 0.f;
#pragma unroll
      for (int s = 0; s < MB; ++s) {
        const uint16_t h = *reinterpret_cast<const uint16_t*>(smem + SM_H1 + kmaj_off(s, o));
        const uint16_t z = f2bf(bf2f(h) > 0.0f ? v[s] : 0.0f);
        zg[size_t(s) * MH] = z;
        db += bf2f(z);
      }
      G[a.o_b1 + o] = db;
      const int64_t e1[1] = {a.o_b1 + o};
      const float g1[1] = {db};
      upd_n(std::integral_constant<int, 1>{}, e1, g1);
    }
  }
  if (tid == 0) bulk_wait<0>();  // the h1 / dz2 stores have left shared memory
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc<256>(tmem);
  if (tid == 0) MLP_TR(15);
  cluster.sync();  // peers have received every copy out of this CTA's shared memory
  if (tid == 0) MLP_TR(16);
}

// ---------------------------------------------------- fused wgrad + update --
// dW^T[f][o] = sum_s act[s][f] dz[s][o] (M = 128 input features f, N = 128
// outputs o, K = batch; both operands MN-major) with the optimizer update as
// the epilogue, the CNN's fc1 wgrad + Adam design (cnn.cu) over the MLP's
// two big tensors: W1 (7 f-tiles x 8 o-tiles of 64 per lane) and W2 (4 x 8).
// Persistent; warp 0 streams the operand boxes and the tile's p, m, v in four
// [32 o][128 f] fp32 chunks into a 4-slot ring, warp 1 issues the MMA
// (accumulator double-buffered in TMEM), 16 update warps apply the update and
// store full 128-B lines.  The last of a lane's 88 x 16 update-warp tiles
// ends the lane's step.
constexpr int MW_SLOTS = 4, MW_UPD = 16;
constexpr int MW_ON = 64, MW_CH = MW_ON / 32;  // outputs per tile, 32-output chunks per tile
constexpr int MW_STAGE = 3 * 8192;             // two act boxes + one dz box (64 x 64 bf16)
constexpr int MW_CHUNK = 32 * 128 * 4;
constexpr int MW_SLOT = 3 * MW_CHUNK;
constexpr int MW_SMEM = MW_STAGE + MW_SLOTS * MW_SLOT + 1024;
constexpr int MW_THREADS = (2 + MW_UPD) * 32;
constexpr int MW_OT = MH / MW_ON;                         // o-tiles per tensor
constexpr int MW_T1 = 7 * MW_OT, MW_TPL = MW_T1 + 4 * MW_OT;  // W1 tiles, tiles per lane

struct MlpWArgs {
  CUtensorMap x, h1, dz1, dz2;           // [lane][64][width] bf16, boxes {64 units, 64 samples}
  CUtensorMap p1, q1, v1, p2, q2, v2;    // fp32 W1 / W2 params, m, v: [lane][512 o][in], box {128 f, 32 o}
  LaneState* lanes;
  float *params, *m1, *m2, *grads;
  uint16_t* wbf;
  int64_t stride, o_w1, o_w2;
  int write_grads, ntiles;
};

struct MwTile {
  int j, w1, f0, o0, in;
};
TLK_DEV MwTile mw_tile(int t) {
  MwTile r;
  r.j = t / MW_TPL;
  const int u = t % MW_TPL;
  r.w1 = u < MW_T1;
  const int v = r.w1 ? u : u - MW_T1;
  r.f0 = (v / MW_OT) * 128;
  r.o0 = (v % MW_OT) * MW_ON;
  r.in = r.w1 ? MIN : MH;
  return r;
}

__global__ void __launch_bounds__(MW_THREADS, 1) mlp_wgrad_adam_kernel(const __grid_constant__ MlpWArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t gfull, gempty, tfull[2], tempty[2], sfull[MW_SLOTS], sempty[MW_SLOTS];
  __shared__ uint32_t tmem_s;
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem), slot_base = sbase + MW_STAGE;
  const uint8_t* slot_ptr = smem + MW_STAGE;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&gfull, 1);
    mbar_init(&gempty, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], MW_UPD);
    }
    for (int s = 0; s < MW_SLOTS; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], MW_UPD);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<2 * MW_ON>(&tmem_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_begin();
  const uint32_t tmem = tmem_s;
  constexpr uint32_t IDESC = umma_idesc_bf16(128, MW_ON, true, true);

  if (warp == 0) {
    if (lane == 0) {  // producer
      int it = 0, cs = 0;
      for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
        const MwTile w = mw_tile(t);
        if (!a.lanes[w.j].active) continue;
        const bool a_hi = w.f0 + 64 < w.in;  // a wholly out-of-range box would never complete
        if (it >= 1) mwait(&gempty, (it - 1) & 1, 20);
        mbar_expect_tx(&gfull, (a_hi ? 3 : 2) * 8192);
        const CUtensorMap* am = w.w1 ? &a.x : &a.h1;
        const CUtensorMap* bm = w.w1 ? &a.dz1 : &a.dz2;
        tma_load_3d(sbase, am, w.f0, 0, w.j, &gfull);
        if (a_hi) tma_load_3d(sbase + 8192, am, w.f0 + 64, 0, w.j, &gfull);
        tma_load_3d(sbase + 16384, bm, w.o0, 0, w.j, &gfull);
        ++it;
        const CUtensorMap* tp = w.w1 ? &a.p1 : &a.p2;
        const CUtensorMap* tm = w.w1 ? &a.q1 : &a.q2;
        const CUtensorMap* tv = w.w1 ? &a.v1 : &a.v2;
        for (int c = 0; c < MW_CH; ++c, ++cs) {
          const int sl = cs % MW_SLOTS;
          if (cs >= MW_SLOTS) mwait(&sempty[sl], ((cs / MW_SLOTS) - 1) & 1, 21);
          const uint32_t d = slot_base + sl * MW_SLOT;
          mbar_expect_tx(&sfull[sl], MW_SLOT);
          tma_load_3d(d, tp, w.f0, w.o0 + 32 * c, w.j, &sfull[sl]);
          tma_load_3d(d + MW_CHUNK, tm, w.f0, w.o0 + 32 * c, w.j, &sfull[sl]);
          tma_load_3d(d + 2 * MW_CHUNK, tv, w.f0, w.o0 + 32 * c, w.j, &sfull[sl]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int it = 0, lt = 0;
      for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
        const MwTile w = mw_tile(t);
        if (!a.lanes[w.j].active) continue;
        const int acc = lt & 1;
        if (lt >= 2) mwait(&tempty[acc], ((lt >> 1) - 1) & 1, 22);
        mwait(&gfull, it & 1, 23);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16(tmem + acc * MW_ON, umma_desc_sw128(sbase + kk * 2048, 8192, 1024),
                   umma_desc_sw128(sbase + 16384 + kk * 2048, 8192, 1024), IDESC, kk > 0 ? 1u : 0u);
        mma_commit(&gempty);
        mma_commit(&tfull[acc]);
        ++it;
        ++lt;
      }
    }
  } else {  // update warps: TMEM lane quarter q = warp & 3 -> f; og = 8-output group
    const int q = warp & 3, og = (warp - 2) >> 2, fl = q * 32 + lane;
    int lt = 0, cs = 0;
    for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
      const MwTile w = mw_tile(t);
      LaneState* lsp = a.lanes + w.j;
      if (!lsp->active) continue;
      const LaneState s = *lsp;
      const int acc = lt & 1;
      const bool live = w.f0 + fl < w.in;
      mwait(&tfull[acc], (lt >> 1) & 1, 24);
      tc_fence_after();
      for (int c = 0; c < MW_CH; ++c, ++cs) {
        const int o0 = 32 * c + 8 * og;  // this thread's outputs w.o0 + o0 .. +7
        float g[8];
        tmem_ld8(tmem + acc * MW_ON + o0 + (uint32_t(q * 32) << 16), g);
        if (c == MW_CH - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        const int sl = cs % MW_SLOTS;
        mwait(&sfull[sl], (cs / MW_SLOTS) & 1, 25);
        const float* Ps = reinterpret_cast<const float*>(slot_ptr + sl * MW_SLOT);
        float pv[8], mv[8], vv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int off = (8 * og + i) * 128 + fl;  // [32 o][128 f]
          pv[i] = Ps[off];
          mv[i] = Ps[MW_CHUNK / 4 + off];
          vv[i] = Ps[MW_CHUNK / 2 + off];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[sl]);  // the slot is refillable once read
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
        if (live) {
          const int64_t e = w.j * a.stride + (w.w1 ? a.o_w1 : a.o_w2) + int64_t(w.o0 + o0) * w.in + w.f0 + fl;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            a.params[e + int64_t(i) * w.in] = pv[i];
            a.m1[e + int64_t(i) * w.in] = mv[i];
            a.m2[e + int64_t(i) * w.in] = vv[i];
            a.wbf[e + int64_t(i) * w.in] = f2bf(pv[i]);
          }
          if (a.write_grads) {
#pragma unroll
            for (int i = 0; i < 8; ++i) a.grads[e + int64_t(i) * w.in] = g[i];
          }
        }
      }
      // the last update warp of the lane's last tile ends the lane's step
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(&lsp->done_ctas, 1u);
        if (prev == MW_TPL * MW_UPD - 1) {
          __threadfence();
          lsp->done_ctas = 0;
          lane_end_step(*lsp);
        }
      }
      ++lt;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<2 * MW_ON>(tmem);
}

struct Mlp2 {
  MlpArgs k1;
  MlpWArgs k2;
};

}  // namespace

bool mlp2_enabled(const Pack& p) {
  static const char* e = getenv("TLK_MLP_V1");  // 1: the 8-kernel path for every MLP pack
  return p.batch == MB && !(e && e[0] == '1');
}

int mlp2_enqueue_step(Pack& p, cudaStream_t st, uint16_t* h1, uint16_t* h2, uint16_t* dz1, uint16_t* dz2) {
  const ModelDef& d = *p.def;
  const int L = p.lanes;
  MlpArgs k{};
  const int64_t o_w1 = tensor_offset(d, 0), o_w2 = tensor_offset(d, 2);
  int rc = make_tmap_bf16_3d(&k.w1, p.wbf + o_w1, MIN, MH, L, MIN * 2, uint64_t(p.stride) * 2, 64, 128);
  if (!rc) rc = make_tmap_bf16_3d(&k.h1m, h1, MH, MB, L, MH * 2, uint64_t(MB) * MH * 2, 64, 64);
  if (!rc) rc = make_tmap_bf16_3d(&k.dz2m, dz2, MH, MB, L, MH * 2, uint64_t(MB) * MH * 2, 64, 64);
  if (!rc) rc = make_tmap_bf16_3d(&k.w2, p.wbf + o_w2, MH, MH, L, MH * 2, uint64_t(p.stride) * 2, 64, 128);
  if (!rc) rc = make_tmap_bf16_3d(&k.w2t, p.wbf + o_w2, MH, MH, L, MH * 2, uint64_t(p.stride) * 2, 64, 64);
  if (rc) return rc;
  k.lanes = p.lane_dev;
  k.teacher = p.teacher;
  k.px = p.pixels;
  k.labels = p.labels;
  k.x = p.x;
  k.params = p.params;
  k.grads = p.grads;
  k.m1 = p.mom1;
  k.m2 = p.mom2;
  k.wbf = p.wbf;
  k.stride = p.stride;
  k.o_b1 = tensor_offset(d, 1);
  k.o_b2 = tensor_offset(d, 3);
  k.o_w3 = tensor_offset(d, 4);
  k.o_b3 = tensor_offset(d, 5);
  k.h1 = h1;
  k.h2 = h2;
  k.dz1 = dz1;
  k.dz2 = dz2;
  k.loss = p.loss;
  k.last_loss = p.last_loss;
  k.max_steps = p.max_steps;
  k.host_input = p.host_input;
  k.trace = nullptr;
  for (auto& nb : p.named)  // debug timeline buffer (mlp_setup, TLK_MLP_TRACE=1)
    if (nb.name == "mlp.trace") k.trace = static_cast<unsigned long long*>(nb.ptr);
  static bool configured = false;
  if (!configured) {
    TLK_CUDA(cudaFuncSetAttribute(mlp_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, M_SMEM));
    configured = true;
  }
  static const char* only = getenv("TLK_MLP2_ONLY");  // debug: 1 / 2 = launch only that kernel
  if (!only || only[0] != '2') {
    TLK_CUDA(launch(mlp_step_kernel, dim3(MC, L), M_THREADS, M_SMEM, st, k));
    p.mark(st, "mlp_step");
  }
  if (only && only[0] == '1') return TLK_OK;

  MlpWArgs w{};
  const uint64_t ls = uint64_t(MB) * MH * 2;
  rc = make_tmap_bf16_3d(&w.x, p.x, MIN, MB, L, MIN * 2, uint64_t(MB) * MIN * 2, 64, 64);
  if (!rc) rc = make_tmap_bf16_3d(&w.h1, h1, MH, MB, L, MH * 2, ls, 64, 64);
  if (!rc) rc = make_tmap_bf16_3d(&w.dz1, dz1, MH, MB, L, MH * 2, ls, 64, 64);
  if (!rc) rc = make_tmap_bf16_3d(&w.dz2, dz2, MH, MB, L, MH * 2, ls, 64, 64);
  const CUtensorMapDataType F32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const CUtensorMapSwizzle NS = CU_TENSOR_MAP_SWIZZLE_NONE;
  const uint64_t ps = uint64_t(p.stride) * 4;
  if (!rc) rc = make_tmap_3d(&w.p1, F32, p.params + o_w1, MIN, MH, L, MIN * 4, ps, 128, 32, NS);
  if (!rc) rc = make_tmap_3d(&w.q1, F32, p.mom1 + o_w1, MIN, MH, L, MIN * 4, ps, 128, 32, NS);
  if (!rc) rc = make_tmap_3d(&w.v1, F32, p.mom2 + o_w1, MIN, MH, L, MIN * 4, ps, 128, 32, NS);
  if (!rc) rc = make_tmap_3d(&w.p2, F32, p.params + o_w2, MH, MH, L, MH * 4, ps, 128, 32, NS);
  if (!rc) rc = make_tmap_3d(&w.q2, F32, p.mom1 + o_w2, MH, MH, L, MH * 4, ps, 128, 32, NS);
  if (!rc) rc = make_tmap_3d(&w.v2, F32, p.mom2 + o_w2, MH, MH, L, MH * 4, ps, 128, 32, NS);
  if (rc) return rc;
  w.lanes = p.lane_dev;
  w.params = p.params;
  w.grads = p.grads;
  w.m1 = p.mom1;
  w.m2 = p.mom2;
  w.wbf = p.wbf;
  w.stride = p.stride;
  w.o_w1 = o_w1;
  w.o_w2 = o_w2;
  w.write_grads = (p.flags & TLK_PACK_WRITE_ALL_GRADS) ? 1 : 0;
  w.ntiles = L * MW_TPL;
  static bool wconf = false;
  if (!wconf) {
    TLK_CUDA(cudaFuncSetAttribute(mlp_wgrad_adam_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MW_SMEM));
    wconf = true;
  }
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  TLK_CUDA(launch(mlp_wgrad_adam_kernel, dim3(std::min(w.ntiles, sms)), MW_THREADS, MW_SMEM, st, w));
  p.mark(st, "mlp_wgrad_adam");
  TLK_CUDA(cudaGetLastError());
  return TLK_OK;
}

}  // namespace tlk
