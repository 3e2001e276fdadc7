// Grouped tcgen05 GEMM for packed jobs: D[128 x BN] tiles accumulated in TMEM.
//
//   D[m, n] = sum_k A[m, k] * B[n, k]        (bf16 operands, fp32 accumulate)
//
// One CTA = one (job, m-tile, n-tile, k-split) work item; blockIdx.z enumerates
// jobs x k-splits, so all K co-resident jobs of a pack run in ONE launch.
//
// Operands are gathered global->shared with 16-byte cp.async chunks into the
// UMMA SWIZZLE_128B canonical layout.  A problem type `P` supplies, per chunk,
// the global address of 8 contiguous bf16 (along K for a K-major operand,
// along M/N for an MN-major one) or nullptr for zero fill.  That single hook
// expresses plain row-major operands, transposed operands (wgrad/dgrad),
// im2col gathers (conv fwd), flipped-tap gathers (conv dgrad) and padding.
//
// Pipeline (STAGES-deep ring):
//   all 128 threads: wait empty[s] -> cp.async chunks of stage s -> commit group
//   then for the oldest stage: cp.async.wait_group -> fence.proxy.async ->
//   __syncthreads -> thread 0 issues 4 x tcgen05.mma (K=16 each) and
//   tcgen05.commit -> empty[s].  After the last k-block a commit on `done`
//   releases the epilogue: each warp tcgen05.ld's its 32 TMEM lanes (rows) in
//   32-column chunks and hands them to P::epilogue.
#pragma once
#include "tma.cuh"
#include "tlk_ptx.cuh"

namespace tlk {

constexpr int GEMM_BM = 128;       // UMMA M (cta_group::1)
constexpr int GEMM_BK = 64;        // one 128-byte swizzle row of bf16
constexpr int GEMM_THREADS = 128;  // 4 warps: producers + epilogue; thread 0 issues MMA

template <int BN>
struct TmemCols {
  static constexpr uint32_t value = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
};

template <class P>
struct GemmSmem {
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr int B_BYTES = P::BN * GEMM_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BYTES = P::STAGES * STAGE_BYTES + 1024;  // + alignment slack
};

// Where chunk `i` of a ROWS x 64 (K-major) or 64 x ROWS (MN-major) stage tile
// lives in shared memory, and which (mn, k) element it starts at.
template <int ROWS, bool MN_MAJOR>
TLK_DEV void chunk_coord(int i, int& mn, int& k, uint32_t& soff) {
  if (!MN_MAJOR) {
    int r = i >> 3, c = i & 7;
    mn = r;
    k = c * 8;
    soff = sw128(r, c);
  } else {
    int atom = i >> 6, w = i & 63, kr = w >> 3, c = w & 7;
    constexpr int NB = ROWS / 64;  // 64-wide MN blocks per 8-deep K group
    int kg = atom / NB, mb = atom % NB;
    mn = mb * 64 + c * 8;
    k = kg * 8 + kr;
    soff = atom * 1024 + sw128(kr, c);
  }
}

template <int ROWS, bool MN_MAJOR>
TLK_DEV uint64_t stage_desc(uint32_t base, int kk) {
  if (!MN_MAJOR) return umma_desc_sw128(base + kk * 32, 16, 1024);
  constexpr uint32_t SBO = (ROWS / 64) * 1024;
  return umma_desc_sw128(base + kk * 2 * SBO, 1024, SBO);
}

template <class P>
struct GemmThreads {  // problems may ask for 256 threads (extra epilogue warps)
  template <class Q>
  static constexpr int get(decltype(Q::THREADS)*) { return Q::THREADS; }
  template <class Q>
  static constexpr int get(...) { return GEMM_THREADS; }
  static constexpr int value = get<P>(nullptr);
};

// Epilogue shared by both mainloops: TMEM -> registers -> problem functor
// (per-row chunks), or -> shared fp32 tile -> problem tile functor.
template <class P>
TLK_DEV void gemm_epilogue(const P& p, const typename P::Work& w, uint32_t tmem, uint8_t* smem) {
  constexpr int BN = P::BN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row = warp * 32 + lane;
  if constexpr (P::TILE_EPILOGUE) {
    static_assert(GEMM_BM * (BN + 4) * 4 <= P::STAGES * GemmSmem<P>::STAGE_BYTES, "tile fits");
    float* tile = reinterpret_cast<float*>(smem);
    if (warp < 4) {
#pragma unroll 1
      for (int cc = 0; cc < BN / 32; ++cc) {
        float v[32];
        tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + cc * 32, v);
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(tile + row * (BN + 4) + cc * 32 + i) =
              make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
    }
    __syncthreads();
    p.tile_epilogue(w, tile, BN + 4);  // may __syncthreads(): all threads call it
  } else if (warp < 4) {
    typename P::Carry carry{};
#pragma unroll 1
    for (int cc = 0; cc < BN / 32; ++cc) {
      float v[32];
      tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + cc * 32, v);
      p.epilogue(w, w.m0 + row, w.n0 + cc * 32, v, carry);
    }
    p.finish(w, w.m0 + row, carry);
  }
}

template <class P>
__global__ void __launch_bounds__(GemmThreads<P>::value, 1) tc_gemm_kernel(const P p) {
  pdl_begin();
  constexpr int NT = GemmThreads<P>::value;
  constexpr int BN = P::BN;
  constexpr int STAGES = P::STAGES;
  using S = GemmSmem<P>;
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128");
  static_assert(!P::B_MN || BN % 64 == 0, "MN-major B needs 64-wide blocks");
  constexpr uint32_t TCOLS = TmemCols<BN>::value;
  constexpr uint32_t IDESC = umma_idesc_bf16(GEMM_BM, BN, P::A_MN, P::B_MN);

  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t done_bar;
  __shared__ uint32_t tmem_base_s;

  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  typename P::Work w;
  if (!p.work(w)) return;  // uniform per CTA

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&empty_bar[s], 1);
    mbar_init(&done_bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<TCOLS>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  const int nk = w.kb_end - w.kb_begin;
  constexpr int A_CH = GEMM_BM * 8, B_CH = BN * 8;

  for (int it = 0; it < nk + STAGES - 1; ++it) {
    if (it < nk) {
      const int s = it % STAGES;
      if (it >= STAGES) mbar_wait(&empty_bar[s], ((it / STAGES) - 1) & 1);
      const int kb = w.kb_begin + it;
      const uint32_t a_s = sbase + s * S::STAGE_BYTES;
      const uint32_t b_s = a_s + S::A_BYTES;
#pragma unroll 4
      for (int i = tid; i < A_CH; i += NT) {
        int mn, k;
        uint32_t off;
        chunk_coord<GEMM_BM, P::A_MN>(i, mn, k, off);
        const void* src = p.a_src(w, w.m0 + mn, kb * GEMM_BK + k);
        cp_async16(a_s + off, src ? src : p.zero_src(), src ? 16u : 0u);
      }
#pragma unroll 4
      for (int i = tid; i < B_CH; i += NT) {
        int mn, k;
        uint32_t off;
        chunk_coord<BN, P::B_MN>(i, mn, k, off);
        const void* src = p.b_src(w, w.n0 + mn, kb * GEMM_BK + k);
        cp_async16(b_s + off, src ? src : p.zero_src(), src ? 16u : 0u);
      }
    }
    cp_async_commit();
    const int c = it - (STAGES - 1);
    if (c >= 0) {
      cp_async_wait<STAGES - 1>();
      fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const int s = c % STAGES;
        const uint32_t a_s = sbase + s * S::STAGE_BYTES;
        const uint32_t b_s = a_s + S::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < GEMM_BK / 16; ++kk) {
          mma_bf16(tmem, stage_desc<GEMM_BM, P::A_MN>(a_s, kk), stage_desc<BN, P::B_MN>(b_s, kk),
                   IDESC, (c > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&empty_bar[s]);
        if (c == nk - 1) mma_commit(&done_bar);
      }
    }
  }

  mbar_wait(&done_bar, 0);
  tc_fence_after();
  gemm_epilogue<P>(p, w, tmem, smem);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<TCOLS>(tmem);
}

// ---------------------------------------------------------------- TMA path --
// Same tiles, but operands arrive as TMA boxes (cp.async.bulk.tensor) into
// the SWIZZLE_128B layouts; warp 0 lane 0 = producer, warp 1 lane 0 = MMA
// issuer, full/empty mbarrier ring.  MN-major operands are 64-wide boxes
// stacked 8 KB apart (LBO = 8192, SBO = 1024).
template <int ROWS, bool MN_MAJOR>
TLK_DEV uint64_t stage_desc_tma(uint32_t base, int kk) {
  if (!MN_MAJOR) return umma_desc_sw128(base + kk * 32, 16, 1024);
  return umma_desc_sw128(base + kk * 2 * 1024, 8192, 1024);
}

#ifdef TLK_KTRACE
template <class P, class = void>
struct KtId {
  static constexpr int value = -1;
};
template <class P>
struct KtId<P, std::void_t<decltype(P::KT_ID)>> {
  static constexpr int value = P::KT_ID;
};
template <class P>
TLK_DEV int kt_step(const P& p) {
  if constexpr (KtId<P>::value >= 0) return p.lanes[0].steps_done;
  return 0;
}
#endif

template <class P>
__global__ void __launch_bounds__(GemmThreads<P>::value, 1)
    tc_gemm_tma_kernel(const __grid_constant__ P p) {
  constexpr int BN = P::BN;
  constexpr int STAGES = P::STAGES;
  using S = GemmSmem<P>;
  constexpr uint32_t TCOLS = TmemCols<BN>::value;
  constexpr uint32_t IDESC = umma_idesc_bf16(GEMM_BM, BN, P::A_MN, P::B_MN);
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  __shared__ __align__(8) uint64_t done_bar;
  __shared__ uint32_t tmem_base_s;
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  typename P::Work w;
  if (!p.work(w)) return;
  TLK_KT(KtId<P>::value, kt_step(p));
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<TCOLS>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_begin();  // barrier init / TMEM allocation above touch no upstream data
  TLK_KT_WAITED();
  const uint32_t tmem = tmem_base_s;
  const int nk = w.kb_end - w.kb_begin;
  if (warp == 0 && lane == 0) {  // producer
    p.prefetch();
    for (int it = 0; it < nk; ++it) {
      const int s = it % STAGES;
      if (it >= STAGES) mbar_wait(&empty_bar[s], ((it / STAGES) - 1) & 1);
      const uint32_t a_s = sbase + s * S::STAGE_BYTES;
      mbar_expect_tx(&full_bar[s], S::STAGE_BYTES);
      p.load_a(w, w.kb_begin + it, a_s, &full_bar[s]);
      p.load_b(w, w.kb_begin + it, a_s + S::A_BYTES, &full_bar[s]);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    for (int it = 0; it < nk; ++it) {
      const int s = it % STAGES;
      mbar_wait(&full_bar[s], (it / STAGES) & 1);
      tc_fence_after();
      const uint32_t a_s = sbase + s * S::STAGE_BYTES;
      const uint32_t b_s = a_s + S::A_BYTES;
#pragma unroll
      for (int kk = 0; kk < GEMM_BK / 16; ++kk)
        mma_bf16(tmem, stage_desc_tma<GEMM_BM, P::A_MN>(a_s, kk), stage_desc_tma<BN, P::B_MN>(b_s, kk),
                 IDESC, (it > 0 || kk > 0) ? 1u : 0u);
      mma_commit(&empty_bar[s]);
      if (it == nk - 1) mma_commit(&done_bar);
    }
  }
  mbar_wait(&done_bar, 0);
  tc_fence_after();
  gemm_epilogue<P>(p, w, tmem, smem);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<TCOLS>(tmem);
}

template <class P>
inline cudaError_t launch_gemm_tma(const P& p, dim3 grid, cudaStream_t stream) {
  constexpr int bytes = GemmSmem<P>::BYTES;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_tma_kernel<P>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (cudaError_t le = launch(tc_gemm_tma_kernel<P>, grid, GemmThreads<P>::value, bytes, stream, p); le != cudaSuccess) return le;
  return cudaGetLastError();
}

template <class P>
inline cudaError_t launch_gemm(const P& p, dim3 grid, cudaStream_t stream) {
  static_assert(P::BN % 32 == 0, "epilogue walks 32-column chunks");
  constexpr int bytes = GemmSmem<P>::BYTES;
  static bool configured = false;  // per template instantiation
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<P>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (cudaError_t le = launch(tc_gemm_kernel<P>, grid, GemmThreads<P>::value, bytes, stream, p); le != cudaSuccess) return le;
  return cudaGetLastError();
}

}  // namespace tlk
