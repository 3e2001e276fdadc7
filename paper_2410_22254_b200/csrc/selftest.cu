// Self-test entry points: the generic tcgen05 GEMM on plain operands in all
// four operand-major combinations (tests/test_gpu_gemm.py compares them with a
// torch fp32 matmul of the same bf16 inputs).
#include <cstdio>
#include <cstdlib>

#include "models.cuh"
#include "tc_gemm.cuh"
#include "tlk_common.cuh"

namespace tlk {
namespace {

template <int BN_, bool AMN, bool BMN>
struct PlainGemm {
  static constexpr int BN = BN_;
  static constexpr bool A_MN = AMN, B_MN = BMN;
  static constexpr bool TILE_EPILOGUE = false;
  static constexpr int STAGES = 4;
  struct Work {
    int j, m0, n0, kb_begin, kb_end;
  };
  const uint16_t* A;
  const uint16_t* B;
  float* C;
  int M, N, K;

  TLK_DEV bool work(Work& w) const {
    w.m0 = blockIdx.x * GEMM_BM;
    w.n0 = blockIdx.y * BN;
    w.j = blockIdx.z;
    w.kb_begin = 0;
    w.kb_end = (K + GEMM_BK - 1) / GEMM_BK;
    return true;
  }
  TLK_DEV const void* zero_src() const { return A; }
  TLK_DEV const void* a_src(const Work& w, int m, int k) const {
    if (m >= M || k >= K) return nullptr;
    return AMN ? A + (size_t(w.j) * K + k) * M + m : A + (size_t(w.j) * M + m) * K + k;
  }
  TLK_DEV const void* b_src(const Work& w, int n, int k) const {
    if (n >= N || k >= K) return nullptr;
    return BMN ? B + (size_t(w.j) * K + k) * N + n : B + (size_t(w.j) * N + n) * K + k;
  }
  struct Carry {};
  TLK_DEV void finish(const Work&, int, Carry&) const {}
  TLK_DEV void epilogue(const Work& w, int m, int n0, const float (&v)[32], Carry&) const {
    if (m >= M) return;
    float* c = C + (size_t(w.j) * M + m) * N;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (n0 + i < N) c[n0 + i] = v[i];
  }
};

template <int BN, bool AMN, bool BMN>
int run_plain(const void* A, const void* B, float* C, int batch, int M, int N, int K,
              cudaStream_t st) {
  PlainGemm<BN, AMN, BMN> p{static_cast<const uint16_t*>(A), static_cast<const uint16_t*>(B), C,
                            M, N, K};
  dim3 grid((M + GEMM_BM - 1) / GEMM_BM, (N + BN - 1) / BN, batch);
  TLK_CUDA(launch_gemm(p, grid, st));
  return TLK_OK;
}

template <int BN>
int dispatch_major(int amn, int bmn, const void* A, const void* B, float* C, int batch, int M,
                   int N, int K, cudaStream_t st) {
  if (!amn && !bmn) return run_plain<BN, false, false>(A, B, C, batch, M, N, K, st);
  if (amn && !bmn) return run_plain<BN, true, false>(A, B, C, batch, M, N, K, st);
  if constexpr (BN % 64 == 0) {
    if (!amn && bmn) return run_plain<BN, false, true>(A, B, C, batch, M, N, K, st);
    return run_plain<BN, true, true>(A, B, C, batch, M, N, K, st);
  }
  return fail(TLK_EINVAL, "MN-major B needs bn %% 64 == 0");
}

}  // namespace
}  // namespace tlk

extern "C" int tlk_selftest_gemm(int32_t a_mn, int32_t b_mn, int32_t bn, const void* A,
                                 const void* B, float* C, int32_t batch, int32_t M, int32_t N,
                                 int32_t K, void* stream) {
  using namespace tlk;
  TLK_CHECK(A && B && C && batch > 0 && M > 0 && N > 0 && K > 0, TLK_EINVAL,
            "selftest_gemm: bad arguments");
  TLK_CHECK(K % 8 == 0 && (!a_mn || M % 8 == 0) && (!b_mn || N % 8 == 0), TLK_EINVAL,
            "selftest_gemm: contiguous extents must be multiples of 8");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (bn) {
    case 32: return dispatch_major<32>(a_mn, b_mn, A, B, C, batch, M, N, K, st);
    case 64: return dispatch_major<64>(a_mn, b_mn, A, B, C, batch, M, N, K, st);
    case 128: return dispatch_major<128>(a_mn, b_mn, A, B, C, batch, M, N, K, st);
    case 256: return dispatch_major<256>(a_mn, b_mn, A, B, C, batch, M, N, K, st);
    default: return fail(TLK_EINVAL, "selftest_gemm: bn must be 32/64/128/256");
  }
}

// ------------------------------------------------ optimizer equivalence --
// opt_update_k (straight-line fast-path sqrt / div) against opt_update_ref
// (library __fsqrt_rn / __fdiv_rn) on random states whose exponents span the
// whole float range (zeros, denormals, tiny and large values, both signs):
// every output bit must agree.
namespace tlk {
namespace {
__device__ __forceinline__ uint64_t st_mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ float st_float(uint64_t h, bool nonneg) {
  const uint32_t kind = uint32_t(h >> 60);
  if (kind == 0) return 0.0f;
  const int e = int((h >> 40) % 157) - 150;  // 2^-150 .. 2^6
  float v = ldexpf(1.0f + float(h & 0xFFFFFF) * 0x1p-24f, e);
  if (!nonneg && (h & 0x1000000)) v = -v;
  return v;
}
__device__ float g_first_bad[12];
template <int KIND>
__global__ void opt_equiv_kernel(uint64_t seed, int64_t n, unsigned long long* bad) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t h0 = st_mix(seed ^ (uint64_t(i) * 4 + 0)), h1 = st_mix(seed ^ (uint64_t(i) * 4 + 1));
    const uint64_t h2 = st_mix(seed ^ (uint64_t(i) * 4 + 2)), h3 = st_mix(seed ^ (uint64_t(i) * 4 + 3));
    LaneState s{};
    s.optimizer = KIND;
    const float lrs[4] = {1e-4f, 1e-3f, 3e-3f, 2e-2f};
    s.lr = lrs[h0 & 3];
    s.beta1 = 0.9f;
    s.beta2 = (h0 & 4) ? 0.95f : 0.999f;
    s.eps = 1e-8f;
    s.wd = (h0 & 8) ? 0.01f : 0.0f;
    const int t = int((h1 >> 50) % 5000);
    s.b1t = pow(double(s.beta1), double(t));
    s.b2t = pow(double(s.beta2), double(t));
    lane_step_scalars(s);
    float p = st_float(h0, false), g = st_float(h1, false), m = st_float(h2, false), v = st_float(h3, true);
    float p2 = p, m2 = m, v2 = v;
    opt_update_k<KIND>(s, p, g, m, v);
    opt_update_ref<KIND>(s, p2, g, m2, v2);
    if (__float_as_uint(p) != __float_as_uint(p2) || __float_as_uint(m) != __float_as_uint(m2) ||
        __float_as_uint(v) != __float_as_uint(v2)) {
      if (local == 0 && atomicAdd(bad + 1, 1ull) == 0) {
        const float in[12] = {st_float(h0, false), g, st_float(h2, false), st_float(h3, true), p, m, v, p2, m2, v2,
                              s.bc2s, s.step_size};
        for (int k = 0; k < 12; ++k) g_first_bad[k] = in[k];
      }
      ++local;
    }
  }
  if (local) atomicAdd(bad, local);
}
}  // namespace
}  // namespace tlk

extern "C" int tlk_selftest_optimizer(int32_t kind, uint64_t seed, int64_t n, uint64_t* mismatches) {
  using namespace tlk;
  TLK_CHECK(mismatches && n > 0, TLK_EINVAL, "selftest_optimizer: bad arguments");
  unsigned long long* d = nullptr;
  TLK_CUDA(cudaMalloc(&d, 2 * sizeof(*d)));
  TLK_CUDA(cudaMemset(d, 0, 2 * sizeof(*d)));
  if (kind == TLK_OPT_ADAMW)
    opt_equiv_kernel<TLK_OPT_ADAMW><<<1184, 256>>>(seed, n, d);
  else if (kind == TLK_OPT_SGD)
    opt_equiv_kernel<TLK_OPT_SGD><<<1184, 256>>>(seed, n, d);
  else
    opt_equiv_kernel<TLK_OPT_ADAM><<<1184, 256>>>(seed, n, d);
  cudaError_t e = cudaGetLastError();
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  TLK_CUDA(e);
  *mismatches = h;
  if (h && getenv("TLK_SELFTEST_VERBOSE")) {
    float fb[12];
    cudaMemcpyFromSymbol(fb, g_first_bad, sizeof(fb));
    fprintf(stderr, "first mismatch: p=%a g=%a m=%a v=%a | new p=%a m=%a v=%a | ref p=%a m=%a v=%a | bc2s=%a step=%a\n",
            fb[0], fb[1], fb[2], fb[3], fb[4], fb[5], fb[6], fb[7], fb[8], fb[9], fb[10], fb[11]);
  }
  return TLK_OK;
}
