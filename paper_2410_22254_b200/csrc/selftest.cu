// Self-test entry points: the generic tcgen05 GEMM on plain operands in all
// four operand-major combinations (tests/test_gpu_gemm.py compares them with a
// torch fp32 matmul of the same bf16 inputs).
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
