// Host side of the TMA tensor maps (see tma.cuh).
#include <mutex>

#include "tma.cuh"

namespace tlk {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int make_tmap_bf16_3d(CUtensorMap* out, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                      uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1) {
  EncodeTiledFn fn = encode_fn();
  TLK_CHECK(fn, TLK_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  const cuuint32_t box[3] = {b0, b1, 1};
  const cuuint32_t estride[3] = {1, 1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TLK_CHECK(r == CUDA_SUCCESS, TLK_ECUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return TLK_OK;
}

int make_tmap_bf16_5d(CUtensorMap* out, const void* base, const uint64_t dims[5],
                      const uint64_t strides_bytes[4], uint32_t b0, uint32_t b1, uint32_t b2,
                      uint32_t b3) {
  EncodeTiledFn fn = encode_fn();
  TLK_CHECK(fn, TLK_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t d[5], st[4];
  for (int i = 0; i < 5; ++i) d[i] = dims[i] ? dims[i] : 1;
  for (int i = 0; i < 4; ++i) {
    st[i] = strides_bytes[i];
    if (d[i + 1] == 1 || st[i] == 0) st[i] = 16;  // never stepped: any legal stride
    TLK_CHECK(st[i] % 16 == 0 && st[i] < (uint64_t(1) << 40), TLK_EINVAL,
              "tensor map stride %llu of dim %d not a multiple of 16 bytes",
              (unsigned long long)st[i], i + 1);
  }
  TLK_CHECK(reinterpret_cast<uintptr_t>(base) % 16 == 0, TLK_EINVAL, "tensor map base not 16-byte aligned");
  const cuuint32_t box[5] = {b0, b1, b2, b3, 1};
  const cuuint32_t estride[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), d, st, box,
                  estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TLK_CHECK(r == CUDA_SUCCESS, TLK_ECUDA, "cuTensorMapEncodeTiled (5d) failed (%d)", int(r));
  return TLK_OK;
}

int make_tmap_5d(CUtensorMap* out, CUtensorMapDataType dt, const void* base, const uint64_t dims[5],
                 const uint64_t strides_bytes[4], uint32_t b0, uint32_t b1, CUtensorMapSwizzle sw) {
  EncodeTiledFn fn = encode_fn();
  TLK_CHECK(fn, TLK_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t d[5], st[4];
  for (int i = 0; i < 5; ++i) d[i] = dims[i] ? dims[i] : 1;
  for (int i = 0; i < 4; ++i) {
    st[i] = strides_bytes[i];
    if (d[i + 1] == 1 || st[i] == 0) st[i] = 16;  // never stepped: any legal stride
    TLK_CHECK(st[i] % 16 == 0 && st[i] < (uint64_t(1) << 40), TLK_EINVAL,
              "tensor map stride %llu of dim %d not a multiple of 16 bytes", (unsigned long long)st[i], i + 1);
  }
  TLK_CHECK(reinterpret_cast<uintptr_t>(base) % 16 == 0, TLK_EINVAL, "tensor map base not 16-byte aligned");
  const cuuint32_t box[5] = {b0, b1, 1, 1, 1};
  const cuuint32_t estride[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(out, dt, 5, const_cast<void*>(base), d, st, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TLK_CHECK(r == CUDA_SUCCESS, TLK_ECUDA, "cuTensorMapEncodeTiled (5d, dt %d) failed (%d)", int(dt), int(r));
  return TLK_OK;
}

int make_tmap_3d(CUtensorMap* out, CUtensorMapDataType dt, const void* base, uint64_t d0, uint64_t d1,
                 uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1,
                 CUtensorMapSwizzle sw) {
  EncodeTiledFn fn = encode_fn();
  TLK_CHECK(fn, TLK_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  TLK_CHECK(reinterpret_cast<uintptr_t>(base) % 16 == 0 && stride1_bytes % 16 == 0 && stride2_bytes % 16 == 0,
            TLK_EINVAL, "tensor map base/strides not 16-byte aligned");
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  const cuuint32_t box[3] = {b0, b1, 1};
  const cuuint32_t estride[3] = {1, 1, 1};
  CUresult r = fn(out, dt, 3, const_cast<void*>(base), dims, strides, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TLK_CHECK(r == CUDA_SUCCESS, TLK_ECUDA, "cuTensorMapEncodeTiled (3d) failed (%d)", int(r));
  return TLK_OK;
}

}  // namespace tlk
