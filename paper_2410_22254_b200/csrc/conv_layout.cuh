// P28 activation layout + conv2 weight-operand layouts (shared by the conv
// kernels in conv_tc.cuh and the optimizer's weight-shadow hook).
//
// Gather-free 3x3 convolutions on tcgen05 for the MNIST-CNN pack.
//
// Layout "P28": every per-image activation lives on a 28x28 position grid
// with a zero border, channels split into 8-wide chunks stored as planes:
//   buf[lane][chunk][32 + b*784 + r*28 + c][8]  (bf16, 16 B per position)
// (32 leading / 64 trailing pad positions per plane).  h1 (conv1 output,
// 26x26) sits at (r, c) = (ih+1, iw+1); dz2 (conv2 output grad, 24x24) and
// the conv2 output rows sit at (oh+2, ow+2).  With that placement every tap
// (kh, kw) of every conv2 GEMM is a CONSTANT position offset:
//   fwd / wgrad:  h1 position  = z2 position + (kh-1)*28 + (kw-1)
//   dgrad:        dz2 position = h1 position + (1-kh)*28 + (1-kw)
// so a tile's input patch is staged ONCE per CTA with TMA bulk copies (one
// contiguous range per chunk plane) and each tap's A (or B) operand is the
// same shared-memory patch with the UMMA descriptor start moved by
// offset*16 B (SWIZZLE_NONE canonical layout: a position is one 16-B core-
// matrix row; consecutive positions are consecutive rows).  No im2col, no
// per-element address math, no re-fetch of the 9 overlapping windows.
#pragma once
#include <cstdint>

namespace tlk {

constexpr int P28 = 28;
constexpr int P28_IMG = 784;
constexpr int P28_FRONT = 32;  // pad positions before image 0
constexpr int P28_BACK = 64;   // pad positions after the last image
constexpr int HALO = 29;       // max |tap offset| = 28 + 1
constexpr int PATCH = 128 + 2 * HALO;  // 186 positions staged per 128-row tile
constexpr int PATCH_BYTES = PATCH * 16;  // 2976

__host__ __device__ constexpr int64_t p28_npos(int batch) {
  return P28_FRONT + int64_t(batch) * P28_IMG + P28_BACK;
}
__host__ __device__ constexpr int tap_off_fwd(int t) { return (t / 3 - 1) * P28 + (t % 3 - 1); }
__host__ __device__ constexpr int tap_off_dgrad(int t) { return (1 - t / 3) * P28 + (1 - t % 3); }

// Weight shadows written by the optimizer (one bf16 copy each, per lane):
//   wf[tap][ic_chunk 4][oc 64][8 ic]  : conv2 fwd B operand, K-major
//   wd[tap][oc_chunk 8][ic 32][8 oc]  : conv2 dgrad B operand, K-major
constexpr int CONV2_W = 64 * 288;
__host__ __device__ constexpr int wf_index(int oc, int tap, int ic) {
  return ((tap * 4 + (ic >> 3)) * 64 + oc) * 8 + (ic & 7);
}
__host__ __device__ constexpr int wd_index(int oc, int tap, int ic) {
  return CONV2_W + ((tap * 8 + (oc >> 3)) * 32 + ic) * 8 + (oc & 7);
}


// Optimizer hook: refresh the transposed conv2.w copies wherever the bf16
// shadow of an element is written (kernels.cu optimizer, cnn.cu cnn_opt).
struct WtHook {
  uint16_t* wt;
  int64_t wt_stride;
  int64_t off;    // start of the source tensor in the arena
  int64_t count;  // its element count
};
__device__ __forceinline__ void wt_write(const WtHook& h, int lane, int64_t e, uint16_t b) {
  if (!h.wt) return;
  int64_t r = e - h.off;
  if (r < 0 || r >= h.count) return;
  const int oc = int(r / 288), t = int(r % 288), tap = t >> 5, ic = t & 31;
  uint16_t* w = h.wt + lane * h.wt_stride;
  w[wf_index(oc, tap, ic)] = b;  // conv2 fwd B operand
  w[wd_index(oc, tap, ic)] = b;  // conv2 dgrad B operand
}
}  // namespace tlk
