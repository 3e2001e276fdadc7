// One MNIST-shaped sample of a lane's step, produced by a whole CTA: the 784
// pixel codes (counter RNG, or the host-input buffer), their bf16 k/256 copy
// and the exact int32 teacher label (oracle/rng.py: data + teacher_label).
// Shared by the generic inputs kernel (kernels.cu) and the CNN's fused
// inputs + conv1 kernel (cnn.cu).  pix: CTA shared buffer of PIXELS bytes
// (16-byte aligned); part: NW x CLASSES ints of shared scratch.
#pragma once
#include "pack.cuh"
#include "rng.cuh"
#include "tlk_ptx.cuh"

namespace tlk {

struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct GroupSync {  // a named barrier over one thread group of a CTA
  int id, n;
  __device__ __forceinline__ void operator()() const { named_bar_sync(id, n); }
};

// NT threads (tid 0..NT-1 of the group, synchronised by `sync`) produce the sample.
template <int NT, class Sync>
__device__ __forceinline__ void sample_inputs_g(int tid, Sync sync, uint64_t seed, int step, int s, size_t row,
                                                int host_input, const int8_t* teacher, uint8_t* px,
                                                int32_t* labels, uint16_t* x, uint8_t* pix, int (*part)[CLASSES]) {
  uint64_t* px_row = reinterpret_cast<uint64_t*>(px + row * PIXELS);
  if (!host_input) {
    const uint64_t key = rng_key(seed, STREAM_DATA, uint64_t(step));
    for (int q = tid; q < WORDS_PER_SAMPLE; q += NT) {
      uint64_t h = rng_bits(key, uint64_t(s) * WORDS_PER_SAMPLE + q);
      reinterpret_cast<uint64_t*>(pix)[q] = h;
      px_row[q] = h;
    }
  } else {
    for (int q = tid; q < WORDS_PER_SAMPLE; q += NT) reinterpret_cast<uint64_t*>(pix)[q] = px_row[q];
  }
  sync();
  if (x) {
    uint4* xr = reinterpret_cast<uint4*>(x + row * PIXELS);
    for (int q = tid; q < WORDS_PER_SAMPLE; q += NT) {
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        w[i] = pack_bf2(float(pix[q * 8 + 2 * i]) * (1.0f / 256.0f), float(pix[q * 8 + 2 * i + 1]) * (1.0f / 256.0f));
      xr[q] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  if (host_input) return;
  // label = argmax_c sum_i t[c][i] (2 p_i - 255) = 2 sum t p - 255 sum t, four
  // pixels per dp4a (signed teacher bytes x unsigned pixel bytes): exact
  int acc[CLASSES];
#pragma unroll
  for (int c = 0; c < CLASSES; ++c) acc[c] = 0;
  for (int q = tid; q < PIXELS / 4; q += NT) {
    const uint32_t pw = reinterpret_cast<const uint32_t*>(pix)[q];
#pragma unroll
    for (int c = 0; c < CLASSES; ++c) {
      const int tw = reinterpret_cast<const int*>(teacher + c * PIXELS)[q];
      int tp, ts;
      asm("dp4a.s32.u32 %0, %1, %2, %3;" : "=r"(tp) : "r"(tw), "r"(pw), "r"(0));
      asm("dp4a.s32.u32 %0, %1, %2, %3;" : "=r"(ts) : "r"(tw), "r"(0x01010101u), "r"(0));
      acc[c] += 2 * tp - 255 * ts;
    }
  }
#pragma unroll
  for (int c = 0; c < CLASSES; ++c) {
    int a = acc[c];
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if ((tid & 31) == 0) part[tid >> 5][c] = a;
  }
  sync();
  if (tid == 0) {
    int best = 0, bestv = 0;
    for (int c = 0; c < CLASSES; ++c) {
      int v = 0;
      for (int w = 0; w < NT / 32; ++w) v += part[w][c];
      if (c == 0 || v > bestv) {
        best = c;
        bestv = v;
      }
    }
    labels[row] = best;
  }
}

template <int NT>
__device__ __forceinline__ void sample_inputs(uint64_t seed, int step, int s, size_t row, int host_input,
                                              const int8_t* __restrict__ teacher, uint8_t* __restrict__ px,
                                              int32_t* __restrict__ labels, uint16_t* __restrict__ x,
                                              uint8_t* pix, int (*part)[CLASSES]) {
  sample_inputs_g<NT>(int(threadIdx.x), CtaSync{}, seed, step, s, row, host_input, teacher, px, labels, x, pix,
                      part);
}

}  // namespace tlk
