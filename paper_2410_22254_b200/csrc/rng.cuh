// Counter-based RNG + synthetic MNIST-shaped batches (device side).
// Bit-identical restatement target: oracle/rng.py (see its docstring for the
// exact definitions; tests/test_gpu_parity.py checks bit equality).
#pragma once
#include <cstdint>

namespace tlk {

constexpr uint64_t RNG_GAMMA = 0x9E3779B97F4A7C15ull;
constexpr uint64_t RNG_G2 = 0xD1B54A32D192ED03ull;
constexpr uint32_t STREAM_DATA = 1, STREAM_TEACHER = 2, STREAM_INIT = 16;
constexpr uint64_t TEACHER_SEED = 0x5EED7EACull;
constexpr int PIXELS = 784, WORDS_PER_SAMPLE = 98, CLASSES = 10;

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += RNG_GAMMA;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t rng_key(uint64_t seed, uint64_t stream, uint64_t step) {
  return splitmix64(splitmix64(seed + stream * RNG_G2) + step);
}
__host__ __device__ __forceinline__ uint64_t rng_bits(uint64_t key, uint64_t i) {
  return splitmix64(key + i);
}
// Uniform(-bound, bound) init value, exactly as oracle.rng.init_uniform.
__device__ __forceinline__ float init_value(uint64_t key, uint64_t e, float bound) {
  float u = __fmul_rn(float(uint32_t(rng_bits(key, e) >> 40)), 0x1p-24f);
  return __fmul_rn(__fsub_rn(__fmul_rn(u, 2.0f), 1.0f), bound);
}

}  // namespace tlk
