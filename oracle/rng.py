"""Counter-based RNG and synthetic MNIST-shaped data (oracle restatement).

Bit-identical with ``paper_2410_22254_b200/csrc/rng.cuh`` (checked by
``tests/test_gpu_parity.py::test_datagen_bit_exact``).  The reference has no
data path (its tasks are opaque argv, executor.py:199); SURVEY.md §7 step 3
asks for counter-based synthetic data shared bit-exactly by CPU and GPU.

    splitmix64(z):  z += 0x9E3779B97F4A7C15
                    z  = (z ^ z>>30) * 0xBF58476D1CE4E5B9
                    z  = (z ^ z>>27) * 0x94D049BB133111EB
                    return z ^ z>>31
    key(seed, stream, step) = splitmix64(splitmix64(seed + stream*G2) + step)
    bits(key, i)            = splitmix64(key + i)

Pixels: sample s of step t uses words bits(key(seed, DATA, t), s*98 + q),
q = 0..97; pixel i = byte (i % 8) of word i // 8 (little-endian), value k/256.
Labels: argmax_c sum_i T[c,i] * (2 k_i - 255) (exact int32; first max wins)
with a fixed global int4 teacher T[10,784] = ((bits(key(TEACHER_SEED,
TEACHER, 0), c*784+i) >> 60) & 15) - 8.
Init: tensor t of a job: w = (2u - 1) * f32(1/sqrt(fan_in)),
u = (bits(key(seed, INIT+t, 0), e) >> 40) * 2^-24.
"""

from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
G2 = 0xD1B54A32D192ED03
STREAM_DATA = 1
STREAM_TEACHER = 2
STREAM_INIT = 16
TEACHER_SEED = 0x5EED7EAC
PIXELS = 784
WORDS_PER_SAMPLE = PIXELS // 8
CLASSES = 10


def splitmix64_int(z: int) -> int:
    z = (z + GAMMA) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def key(seed: int, stream: int, step: int) -> int:
    inner = splitmix64_int((seed + stream * G2) & M64)
    return splitmix64_int((inner + step) & M64)


def splitmix64_np(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z += np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def bits(k: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        return splitmix64_np(np.uint64(k) + idx.astype(np.uint64))


_TEACHER = None


def teacher() -> np.ndarray:
    """int32 [10, 784] in [-8, 7]."""
    global _TEACHER
    if _TEACHER is None:
        w = bits(key(TEACHER_SEED, STREAM_TEACHER, 0), np.arange(CLASSES * PIXELS))
        _TEACHER = (((w >> np.uint64(60)) & np.uint64(15)).astype(np.int32) - 8).reshape(
            CLASSES, PIXELS
        )
    return _TEACHER


def pixels(seed: int, step: int, batch: int) -> np.ndarray:
    """uint8 [batch, 784] raw pixel codes k (value = k / 256)."""
    words = bits(key(seed, STREAM_DATA, step), np.arange(batch * WORDS_PER_SAMPLE))
    return words.view(np.uint8).reshape(batch, PIXELS).copy()  # little-endian bytes


def labels_for(px: np.ndarray) -> np.ndarray:
    """int32 [batch] teacher labels of uint8 pixel codes."""
    centered = 2 * px.astype(np.int32) - 255
    scores = centered @ teacher().T  # exact int32 arithmetic
    return np.argmax(scores, axis=1).astype(np.int32)


def batch(seed: int, step: int, n: int):
    px = pixels(seed, step, n)
    return px, labels_for(px)


def init_uniform(seed: int, tensor_index: int, count: int, fan_in: int) -> np.ndarray:
    bound = np.float32(1.0 / np.sqrt(np.float64(fan_in)))
    h = bits(key(seed, STREAM_INIT + tensor_index, 0), np.arange(count))
    u = (h >> np.uint64(40)).astype(np.float32) * np.float32(2.0**-24)
    return (u * np.float32(2.0) - np.float32(1.0)) * bound
