"""bf16 round-to-nearest-even emulation on fp32 numpy arrays (oracle).

Matches ``__float2bfloat16_rn`` for finite values; results stay fp32 arrays
holding bf16-representable values.
"""

import numpy as np


def round_bf16(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    return (round_bf16(x).view(np.uint32) >> 16).astype(np.uint16)
