"""Small numpy helpers shared by the tests (bf16 round-trips)."""
import numpy as np


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def rand_bf16(rng: np.random.Generator, shape, scale=1.0):
    bits = f32_to_bf16_bits(rng.standard_normal(shape).astype(np.float32) * scale)
    return bits, bf16_bits_to_f32(bits)
