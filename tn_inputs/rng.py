"""Counter-based 64-bit generator shared by every seeded input.

This module holds NO arithmetic of the method: it only turns (seed, tag, counter)
into pseudo-random 64-bit words.  Both the product path (tests/bench feed its
outputs to the C ABI) and the oracle consume these inputs; neither side
re-implements them.

    key(seed, tag)          = mix64(seed ^ (tag * 0xD1B54A32D192ED03))
    word(key, i)            = mix64(key + (i + 1) * 0x9E3779B97F4A7C15)
    uniform01(key, i)       = (word(key, i) >> 11) * 2^-53          in [0, 1)

mix64 is the splitmix64 finaliser.  All arithmetic is mod 2^64.
"""
from __future__ import annotations

import numpy as np

MASK = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
TAGMUL = 0xD1B54A32D192ED03

# tags separating independent streams drawn from one seed
TAG_GATES = 1
TAG_FSIM = 2
TAG_BITS = 3
TAG_SAMPLER = 4
TAG_METROPOLIS = 5


def mix64(z: int) -> int:
    z &= MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def key(seed: int, tag: int) -> int:
    return mix64((seed & MASK) ^ ((tag * TAGMUL) & MASK))


def word(k: int, i: int) -> int:
    return mix64((k + ((i + 1) * GOLDEN)) & MASK)


def uniform01(k: int, i: int) -> float:
    return (word(k, i) >> 11) * (1.0 / (1 << 53))


def mix64_np(z: np.ndarray) -> np.ndarray:
    """Vectorised mix64 over a uint64 array (numpy wraps uint64 arithmetic mod 2^64)."""
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def words_np(k: int, idx: np.ndarray) -> np.ndarray:
    """word(k, i) for every i in idx (uint64 array)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = np.uint64(k) + (idx + np.uint64(1)) * np.uint64(GOLDEN)
    return mix64_np(x)
