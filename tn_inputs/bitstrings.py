"""Seeded sparse-state requests: L groups x l correlated bitstrings (input data only).

PAPER.md L183-L186 (Supplement "The sparse-state method"): L sub-bitstrings s1 are drawn
uniformly by flipping a coin for each bit; each s1 is concatenated with all 2^|O|
configurations s2 of the open qubits, giving L*l bitstrings.  L225: the open qubits.

Conventions: a bitstring is a uint64 with bit (n-1-q) = value of qubit q
(qubit 0 = MSB), so the value equals the state-vector index.  Within a group the open
configurations run in ascending order of the open bits packed with the lowest open qubit
id as MSB.  open_mask uses the same bit convention.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np

from . import rng


def qubit_mask(n: int, qubits: Sequence[int]) -> int:
    m = 0
    for q in qubits:
        m |= 1 << (n - 1 - q)
    return m


def generate_groups(n: int, open_qubits: Sequence[int], L: int, seed: int) -> np.ndarray:
    """Return the M = L * 2^|O| requested bitstrings (uint64), grouped."""
    open_qubits = sorted(open_qubits)
    fixed = [q for q in range(n) if q not in set(open_qubits)]
    k = rng.key(seed, rng.TAG_BITS)
    g = np.arange(L, dtype=np.uint64)
    fixed_val = np.zeros(L, dtype=np.uint64)
    for q in fixed:  # one coin per (group, qubit): counter = g * n + q
        w = rng.words_np(k, g * np.uint64(n) + np.uint64(q))
        bit = w >> np.uint64(63)
        fixed_val |= bit << np.uint64(n - 1 - q)
    l = 1 << len(open_qubits)
    opens = np.zeros(l, dtype=np.uint64)
    for mu in range(l):
        v = 0
        for i, q in enumerate(open_qubits):  # lowest open qubit id = MSB of mu
            b = (mu >> (len(open_qubits) - 1 - i)) & 1
            v |= b << (n - 1 - q)
        opens[mu] = v
    return (fixed_val[:, None] | opens[None, :]).reshape(-1)


def all_bitstrings(n: int) -> np.ndarray:
    return np.arange(1 << n, dtype=np.uint64)
