"""Sparse-state bookkeeping recomputed independently.

TEST INFRASTRUCTURE ONLY.  PAPER.md L202-L210 (Supplement, the 3-qubit worked example):
"when contracting two tensors involving qubits at the final state, one should always refer
to the target bitstrings and find out which entries of the merged dimension are required".

For a tensor whose fixed final qubits are Q (ascending ids) the required entries are the
DISTINCT projections of the requested bitstrings onto Q, packed with the lowest qubit id as
the most significant bit and sorted ascending.  A parent map sends each
row of the merged tensor to the row of an operand that holds its projection.
Written with numpy.unique only.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np


def project(bitstrings: np.ndarray, n: int, Q: Sequence[int]) -> np.ndarray:
    """Packed projection onto Q (lowest qubit id -> MSB)."""
    b = np.asarray(bitstrings, dtype=np.uint64)
    key = np.zeros(len(b), dtype=np.uint64)
    for q in sorted(Q):
        key = (key << np.uint64(1)) | ((b >> np.uint64(n - 1 - q)) & np.uint64(1))
    return key


def rows(bitstrings: np.ndarray, n: int, Q: Sequence[int]) -> np.ndarray:
    """Sorted distinct projections onto Q (the rows actually computed)."""
    return np.unique(project(bitstrings, n, Q))


def parent_map(bitstrings: np.ndarray, n: int, Q_child: Sequence[int], Q_parent: Sequence[int]) -> np.ndarray:
    """For each row of the merged tensor (fixed set Q_child, a superset of Q_parent), the index
    of the parent's row holding the same projection onto Q_parent."""
    if not set(Q_parent) <= set(Q_child):
        raise ValueError("parent set must be a subset")
    child_rows = rows(bitstrings, n, Q_child)
    # unpack child rows to full-width bitstrings, then re-project
    Qc = sorted(Q_child)
    full = np.zeros(len(child_rows), dtype=np.uint64)
    for i, q in enumerate(Qc):
        bit = (child_rows >> np.uint64(len(Qc) - 1 - i)) & np.uint64(1)
        full |= bit << np.uint64(n - 1 - q)
    pk = project(full, n, Q_parent)
    prows = rows(bitstrings, n, Q_parent)
    idx = np.searchsorted(prows, pk)
    assert np.all(prows[idx] == pk)
    return idx.astype(np.int32)


def readout_rows(bitstrings: np.ndarray, n: int, fixed_qubits: Sequence[int]) -> np.ndarray:
    """Row of the final tensor that holds each requested bitstring."""
    r = rows(bitstrings, n, fixed_qubits)
    return np.searchsorted(r, project(bitstrings, n, fixed_qubits)).astype(np.int32)
