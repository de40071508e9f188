"""Closed-network contraction of single amplitudes (SURVEY §8(c) "53q amplitudes": recompute a few x_j for one
slice on the CPU via a closed-network contraction with an independent order).

TEST INFRASTRUCTURE ONLY.  Independent of the product: the network is written from PAPER.md L57-L60 in numpy
(one tensor per gate: Eq. (1) fSim as a 4-index tensor U[o_a, o_b, i_a, i_b], single-qubit gates as U[out,in],
<0| on every input wire, <x_q| on every output wire) and contracted pairwise with np.tensordot in a plain
greedy order (smallest result first).  A sliced wire (q, k) with value v is the projector Pi_v = |v><v| on the
segment of qubit q after its k-th gate.  fp64 complex.

    amplitude(circuit, x, {(q, k): v, ...}) = <x| U_Pi |0^n>

Pinned in tests/test_oracle.py against the state-vector oracle (sv.c) with projectors, n <= 12.
"""
from __future__ import annotations

from typing import Dict, List, Tuple

import numpy as np

from oracle.tn_brute import fsim
from tn_inputs import circuits as cc


def network(circuit: dict, x: int, fixed: Dict[Tuple[int, int], int] = None):
    """Tensors (array, labels) of the closed network for bitstring x (qubit 0 = MSB)."""
    n = circuit["n"]
    fixed = dict(fixed or {})
    seg = [0] * n                       # gates applied so far on each qubit (the wire segment index k)
    cur = [("w", q, 0) for q in range(n)]  # dangling label of each qubit's wire
    T: List[Tuple[np.ndarray, list]] = []
    for q in range(n):  # <0| inputs
        T.append((np.array([1.0, 0.0], dtype=complex), [cur[q]]))
    for g in cc.gate_list(circuit):
        qs = [g["target"]] if g["type"] == "single" else list(g["targets"])
        new = []
        for q in qs:
            seg[q] += 1
            new.append(("w", q, seg[q]))
        if g["type"] == "single":
            T.append((np.asarray(g["matrix"], dtype=complex), [new[0], cur[qs[0]]]))   # U[out][in]
        else:
            U = fsim(g["theta"], g["phi"]).reshape(2, 2, 2, 2)  # [o_a, o_b, i_a, i_b]
            T.append((U, [new[0], new[1], cur[qs[0]], cur[qs[1]]]))
        for q, lab in zip(qs, new):
            cur[q] = lab
            if (q, seg[q]) in fixed:  # Pi_v on the segment right after this gate
                e = np.zeros(2, dtype=complex)
                e[fixed[(q, seg[q])]] = 1.0
                p = ("p", q, seg[q])
                T.append((np.diag(e), [p, lab]))
                cur[q] = p
    for q in range(n):  # <x_q| outputs
        e = np.zeros(2, dtype=complex)
        e[(x >> (n - 1 - q)) & 1] = 1.0
        T.append((e, [cur[q]]))
    return T


def contract(T) -> complex:
    """Greedy pairwise contraction (np.tensordot) of a closed network to a scalar: repeatedly contract the pair
    of tensors sharing a wire that minimises size(result) - size(operands)."""
    ts = {i: (np.asarray(a), list(l)) for i, (a, l) in enumerate(T)}
    nxt = len(ts)
    while len(ts) > 1:
        where = {}
        for i, (_, labs) in ts.items():
            for lab in labs:
                where.setdefault(lab, []).append(i)
        best = None
        for lab, ij in where.items():
            if len(ij) != 2:
                continue
            i, j = ij
            (A, la), (B, lb) = ts[i], ts[j]
            sh = len(set(la).intersection(lb))
            out = len(la) + len(lb) - 2 * sh
            key = ((2.0 ** out) - A.size - B.size, out)
            if best is None or key < best[0]:
                best = (key, i, j)
        if best is None:  # disconnected pieces: multiply scalars / outer products
            i, j = sorted(ts)[:2]
        else:
            _, i, j = best
        (A, la), (B, lb) = ts.pop(i), ts.pop(j)
        sh = [x for x in la if x in lb]
        C = np.tensordot(A, B, axes=([la.index(x) for x in sh], [lb.index(x) for x in sh]))
        ts[nxt] = (C, [x for x in la if x not in sh] + [x for x in lb if x not in sh])
        nxt += 1
    (A, la), = ts.values()
    assert A.ndim == 0, la
    return complex(A)


def amplitude(circuit: dict, x: int, fixed: Dict[Tuple[int, int], int] = None) -> complex:
    return contract(network(circuit, int(x), fixed))
