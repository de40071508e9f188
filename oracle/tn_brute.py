"""Brute-force tensor-network enumeration for tiny circuits.

TEST INFRASTRUCTURE ONLY.  Independent of oracle/sv.c: it writes Eq. (1) again in numpy
and evaluates the network of PAPER.md L57-L60 by its definition:

  amp(x) = sum over every assignment of the internal wire values of
           prod_g  U_g[outputs of g][inputs of g],

with <0| input boundaries, the output boundary fixed to the bits of x, and every sliced
wire fixed to its slice value.  Wire (q, k) = segment of qubit q after
its k-th gate; (q, 0) is the input, (q, G_q) the output.
Pure numpy over all 2^W assignments: only for W <= ~20 internal wires.
"""
from __future__ import annotations

import math
from typing import Dict, Tuple

import numpy as np

from tn_inputs import circuits as cc


def fsim(theta: float, phi: float) -> np.ndarray:
    """PAPER.md Eq. (1), L96-L102."""
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[1, 0, 0, 0],
                     [0, c, -1j * s, 0],
                     [0, -1j * s, c, 0],
                     [0, 0, 0, np.exp(-1j * phi)]], dtype=complex)


def amplitude(circuit: dict, x: int, fixed_wires: Dict[Tuple[int, int], int] = None) -> complex:
    n = circuit["n"]
    gates = cc.gate_list(circuit)
    fixed_wires = dict(fixed_wires or {})
    count = [0] * n
    ops = []  # (matrix, [(q,k_out)...], [(q,k_in)...])
    for g in gates:
        if g["type"] == "single":
            q = g["target"]
            count[q] += 1
            ops.append((np.asarray(g["matrix"], dtype=complex), [(q, count[q])], [(q, count[q] - 1)]))
        else:
            a, b = g["targets"]
            count[a] += 1
            count[b] += 1
            ops.append((fsim(g["theta"], g["phi"]), [(a, count[a]), (b, count[b])],
                        [(a, count[a] - 1), (b, count[b] - 1)]))
    value: Dict[Tuple[int, int], object] = {}
    for q in range(n):
        value[(q, 0)] = 0                                   # <0| input boundary
        value[(q, count[q])] = (x >> (n - 1 - q)) & 1       # output boundary = bits of x
    for w, v in fixed_wires.items():
        q, k = w
        if not (1 <= k < count[q]):
            raise ValueError(f"wire {w} is not internal")
        value[w] = v
    internal = [(q, k) for q in range(n) for k in range(1, count[q]) if (q, k) not in value]
    W = len(internal)
    if W > 22:
        raise ValueError("too many internal wires for brute force")
    assign = ((np.arange(1 << W)[:, None] >> np.arange(W)[None, :]) & 1) if W else np.zeros((1, 0), int)
    col = {w: i for i, w in enumerate(internal)}

    def val(w):
        if w in col:
            return assign[:, col[w]]
        return np.full(assign.shape[0], value[w])

    prod = np.ones(assign.shape[0], dtype=complex)
    for U, outs, ins in ops:
        if len(outs) == 1:
            prod *= U[val(outs[0]), val(ins[0])]
        else:
            o = 2 * val(outs[0]) + val(outs[1])
            i = 2 * val(ins[0]) + val(ins[1])
            prod *= U[o, i]
    return complex(prod.sum())


def internal_wires(circuit: dict):
    n = circuit["n"]
    count = [0] * n
    for g in cc.gate_list(circuit):
        for q in ([g["target"]] if g["type"] == "single" else g["targets"]):
            count[q] += 1
    return [(q, k) for q in range(n) for k in range(1, count[q])], count
