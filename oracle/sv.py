"""Python wrapper of the fp64 state-vector oracle (oracle/sv.c).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares nothing with the product.

Slicing semantics (SURVEY §8(c) Definition, App. A.4): for the ordered sliced-wire list
W = (w_0 .. w_{s-1}) exported by the product's planner and a slice subset S,

    amp_S(x_j) = sum_{sigma in S, ascending} <x_j | U_sigma | 0^n>,

where U_sigma is the circuit with the projector Pi_v inserted on wire w_i,
v = (sigma >> (s-1-i)) & 1  (each choice of sliced-index values is a
"sliced copy", and their sum returns the original contraction).
Prefix shortcut: S = [0, 2^(s-j)) is Pi_0 on w_0..w_{j-1} only.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

from tn_inputs import circuits as cc

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_sv.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/sv.c with gcc (plain C, OpenMP)."""
    src = os.path.join(_HERE, "sv.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", src, "-o", _SO, "-lm"])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.POINTER
        ci, cd = ctypes.c_int, ctypes.c_double
        L.sv_run.argtypes = [ci, ci, P(ci), P(ci), P(ci), P(cd), P(cd), P(cd), ci, P(ci), P(ci), P(ci), ci, P(cd)]
        L.sv_run.restype = ci
        L.sv_run_amps.argtypes = [ci, ci, P(ci), P(ci), P(ci), P(cd), P(cd), P(cd), ci, P(ci), P(ci), P(ci), ci,
                                  ctypes.c_int64, P(ctypes.c_uint64), P(cd), P(cd)]
        L.sv_run_amps.restype = ci
        L.sv_fsim_matrix.argtypes = [cd, cd, P(cd)]
        L.sv_fsim_matrix.restype = None
        _lib = L
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def _arrays(circuit: dict):
    gates = cc.gate_list(circuit)
    G = len(gates)
    kind = np.zeros(G, np.int32)
    q0 = np.zeros(G, np.int32)
    q1 = np.full(G, -1, np.int32)
    th = np.zeros(G)
    ph = np.zeros(G)
    u = np.zeros(8 * G)
    for g, gate in enumerate(gates):
        if gate["type"] == "single":
            kind[g] = 0
            q0[g] = gate["target"]
            m = np.asarray(gate["matrix"], dtype=complex).reshape(4)
            u[8 * g:8 * g + 8:2] = m.real
            u[8 * g + 1:8 * g + 8:2] = m.imag
        else:
            kind[g] = 1
            q0[g], q1[g] = gate["targets"]
            th[g] = gate["theta"]
            ph[g] = gate["phi"]
    return G, kind, q0, q1, th, ph, u


def _ins_arrays(insertions: Sequence[Tuple[int, int, int]]):
    n = len(insertions)
    iq = np.array([t[0] for t in insertions] or [0], np.int32)
    ik = np.array([t[1] for t in insertions] or [0], np.int32)
    io = np.array([t[2] for t in insertions] or [0], np.int32)
    return n, iq, ik, io


def fsim_matrix(theta: float, phi: float) -> np.ndarray:
    out = np.zeros(32)
    lib().sv_fsim_matrix(theta, phi, _ptr(out, ctypes.c_double))
    return (out[0::2] + 1j * out[1::2]).reshape(4, 4)


def statevector(circuit: dict, insertions: Sequence[Tuple[int, int, int]] = (), threads: int = 0) -> np.ndarray:
    """Final state psi (complex128, length 2^n) with insertions (q, k, op); op 0/1 = Pi_0/Pi_1,
    2 = sigma_z, applied right after the k-th gate on qubit q."""
    n = circuit["n"]
    G, kind, q0, q1, th, ph, u = _arrays(circuit)
    ni, iq, ik, io = _ins_arrays(insertions)
    psi = np.zeros(2 << n)
    ci, cd = ctypes.c_int, ctypes.c_double
    rc = lib().sv_run(n, G, _ptr(kind, ci), _ptr(q0, ci), _ptr(q1, ci), _ptr(th, cd), _ptr(ph, cd), _ptr(u, cd),
                      ni, _ptr(iq, ci), _ptr(ik, ci), _ptr(io, ci), threads, _ptr(psi, cd))
    if rc != 0:
        raise ValueError(f"sv_run failed rc={rc}")
    return psi[0::2] + 1j * psi[1::2]


def amplitudes(circuit: dict, bitstrings: np.ndarray, insertions: Sequence[Tuple[int, int, int]] = (),
               threads: int = 0) -> Tuple[np.ndarray, float]:
    """psi(x_j) for the requested bitstrings (uint64 state indices) and ||psi||^2."""
    n = circuit["n"]
    G, kind, q0, q1, th, ph, u = _arrays(circuit)
    ni, iq, ik, io = _ins_arrays(insertions)
    idx = np.ascontiguousarray(bitstrings, dtype=np.uint64)
    out = np.zeros(2 * len(idx))
    nrm = ctypes.c_double(0.0)
    ci, cd = ctypes.c_int, ctypes.c_double
    rc = lib().sv_run_amps(n, G, _ptr(kind, ci), _ptr(q0, ci), _ptr(q1, ci), _ptr(th, cd), _ptr(ph, cd),
                           _ptr(u, cd), ni, _ptr(iq, ci), _ptr(ik, ci), _ptr(io, ci), threads,
                           len(idx), _ptr(idx, ctypes.c_uint64), _ptr(out, cd), ctypes.byref(nrm))
    if rc != 0:
        raise ValueError(f"sv_run_amps failed rc={rc}")
    return out[0::2] + 1j * out[1::2], nrm.value


def slice_values(sigma: int, s: int) -> List[int]:
    """e_i <- (sigma >> (s-1-i)) & 1 (MSB-first)."""
    return [(sigma >> (s - 1 - i)) & 1 for i in range(s)]


def slice_insertions(wires: Sequence[Tuple[int, int]], sigma: int) -> List[Tuple[int, int, int]]:
    s = len(wires)
    return [(q, k, v) for (q, k), v in zip(wires, slice_values(sigma, s))]


def hole_insertions(circuit: dict, holes: Sequence[int]) -> List[Tuple[int, int, int]]:
    """A drilled hole (Fig. 1) breaks both input edges of one fSim gate: E = (1,0)x(1,0),
    i.e. Pi_0 on each of its two qubits right before the gate (after the gates already on the wire).
    holes index the circuit's gates flattened moment by moment."""
    flat = [g for m in circuit["moments"] for g in m]
    ins = []
    for h in holes:
        g = flat[h]
        if g["type"] != "fsim":
            raise ValueError("a hole must be an fSim gate")
        for q in g["targets"]:
            before = sum(1 for x in flat[:h] if (x["target"] == q if x["type"] == "single" else q in x["targets"]))
            ins.append((q, before, 0))
    return ins


def companion_of(circuit: dict, wire: Tuple[int, int]) -> Optional[Tuple[int, int]]:
    """Companion of a sliced wire (supplement "singular values of the sliced fSim
    gate"): if wire (q, k) is the output on q of an fSim gate G (G = the k-th gate on q) on qubits (q, b),
    the companion edge is G's other input; the rank-one truncation keeps the dominant singular vector e_v,
    i.e. Pi_v on qubit b right before G: wire (b, number of gates on b before G).  None otherwise."""
    q, k = wire
    flat = [g for m in circuit["moments"] for g in m]
    seen = 0
    for h, g in enumerate(flat):
        on_q = g["target"] == q if g["type"] == "single" else q in g["targets"]
        if not on_q:
            continue
        seen += 1
        if seen == k:
            if g["type"] != "fsim":
                return None
            b = g["targets"][1] if g["targets"][0] == q else g["targets"][0]
            before = sum(1 for x in flat[:h] if (x["target"] == b if x["type"] == "single" else b in x["targets"]))
            return (b, before)
    return None


def sliced_amplitudes(circuit: dict, bitstrings: np.ndarray, wires: Sequence[Tuple[int, int]],
                      subset: Iterable[int], threads: int = 0,
                      extra: Sequence[Tuple[int, int, int]] = (),
                      companions: Sequence[Tuple[int, int, int]] = ()) -> np.ndarray:
    """amp_S(x_j) = sum over sigma in S (ascending) of <x_j|U_sigma|0> (one state-vector run per sigma);
    `extra` insertions (e.g. drilled holes) apply to every run; `companions` (q, k, i) put Pi_v on wire
    (q, k) with v the value of sliced wire i."""
    acc = np.zeros(len(bitstrings), dtype=complex)
    for sigma in sorted(set(int(x) for x in subset)):
        ins = slice_insertions(wires, sigma)
        # companions: (q, k, i) -> Pi_v on (q, k) with v the value of sliced wire i in this slice
        ins += [(cq, ck, ins[i][2]) for (cq, ck, i) in companions]
        a, _ = amplitudes(circuit, bitstrings, list(extra) + ins, threads)
        acc += a
    return acc


def prefix_amplitudes(circuit: dict, bitstrings: np.ndarray, wires: Sequence[Tuple[int, int]], j: int,
                      threads: int = 0) -> Tuple[np.ndarray, float]:
    """S = [0, 2^(s-j)): Pi_0 on w_0..w_{j-1} only."""
    ins = [(q, k, 0) for (q, k) in list(wires)[:j]]
    return amplitudes(circuit, bitstrings, ins, threads)
