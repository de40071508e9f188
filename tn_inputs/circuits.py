"""Seeded synthetic Sycamore-style circuits (input data only).

What the paper fixes and what is our reading:
  * two-qubit gates are fSim(theta, phi) (Eq. (1)) with
    theta ~ pi/2 (L104); we draw theta ~ U(pi/2 +- 0.15), phi ~ U(pi/6 +- 0.15)
    (SPEC.md L75).  The circuit stores (theta, phi) only:
    turning them into a matrix is method arithmetic, done independently by the
    oracle (oracle/sv.c) and by the product builder (csrc/network.cpp).
  * single-qubit gates are sqrt(X), sqrt(Y), sqrt(W) written
    out explicitly as 2x2 matrices U[out][in] - they are input data, the paper
    never lists them.  First cycle: uniform over the 3; afterwards uniform over the
    2 gates differing from the previous one on that qubit.
  * layout: rectangular patches and the Sycamore grid of SURVEY App. B; coupler
    patterns A-H are cirq-style GridInteractionLayer(col_offset, vertical, stagger)
    (SURVEY App. B), stored as data.
  * a cycle = one single-qubit moment + one fSim moment (pattern letter
    sequence[c % len(sequence)]); an optional final single-qubit moment
    (default on).

Circuit dict (SPEC.md L81 schema, plus "final_layer"):
  {"n": int, "qubits": [(row, col)], "sequence": str, "cycles": int,
   "final_layer": bool,
   "moments": [[gate, ...], ...]}
  gate = {"type": "single", "target": q, "matrix": 2x2 complex nested list}
       | {"type": "fsim", "targets": [a, b], "theta": t, "phi": p}
"""
from __future__ import annotations

import cmath
import math
from typing import Dict, List, Sequence, Tuple

from . import rng

# ----------------------------------------------------------------------------
# layouts
# ----------------------------------------------------------------------------

# cirq-style Sycamore grid, '-' = no qubit, letters = qubit sites.
SYCAMORE_DIAGRAM = (
    "-----AB---",
    "----ABCD--",
    "---ABCDEF-",
    "--ABCDEFGH",
    "-ABCDEFGHI",
    "ABCDEFGHI-",
    "-CDEFGHI--",
    "--EFGHI---",
    "---GHI----",
    "----I-----",
)


def rect_layout(rows: int, cols: int) -> List[Tuple[int, int]]:
    return [(r, c) for r in range(rows) for c in range(cols)]


def sycamore_sites() -> List[Tuple[int, int]]:
    return [(r, c) for r, line in enumerate(SYCAMORE_DIAGRAM) for c, ch in enumerate(line) if ch != "-"]


def couplers(sites: Sequence[Tuple[int, int]]) -> List[Tuple[Tuple[int, int], Tuple[int, int]]]:
    s = set(sites)
    out = []
    for (r, c) in sorted(s):
        if (r, c + 1) in s:
            out.append(((r, c), (r, c + 1)))
        if (r + 1, c) in s:
            out.append(((r, c), (r + 1, c)))
    return out


def sycamore53_layout() -> List[Tuple[int, int]]:
    """54 Sycamore sites minus one degree-2 site (the first in row-major order).

    Which site Google dropped is not in PAPER.md; any choice gives
    53 qubits / 86 couplers and is irrelevant to parity."""
    sites = sycamore_sites()
    s = set(sites)

    def deg(p):
        r, c = p
        return sum((q in s) for q in ((r - 1, c), (r + 1, c), (r, c - 1), (r, c + 1)))

    drop = next(p for p in sites if deg(p) == 2)
    return [p for p in sites if p != drop]


# ----------------------------------------------------------------------------
# coupler patterns
# ----------------------------------------------------------------------------

PATTERNS: Dict[str, Tuple[int, bool, bool]] = {
    "A": (0, True, True),
    "B": (1, True, True),
    "C": (1, False, True),
    "D": (0, False, True),
    "E": (1, False, False),
    "F": (0, False, False),
    "G": (0, True, False),
    "H": (1, True, False),
}


def in_layer(pair, col_offset: int, vertical: bool, stagger: bool) -> bool:
    (r0, c0), (r1, c1) = pair
    if vertical:  # transpose coordinates for the vertical orientation
        r0, c0, r1, c1 = c0, r0, c1, r1
    if r0 != r1 or abs(c0 - c1) != 1:
        return False
    c = min(c0, c1)
    return (c + col_offset + (r0 if stagger else 0)) % 2 == 0


def pattern_couplers(layout: Sequence[Tuple[int, int]], letter: str):
    if letter not in PATTERNS:
        raise ValueError(f"unknown pattern letter {letter!r}")
    off, vert, stag = PATTERNS[letter]
    idx = {p: i for i, p in enumerate(layout)}
    pairs = []
    for a, b in couplers(layout):
        if in_layer((a, b), off, vert, stag):
            pairs.append((idx[a], idx[b]))
    return sorted(pairs)


# ----------------------------------------------------------------------------
# single-qubit gate set (input data)
# ----------------------------------------------------------------------------

_S = 1.0 / math.sqrt(2.0)
SQRT_X = [[_S, -1j * _S], [-1j * _S, _S]]
SQRT_Y = [[_S, -_S], [_S, _S]]
SQRT_W = [[_S, -cmath.exp(1j * math.pi / 4) * _S], [cmath.exp(-1j * math.pi / 4) * _S, _S]]
SINGLE_GATES = (SQRT_X, SQRT_Y, SQRT_W)
SINGLE_NAMES = ("sqrtX", "sqrtY", "sqrtW")


def generate_circuit(layout: Sequence[Tuple[int, int]], cycles: int, sequence: str, seed: int,
                     final_layer: bool = True, theta_center: float = math.pi / 2,
                     phi_center: float = math.pi / 6, jitter: float = 0.15) -> dict:
    n = len(layout)
    if n < 1 or cycles < 0:
        raise ValueError("bad circuit size")
    kg = rng.key(seed, rng.TAG_GATES)
    kf = rng.key(seed, rng.TAG_FSIM)
    gi = 0  # counter in the single-gate stream
    fi = 0  # counter in the fSim stream
    prev = [-1] * n
    moments: List[list] = []

    def single_layer():
        nonlocal gi
        m = []
        for q in range(n):
            w = rng.word(kg, gi)
            gi += 1
            if prev[q] < 0:
                choice = int(w % 3)
            else:
                others = [g for g in range(3) if g != prev[q]]
                choice = others[int(w % 2)]
            prev[q] = choice
            m.append({"type": "single", "target": q, "matrix": SINGLE_GATES[choice], "name": SINGLE_NAMES[choice]})
        moments.append(m)

    for c in range(cycles):
        single_layer()
        letter = sequence[c % len(sequence)]
        m = []
        for a, b in pattern_couplers(layout, letter):
            th = theta_center + jitter * (2.0 * rng.uniform01(kf, fi) - 1.0)
            ph = phi_center + jitter * (2.0 * rng.uniform01(kf, fi + 1) - 1.0)
            fi += 2
            m.append({"type": "fsim", "targets": [a, b], "theta": th, "phi": ph})
        moments.append(m)
    if final_layer:
        single_layer()
    return {"n": n, "qubits": [tuple(p) for p in layout], "sequence": sequence, "cycles": cycles,
            "final_layer": final_layer, "seed": seed, "moments": moments}


def gate_list(circuit: dict) -> List[dict]:
    """Gates flattened in circuit order (moment by moment)."""
    return [g for m in circuit["moments"] for g in m]


def count_fsim(circuit: dict) -> int:
    return sum(1 for g in gate_list(circuit) if g["type"] == "fsim")
