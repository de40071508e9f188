"""Shared helpers for the parity tests (tolerances derived in DESIGN.md §Tolerances)."""
import numpy as np

# Amplitudes: relative L2 error <= 1e-4 (BASELINE.json north_star), and element by element
# |a_j - o_j| <= 1e-4 * rms(o) (complex64 storage, fp32 arithmetic with 3xTF32 products over
# O(100) pairwise steps gives ~1e-6 relative; 1e-4 leaves two orders of margin).
REL_L2 = 1e-4
ELEM = 1e-4


def rel_l2(a, o):
    a = np.asarray(a, dtype=complex)
    o = np.asarray(o, dtype=complex)
    return float(np.linalg.norm(a - o) / np.linalg.norm(o))


def assert_amps_close(a, o, rel=REL_L2, elem=ELEM):
    a = np.asarray(a, dtype=complex)
    o = np.asarray(o, dtype=complex)
    assert a.shape == o.shape
    e = rel_l2(a, o)
    assert e <= rel, f"rel L2 {e:.3e} > {rel}"
    rms = np.sqrt(np.mean(np.abs(o) ** 2))
    worst = float(np.max(np.abs(a - o)) / rms)
    assert worst <= elem, f"max |a-o|/rms {worst:.3e} > {elem}"
    return e, worst
