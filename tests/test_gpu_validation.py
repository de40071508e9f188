"""The supplement's validation claims on a 20-qubit m=14 EFGH
circuit, through the product path: fidelity estimates coincide with the true fidelity of the approximate
state, the XEB of one sample per group follows it, the sample entropy equals the state entropy, and the
sparse state is Porter-Thomas.  Statistical checks at fixed seeds (tools/validation.py prints the full
table; profiles/r01_validation_24q.json holds the 24-qubit run)."""
import numpy as np
import pytest

from tn_inputs import bitstrings as bs
from tn_inputs import circuits as cc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import paper_2111_03011_b200 as T
    return T


def test_validation_fidelity_xeb_entropy(T):
    circ = cc.generate_circuit(cc.rect_layout(4, 5), 14, "EFGH", 7)
    n = circ["n"]
    opens = list(range(n - 6, n))
    bits = bs.generate_groups(n, opens, 8192, 8)
    ss = T.SparseState(circ, bits, bs.qubit_mask(n, opens))
    info = ss.plan(1 << 20, n_sliced=6, seed=1, trials=8, time_budget_s=300)
    s = info["s"]
    ss.bind(0, pipelines=4)
    exact = ss.contract(range(1 << s)).cpu().numpy()
    for k in range(0, s + 1, 2):  # k sliced wires pinned to 0: fraction f = 2^-k
        nS = 1 << (s - k)
        f = nS / (1 << s)
        approx = ss.contract(range(nS)).cpu().numpy()
        a, b = exact.astype(complex), approx.astype(complex)
        F = abs(np.vdot(a, b)) ** 2 / (np.vdot(a, a).real * np.vdot(b, b).real)
        xs = []
        for sampler in ("categorical", "metropolis"):
            _, _, r = ss.sample_report(approx, nS, 100 + k, sampler=sampler, steps=1000, ideal=exact)
            xs.append(r["xeb"])
            # F_norm and f estimate the fidelity of the approximate state
            assert abs(r["F_norm"] - F) < 0.1 * F + 0.003, (k, r["F_norm"], F)
            assert abs(f - F) < 0.1 * F + 0.003, (k, f, F)
            # entropy of the samples vs the distribution they came from: within 1 %
            assert abs(r["entropy_samples"] / r["entropy_state"] - 1) < 0.01
            assert r["pt_ks"] < 0.03  # Porter-Thomas
        # linear XEB of 8192 samples ~ F * l/(l+1) (finite-group bias, l = 64); 1/sqrt(L) noise
        for x in xs:
            assert abs(x - F * 64 / 65) < 0.05 * F + 0.04, (k, x, F)
    ss.close()
