"""Fidelity estimators, XEB and the within-group sampler.

TEST INFRASTRUCTURE ONLY.  Plain numpy fp64.

  F_exact(psi, psi_hat) = |<psi|psi_hat>|^2 / (<psi|psi> <psi_hat|psi_hat>)
  F_norm(amps)         = (2^n / M) * sum_j |amp_j|^2
  F_sparse(a, a_hat)   = |sum_j a_j^* a_hat_j|^2 / (sum|a_j|^2 sum|a_hat_j|^2)
  f                    = nS / 2^s
  XEB                  = (2^n / L) sum_i P(s_i) - 1
  sampler: per group g, weights w_mu = |a_{g,mu}|^2; u = (word(key(seed,TAG_SAMPLER), g) >> 11)
           * 2^-53; draw the smallest mu whose cumulative weight exceeds u * sum(w)
           (categorical = frugal within a group).
"""
from __future__ import annotations

import numpy as np

from tn_inputs import rng


def f_exact(psi: np.ndarray, psi_hat: np.ndarray) -> float:
    num = abs(np.vdot(psi, psi_hat)) ** 2
    den = np.vdot(psi, psi).real * np.vdot(psi_hat, psi_hat).real
    if den == 0:
        raise ZeroDivisionError("zero-norm state")
    return float(num / den)


def f_norm(amps: np.ndarray, n: int) -> float:
    a = np.asarray(amps, dtype=complex)
    return float((2.0 ** n / len(a)) * np.sum(np.abs(a) ** 2))


def f_sparse(a: np.ndarray, a_hat: np.ndarray) -> float:
    a = np.asarray(a, dtype=complex)
    a_hat = np.asarray(a_hat, dtype=complex)
    return float(abs(np.vdot(a, a_hat)) ** 2 / (np.sum(np.abs(a) ** 2) * np.sum(np.abs(a_hat) ** 2)))


def linear_xeb(ideal_probs_of_samples: np.ndarray, n: int) -> float:
    p = np.asarray(ideal_probs_of_samples, dtype=float)
    return float((2.0 ** n / len(p)) * p.sum() - 1.0)


def sample_groups(amps: np.ndarray, l: int, seed: int) -> np.ndarray:
    """Index j (into the M requested bitstrings) of the one sample drawn per group."""
    a = np.asarray(amps)
    M = len(a)
    L = M // l
    k = rng.key(seed, rng.TAG_SAMPLER)
    out = np.zeros(L, dtype=np.int64)
    for g in range(L):
        z = a[g * l:(g + 1) * l].astype(complex)
        w = z.real * z.real + z.imag * z.imag  # fp64, re^2 + im^2 (no hypot), same as the product
        tot = 0.0
        for x in w:
            tot += float(x)
        if tot == 0.0:
            raise ZeroDivisionError(f"all-zero group {g}")
        u = (rng.word(k, g) >> 11) * (1.0 / (1 << 53))
        thr = u * tot
        c = 0.0
        pick = l - 1
        for mu in range(l):
            c += float(w[mu])
            if c > thr:
                pick = mu
                break
        out[g] = g * l + pick
    return out
