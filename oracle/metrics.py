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

Validation suite:
  Metropolis  : per group a uniform-proposal chain over the l indices ("a Markov chain ...
                using the Metropolis algorithm"); the move x -> y is taken when u * w(x) < w(y), i.e. with
                probability min(1, w(y)/w(x)); the sample is the chain state after `steps` steps.  Random
                words: u_c = (word(key(seed, TAG_METROPOLIS), c) >> 11) * 2^-53, c = g*(2*steps+1) + t; start
                floor(u_{c0} * l), proposal t floor(u_{c0+2t-1} * l), acceptance u_{c0+2t}.
  log-XEB     : <ln(2^n P(s_i))> + gamma_Euler (PAPER.md L393 cites it; definition of the cited experiment,
                SPEC.md L539 ledger)
  entropies   : H_samples = -<ln phat(s_i)>, H_state = -(2^n/M) sum_j phat_j ln phat_j, with
                phat_j = |a_j|^2 / F_norm
  Porter-Thomas: Kolmogorov-Smirnov distance of {2^n phat_j} to Exp(1)
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


EULER_GAMMA = 0.57721566490153286061


def metropolis_groups(amps: np.ndarray, l: int, seed: int, steps: int) -> np.ndarray:
    """Index j of the one sample per group drawn by the uniform-proposal Metropolis chain (see header);
    vectorised over groups, one chain step at a time."""
    a = np.asarray(amps).astype(complex)
    w = (a.real * a.real + a.imag * a.imag).reshape(-1, l)   # fp64 weights per group
    L = w.shape[0]
    k = rng.key(seed, rng.TAG_METROPOLIS)
    c0 = np.arange(L, dtype=np.uint64) * np.uint64(2 * steps + 1)

    def u(c):
        return (rng.words_np(k, c) >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))

    rows = np.arange(L)
    x = np.minimum((u(c0) * l).astype(np.int64), l - 1)
    for t in range(1, steps + 1):
        y = np.minimum((u(c0 + np.uint64(2 * t - 1)) * l).astype(np.int64), l - 1)
        move = u(c0 + np.uint64(2 * t)) * w[rows, x] < w[rows, y]
        x = np.where(move, y, x)
    return rows * l + x


def log_xeb(ideal_probs_of_samples: np.ndarray, n: int) -> float:
    p = np.asarray(ideal_probs_of_samples, dtype=float)
    return float(np.mean(np.log((2.0 ** n) * p)) + EULER_GAMMA)


def phat(amps: np.ndarray, n: int) -> np.ndarray:
    """|a_j|^2 / F_norm: the approximate distribution over all 2^n bitstrings, normalised by the paper's
    estimate (2^n/M) sum |a|^2."""
    a = np.asarray(amps).astype(complex)
    w = a.real * a.real + a.imag * a.imag
    return w / ((2.0 ** n / len(a)) * w.sum())


def entropy_samples(phat_of_samples: np.ndarray) -> float:
    return float(-np.mean(np.log(np.asarray(phat_of_samples, dtype=float))))


def entropy_state(phat_all: np.ndarray, n: int) -> float:
    p = np.asarray(phat_all, dtype=float)
    nz = p[p > 0]
    return float(-(2.0 ** n / len(p)) * np.sum(nz * np.log(nz)))


def porter_thomas_ks(x: np.ndarray) -> float:
    """KS distance between the empirical distribution of x (= 2^n p) and Exp(1)."""
    xs = np.sort(np.asarray(x, dtype=float))
    m = len(xs)
    F = -np.expm1(-xs)
    i = np.arange(m)
    return float(max(np.max((i + 1) / m - F), np.max(F - i / m)))
