"""Pins for the oracle (SURVEY §8(c) "What pins each part").  CPU only.

Each test fixes the oracle to something other than itself: a value the paper prints or
that Eq. (1) gives in closed form at special angles, an invariant, a textbook dense
construction, or brute-force enumeration of the network.  A plausible mistake (a dropped
term, a sign, a transposed U[out][in], a wrong bit order, a projector on the wrong wire
segment) fails at least one of them (see the comment on each test).
"""
import math
import os

import numpy as np
import pytest

from tn_inputs import circuits as cc
from tn_inputs import bitstrings as bs
from tn_inputs import configs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def small_circuit(rows, cols, cycles, seed, seq="ABCDCDAB", final=True):
    return cc.generate_circuit(cc.rect_layout(rows, cols), cycles, seq, seed, final)


def load_golden_fsim():
    U = np.zeros((4, 4), complex)
    for line in open(os.path.join(GOLD, "fsim_theta_pi2_phi_pi6.txt")):
        if line.startswith("#") or not line.strip():
            continue
        r, c, re, im = line.split()
        U[int(r), int(c)] = float(re) + 1j * float(im)
    return U


# --------------------------------------------------------------------------- gates

def test_fsim_special_angles(oracle_built):
    """Eq. (1) at theta=pi/2, phi=pi/6 (golden, worked by hand) and fSim(0,0) = I.
    Catches a wrong sign of -i sin, a swapped e^{-i phi} conjugation, misplaced entries."""
    from oracle import sv
    np.testing.assert_allclose(sv.fsim_matrix(math.pi / 2, math.pi / 6), load_golden_fsim(), atol=1e-15)
    np.testing.assert_allclose(sv.fsim_matrix(0.0, 0.0), np.eye(4), atol=1e-15)


def test_fsim_unitary(oracle_built):
    from oracle import sv
    r = np.random.default_rng(1)
    for _ in range(50):
        U = sv.fsim_matrix(*r.uniform(-3, 3, 2))
        assert np.abs(U.conj().T @ U - np.eye(4)).max() < 1e-12


def test_pinned_fsim_singular_values(oracle_built):
    """pinning one input of fSim gives squared singular values
    {1+sin^2 t, cos^2 t}; at t = pi/3 these are {1.75, 0.25} (golden).  All four pinning cases.
    Pins the magnitudes and positions of the cos/sin entries of the oracle's Eq. (1)."""
    from oracle import sv
    vals = open(os.path.join(GOLD, "pinned_fsim_singular_values.txt")).read().split("squared_singular_values")[1].split()
    want = sorted(map(float, vals), reverse=True)
    for theta, phi, expect in [(math.pi / 3, 0.7, want)] + [
            (t, p, [1 + math.sin(t) ** 2, math.cos(t) ** 2]) for t, p in np.random.default_rng(2).uniform(0, 3, (20, 2))]:
        U = sv.fsim_matrix(theta, phi)          # U[out=(oa,ob)][in=(ia,ib)]
        T = U.reshape(2, 2, 2, 2)               # [oa, ob, ia, ib]
        for which in ("ia", "ib"):
            for v in (0, 1):
                E = T[:, :, v, :] if which == "ia" else T[:, :, :, v]   # [oa, ob, other_in]
                # L323/L333: group (pinned input, other input, one output) against the companion
                # output omega, which is the output of the OTHER qubit (ob when ia is pinned,
                # oa after "swapping the third and the fourth dimension" when ib is pinned)
                comp = 1 if which == "ia" else 0
                F = np.moveaxis(E, comp, -1).reshape(4, 2)
                s2 = np.sort(np.linalg.svd(F, compute_uv=False) ** 2)[::-1]
                np.testing.assert_allclose(s2, sorted(expect, reverse=True), atol=1e-12)


# --------------------------------------------------------------------------- state vector

def kron_reference(circuit):
    """Textbook construction (n <= 6): each gate as a full 2^n x 2^n matrix, psi = prod M_g e_0.
    Uses tn_brute's independent Eq. (1).  Qubit 0 = MSB; U[out][in]; fSim local index 2*x_a+x_b."""
    from oracle.tn_brute import fsim
    n = circuit["n"]
    N = 1 << n
    psi = np.zeros(N, complex)
    psi[0] = 1
    for g in cc.gate_list(circuit):
        M = np.zeros((N, N), complex)
        if g["type"] == "single":
            q = g["target"]
            ops = [np.eye(2)] * n
            ops = list(ops)
            ops[q] = np.asarray(g["matrix"], complex)
            M = ops[0]
            for o in ops[1:]:
                M = np.kron(M, o)
        else:
            a, b = g["targets"]
            U = fsim(g["theta"], g["phi"])
            ma, mb = 1 << (n - 1 - a), 1 << (n - 1 - b)
            for i in range(N):
                for o in range(N):
                    if (i & ~(ma | mb)) != (o & ~(ma | mb)):
                        continue
                    li = 2 * bool(i & ma) + bool(i & mb)
                    lo = 2 * bool(o & ma) + bool(o & mb)
                    M[o, i] = U[lo, li]
        psi = M @ psi
    return psi


@pytest.mark.parametrize("shape,cycles,seed", [((2, 2), 3, 11), ((2, 3), 4, 12), ((1, 5), 5, 13), ((2, 3), 6, 14)])
def test_statevector_matches_kron(oracle_built, shape, cycles, seed):
    """Catches transposed U[out][in] (sqrtY/sqrtW are not symmetric), LSB/MSB bit order, and the
    2*x_a + x_b local index of the fSim."""
    from oracle import sv
    c = small_circuit(*shape, cycles, seed)
    np.testing.assert_allclose(sv.statevector(c), kron_reference(c), atol=1e-12)


def test_statevector_norm(oracle_built):
    from oracle import sv
    for seed in range(5):
        psi = sv.statevector(small_circuit(3, 4, 6, 100 + seed))
        assert abs(np.vdot(psi, psi).real - 1) < 1e-12


def test_product_state_closed_form(oracle_built):
    """Single-qubit-only circuit: psi = kron_q (U_q,last ... U_q,1 |0>)."""
    from oracle import sv
    c = cc.generate_circuit(cc.rect_layout(1, 5), 0, "A", 7, final_layer=True)
    c["moments"] += cc.generate_circuit(cc.rect_layout(1, 5), 0, "A", 8, final_layer=True)["moments"]
    per_q = []
    for q in range(5):
        v = np.array([1, 0], complex)
        for g in cc.gate_list(c):
            if g["target"] == q:
                v = np.asarray(g["matrix"], complex) @ v
        per_q.append(v)
    want = per_q[0]
    for v in per_q[1:]:
        want = np.kron(want, v)
    np.testing.assert_allclose(sv.statevector(c), want, atol=1e-14)


def test_single_fsim_on_00(oracle_built):
    """a single fSim on |00> gives the first column of Eq. (1) = e_0."""
    from oracle import sv
    c = {"n": 2, "moments": [[{"type": "fsim", "targets": [0, 1], "theta": 1.1, "phi": 0.4}]]}
    np.testing.assert_allclose(sv.statevector(c), [1, 0, 0, 0], atol=1e-15)


# --------------------------------------------------------------------------- brute-force network

@pytest.mark.parametrize("shape,cycles,seed,nfix", [((2, 2), 2, 21, 0), ((2, 2), 3, 22, 2), ((1, 3), 3, 23, 3),
                                                     ((2, 2), 2, 24, 4)])
def test_statevector_matches_bruteforce_network(oracle_built, shape, cycles, seed, nfix):
    """O6: the network evaluated by definition (sum over internal wire values of products of gate
    entries) equals the state vector; with sliced wires fixed to v it equals the state vector
    with Pi_v inserted after the k-th gate on q (pins the wire-segment convention of App. A.2)."""
    from oracle import sv, tn_brute
    c = small_circuit(*shape, cycles, seed)
    wires, _ = tn_brute.internal_wires(c)
    r = np.random.default_rng(seed)
    pick = [wires[i] for i in r.choice(len(wires), size=nfix, replace=False)] if nfix else []
    vals = list(r.integers(0, 2, size=nfix))
    fixed = {w: int(v) for w, v in zip(pick, vals)}
    psi = sv.statevector(c, [(q, k, v) for (q, k), v in fixed.items()])
    n = c["n"]
    for x in range(1 << n):
        assert abs(tn_brute.amplitude(c, x, fixed) - psi[x]) < 1e-12


# --------------------------------------------------------------------------- slicing identities

def fsim_wires(circuit):
    """(q,k) right after each fSim (the wire segments a simplified network can slice)."""
    n = circuit["n"]
    count = [0] * n
    out = []
    gl = cc.gate_list(circuit)
    tot = [0] * n
    for g in gl:
        for q in ([g["target"]] if g["type"] == "single" else g["targets"]):
            tot[q] += 1
    for g in gl:
        qs = [g["target"]] if g["type"] == "single" else g["targets"]
        for q in qs:
            count[q] += 1
            if g["type"] == "fsim" and count[q] < tot[q]:
                out.append((q, count[q]))
    return out


def test_sum_over_all_slices_is_unsliced(oracle_built):
    """the sum of all sub-task results returns the original contraction."""
    from oracle import sv
    c = small_circuit(3, 3, 6, 31)
    W = fsim_wires(c)
    r = np.random.default_rng(3)
    wires = [W[i] for i in r.choice(len(W), 4, replace=False)]
    x = np.arange(1 << c["n"], dtype=np.uint64)
    full, _ = sv.amplitudes(c, x)
    tot = sv.sliced_amplitudes(c, x, wires, range(16))
    np.testing.assert_allclose(tot, full, atol=1e-12)


def test_prefix_equals_pinned(oracle_built):
    """S = [0, 2^(s-j)) equals Pi_0 on w_0..w_{j-1} only."""
    from oracle import sv
    c = small_circuit(3, 3, 6, 32)
    W = fsim_wires(c)
    wires = W[3:8]
    x = np.arange(1 << c["n"], dtype=np.uint64)
    s = len(wires)
    for j in range(s + 1):
        a, _ = sv.prefix_amplitudes(c, x, wires, j)
        b = sv.sliced_amplitudes(c, x, wires, range(1 << (s - j)))
        np.testing.assert_allclose(a, b, atol=1e-12)


def test_edge_breaking_pauli_split(oracle_built):
    """E = (1,0)x(1,0) = I/2 + sigma_z/2, so psi_{Pi_0} = psi/2 + psi_{sigma_z}/2."""
    from oracle import sv
    c = small_circuit(3, 3, 5, 33)
    for (q, k) in fsim_wires(c)[:6]:
        p0 = sv.statevector(c, [(q, k, 0)])
        pz = sv.statevector(c, [(q, k, 2)])
        np.testing.assert_allclose(p0, 0.5 * sv.statevector(c) + 0.5 * pz, atol=1e-13)


def test_slices_orthogonal_on_latest_wire(oracle_built):
    """SURVEY §8(c) item 11 (derived from PAPER.md L248): <psi_s|psi_t> = 0 exactly when s, t
    differ on the latest sliced wire (U^dag U cancels after it; Pi_a Pi_b = delta_ab Pi_a)."""
    from oracle import sv
    c = small_circuit(3, 3, 6, 34)
    W = fsim_wires(c)
    gl_index = {}
    # order wires by time: the wire list is produced in circuit order already
    early, late = W[2], W[-3]
    wires = [early, late]
    psis = [sv.statevector(c, sv.slice_insertions(wires, s)) for s in range(4)]
    # sigma bit1 (LSB) = late wire value
    assert abs(np.vdot(psis[0], psis[1])) < 1e-13
    assert abs(np.vdot(psis[2], psis[3])) < 1e-13
    assert abs(np.vdot(psis[0], psis[3])) < 1e-13


# --------------------------------------------------------------------------- rows (O7)

def test_paper_three_qubit_example():
    """request {111, 010, 000}; merging qubits 2 and 3 needs only {11, 10, 00}."""
    from oracle import rows
    lines = dict(l.split(None, 1) for l in open(os.path.join(GOLD, "paper_3qubit_example.txt"))
                 if l.strip() and not l.startswith("#"))
    req = np.array([int(s, 2) for s in lines["request"].split()], np.uint64)
    Q = [int(t) for t in lines["merged_qubits"].split()]
    got = rows.rows(req, 3, Q)
    assert [format(int(v), "02b") for v in got] == lines["rows"].split()
    assert [format(int(v), "03b") for v in rows.rows(req, 3, [0, 1, 2])] == lines["final_rows"].split()


def test_readout_rows_paper_example_and_bruteforce():
    """readout_rows: PAPER.md L202's request {111, 010, 000} reads rows {000, 010, 111} -> [2, 1, 0]; and on a
    random grouped request every amplitude's row holds its projection, computed bit by bit here."""
    from oracle import rows
    req = np.array([0b111, 0b010, 0b000], np.uint64)
    np.testing.assert_array_equal(rows.readout_rows(req, 3, [0, 1, 2]), [2, 1, 0])
    np.testing.assert_array_equal(rows.readout_rows(req, 3, [1, 2]), [2, 1, 0])   # rows {00, 10, 11}
    np.testing.assert_array_equal(rows.readout_rows(req, 3, [0]), [1, 0, 0])      # rows {0, 1}
    n = 9
    x = bs.generate_groups(n, [7, 8], 30, 11)
    Q = [0, 2, 3, 6]
    table = rows.rows(x, n, Q)
    idx = rows.readout_rows(x, n, Q)
    for j, b in enumerate(x):
        key = 0
        for q in Q:
            key = 2 * key + ((int(b) >> (n - 1 - q)) & 1)
        assert int(table[idx[j]]) == key


def test_rows_full_request_is_dense():
    """request = all 2^n bitstrings degenerates to the dense case."""
    from oracle import rows
    n = 6
    x = bs.all_bitstrings(n)
    for Q in ([0], [1, 4], [0, 2, 3, 5]):
        np.testing.assert_array_equal(rows.rows(x, n, Q), np.arange(1 << len(Q)))


def test_parent_map_bruteforce():
    from oracle import rows
    n = 10
    x = bs.generate_groups(n, [8, 9], 40, 5)
    Qc, Qp = [1, 3, 4, 7], [3, 7]
    rc = rows.rows(x, n, Qc)
    rp = rows.rows(x, n, Qp)
    pm = rows.parent_map(x, n, Qc, Qp)
    for r, p in zip(rc, pm):
        bits = {q: (int(r) >> (len(Qc) - 1 - i)) & 1 for i, q in enumerate(Qc)}
        key = 0
        for q in Qp:
            key = 2 * key + bits[q]
        assert int(rp[p]) == key


# --------------------------------------------------------------------------- metrics / sampler

def test_fidelity_definitions(oracle_built):
    from oracle import metrics, sv
    psi = sv.statevector(small_circuit(2, 3, 5, 41))
    assert abs(metrics.f_exact(psi, psi) - 1) < 1e-12
    assert abs(metrics.f_exact(psi, np.exp(0.7j) * 3 * psi) - 1) < 1e-12     # phase/scale invariant
    orth = np.zeros_like(psi)
    i = np.argmax(np.abs(psi))
    orth[i] = -np.conj(psi[(i + 1) % len(psi)])
    orth[(i + 1) % len(psi)] = np.conj(psi[i])
    assert metrics.f_exact(psi, orth) < 1e-25
    assert abs(metrics.f_norm(psi, 6) - 1) < 1e-12                            # full request, exact state


def test_f_sparse_closed_forms(oracle_built):
    """F_sparse(a, b) = |sum a_j^* b_j|^2 / (sum |a_j|^2 sum |b_j|^2).  Identity -> 1;
    global phase and scale -> 1; orthogonal -> 0; hand-worked 2-vectors; on a full request it is F_exact."""
    from oracle import metrics, sv
    a = np.array([1.0, 0.0], complex)
    assert abs(metrics.f_sparse(a, np.array([1.0, 1.0])) - 0.5) < 1e-15          # |1|^2 / (1 * 2)
    assert abs(metrics.f_sparse(np.array([1.0, 1j]), np.array([1.0, 1.0])) - 0.5) < 1e-15  # |1 - i|^2 / 4
    assert abs(metrics.f_sparse(np.array([3.0, 4.0]), np.array([4.0, -3.0]))) < 1e-15     # orthogonal
    # a = (1, 2i), b = (2, i): sum a^* b = 2 + (-2i)(i) = 4; |4|^2 / (5 * 5) = 16/25
    assert abs(metrics.f_sparse(np.array([1.0, 2j]), np.array([2.0, 1j])) - 0.64) < 1e-15
    psi = sv.statevector(small_circuit(2, 3, 4, 43))
    amps = psi[:17]
    assert abs(metrics.f_sparse(amps, amps) - 1) < 1e-12
    assert abs(metrics.f_sparse(amps, 0.3 * np.exp(-1.1j) * amps) - 1) < 1e-12
    phi = sv.statevector(small_circuit(2, 3, 4, 44))
    assert abs(metrics.f_sparse(psi, phi) - metrics.f_exact(psi, phi)) < 1e-12


def test_xeb_uniform_and_exact(oracle_built):
    """F_XEB = (2^n/L) sum P(s_i) - 1: ~1 for exact samples of a Porter-Thomas
    state, ~0 for uniform samples."""
    from oracle import metrics, sv
    c = small_circuit(3, 4, 12, 42)
    n = c["n"]
    p = np.abs(sv.statevector(c)) ** 2
    r = np.random.default_rng(0)
    L = 1 << 15
    exact = r.choice(len(p), size=L, p=p / p.sum())
    unif = r.integers(0, len(p), size=L)
    assert abs(metrics.linear_xeb(p[exact], n) - 1) < 0.1
    assert abs(metrics.linear_xeb(p[unif], n)) < 0.05


def test_sampler_distribution():
    """Categorical within a group: empirical frequencies match |a|^2 / sum (chi^2), one
    non-zero amplitude is always drawn, l = 1 draws the only bitstring."""
    from oracle import metrics
    l = 8
    r = np.random.default_rng(5)
    a = (r.normal(size=l) + 1j * r.normal(size=l)).astype(np.complex64)
    p = np.abs(a.astype(complex)) ** 2
    p /= p.sum()
    G = 20000
    amps = np.tile(a, G)
    picks = metrics.sample_groups(amps, l, seed=123) % l
    cnt = np.bincount(picks, minlength=l)
    chi2 = ((cnt - G * p) ** 2 / (G * p)).sum()
    assert chi2 < 30  # 7 dof, p ~ 1e-4
    one = np.zeros(l, np.complex64)
    one[5] = 0.3
    assert set(metrics.sample_groups(np.tile(one, 50), l, 9) % l) == {5}
    np.testing.assert_array_equal(metrics.sample_groups(a, 1, 3), np.arange(l))


@pytest.mark.parametrize("seed", [51, 52, 53, 54, 55, 56])
def test_one_broken_edge_halves_fidelity(oracle_built, seed):
    """breaking an edge (Pi_0 insertion) mid-circuit gives F ~ 1/2
    (statistical; checked on the ensemble mean below with a loose per-circuit bound)."""
    from oracle import metrics, sv
    c = small_circuit(3, 4, 10, seed)
    W = fsim_wires(c)
    mid = W[len(W) // 2]
    F = metrics.f_exact(sv.statevector(c), sv.statevector(c, [(mid[0], mid[1], 0)]))
    assert 0.25 < F < 0.75


def test_porter_thomas(oracle_built):
    """deep random circuits are Porter-Thomas: 2^n p ~ Exp(1) (KS statistic)."""
    from oracle import sv
    c = small_circuit(4, 4, 14, 61)
    N = 1 << c["n"]
    x = np.sort(N * np.abs(sv.statevector(c)) ** 2)
    ecdf = np.arange(1, N + 1) / N
    ks = np.max(np.abs(ecdf - (1 - np.exp(-x))))
    assert ks < 0.02


def test_config_structure():
    """Generator structure."""
    s = cc.sycamore_sites()
    assert len(s) == 54 and len(cc.couplers(s)) == 88
    l53 = cc.sycamore53_layout()
    assert len(l53) == 53 and len(cc.couplers(l53)) == 86
    assert [cc.count_fsim(configs.get(k).circuit()) for k in (1, 2, 3, 4, 5)] == [17, 62, 147, 301, 430]
    b = configs.get(2).bitstrings(20)
    assert len(b) == 4096 and len(np.unique(b)) == 4096


# ------------------------------------------------------------------------------ validation suite (NEXT-4)

def test_metropolis_degenerate_group():
    """l=2 with p=(1,0) -> always index 0 (a chain that starts on the zero-weight index
    moves as soon as index 0 is proposed and never leaves it)."""
    from oracle import metrics
    amps = np.tile(np.array([1.0, 0.0], dtype=np.complex64), 4096)
    idx = metrics.metropolis_groups(amps, 2, seed=11, steps=64)
    assert np.all(idx % 2 == 0)


def test_metropolis_stationary_distribution():
    """the chain's stationary distribution is p (detailed balance of min(1, p'/p) with a
    symmetric proposal): l=4, p=(.4,.3,.2,.1), total variation of the empirical sample distribution."""
    from oracle import metrics
    p = np.array([0.4, 0.3, 0.2, 0.1])
    G = 20000
    amps = np.tile(np.sqrt(p).astype(np.complex64), G)
    idx = metrics.metropolis_groups(amps, 4, seed=5, steps=50)
    emp = np.bincount(idx % 4, minlength=4) / G
    assert 0.5 * np.abs(emp - p).sum() < 0.02
    # and it mixes: with 1 step the start (uniform) is still visible
    emp1 = np.bincount(metrics.metropolis_groups(amps, 4, seed=5, steps=1) % 4, minlength=4) / G
    assert 0.5 * np.abs(emp1 - p).sum() > 0.05


def test_metropolis_agrees_with_categorical_on_pt_groups():
    """Metropolis and the categorical draw agree in distribution on random (Porter-Thomas)
    groups: the linear XEB of both sample sets under the source state agree (both ~ 1)."""
    from oracle import metrics
    r = np.random.default_rng(3)
    l, G, n = 64, 4000, 12
    amps = ((r.normal(size=l * G) + 1j * r.normal(size=l * G)) / np.sqrt(2 * (1 << n))).astype(np.complex64)
    ph = metrics.phat(amps, n)
    x_cat = metrics.linear_xeb(ph[metrics.sample_groups(amps, l, 7)], n)
    x_met = metrics.linear_xeb(ph[metrics.metropolis_groups(amps, l, 7, 200)], n)
    assert abs(x_cat - 1.0) < 0.1 and abs(x_met - 1.0) < 0.1 and abs(x_cat - x_met) < 0.1


def test_log_xeb_closed_forms():
    """log XEB = <ln(N P)> + gamma: perfect Porter-Thomas sampling (N P ~ Gamma(2,1), size-biased Exp)
    gives psi(2) + gamma = 1; uniform sampling (N P ~ Exp(1)) gives psi(1) + gamma = 0."""
    from oracle import metrics
    r = np.random.default_rng(9)
    n, L = 20, 200000
    N = 2.0 ** n
    assert abs(metrics.log_xeb(r.gamma(2.0, 1.0, L) / N, n) - 1.0) < 0.01
    assert abs(metrics.log_xeb(r.exponential(1.0, L) / N, n)) < 0.01


def test_entropy_closed_forms():
    """Uniform distribution over the 2^n strings, observed on a subset of M = 256 of them (the sparse
    state): H_state = H_samples = n ln 2 (this needs the 2^n/M factor); a delta: 0."""
    from oracle import metrics
    n = 10
    amps = np.full(256, 2.0 ** (-n / 2), dtype=np.complex64)
    ph = metrics.phat(amps, n)
    assert abs(metrics.entropy_state(ph, n) - n * math.log(2)) < 1e-9
    assert abs(metrics.entropy_samples(ph[:100]) - n * math.log(2)) < 1e-9
    d = np.zeros(1 << n, dtype=np.complex64)
    d[5] = 1
    pd = metrics.phat(d, n)
    assert abs(metrics.entropy_state(pd, n)) < 1e-12 and abs(metrics.entropy_samples(pd[[5]])) < 1e-12


def test_porter_thomas_ks_closed_forms():
    """KS distance to Exp(1): exact Exp(1) draws -> small (< 1.63/sqrt(m) at 1 %); a constant x = 1 ->
    max(F(1), 1 - F(1)) = F(1) = 1 - e^-1 = 0.632."""
    from oracle import metrics
    r = np.random.default_rng(2)
    assert metrics.porter_thomas_ks(r.exponential(1.0, 100000)) < 1.63 / math.sqrt(100000)
    assert abs(metrics.porter_thomas_ks(np.ones(1000)) - (1 - math.exp(-1))) < 1e-12


# ------------------------------------------------------------------------------ drilled holes (NEXT-3)

def _fsim_indices(circuit):
    flat = [g for m in circuit["moments"] for g in m]
    return [i for i, g in enumerate(flat) if g["type"] == "fsim"]


def _without_gate(circuit, h):
    """The same circuit with flattened gate h deleted."""
    out, i = [], 0
    for m in circuit["moments"]:
        mm = []
        for g in m:
            if i != h:
                mm.append(g)
            i += 1
        out.append(mm)
    c = dict(circuit)
    c["moments"] = out
    return c


def test_hole_removes_the_gate_exactly(oracle_built):
    """PAPER.md L106-L109, case (i): with both input edges of an fSim broken (Pi_0 (x) Pi_0 right before
    it), the gate evaluates to |00><00| -- it can be replaced by (1,0) vectors: the state equals that of
    the circuit with the gate deleted and the same two projectors."""
    from oracle import sv
    c = small_circuit(3, 3, 8, 71)
    fs = _fsim_indices(c)
    for h in (fs[len(fs) // 3], fs[2 * len(fs) // 3]):
        ins = sv.hole_insertions(c, [h])
        a = sv.statevector(c, ins)
        b = sv.statevector(_without_gate(c, h), ins)
        assert np.max(np.abs(a - b)) < 1e-12
        assert np.linalg.norm(a) > 0.05  # a nontrivial state survives


def test_hole_fidelity_quarter(oracle_built):
    """PAPER.md L73 / Fig. 1: each broken edge halves the fidelity, so one hole (two edges) gives
    F ~ 1/4; ensemble mean over random 12-qubit circuits with a hole mid-circuit."""
    from oracle import metrics, sv
    Fs = []
    for seed in range(10):
        c = small_circuit(3, 4, 12, 300 + seed)
        fs = _fsim_indices(c)
        h = fs[len(fs) // 2]
        Fs.append(metrics.f_exact(sv.statevector(c), sv.statevector(c, sv.hole_insertions(c, [h]))))
    assert 0.15 < np.mean(Fs) < 0.4, Fs


# ------------------------------------------------------------------------------ companion edges (NEXT-3)

@pytest.mark.parametrize("theta", [math.pi / 2, math.pi / 3, 1.4])
@pytest.mark.parametrize("v", [0, 1])
def test_companion_truncation_is_the_input_projector(theta, v):
    """Supplement: with one output of fSim pinned to v, the 3-way remainder reshaped
    with the OTHER qubit's input as columns has squared singular values {1 + sin^2, cos^2}; its rank-one
    truncation (SVD, keep the dominant pair) equals pinning that input to the same v (Pi_v), and keeps
    (1 + sin^2 theta)/2 of the squared norm.  (Pinning an output and cutting the other input is the
    transpose of the paper's cases: fSim is a symmetric matrix.)"""
    from oracle import sv
    F = sv.fsim_matrix(theta, math.pi / 6).reshape(2, 2, 2, 2)   # [o_a, o_b, i_a, i_b]
    M = F[v].reshape(4, 2)                                       # rows (o_b, i_a), columns i_b
    U, S, Vh = np.linalg.svd(M, full_matrices=False)
    assert np.allclose(np.sort(S ** 2), np.sort([1 + math.sin(theta) ** 2, math.cos(theta) ** 2]))
    rank1 = S[0] * np.outer(U[:, 0], Vh[0])
    pin = M.copy()
    pin[:, 1 - v] = 0                                            # Pi_v on the input i_b
    assert np.allclose(rank1, pin)
    assert abs(np.sum(np.abs(pin) ** 2) / 2 - (1 + math.sin(theta) ** 2) / 2) < 1e-12


def _set_theta(circuit, wire, theta):
    """Copy of the circuit with the fSim that ends sliced wire `wire` set to angle theta."""
    import copy
    c = copy.deepcopy(circuit)
    q, k = wire
    seen = 0
    for m in c["moments"]:
        for g in m:
            if (g["target"] == q if g["type"] == "single" else q in g["targets"]):
                seen += 1
                if seen == k:
                    g["theta"] = theta
                    return c
    raise AssertionError


def test_companion_fidelity_factor(oracle_built):
    """the companion truncation costs (1 + sin^2 theta)/2 of fidelity: exactly 1 at
    theta = pi/2 (nothing truncated, cos theta = 0); ~0.875 at theta = pi/3 (ensemble)."""
    from oracle import metrics, sv
    Fs = {math.pi / 2: [], math.pi / 3: []}
    for seed in range(8):
        c0 = small_circuit(3, 4, 10, 500 + seed)
        w = fsim_wires(c0)[len(fsim_wires(c0)) // 2]
        for th in Fs:
            c = _set_theta(c0, w, th)
            comp = sv.companion_of(c, w)
            psi = sv.statevector(c)
            approx = sum(sv.statevector(c, [(w[0], w[1], v), (comp[0], comp[1], v)]) for v in (0, 1))
            Fs[th].append(metrics.f_exact(psi, approx))
    assert min(Fs[math.pi / 2]) > 1 - 1e-12
    assert abs(np.mean(Fs[math.pi / 3]) - 0.875) < 0.06, Fs[math.pi / 3]


@pytest.mark.parametrize("seed", [5, 9])
def test_closed_network_matches_statevector(oracle_built, seed):
    """oracle/tn_einsum (closed-network contraction, numpy tensordot) = the state-vector oracle with the same
    projectors inserted (12 qubits, 6 cycles, three sliced wires), for several bitstrings."""
    from oracle import sv, tn_einsum
    circ = cc.generate_circuit(cc.rect_layout(3, 4), 6, "ABCDCDAB", seed)
    x = np.array([5, 1234, 4095, 77, 2048], np.uint64)
    wires = [(1, 3, 1), (5, 4, 0), (7, 5, 1)]
    want, _ = sv.amplitudes(circ, x, wires)
    got = np.array([tn_einsum.amplitude(circ, int(v), {(q, k): b for q, k, b in wires}) for v in x])
    assert np.abs(got - want).max() < 1e-14
    # and without projectors (the unsliced amplitude)
    want0, _ = sv.amplitudes(circ, x)
    got0 = np.array([tn_einsum.amplitude(circ, int(v)) for v in x])
    assert np.abs(got0 - want0).max() < 1e-14
