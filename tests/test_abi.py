"""CPU tests of the C ABI library: exports, validation/error codes, host planning, structural bit-exact
row tables and the host sampler against the oracle.  No GPU needed."""
import json
import os
import re
import ctypes

import numpy as np
import pytest

from tn_inputs import bitstrings as bs
from tn_inputs import circuits as cc
from tn_inputs import configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def T():
    from paper_2111_03011_b200 import build
    build.build()
    import paper_2111_03011_b200 as T
    T.lib()
    return T


def header_functions():
    names = set()
    for h in ("tn.h", "tn_debug.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(tn_[a-z_0-9]+)\s*\(", src):
            names.add(m.group(1))
    return names


def test_exports_every_declared_symbol(T):
    L = T.lib()
    names = header_functions()
    assert {"tn_build", "tn_plan", "tn_bind_device", "tn_contract", "tn_sample"} <= names
    for name in sorted(names):
        assert hasattr(L, name), f"{name} declared in include/ but not exported"
    assert set(T.EXPORTS) == names


def test_version(T):
    assert b"sm_100a" in T.lib().tn_version()


# ------------------------------------------------------------------------------ validation

def _small():
    circ = cc.generate_circuit(cc.rect_layout(2, 3), 4, "ABCD", 5)
    bits = bs.generate_groups(6, [5], 8, 6)
    return circ, bits, bs.qubit_mask(6, [5])


def test_build_rejects_bad_inputs(T):
    circ, bits, om = _small()
    with pytest.raises(T.TnError) as e:
        T.SparseState(circ, np.array([1 << 6], np.uint64), 0)
    assert e.value.status == T.TN_EINVAL and "bits beyond" in str(e.value)
    with pytest.raises(T.TnError) as e:                       # broken group structure
        T.SparseState(circ, bits[::-1].copy(), om)
    assert e.value.status == T.TN_EINVAL and "group" in str(e.value)
    bad = dict(circ)
    bad["moments"] = [[{"type": "fsim", "targets": [0, 5], "theta": 1.0, "phi": 0.5}]]
    with pytest.raises(T.TnError) as e:                       # (0,0)-(1,2) are not neighbours
        T.SparseState(bad, bits, om)
    assert "neighbours" in str(e.value)
    bad["moments"] = [[{"type": "fsim", "targets": [0, 1], "theta": 1.0, "phi": 0.5},
                       {"type": "single", "target": 1, "matrix": [[1, 0], [0, 1]]}]]
    with pytest.raises(T.TnError) as e:
        T.SparseState(bad, bits, om)
    assert "twice" in str(e.value)


def test_call_order_and_infeasible(T):
    circ, bits, om = _small()
    ss = T.SparseState(circ, bits, om)
    with pytest.raises(T.TnError) as e:
        ss.contract_host([0])
    assert e.value.status == T.TN_EINVAL and "bind" in str(e.value)
    with pytest.raises(T.TnError) as e:
        ss.plan(1, n_sliced=0)                                # bound 1 with no slicing: infeasible
    assert e.value.status == T.TN_EINFEASIBLE
    with pytest.raises(T.TnError) as e:
        ss.plan(1 << 10, forced_wires=[(0, 0)])
    assert e.value.status == T.TN_EINVAL


def test_bind_without_gpu_fails_cleanly(T):
    from tests.conftest import has_gpu
    if has_gpu():
        pytest.skip("GPU present")
    circ, bits, om = _small()
    ss = T.SparseState(circ, bits, om)
    ss.plan(1 << 10)
    ws = ctypes.c_void_p(0)
    rc = T.lib().tn_bind_device(ss._ctx, 0, ws, 0, None)
    assert rc == T.TN_ECUDA


# ------------------------------------------------------------------------------ network + plan structure

def test_simplified_network_sizes(T):
    """P:L130 simplification; 13 / 54 / 135 tensors for configs 1-3."""
    for k, want in ((1, 13), (2, 54), (3, 135)):
        c = configs.get(k)
        circ = c.circuit()
        n = circ["n"]
        ss = T.SparseState(circ, c.bitstrings(n), c.open_mask(n))
        assert ss.network_size()["tensors"] == want


def gate_counts(circ):
    n = circ["n"]
    seq = [[] for _ in range(n)]
    for g in cc.gate_list(circ):
        for q in ([g["target"]] if g["type"] == "single" else g["targets"]):
            seq[q].append(g["type"])
    return seq


@pytest.mark.parametrize("k", [2, 3])
def test_plan_rows_bit_exact(T, tmp_path, k):
    """O7: every sparse row table and parent map in the plan equals the oracle's independent
    recomputation (oracle/rows.py); sliced wires are internal wires right after an fSim."""
    from oracle import rows
    c = configs.get(k)
    circ = c.circuit()
    n = circ["n"]
    bits = c.bitstrings(n)
    ss = T.SparseState(circ, bits, c.open_mask(n))
    info = ss.plan(1 << c.log2_tmax, n_sliced=c.n_sliced)
    p = tmp_path / "plan.json"
    ss.dump(str(p))
    d = json.load(open(p))
    assert [tuple(w) for w in d["sliced_wires"]] == info["sliced_wires"]
    seq = gate_counts(circ)
    for q, kk in info["sliced_wires"]:
        assert 1 <= kk < len(seq[q]) and seq[q][kk - 1] == "fsim" and "fsim" in seq[q][kk:]

    def qubits(mask):
        return [q for q in range(n) if (mask >> (n - 1 - q)) & 1]

    checked = 0
    for st in d["steps"]:
        if "row_keys" not in st:
            continue
        Q = qubits(st["qmask"])
        got = rows.project(np.array(st["row_keys"], np.uint64), n, Q)
        np.testing.assert_array_equal(got, rows.rows(bits, n, Q))
        for side in ("a", "b"):
            Qp = qubits(st[f"qmask_{side}"])
            if Qp:
                np.testing.assert_array_equal(np.array(st[f"map_{side}"]), rows.parent_map(bits, n, Q, Qp))
        checked += 1
    assert checked > 5
    fin = d["final"]
    Qf = qubits(fin["qmask"])
    assert sorted(Qf) == sorted(set(range(n)) - set(c.open_ids(n)))
    np.testing.assert_array_equal(rows.project(np.array(fin["row_keys"], np.uint64), n, Qf), rows.rows(bits, n, Qf))
    # readout: amplitude j reads the final row holding its fixed part
    keys = np.array(fin["row_keys"], np.uint64)
    mask = np.uint64(fin["qmask"])
    np.testing.assert_array_equal(keys[rows.readout_rows(bits, n, Qf)], bits & mask)


def test_mac_count_identity(T, tmp_path):
    """MACs of a pairwise step = prod(output dims) x prod(shared dims) (rows x 2^(fa+fb+k))."""
    c = configs.get(2)
    circ = c.circuit()
    n = circ["n"]
    ss = T.SparseState(circ, c.bitstrings(n), c.open_mask(n))
    info = ss.plan(1 << c.log2_tmax, n_sliced=c.n_sliced)
    ss.dump(str(tmp_path / "p.json"))
    d = json.load(open(tmp_path / "p.json"))
    tot = inv = 0.0
    for st in d["steps"]:
        assert st["cmac"] == st["rows"] * 2.0 ** (st["fa"] + st["fb"] + st["k"])
        if st["invariant"]:
            inv += st["cmac"]
        else:
            tot += st["cmac"]
    assert tot == info["cmac_per_slice"]
    assert inv == info["invariant_cmac"]
    assert sum(st["invariant"] for st in d["steps"]) == info["n_invariant_steps"]


def test_plan_deterministic(T, tmp_path):
    c = configs.get(2)
    circ = c.circuit()
    n = circ["n"]
    outs = []
    for i in range(2):
        ss = T.SparseState(circ, c.bitstrings(n), c.open_mask(n))
        ss.plan(1 << c.log2_tmax, n_sliced=c.n_sliced, seed=7)
        ss.dump(str(tmp_path / f"p{i}.json"))
        outs.append(open(tmp_path / f"p{i}.json").read())
    assert outs[0] == outs[1]


# ------------------------------------------------------------------------------ tn_sample (host)

def test_host_sampler_matches_oracle(T):
    """tn_sample's categorical draw equals the oracle's on the same amplitudes (same counter-based
    generator, same fp64 decision), and its estimators equal the oracle metrics."""
    from oracle import metrics
    c = configs.get(2)
    circ = c.circuit()
    n = circ["n"]
    bits = c.bitstrings(n)
    ss = T.SparseState(circ, bits, c.open_mask(n))
    info = ss.plan(1 << c.log2_tmax, n_sliced=c.n_sliced)
    r = np.random.default_rng(9)
    amps = ((r.normal(size=len(bits)) + 1j * r.normal(size=len(bits))) * 2 ** -10).astype(np.complex64)
    ideal = ((r.normal(size=len(bits)) + 1j * r.normal(size=len(bits))) * 2 ** -10).astype(np.complex64)
    for seed in (0, 3001, 2 ** 63 + 5):
        samples, est = ss.sample(amps, 4, seed, ideal=ideal)
        idx = metrics.sample_groups(amps, 64, seed)
        np.testing.assert_array_equal(samples, bits[idx])
    assert est["fraction"] == 4 / 16
    assert abs(est["F_norm"] / metrics.f_norm(amps, n) - 1) < 1e-12
    p = ideal.real.astype(float) ** 2 + ideal.imag.astype(float) ** 2
    assert abs(est["xeb"] - metrics.linear_xeb(p[idx], n)) < 1e-9 * abs(est["xeb"]) + 1e-9
    zero = amps.copy()
    zero[:64] = 0
    with pytest.raises(T.TnError) as e:
        ss.sample(zero, 1, 0)
    assert e.value.status == T.TN_ENUMERIC


def test_sample_report_matches_oracle(T):
    """tn_sample_report (NEXT-4 validation suite) against the oracle on the same amplitudes: the
    categorical and the Metropolis samples are bit-exact (same counter-based generator, same fp64
    decisions); every estimator equals the oracle's definition."""
    from oracle import metrics
    c = configs.get(2)
    circ = c.circuit()
    n = circ["n"]
    bits = c.bitstrings(n)
    ss = T.SparseState(circ, bits, c.open_mask(n))
    ss.plan(1 << c.log2_tmax, n_sliced=c.n_sliced)
    r = np.random.default_rng(21)
    M = len(bits)
    amps = ((r.normal(size=M) + 1j * r.normal(size=M)) * 2 ** -10).astype(np.complex64)
    ideal = ((r.normal(size=M) + 1j * r.normal(size=M)) * 2 ** -10).astype(np.complex64)
    l = 64
    ph = metrics.phat(amps, n)
    P = ideal.real.astype(float) ** 2 + ideal.imag.astype(float) ** 2
    for sampler, steps in (("categorical", 0), ("metropolis", 1), ("metropolis", 200)):
        samples, idx, rep = ss.sample_report(amps, 16, 3001, sampler=sampler, steps=steps, ideal=ideal)
        want = (metrics.sample_groups(amps, l, 3001) if sampler == "categorical"
                else metrics.metropolis_groups(amps, l, 3001, steps))
        np.testing.assert_array_equal(idx, want)
        np.testing.assert_array_equal(samples, bits[want])
        assert rep["f"] == 1.0
        assert abs(rep["F_norm"] / metrics.f_norm(amps, n) - 1) < 1e-12
        assert abs(rep["xeb"] - metrics.linear_xeb(P[want], n)) < 1e-9 * (1 + abs(rep["xeb"]))
        assert abs(rep["log_xeb"] - metrics.log_xeb(P[want], n)) < 1e-9
        assert abs(rep["entropy_samples"] / metrics.entropy_samples(ph[want]) - 1) < 1e-12
        assert abs(rep["entropy_state"] / metrics.entropy_state(ph, n) - 1) < 1e-12
        assert abs(rep["pt_ks"] - metrics.porter_thomas_ks((2.0 ** n) * ph)) < 1e-12
    _, _, rep = ss.sample_report(amps, 16, 1, sampler="metropolis", steps=10)
    assert np.isnan(rep["xeb"]) and np.isnan(rep["log_xeb"])
    with pytest.raises(T.TnError) as e:
        ss.sample_report(amps, 16, 1, sampler="metropolis", steps=0)
    assert e.value.status == T.TN_EINVAL


def test_drilled_holes_shrink_the_network(T):
    """tn_build_drilled (NEXT-3): drilling fSim gates removes them from the network (fewer
    tensors and sliceable edges); bad hole lists are rejected."""
    c = configs.get(3)
    circ = c.circuit()
    n = circ["n"]
    flat = [g for m in circ["moments"] for g in m]
    fs = [i for i, g in enumerate(flat) if g["type"] == "fsim"]
    holes = [fs[len(fs) // 2 - 3], fs[len(fs) // 2 + 3]]
    base = T.SparseState(circ, c.bitstrings(n), c.open_mask(n))
    drilled = T.SparseState(circ, c.bitstrings(n), c.open_mask(n), holes=holes)
    a, b = base.network_size(), drilled.network_size()
    assert b["tensors"] < a["tensors"] and b["internal_edges"] < a["internal_edges"]
    for bad in ([0], [holes[0], holes[0]], [len(flat)]):  # gate 0 is a single-qubit gate
        with pytest.raises(T.TnError) as e:
            T.SparseState(circ, c.bitstrings(n), c.open_mask(n), holes=bad)
        assert e.value.status == T.TN_EINVAL


def test_companion_plan_report(T):
    """tn_slicing.companions: every companion is the oracle's companion of its tied sliced wire (the other
    input of the fSim that ends that wire) and companion_fidelity = prod (1 + sin^2 theta_i)/2 over those
    gates, with theta read from the circuit."""
    import math
    from oracle import sv
    c = configs.get(3)
    circ = c.circuit()
    n = circ["n"]
    ss = T.SparseState(circ, c.bitstrings(n), c.open_mask(n))
    info = ss.plan(1 << c.log2_tmax, n_sliced=c.n_sliced, seed=3, trials=8, time_budget_s=300, companions=True)
    wires = info["sliced_wires"]
    assert info["companions"]
    flat = [g for m in circ["moments"] for g in m]
    want = 1.0
    for (q, k, i) in info["companions"]:
        assert 0 <= i < info["s"]
        assert sv.companion_of(circ, wires[i]) == (q, k)
        # the gate: the (k+1)-th gate on q
        seen, theta = 0, None
        for g in flat:
            if (g["target"] == q if g["type"] == "single" else q in g["targets"]):
                seen += 1
                if seen == k + 1:
                    theta = g["theta"]
                    break
        want *= (1 + math.sin(theta) ** 2) / 2
    assert abs(info["companion_fidelity"] - want) < 1e-12


def test_loop_program_companions_and_plan_file_flag(T, tmp_path):
    """Loop programs accept companion edges: each companion is the oracle's companion of its partner,
    indexed in sliced_wires + local_wires; the plan file records the flag, and importing it with a different
    tn_slicing.companions is refused (the tied edges change the lowered network)."""
    from oracle import sv
    c = configs.get(2)
    circ = c.circuit()
    n = circ["n"]
    bits = c.bitstrings(n)
    ss = T.SparseState(circ, bits, c.open_mask(n))
    info = ss.plan(1 << 12, n_sliced=2, method=2, max_segments=8, seed=1, time_budget_s=5.0, companions=True)
    W = info["sliced_wires"] + info["local_wires"]
    assert info["companions"] and info["s_local"] >= 1
    for (q, k, i) in info["companions"]:
        assert sv.companion_of(circ, W[i]) == (q, k)
    p = str(tmp_path / "plan.json")
    ss.save_plan(p)
    ss2 = T.SparseState(circ, bits, c.open_mask(n))
    with pytest.raises(T.TnError) as e:
        ss2.plan(1 << 12, plan_path=p)
    assert e.value.status == T.TN_EINVAL
    info2 = ss2.plan(1 << 12, plan_path=p, companions=True)
    assert info2["companions"] == info["companions"] and info2["total_cmac"] == info["total_cmac"]
