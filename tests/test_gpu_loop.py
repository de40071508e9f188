"""Loop programs (tn_slicing.method = 2: stem sweep, local slices summed inside the program, checkpointed
segments reusing the head across slices -- PAPER.md L89-L91, L131-L136) vs the oracle through the C ABI.

A slice id of a loop program is a global slice: its local wires are summed inside tn_contract, so the
oracle projects only the exported (global) wires (Sigma_v Pi_v = I on the local ones).  Expected values
come only from oracle/."""
import numpy as np
import pytest

from tests.helpers import assert_amps_close
from tn_inputs import bitstrings as bs
from tn_inputs import circuits as cc
from tn_inputs import configs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2111_03011_b200 as T
    T.lib()
    return T


def loop_plan(T, circ, bits, om, tmax, n_global=2, segs=8, seed=1, pipelines=4):
    ss = T.SparseState(circ, bits, om)
    info = ss.plan(tmax, n_sliced=n_global, method=2, max_segments=segs, seed=seed, time_budget_s=5.0)
    ss.bind(0, pipelines=pipelines)
    return ss, info


@pytest.fixture(scope="module")
def cfg2():
    c = configs.get(2)
    circ = c.circuit()
    n = circ["n"]
    return c, circ, c.bitstrings(n), c.open_mask(n)


def test_loop_program_all_slices_match_statevector(T, oracle_built, cfg2):
    """Config 2 (20q m=8, M=4096) planned as a loop program at max_tensor_size 2^12, so that local slices,
    summations and several segments occur; the sum over every global slice is the exact state."""
    from oracle import sv
    c, circ, bits, om = cfg2
    ss, info = loop_plan(T, circ, bits, om, 1 << 12)
    assert info["s_local"] >= 1 and info["n_segments"] >= 2, info
    amps = ss.contract(range(1 << info["s"])).cpu().numpy()
    want, _ = sv.amplitudes(circ, bits)
    assert_amps_close(amps, want)


@pytest.mark.parametrize("j", [1, 2])
def test_loop_program_prefix_and_subset(T, oracle_built, cfg2, j):
    """Prefix [0, 2^(s-j)) of the global slices = Pi_0 on the first j global wires (App. A.4), and an
    arbitrary subset = the per-slice projector sum; local wires are never projected."""
    from oracle import sv
    c, circ, bits, om = cfg2
    ss, info = loop_plan(T, circ, bits, om, 1 << 12)
    s = info["s"]
    W = info["sliced_wires"]
    amps = ss.contract(range(1 << (s - j))).cpu().numpy()
    assert_amps_close(amps, sv.prefix_amplitudes(circ, bits, W, j)[0])
    sub = [x for x in range(1 << s) if (x * 2654435761) % 7 < 3]
    amps = ss.contract(sub).cpu().numpy()
    assert_amps_close(amps, sv.sliced_amplitudes(circ, bits, W, sub))


def test_loop_program_plan_file_roundtrip(T, tmp_path, cfg2):
    """tn_plan_save -> tn_plan(plan_path): the imported plan reproduces the amplitudes bit for bit."""
    c, circ, bits, om = cfg2
    ss, info = loop_plan(T, circ, bits, om, 1 << 12)
    p = str(tmp_path / "plan.json")
    ss.save_plan(p)
    a = ss.contract(range(1 << info["s"])).cpu().numpy()
    ss2 = T.SparseState(circ, bits, om)
    info2 = ss2.plan(1 << 12, plan_path=p)
    ss2.bind(0, pipelines=4)
    assert info2["sliced_wires"] == info["sliced_wires"] and info2["local_wires"] == info["local_wires"]
    b = ss2.contract(range(1 << info2["s"])).cpu().numpy()
    assert np.array_equal(a, b)


def test_loop_program_pipelines_agree(T, oracle_built, cfg2):
    """One pipeline vs several (different slice blocks, each with its own head reuse): same amplitudes
    within fp32 rounding of the pipeline sum."""
    c, circ, bits, om = cfg2
    ss1, info = loop_plan(T, circ, bits, om, 1 << 12, pipelines=1)
    ssn, _ = loop_plan(T, circ, bits, om, 1 << 12, pipelines=8)
    a = ss1.contract(range(1 << info["s"])).cpu().numpy()
    b = ssn.contract(range(1 << info["s"])).cpu().numpy()
    assert_amps_close(b, a, rel=1e-6, elem=1e-5)


def test_loop_program_24q_random_circuit(T, oracle_built):
    """24 qubits (4x6, m=10, ABCDCDAB), 256 groups x 64: a loop program with tensor-core steps."""
    from oracle import sv
    circ = cc.generate_circuit(cc.rect_layout(4, 6), 10, "ABCDCDAB", 4242)
    n = circ["n"]
    openq = list(range(n - 6, n))
    bits = bs.generate_groups(n, openq, 256, 4343)
    ss, info = loop_plan(T, circ, bits, bs.qubit_mask(n, openq), 1 << 16, n_global=3)
    amps = ss.contract(range(1 << info["s"])).cpu().numpy()
    want, _ = sv.amplitudes(circ, bits)
    assert_amps_close(amps, want)


def test_loop_program_with_companions(T, oracle_built, cfg2):
    """Loop program with companion-edge truncation ("rank one approximation to companion
    edges" of the interface): every companion is Pi_v on the oracle's companion wire with v the value of its
    partner (global or local), so the oracle enumerates the local wires too and sums their values itself
    (Sigma_v Pi_v x Pi_v != I on a tied pair)."""
    from oracle import sv
    c, circ, bits, om = cfg2
    ss = T.SparseState(circ, bits, om)
    info = ss.plan(1 << 12, n_sliced=2, method=2, max_segments=8, seed=1, time_budget_s=5.0, companions=True)
    comps = info["companions"]
    assert len(comps) >= 1 and info["s_local"] >= 1, info
    W = info["sliced_wires"] + info["local_wires"]
    for (q, k, i) in comps:
        assert sv.companion_of(circ, W[i]) == (q, k)
    ss.bind(0, pipelines=4)
    s, sl = info["s"], info["s_local"]
    for glob in (range(1 << s), [1]):
        ids = [(g << sl) | lam for g in glob for lam in range(1 << sl)]
        want = sv.sliced_amplitudes(circ, bits, W, ids, companions=comps)
        assert_amps_close(ss.contract(glob).cpu().numpy(), want)
    assert 0.9 < info["companion_fidelity"] <= 1.0


@pytest.mark.parametrize("log2_tmax,method", [(12, 2), (16, 2), (20, 1)])
def test_gate_kernel_all_modes_match_statevector(T, oracle_built, cfg2, monkeypatch, log2_tmax, method):
    """The tensor-core gate kernel (gate_tc.cuh) in all three modes -- rowless gate (0), gate per B row (1),
    A-row groups with the members' B rows as gate columns (2) -- on config 2 with TNB_GATE_ANY=1, which sends
    every structurally eligible step to it regardless of size (the production thresholds only pick the big
    ones).  The sum over all slices equals the oracle's exact state."""
    import json
    from oracle import sv
    c, circ, bits, om = cfg2
    monkeypatch.setenv("TNB_GATE_ANY", "1")
    ss = T.SparseState(circ, bits, om)
    info = ss.plan(1 << log2_tmax, n_sliced=2 if method == 2 else 4, method=method, seed=1, time_budget_s=5.0)
    monkeypatch.delenv("TNB_GATE_ANY")
    import tempfile, os
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "dump.json")
        ss.dump(p)
        modes = {s["gate_tc"] for s in json.load(open(p))["steps"] if "gate_tc" in s}
    assert {0, 2} <= modes, modes
    if log2_tmax == 16:
        assert 1 in modes, modes
    ss.bind(0, pipelines=2)
    amps = ss.contract(range(1 << info["s"])).cpu().numpy()
    want, _ = sv.amplitudes(circ, bits)
    assert_amps_close(amps, want)
