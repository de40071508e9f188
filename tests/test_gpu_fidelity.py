"""North-star check "partial-slice fidelity within 1e-3 of the oracle's value" (BASELINE.json; SURVEY §8(c)
item 16; "by summing over 2^16 paths ... the fidelity", L250 "sum 1/2^8 of the overall
sub-tasks").  For each prefix S = [0, 2^(s-j)) of the slice ids (= Pi_0 on the first j sliced wires, SURVEY
App. A.4) the SAME estimators are evaluated on the GPU's amplitudes and on the oracle's:
    F_norm(S)   = (2^n / M) sum_j |psi_S(x_j)|^2
    F_sparse(S) = |sum_j psi(x_j)^* psi_S(x_j)|^2 / (sum |psi(x_j)|^2 sum |psi_S(x_j)|^2)
where psi(x_j) is each side's own all-slices result.  Both must agree within 1e-3 (absolute)."""
import numpy as np
import pytest

from tn_inputs import configs

pytestmark = pytest.mark.gpu

TOL = 1e-3


@pytest.fixture(scope="module")
def T():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2111_03011_b200 as T
    T.lib()
    return T


def check_prefixes(T, cfg, js, plan_kwargs, tmax):
    from oracle import metrics, sv
    c = configs.get(cfg)
    circ = c.circuit()
    n = circ["n"]
    bits = c.bitstrings(n)
    ss = T.SparseState(circ, bits, c.open_mask(n))
    info = ss.plan(tmax, **plan_kwargs)
    ss.bind(0)
    s = info["s"]
    W = info["sliced_wires"]
    gpu_all = ss.contract(range(1 << s)).cpu().numpy().astype(complex)
    ora_all, _ = sv.amplitudes(circ, bits)
    rows = []
    for j in js:
        if j > s:
            continue
        gpu = gpu_all if j == 0 else ss.contract(range(1 << (s - j))).cpu().numpy().astype(complex)
        ora = ora_all if j == 0 else sv.prefix_amplitudes(circ, bits, W, j)[0]
        fn_g, fn_o = metrics.f_norm(gpu, n), metrics.f_norm(ora, n)
        fs_g, fs_o = metrics.f_sparse(gpu_all, gpu), metrics.f_sparse(ora_all, ora)
        rows.append((j, fn_g, fn_o, fs_g, fs_o))
        assert abs(fn_g - fn_o) <= TOL, f"F_norm j={j}: gpu {fn_g:.6f} oracle {fn_o:.6f}"
        assert abs(fs_g - fs_o) <= TOL, f"F_sparse j={j}: gpu {fs_g:.6f} oracle {fs_o:.6f}"
    return rows


def test_partial_fidelity_config2_every_prefix(T, oracle_built):
    """Config 2 (20q m=8, M=4096, 2^4 slices): every prefix j = 0..4."""
    c = configs.get(2)
    rows = check_prefixes(T, 2, range(0, 5), {"n_sliced": c.n_sliced}, 1 << c.log2_tmax)
    assert len(rows) == 5
    # the fraction of slices tracks the fidelity (statistical): F_norm halves per pinned wire
    for j, fn_g, _, _, _ in rows:
        assert 0.5 ** j * 0.5 < fn_g < 0.5 ** j * 2.0


@pytest.mark.slow
def test_partial_fidelity_config3_prefixes(T, oracle_built):
    """Config 3 (30q m=12, M=65536, 2^8 slices, the bench plan): prefixes j = 0, 1, 2 (one 2^30 fp64
    state-vector run on the host per prefix)."""
    c = configs.get(3)
    rows = check_prefixes(T, 3, range(0, 3), c.plan_kwargs(), 1 << c.log2_tmax)
    assert len(rows) == 3
