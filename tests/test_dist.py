"""Host-side multi-GPU logic on CPU (gloo, world_size 2): slice partitioning and the amplitude all-reduce
(SURVEY §8(a) row a8, §8(e))."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2111_03011_b200.dist import allreduce_amplitudes, partition


def test_partition_covers_each_slice_once():
    for nS in (1, 7, 16, 256, 4096):
        for world in (1, 2, 3, 4, 8):
            blocks = [partition(range(nS), world, r) for r in range(world)]
            flat = [x for b in blocks for x in b]
            assert flat == list(range(nS))
            sizes = [len(b) for b in blocks]
            assert max(sizes) - min(sizes) <= 1
    assert partition([9, 3, 5], 2, 0) == [3, 5]
    with pytest.raises(ValueError):
        partition([1, 1], 2, 0)


def fake_slice_amps(sigma, M):
    """Stand-in for one slice's contraction output (deterministic per slice id)."""
    r = np.random.default_rng(1000 + sigma)
    return (r.normal(size=M) + 1j * r.normal(size=M)).astype(np.complex64)


def _worker(rank, world, port, M, nS, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    block = partition(range(nS), world, rank)
    acc = np.zeros(M, np.complex64)
    for s in block:
        acc += fake_slice_amps(s, M)
    t = torch.from_numpy(acc.copy())
    allreduce_amplitudes(t)
    q.put((rank, t.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_allreduce_two_ranks():
    world, M, nS = 2, 1000, 13
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, nS, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    want = sum(fake_slice_amps(s, M).astype(complex) for s in range(nS))
    for r in range(world):
        np.testing.assert_allclose(res[r], want, rtol=0, atol=1e-4 * np.abs(want).max())
    np.testing.assert_array_equal(res[0], res[1])


def _fp_worker(rank, world, port, infos, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2111_03011_b200.dist import check_same_plan
    try:
        check_same_plan(infos[rank])
        q.put((rank, "ok"))
    except RuntimeError as e:
        q.put((rank, "mismatch" if "different plans" in str(e) else str(e)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("same", [True, False])
def test_ranks_must_hold_the_same_plan(same):
    """contract_distributed all-gathers a plan fingerprint first: ranks with different plans raise instead of
    adding slices of different networks."""
    base = {"s": 4, "sliced_wires": [(1, 2), (3, 4), (5, 6), (7, 8)], "s_local": 0, "local_wires": [],
            "n_segments": 1, "n_steps": 53, "n_tensors": 54}
    other = dict(base, sliced_wires=[(1, 2), (3, 4), (5, 6), (7, 9)])
    infos = [base, base if same else other]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_fp_worker, args=(r, 2, port, infos, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert set(res.values()) == ({"ok"} if same else {"mismatch"})


def _gpu_worker(rank, world, port, plan_path, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2111_03011_b200 as T
    from paper_2111_03011_b200.dist import contract_distributed
    from tn_inputs import configs
    c = configs.get(2)
    circ = c.circuit()
    n = circ["n"]
    ss = T.SparseState(circ, c.bitstrings(n), c.open_mask(n))
    info = ss.plan(1 << 12, plan_path=plan_path)
    ss.bind(0, pipelines=2)
    amps = contract_distributed(ss, range(1 << info["s"]))
    q.put((rank, amps.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("method", [1, 2])
def test_contract_distributed_two_ranks_on_one_gpu(tmp_path, oracle_built, method):
    """contract_distributed (each rank tn_contract's its contiguous block of global slices, then the
    all-reduce) with world_size 2 on one GPU over gloo, for a flat plan and a loop program, vs the oracle's
    exact amplitudes (all slices summed).  The plan is made once and imported by both ranks (plan file)."""
    import paper_2111_03011_b200 as T
    from oracle import sv
    from tests.helpers import assert_amps_close
    from tn_inputs import configs
    c = configs.get(2)
    circ = c.circuit()
    n = circ["n"]
    bits = c.bitstrings(n)
    ss = T.SparseState(circ, bits, c.open_mask(n))
    ss.plan(1 << 12, n_sliced=(-1 if method == 1 else 3), method=method, time_budget_s=3.0)
    p = str(tmp_path / "plan.json")
    ss.save_plan(p)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, p, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
    want, _ = sv.amplitudes(circ, bits)
    for r in range(2):
        assert_amps_close(res[r], want)
    np.testing.assert_array_equal(res[0], res[1])
