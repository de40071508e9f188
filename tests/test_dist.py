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
