"""Multi-GPU slice partitioning and the cross-GPU amplitude sum.

Slices are independent sub-tasks ("creating 2^16 subtasks", P:L149 512 GPUs); the only exchange
is the sum of the per-rank partial amplitude vectors ("By summing over 2^16 paths"), done once
per tn_contract as one NCCL all-reduce over NVLink/NVSwitch (torch.distributed plumbing).
"""
from __future__ import annotations

from typing import List, Sequence


def partition(slice_ids: Sequence[int], world: int, rank: int) -> List[int]:
    """Contiguous block of the ascending slice subset for `rank` (sizes differ by at most one; every
    slice has the same shapes, so a static split balances the work)."""
    ids = sorted(int(x) for x in slice_ids)
    if len(set(ids)) != len(ids):
        raise ValueError("duplicate slice ids")
    n = len(ids)
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    size = base + (1 if rank < extra else 0)
    return ids[start:start + size]


def allreduce_amplitudes(amps, group=None):
    """Sum the complex64 amplitude vectors of all ranks in place (NCCL on GPUs, gloo on CPU tests)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return amps
    dist.all_reduce(torch.view_as_real(amps), op=dist.ReduceOp.SUM, group=group)
    return amps


def contract_distributed(ss, slice_ids: Sequence[int], out=None):
    """Each rank contracts its block of slice_ids on its own GPU (tn_contract), then all ranks
    all-reduce.  Returns the summed amplitudes (complex64 CUDA tensor) on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    block = partition(slice_ids, world, rank)
    if out is None:
        out = torch.empty(ss.M, dtype=torch.complex64, device=torch.device("cuda", ss._dev))
    if block:
        ss.contract(block, out=out)
    else:
        out.zero_()
    return allreduce_amplitudes(out)
