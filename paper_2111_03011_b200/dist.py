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


def plan_fingerprint(info: dict) -> str:
    """Identity of a plan as the slice-id space sees it: the global and local sliced wires, the segment count
    and the step count.  Ranks that sum partial amplitudes must hold the same plan (else the all-reduce adds
    slices of different networks)."""
    import hashlib
    key = repr((info["s"], info["sliced_wires"], info.get("s_local", 0), info.get("local_wires", []),
                info.get("n_segments", 1), info["n_steps"], info["n_tensors"]))
    return hashlib.sha256(key.encode()).hexdigest()


def check_same_plan(info: dict, group=None) -> None:
    """All-gather the plan fingerprint and raise if any rank planned differently (the planner's search is
    time-budgeted, so independent searches may differ: plan once and import the plan file instead)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    fp = plan_fingerprint(info)
    allfp = [None] * dist.get_world_size(group)
    dist.all_gather_object(allfp, fp, group=group)
    if len(set(allfp)) != 1:
        raise RuntimeError(f"ranks hold different plans (fingerprints {sorted(set(allfp))}); plan on one rank, "
                           "save_plan(), and load it with plan(plan_path=...) on every rank")


def contract_distributed(ss, slice_ids: Sequence[int], out=None, check_plan: bool = True):
    """Each rank contracts its block of slice_ids on its own GPU (tn_contract), then all ranks
    all-reduce.  Returns the summed amplitudes (complex64 CUDA tensor) on every rank.  The ranks'
    plans are compared first (check_same_plan)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    if check_plan:
        check_same_plan(ss.info)
    block = partition(slice_ids, world, rank)
    if out is None:
        out = torch.empty(ss.M, dtype=torch.complex64, device=torch.device("cuda", ss._dev))
    if block:
        ss.contract(block, out=out)
    else:
        out.zero_()
    return allreduce_amplitudes(out)
