"""Multi-GPU parity: torchrun --nproc-per-node N tools/dist_check.py [cfg] [method]
Rank 0 plans (method 1 flat / 2 loop program) and saves the plan file; every rank imports it, contracts its
contiguous block of all (global) slices, NCCL all-reduce (contract_distributed, which also compares the ranks'
plan fingerprints); rank 0 compares with the oracle's exact amplitudes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2111_03011_b200 as T  # noqa: E402
from paper_2111_03011_b200.dist import contract_distributed  # noqa: E402
from tn_inputs import configs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
c = configs.get(cfg)
circ = c.circuit()
n = circ["n"]
bits = c.bitstrings(n)
method = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ss = T.SparseState(circ, bits, c.open_mask(n))
path = f"/tmp/dist_check_plan_{cfg}_{method}.json"
tmax = 1 << (c.log2_tmax if method == 1 else 12)
if rank == 0:
    ss.plan(tmax, **(c.plan_kwargs() if method == 1 else {"n_sliced": 3, "method": 2, "time_budget_s": 5.0}))
    ss.save_plan(path)
dist.barrier()
info = ss.plan(tmax, plan_path=path)
ss.bind(local)
S = list(range(1 << info["s"]))
amps = contract_distributed(ss, S).cpu().numpy()
if rank == 0:
    from oracle import sv
    want = sv.amplitudes(circ, bits)[0] if n <= 24 else None
    single = None
    if want is not None:
        err = np.linalg.norm(amps - want) / np.linalg.norm(want)
        print(f"world={world} cfg={cfg} method={method} slices={len(S)} local bits={info['s_local']} "
              f"rel L2 vs oracle {err:.2e}", flush=True)
        assert err < 1e-4
dist.barrier()
dist.destroy_process_group()
