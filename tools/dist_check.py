"""Multi-GPU parity: torchrun --nproc-per-node N tools/dist_check.py [cfg]
Each rank contracts its contiguous block of all slices, NCCL all-reduce, rank 0 compares with the oracle."""
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
ss = T.SparseState(circ, bits, c.open_mask(n))
info = ss.plan(1 << c.log2_tmax, **c.plan_kwargs())
ss.bind(local)
S = list(range(1 << info["s"]))
amps = contract_distributed(ss, S).cpu().numpy()
if rank == 0:
    from oracle import sv
    want = sv.sliced_amplitudes(circ, bits, info["sliced_wires"], S) if n <= 24 else None
    single = None
    if want is not None:
        err = np.linalg.norm(amps - want) / np.linalg.norm(want)
        print(f"world={world} cfg={cfg} rel L2 vs oracle {err:.2e}", flush=True)
        assert err < 1e-4
dist.barrier()
dist.destroy_process_group()
