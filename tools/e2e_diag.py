"""Per-step wall vs device time of tn_contract on config 3 (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import paper_2111_03011_b200 as T  # noqa: E402
from tn_inputs import configs  # noqa: E402

c = configs.get(3)
circ = c.circuit()
n = circ["n"]
ss = T.SparseState(circ, c.bitstrings(n), c.open_mask(n))
info = ss.plan(1 << c.log2_tmax, **c.plan_kwargs())
ss.bind(0, pipelines=16)
ids = list(range(256))
out = torch.empty(ss.M, dtype=torch.complex64, device="cuda")
host = torch.empty(ss.M, dtype=torch.complex64).pin_memory()
for _ in range(3):
    ss.contract(ids, out=out)
torch.cuda.synchronize()
for i in range(8):
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    ss.contract(ids, out=out)
    torch.cuda.synchronize()
    print(f"untimed step {i}: {1e3 * (time.perf_counter() - w0):7.1f} ms", flush=True)
for i in range(8):
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    _, secs = ss.contract(ids, out=out, timed=True)
    w1 = time.perf_counter()
    host.copy_(out, non_blocking=True)
    torch.cuda.synchronize()
    w2 = time.perf_counter()
    print(f"step {i}: contract-call {1e3 * (w1 - w0):7.1f} ms  device {1e3 * secs:7.1f} ms  total {1e3 * (w2 - w0):7.1f} ms",
          flush=True)
