"""Run config C's plan for a few slices (for ncu captures): python tools/one_slice.py [cfg] [n_slices]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_03011_b200 as T  # noqa: E402
from tn_inputs import configs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 1
c = configs.get(cfg)
circ = c.circuit()
n = circ["n"]
ss = T.SparseState(circ, c.bitstrings(n), c.open_mask(n))
info = ss.plan(1 << c.log2_tmax, **c.plan_kwargs())
ss.bind(0)
amps = ss.contract(range(ns))
torch.cuda.synchronize()
print("ok", info["s"], float(amps.abs().pow(2).sum()))
