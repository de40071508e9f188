"""Config 4 (53q Sycamore, m=14, M=2^20) as a loop program from a plan file: bind, contract a few global
slices, time them (CUDA events) and print the per-kind launch profile of one pass through every segment.
    python tools/syc53_loop.py PLAN_FILE [n_slices] [max_tensor_log2]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_03011_b200 as T  # noqa: E402
from tn_inputs import configs  # noqa: E402

path = sys.argv[1]
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 1
tm = int(sys.argv[3]) if len(sys.argv) > 3 else 30
c = configs.get(4)
circ = c.circuit()
n = circ["n"]
bits = c.bitstrings(n)
t0 = time.time()
ss = T.SparseState(circ, bits, c.open_mask(n))
info = ss.plan(1 << tm, plan_path=path)
print("plan", round(time.time() - t0, 1), "s", {k: v for k, v in info.items()
                                               if k not in ("sliced_wires", "local_wires", "companions")}, flush=True)
ss.bind(0, pipelines=1)
print("bound; workspace GB", ss._work.numel() / 1e9, flush=True)
prof = ss.profile_slice(0)
agg = {}
for p in prof:
    a = agg.setdefault(p["kind"], [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += p["ms"]
    a[2] += p["cmac"]
    a[3] += p["bytes"]
tot = sum(a[1] for a in agg.values())
print(f"one pass through every segment: {tot:.1f} ms, {len(prof)} launches", flush=True)
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:14s} n {a[0]:4d}  {a[1]:9.2f} ms  {a[2] / max(a[1], 1e-9) / 1e9:8.2f} TCMAC/s  "
          f"{a[3] / max(a[1], 1e-9) / 1e9:8.1f} GB/s", flush=True)
top = sorted(prof, key=lambda p: -p["ms"])[:12]
for p in top:
    print("   ", p, flush=True)
torch.cuda.synchronize()
amps, secs = ss.contract(range(ns), timed=True)
a = amps.cpu().numpy()
print(f"{ns} global slices: {secs:.3f} s ({secs / ns:.3f} s per global slice); |a|^2 sum {np.sum(np.abs(a) ** 2):.4e}; "
      f"F_norm of this partial sum {(2.0 ** n / len(a)) * np.sum(np.abs(a) ** 2):.4e}", flush=True)
