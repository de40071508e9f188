"""Measure real per-contraction time of several planner settings on config C (plan selection is setup).
python tools/plan_sweep.py CFG 'seed:trials:budget[:c]' ...   (:c = companion-edge truncation)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import paper_2111_03011_b200 as T  # noqa: E402
from tn_inputs import configs  # noqa: E402

cfg = int(sys.argv[1])
c = configs.get(cfg)
circ = c.circuit()
n = circ["n"]
bits = c.bitstrings(n)
for spec in sys.argv[2:]:
    parts = spec.split(":")
    seed, trials, budget = (int(x) for x in parts[:3])
    comp = len(parts) > 3 and parts[3] == "c"  # 'seed:trials:budget:c' plans with companion edges
    ss = T.SparseState(circ, bits, c.open_mask(n))
    t0 = time.time()
    info = ss.plan(1 << c.log2_tmax, n_sliced=c.n_sliced, seed=seed, trials=trials, time_budget_s=budget,
                   companions=comp)
    tp = time.time() - t0
    ss.bind(0, pipelines=16)
    S = range(1 << info["s"])
    ss.contract(S)
    _, first = ss.contract(S, timed=True)
    if first > 0.3:  # a slow plan: report and move on (keeps long sweeps short)
        print(f"seed={seed} trials={trials} budget={budget} companions={comp}: plan {tp:.1f}s cmac "
              f"{info['cmac_per_slice']:.3g} -> {first * 1e3:.0f} ms (skipped)", flush=True)
        ss.close()
        del ss
        torch.cuda.empty_cache()
        continue
    best = 1e9
    for _ in range(3):
        _, secs = ss.contract(S, timed=True)
        best = min(best, secs)
    print(f"seed={seed} trials={trials} budget={budget} companions={comp}: plan {tp:.1f}s cmac {info['cmac_per_slice']:.3g} "
          f"bytes {info['bytes_per_slice']:.3g} -> {best * 1e3:.1f} ms ({(1 << info['s']) / best:.0f} slices/s)",
          flush=True)
    ss.close()
    del ss
    torch.cuda.empty_cache()
