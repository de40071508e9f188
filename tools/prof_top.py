"""Per-launch device times of one slice (tn_profile_slice) for config C: python tools/prof_top.py [cfg] [top]"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_03011_b200 as T  # noqa: E402
from tn_inputs import configs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = configs.get(cfg)
circ = c.circuit()
n = circ["n"]
ss = T.SparseState(circ, c.bitstrings(n), c.open_mask(n))
info = ss.plan(1 << c.log2_tmax, **c.plan_kwargs())
print({k: v for k, v in info.items() if k != "sliced_wires"})
ss.bind(0)
ss.contract([0])
p = ss.profile_slice(0)
p = ss.profile_slice(0)
agg = defaultdict(lambda: [0, 0.0])
for x in p:
    agg[x["kind"]][0] += 1
    agg[x["kind"]][1] += x["ms"]
tot = sum(x["ms"] for x in p)
print(f"total {tot:.3f} ms in {len(p)} launches")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:14s} {v[0]:4d} launches {v[1]:8.3f} ms {100 * v[1] / tot:5.1f}%")
for x in sorted(p, key=lambda x: -x["ms"])[:top]:
    bw = x["bytes"] / (x["ms"] * 1e-3) / 1e9 if x["ms"] > 0 else 0
    fl = 8 * x["cmac"] / (x["ms"] * 1e-3) / 1e12 if x["ms"] > 0 else 0
    print(f"  {x['kind']:13s} step {x['step']:4d} {x['ms']:8.4f} ms  m={x['m']} n={x['n']} k={x['k']} rows={x['rows']}"
          f"  {bw:7.0f} GB/s  {fl:6.1f} cTFLOP/s")
n_small = sum(1 for x in p if x["ms"] < 0.02)
print("launches < 20us:", n_small, "sum ms", sum(x["ms"] for x in p if x["ms"] < 0.02))
