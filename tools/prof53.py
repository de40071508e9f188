"""Per-launch profile of one slice of the 53-qubit Sycamore m=M run: python tools/prof53.py M LOG2_TMAX [top]"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_03011_b200 as T  # noqa: E402
from tn_inputs import bitstrings as bs  # noqa: E402
from tn_inputs import circuits as cc  # noqa: E402

m, tm = int(sys.argv[1]), int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
n = 53
openq = [11, 19, 28, 29, 37, 44]
circ = cc.generate_circuit(cc.sycamore53_layout(), m, "ABCDCDAB", 1004)
bits = bs.generate_groups(n, openq, 1 << 14, 2004)
ss = T.SparseState(circ, bits, bs.qubit_mask(n, openq))
info = ss.plan(1 << tm, n_sliced=-1, seed=1, time_budget_s=60)
ss.bind(0, pipelines=1)
ss.contract([0])
p = ss.profile_slice(0)
agg = defaultdict(lambda: [0, 0.0, 0.0])
for x in p:
    agg[x["kind"]][0] += 1
    agg[x["kind"]][1] += x["ms"]
    agg[x["kind"]][2] += x["bytes"]
tot = sum(x["ms"] for x in p)
print(f"total {tot:.2f} ms in {len(p)} launches; plan bytes/slice {info['bytes_per_slice'] / 1e9:.1f} GB")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:14s} {v[0]:4d} launches {v[1]:9.2f} ms {100 * v[1] / tot:5.1f}%  {v[2] / max(v[1], 1e-9) / 1e6:7.0f} GB/s")
for x in sorted(p, key=lambda x: -x["ms"])[:top]:
    bw = x["bytes"] / (x["ms"] * 1e-3) / 1e9 if x["ms"] > 0 else 0
    fl = 8 * x["cmac"] / (x["ms"] * 1e-3) / 1e12 if x["ms"] > 0 else 0
    print(f"  {x['kind']:13s} step {x['step']:4d} {x['ms']:8.3f} ms  m={x['m']} n={x['n']} k={x['k']} rows={x['rows']}"
          f"  {bw:7.0f} GB/s  {fl:6.1f} cTFLOP/s")
