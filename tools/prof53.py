"""Weighted launch profile of a loop program (config 4 by default): one pass through every segment with CUDA
events (tn_profile_slice), each launch weighted by its segment's runs in a block of B global slices
(tn_segment_runs); prints the top launches by weighted time with their shapes.
    python tools/prof53.py [plan_file] [B] [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_03011_b200 as T  # noqa: E402
from tn_inputs import configs  # noqa: E402

plan = sys.argv[1] if len(sys.argv) > 1 else "plans/config4.json"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 4
c = configs.get(cfg)
circ = c.circuit()
n = circ["n"]
ss = T.SparseState(circ, c.bitstrings(n), c.open_mask(n))
info = ss.plan(1 << c.log2_tmax, plan_path=plan)
ss.bind(0, pipelines=1)
prof = ss.profile_slice(0)
runs = ss.segment_runs(range(B))
tot = 0.0
rows = []
for i, p in enumerate(prof):
    w = runs[p["seg"]] if p["seg"] >= 0 else B
    tot += p["ms"] * w
    rows.append((p["ms"] * w, i, w, p))
rows.sort(key=lambda r: -r[0])
print(f"block of {B} global slices: weighted {tot:.1f} ms; runs per segment {runs}", flush=True)
acc = 0.0
for wms, i, w, p in rows[:40]:
    acc += wms
    print(f"{wms:9.2f} ms ({100 * wms / tot:5.1f} %, cum {100 * acc / tot:5.1f} %) launch {i:3d} x{w}: {p['kind']:12s} "
          f"step {p['step']:3d} seg {p['seg']} ms {p['ms']:.3f} m {p['m']} n {p['n']} k {p['k']} rows {p['rows']} "
          f"GB {p['bytes'] / 1e9:.2f} GCMAC {p['cmac'] / 1e9:.2f} -> {p['bytes'] / p['ms'] / 1e6:.0f} GB/s", flush=True)

# whole-run and fidelity-prefix extrapolation from the measured per-run segment times (one profiled pass):
# segment j runs 2^|D_j| times over all global slices; over the prefix [0, 2^p) of global slice ids (fidelity
# ~ 2^p / 2^s, PAPER.md L77 / L152) it runs 2^|D_j n (local bits u last p global bits)| times
import json  # noqa: E402
import math  # noqa: E402
import tempfile  # noqa: E402

with tempfile.NamedTemporaryFile(suffix=".json", delete=False) as f:
    pth = f.name
ss.save_plan(pth)
pf = json.load(open(pth))
os.unlink(pth)
ns = len(pf["sliced"])
glob = [i for i in range(ns) if pf["global"][i]]
local = [i for i in range(ns) if not pf["global"][i]]
seg_ms = {}
for p in prof:
    seg_ms[p["seg"]] = seg_ms.get(p["seg"], 0.0) + p["ms"]
bit = lambda r: 1 << (ns - 1 - r)  # noqa: E731
full = sum(seg_ms.get(j, 0.0) * 2.0 ** bin(int(D)).count("1") for j, (D, _, _) in enumerate(pf["segs"]))
print(f"extrapolated whole run (all 2^{len(glob)} global slices, one GPU, serial profile): {full / 1e3:.4g} s")
for F in (0.002, 0.0037):
    pbits = max(0, min(len(glob), math.ceil(math.log2(F * 2 ** len(glob)))))
    free = 0
    for r in local + glob[len(glob) - pbits:]:
        free |= bit(r)
    t = sum(seg_ms.get(j, 0.0) * 2.0 ** bin(int(D) & free).count("1") for j, (D, _, _) in enumerate(pf["segs"]))
    print(f"F ~ {F}: prefix of 2^{pbits} global slices (fraction {2 ** pbits / 2 ** len(glob):.4g}): {t / 1e3:.4g} s "
          f"on one GPU; {t / 8e3:.4g} s on 8 (weak scaling over slices)")
