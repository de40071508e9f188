"""Serialized per-launch GEMM times of one config-3 slice under env variants (A/B of GEMM tile choices)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_03011_b200 as T
from tn_inputs import configs
c = configs.get(int(os.environ.get("CFG", "3"))); circ = c.circuit(); n = circ["n"]
ss = T.SparseState(circ, c.bitstrings(n), c.open_mask(n))
info = ss.plan(1 << c.log2_tmax, **c.plan_kwargs())
for v in sys.argv[1:]:
    for kv in filter(None, v.split(";")):
        k, val = kv.split("="); os.environ[k] = val
    ss.bind(0, pipelines=1)
    ss.contract([0])
    for rep in range(3):
        p = ss.profile_slice(0)
    rows = [x for x in p if x["kind"] == "gemm_tcgen05"]
    tot = sum(x["ms"] for x in rows)
    kinds = {}
    for x in p:
        kinds[x["kind"]] = kinds.get(x["kind"], 0.0) + x["ms"]
    print(f"{v:12s} gemm total {tot:.4f} ms: " + " ".join(f"s{x['step']}:{x['ms']:.4f}" for x in rows), flush=True)
    print("    kinds: " + " ".join(f"{k}:{t:.3f}" for k, t in sorted(kinds.items(), key=lambda kv: -kv[1])) +
          f"  total {sum(kinds.values()):.3f} ms in {len(p)} launches", flush=True)
