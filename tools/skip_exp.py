"""Throughput of variants with concurrent pipelines: each argument is "VAR=val;VAR2=val" env settings read at
bind (e.g. TNB_SKIP=k1 drops launch kind 1: outputs are then wrong, timing only).  Needs a diagnostics build:
TNB_NVCC_FLAGS=-DTNB_DIAG_SKIP python -m paper_2111_03011_b200.build (the product build ignores TNB_SKIP)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_03011_b200 as T
from tn_inputs import configs
cfg = int(os.environ.get("CFG", "3"))
c = configs.get(cfg); circ = c.circuit(); n = circ["n"]
ss = T.SparseState(circ, c.bitstrings(n), c.open_mask(n))
info = ss.plan(1 << c.log2_tmax, **c.plan_kwargs())
ns = 1 << len(info["sliced_wires"])
pipes = int(os.environ.get("PIPES", "16"))
variants = sys.argv[1:] or [""]
if variants == ["each"]:  # every launch of the per-slice graph, skipped one at a time
    ss.bind(0, pipelines=1)
    prof = ss.profile_slice(0)
    kinds = {"instantiate": 0, "apply": 1, "prep_a": 2, "prep_b": 3, "gemm_tcgen05": 4, "readout": 5, "multi": 7}
    variants = [""] + [f"TNB_SKIP=x{kinds[x['kind']]}_{x['step']}" for x in prof if x["ms"] > 0.015]
    ms = {f"TNB_SKIP=x{kinds[x['kind']]}_{x['step']}": x["ms"] for x in prof}
for v in variants:
    for k in ("TNB_SKIP", "TNB_RG"):
        os.environ.pop(k, None)
    for kv in filter(None, v.split(";")):
        k, val = kv.split("=")
        os.environ[k] = val
    ss.bind(0, pipelines=pipes)
    ts = []
    for r in range(6):
        _, sec = ss.contract(range(ns), timed=True)
        ts.append(sec)
    ts = sorted(ts[2:])
    thr = ns / ts[len(ts) // 2]
    if not v:
        base = thr
    extra = ""
    if v and "base" in globals():
        extra = f"  marginal {1e3 / base - 1e3 / thr:.4f} ms/slice"
        if "ms" in globals() and v in ms:
            extra += f"  (serialized {ms[v]:.4f} ms)"
    print(f"{v!r:28s} {thr:8.1f} slices/s  (min {ns/ts[-1]:.1f} max {ns/ts[0]:.1f}){extra}", flush=True)
