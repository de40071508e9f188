"""Throughput of variants with concurrent pipelines: each argument is "VAR=val;VAR2=val" env settings read at
bind (e.g. TNB_SKIP=k1 drops launch kind 1: outputs are then wrong, timing only)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2111_03011_b200 as T
from tn_inputs import configs
cfg = int(os.environ.get("CFG", "3"))
c = configs.get(cfg); circ = c.circuit(); n = circ["n"]
ss = T.SparseState(circ, c.bitstrings(n), c.open_mask(n))
info = ss.plan(1 << c.log2_tmax, **c.plan_kwargs())
ns = 1 << len(info["sliced_wires"])
pipes = int(os.environ.get("PIPES", "16"))
variants = sys.argv[1:] or [""]
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
    print(f"{v!r:28s} {ns / ts[len(ts)//2]:8.1f} slices/s  (min {ns/ts[-1]:.1f} max {ns/ts[0]:.1f})", flush=True)
