"""Diagnostics for loop programs on the GPU: plan config 2 as a loop program with J segments, contract, and
compare with the oracle (prints per-variant rel L2 and the launch profile of one pass)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2111_03011_b200 as T  # noqa: E402
from oracle import sv  # noqa: E402
from tn_inputs import configs  # noqa: E402

c = configs.get(2)
circ = c.circuit()
n = circ["n"]
bits = c.bitstrings(n)
want, _ = sv.amplitudes(circ, bits)
for tm, J, ng, pipes in [(20, 1, 2, 1), (14, 1, 2, 1), (12, 1, 10, 1), (12, 2, 2, 1), (12, 8, 2, 1), (12, 8, 2, 4)]:
    ss = T.SparseState(circ, bits, c.open_mask(n))
    info = ss.plan(1 << tm, n_sliced=ng, method=2, max_segments=J, time_budget_s=2.0)
    ss.bind(0, pipelines=pipes)
    a = ss.contract(range(1 << info["s"])).cpu().numpy()
    err = np.linalg.norm(a - want) / np.linalg.norm(want)
    print(f"tmax 2^{tm} J {J} ng {ng} pipes {pipes}: s {info['s']} local {info['s_local']} segs {info['n_segments']} "
          f"rel L2 {err:.3e} |a| {np.linalg.norm(a):.3e}", flush=True)
    if err > 1e-3 and info["s"] > 0:
        W = info["sliced_wires"]
        a0 = ss.contract([0]).cpu().numpy()
        w0 = sv.sliced_amplitudes(circ, bits, W, [0])
        print("   slice 0 rel", np.linalg.norm(a0 - w0) / np.linalg.norm(w0), "|a0|", np.linalg.norm(a0), flush=True)
        prof = ss.profile_slice(0)
        print("   launches:", [(p["kind"], p["step"], round(p["ms"], 4)) for p in prof][:40], flush=True)
