"""53-qubit Sycamore sparse-state run: python tools/syc53.py M_CYCLES LOG2_TMAX N_SLICES(-1=all) [pipelines]
Prints plan, per-slice time, and F_norm = (2^n/M) sum |a|^2 of the summed slices."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_03011_b200 as T  # noqa: E402
from tn_inputs import bitstrings as bs  # noqa: E402
from tn_inputs import circuits as cc  # noqa: E402

m = int(sys.argv[1])
tm = int(sys.argv[2])
ns = int(sys.argv[3])
pipes = int(sys.argv[4]) if len(sys.argv) > 4 else 8
n = 53
openq = [11, 19, 28, 29, 37, 44]
circ = cc.generate_circuit(cc.sycamore53_layout(), m, "ABCDCDAB", 1004)
bits = bs.generate_groups(n, openq, 1 << 14, 2004)
t0 = time.time()
ss = T.SparseState(circ, bits, bs.qubit_mask(n, openq))
info = ss.plan(1 << tm, n_sliced=-1, seed=1, time_budget_s=60)
print("plan", round(time.time() - t0, 1), "s", {k: v for k, v in info.items() if k != "sliced_wires"}, flush=True)
ss.bind(0, pipelines=pipes)
print("pipelines", ss.pipelines, flush=True)
S = list(range(1 << info["s"])) if ns < 0 else list(range(ns))
ss.contract(S[: max(1, min(len(S), 2 * ss.pipelines))])   # warm-up
torch.cuda.synchronize()
amps, secs = ss.contract(S, timed=True)
a = amps.cpu().numpy().astype(complex)
fn = (2.0 ** n / len(a)) * np.sum(np.abs(a) ** 2)
print(f"m={m} slices={len(S)} of 2^{info['s']}: {secs:.3f} s, {len(S) / secs:.1f} slices/s, "
      f"{8 * info['cmac_per_slice'] * len(S) / secs / 1e12:.1f} complex TFLOP/s, F_norm {fn:.4f} "
      f"(fraction {len(S) / 2 ** info['s']:.4g})", flush=True)
