"""Validation of the sparse-state sampler on a desk-scale Sycamore-style circuit, after the paper's
supplement: for K broken (sliced) edges, compare the
fraction estimate f = 2^-K, the norm estimate F_norm, the true fidelity of the
approximate state over the requested bitstrings, and the linear / logarithmic XEB of one sample per
group (categorical and Metropolis) under the exact state; the entropy of the samples against the
entropy of the sparse state; and XEB as a function of the group size l.

Everything runs through the product (tn_contract, tn_sample_report): the exact amplitudes are the sum of
all 2^s slices, psi_K is the prefix with the first K sliced wires pinned to 0.

    python tools/validation.py [--rows 4 --cols 6 --cycles 14 --seq EFGH --L 65536 --K 8 --reps 4]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_03011_b200 as T  # noqa: E402
from tn_inputs import bitstrings as bs  # noqa: E402
from tn_inputs import circuits as cc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=4)
ap.add_argument("--cols", type=int, default=5)
ap.add_argument("--cycles", type=int, default=14)
ap.add_argument("--seq", default="EFGH")
ap.add_argument("--L", type=int, default=1024)
ap.add_argument("--K", type=int, default=8)
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--seed", type=int, default=7)
ap.add_argument("--steps", type=int, default=1000, help="Metropolis chain length (the paper gives none)")
ap.add_argument("--tmax", type=int, default=22, help="log2 max_tensor_size of the plan")
ap.add_argument("--out", default="")
args = ap.parse_args()

circ = cc.generate_circuit(cc.rect_layout(args.rows, args.cols), args.cycles, args.seq, args.seed)
n = circ["n"]
rows = []


def run(n_open, K, label):
    opens = list(range(n - n_open, n))
    bits = bs.generate_groups(n, opens, args.L, args.seed + 1)
    ss = T.SparseState(circ, bits, bs.qubit_mask(n, opens))
    info = ss.plan(1 << args.tmax, n_sliced=K, seed=1, trials=8, time_budget_s=300)
    s = info["s"]
    ss.bind(0, pipelines=4)
    exact = ss.contract(range(1 << s)).cpu().numpy()
    out = []
    for k in range(0, s + 1):  # k edges broken: slices [0, 2^(s-k)) = first k sliced wires pinned to 0
        nS = 1 << (s - k)
        approx = ss.contract(range(nS)).cpu().numpy()
        a, b = exact.astype(complex), approx.astype(complex)
        f_true = abs(np.vdot(a, b)) ** 2 / (np.vdot(a, a).real * np.vdot(b, b).real)
        row = {"label": label, "n": n, "l": 1 << n_open, "L": args.L, "K": k, "f": nS / (1 << s), "F_true": f_true}
        for sampler in ("categorical", "metropolis"):
            xs, ls, hs, ht = [], [], [], []
            for rep in range(args.reps):
                _, _, r = ss.sample_report(approx, nS, 1000 + rep, sampler=sampler, steps=args.steps, ideal=exact)
                xs.append(r["xeb"])
                ls.append(r["log_xeb"])
                hs.append(r["entropy_samples"])
                ht.append(r["entropy_state"])
                row["F_norm"] = r["F_norm"]
                row["pt_ks"] = r["pt_ks"]
            row[f"xeb_{sampler}"] = float(np.mean(xs))
            row[f"xeb_{sampler}_sem"] = float(np.std(xs) / np.sqrt(len(xs)))
            row[f"log_xeb_{sampler}"] = float(np.mean(ls))
            row[f"log_xeb_{sampler}_sem"] = float(np.std(ls) / np.sqrt(len(ls)))
            row[f"entropy_samples_{sampler}"] = float(np.mean(hs))
            row["entropy_state"] = float(np.mean(ht))
        out.append(row)
        print(json.dumps(row), flush=True)
    ss.close()
    return out


rows += run(6, args.K, "fidelity-vs-K")
for o in (1, 2, 3, 4, 5):  # XEB vs group size l at K broken edges
    rows += [r for r in run(o, args.K, "xeb-vs-l") if r["K"] == args.K]
if args.out:
    with open(args.out, "w") as fh:
        json.dump({"circuit": {"rows": args.rows, "cols": args.cols, "cycles": args.cycles, "seq": args.seq,
                               "seed": args.seed}, "rows": rows}, fh, indent=1)
