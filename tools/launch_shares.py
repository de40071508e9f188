"""Per-kernel shares of an ncu launch list (--metrics gpu__time_duration.sum --csv):
python tools/launch_shares.py launches.csv"""
import csv
import sys
from collections import defaultdict

lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))  # skip ncu's ==PROF== / warning lines
rows = [r for r in csv.DictReader(lines[start:]) if r.get("Metric Name") == "gpu__time_duration.sum"]
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    name = name.split("::")[-1] if "k_gemm" not in name else name.split("tc::")[-1]
    agg[name][0] += 1
    agg[name][1] += float(r["Metric Value"].replace(",", "")) / 1e3  # us
tot = sum(v[1] for v in agg.values())
print(f"{len(rows)} launches, {tot:.1f} us serialized (cold cache, ncu)")
print("kernel | launches | us | share")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k} | {n} | {us:.1f} | {100 * us / tot:.1f}%")
