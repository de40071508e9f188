"""DRAM traffic per launch of one kernel from an ncu --set full report, as JSON for bench.py's
roofline.traffic: python tools/ncu_traffic.py report.ncu-rep <kernel substring> <source label> [name] [last N]
(name: the kernel name bench.py reports, default the substring; last N: average over the last N matching
launches only, e.g. one slice after the prologue)"""
import csv
import io
import json
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
kn = hdr.index("Kernel Name")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
match = [r for r in rows[2:] if sys.argv[2] in r[kn]]
if len(sys.argv) > 5:
    match = match[-int(sys.argv[5]):]
tot = sum(float(r[ir].replace(",", "")) * scale[units[ir]] + float(r[iw].replace(",", "")) * scale[units[iw]]
          for r in match)
n = len(match)
print(json.dumps({"kernel": sys.argv[4] if len(sys.argv) > 4 else sys.argv[2], "launches": n,
                  "dram_bytes_per_launch": tot / max(n, 1), "source": sys.argv[3]}))
