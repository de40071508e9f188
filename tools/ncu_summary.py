"""Summarise an ncu --set full report: per launch duration, DRAM bytes, tensor/FMA pipe, SM throughput.
python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]


def to_num(v, u):
    v = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
    return v * scale.get(u, 1)


out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
idx = {w: hdr.index(w) for w in WANT if w in hdr}
kn = hdr.index("Kernel Name")
gs = hdr.index("Grid Size")
print("kernel | grid | us | DRAM MB (r+w) | DRAM GB/s | dram% | tensor% | fma% | sm% | L2 MB | regs")
for r in rows[2:]:
    d = {w: to_num(r[i], units[i]) for w, i in idx.items()}
    us = d["gpu__time_duration.sum"]
    mb = (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / 1e6
    print(f"{r[kn].split('(')[0][:28]} | {r[gs]} | {us:.1f} | {mb:.1f} | {mb * 1e3 / us:.0f} | "
          f"{d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
          f"{d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
          f"{d.get('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
          f"{d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
          f"{d.get('lts__t_bytes.sum', 0) / 1e6:.1f} | {d.get('launch__registers_per_thread', 0):.0f}")
