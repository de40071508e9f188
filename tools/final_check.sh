#!/bin/bash
# End-of-round measurement on one B200 (run from the repo root under gpurun): DRAM traffic of the dominant kernel
# (k_gate_tc, every launch of one profiled pass of config 4) -> profiles/ncu_traffic.json (read by bench.py's
# roofline.traffic), then the GPU test suite, smoke, the default bench line and the ncu launch list of the bench.
set -u
mkdir -p gpurun_out
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_gate_tc -o gpurun_out/gate_traffic python tools/prof53.py plans/config4.json 1 > gpurun_out/gate_traffic.log 2>&1
python tools/ncu_traffic.py gpurun_out/gate_traffic.ncu-rep k_gate_tc \
    "ncu dram__bytes_{read,write}.sum of every k_gate_tc launch of one profiled pass of config 4 (tools/final_check.sh)" \
    > gpurun_out/gate_traffic.json 2>> gpurun_out/gate_traffic.log
python - <<'PY'
import json
e = json.load(open("gpurun_out/gate_traffic.json"))
e["config"] = 4
json.dump([e], open("profiles/ncu_traffic.json", "w"), indent=1)
print(e)
PY
rm -f gpurun_out/gate_traffic.ncu-rep
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_final.log 2>&1
tail -3 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 400 --csv \
    --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline \
    > gpurun_out/launches_final.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
