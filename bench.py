#!/usr/bin/env python
"""Benchmark of the sliced sparse-state contraction (arXiv:2111.03011) on B200.

    python bench.py [--gpus N --steps K --warmup W --config C --impl {ours,reference}]

A step = one tn_contract over the workload's whole slice set S (slice
instantiate, pairwise contractions, readout+accumulate) plus, for N > 1, the NCCL all-reduce of the M
amplitudes.  S is split into N contiguous blocks (strong scaling: the total work is fixed).
Metric (BASELINE.json): slices/s (aggregate over ranks) with complex TFLOP/s (8 x CMAC/s) and
the roofline fraction of the dominant kernel alongside.

Rank 0 prints ONE JSON line.  Multi-GPU: launched by torch.distributed.run (one rank per GPU, NCCL).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# concurrent slice pipelines use one stream each: give every stream its own hardware queue
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from tn_inputs import configs  # noqa: E402

METRIC = "slices/sec & complex TFLOP/s (frac of peak) at 1/2/4/8 B200; time to 1e6 amplitudes"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16": d["bf16_tflops"], "bf16_sust": d["bf16_tflops_sustained"],
                "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16": 1590.0, "bf16_sust": 1400.0, "src": "fallback (B200_PROFILING.md)"}


# ------------------------------------------------------------------------------ clocks sampler

class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------------ oracle (CPU baseline)

def oracle_sample(cfg, max_seconds: float = 20.0):
    """Time the oracle (oracle/sv.c, fp64 state vector, OpenMP over all host cores) on a bounded sample of
    one slice of the workload: the first G gate passes of the projector-inserted state-vector run of
    slice 0, with G grown until ~max_seconds of CPU work; extrapolated linearly to the whole circuit
    (one slice = one full run over all gates)."""
    from oracle import sv  # test infrastructure: allowed only in this leg
    from tn_inputs import circuits as cc
    circ = cfg.circuit()
    gates = cc.gate_list(circ)
    G = len(gates)
    cores = os.cpu_count() or 1
    take = 4
    t_used = 0.0
    while True:
        sub = dict(circ)
        sub["moments"] = [gates[:take]]
        t0 = time.perf_counter()
        sv.amplitudes(sub, np.zeros(1, np.uint64), threads=cores)
        t_used = time.perf_counter() - t0
        if t_used > max_seconds / 3 or take >= G:
            break
        take = min(G, take * 4)
    # subtract nothing: state allocation + |0> init are part of the oracle run as it stands
    per_slice = t_used * G / take
    return {"kind": "oracle", "cores": cores, "value": 1.0 / per_slice, "unit": "slices/s",
            "sample": f"first {take} of {G} gate passes of one {circ['n']}-qubit slice (fp64 state vector, "
                      f"{cores} OpenMP threads), {t_used:.1f} s, extrapolated linearly to {per_slice:.1f} s/slice"}


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    steps = []
    for _ in range(args.warmup):
        oracle_sample(cfg, max_seconds=args.ref_seconds)
    for _ in range(args.steps):
        steps.append(oracle_sample(cfg, max_seconds=args.ref_seconds))
    v = statistics.median(s["value"] for s in steps)
    s0 = steps[-1]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "slices/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / v, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg),
            "cpu_baseline": {"kind": "oracle", "cores": s0["cores"], "value": v, "unit": "slices/s",
                             "sample": s0["sample"]},
            "e2e": {"value": v, "unit": "slices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ our arm

def workload_config(cfg) -> dict:
    """The workload keys both arms report (the GPU arm adds its run-specific keys)."""
    n = cfg.circuit()["n"]
    M = cfg.L << len(cfg.open_ids(n))
    s = cfg.n_sliced
    return {"workload": f"config{cfg.cfg}: {cfg.name} ({cfg.layout}, m={cfg.cycles}, M={M}, 2^{s} slices all summed)",
            "n_qubits": n, "cycles": cfg.cycles, "M": M, "L": cfg.L, "l": 1 << len(cfg.open_ids(n)),
            "slices": 1 << s, "max_tensor_size": 1 << cfg.log2_tmax}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=20.0)
    ap.add_argument("--trials", type=int, default=0)
    ap.add_argument("--pipelines", type=int, default=16)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = configs.get(args.config)

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    import paper_2111_03011_b200 as T

    # ------------------------------------------------------------ setup (not timed): build, plan, bind
    t0 = time.perf_counter()
    circ = cfg.circuit()
    n = circ["n"]
    bits = cfg.bitstrings(n)
    ss = T.SparseState(circ, bits, cfg.open_mask(n))
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    pk = cfg.plan_kwargs()
    if args.trials:
        pk["trials"] = args.trials
    info = ss.plan(1 << cfg.log2_tmax, **pk)
    t_plan = time.perf_counter() - t0
    if world > 1:  # every rank must contract the same sliced network: compare plan fingerprints
        fp = torch.tensor([float(hash(tuple(info["sliced_wires"])) % (1 << 52)), info["cmac_per_slice"]],
                          dtype=torch.float64, device=dev)
        allfp = [torch.zeros_like(fp) for _ in range(world)]
        dist.all_gather(allfp, fp)
        if any(not torch.equal(allfp[0], x) for x in allfp):
            raise RuntimeError("ranks produced different plans; refusing to sum inconsistent slices")
    t0 = time.perf_counter()
    stream = torch.cuda.current_stream(dev)
    ss.bind(local, stream=stream, pipelines=args.pipelines)
    torch.cuda.synchronize()
    t_bind = time.perf_counter() - t0
    s = info["s"]
    nS = 1 << s
    from paper_2111_03011_b200.dist import partition
    block = partition(range(nS), world, rank)
    M = ss.M

    out = torch.empty(M, dtype=torch.complex64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    def step(dst):
        if block:
            ss.contract(block, out=dst)
        else:
            dst.zero_()
        if world > 1:
            dist.all_reduce(torch.view_as_real(dst), op=dist.ReduceOp.SUM)

    for _ in range(args.warmup):
        step(out)
    torch.cuda.synchronize()

    # ------------------------------------------------------------ device-timed steps
    clk = Clocks(local)
    clk.start()
    total_ms = 0.0
    for _ in range(args.steps):
        flush.zero_()                                   # L2 flush between timed iterations (untimed)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(out)
        e1.record(stream)
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
    clocks = clk.stop()
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    slices_per_s = nS / (ms_per_step * 1e-3)

    def spin_sync():
        """Wait for the device by polling an event (blocking waits on this KVM host wake up late)."""
        ev = torch.cuda.Event()
        ev.record(stream)
        while not ev.query():
            pass

    # ------------------------------------------------------------ end to end through the public API
    # host -> device: the step's slice ids from pinned host memory (inside tn_contract); device -> host:
    # the M amplitudes (pinned); plus the all-reduce for N > 1.
    ids_pinned = torch.tensor(block if block else [0], dtype=torch.int64).pin_memory()
    host_out = torch.empty(M, dtype=torch.complex64).pin_memory()
    e2e_ms = 0.0
    e2e_each = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        w0 = time.perf_counter()
        ids = ids_pinned.numpy().astype(np.uint64) if block else []
        if block:
            ss.contract(ids, out=out)
        else:
            out.zero_()
        if world > 1:
            dist.all_reduce(torch.view_as_real(out), op=dist.ReduceOp.SUM)
        host_out.copy_(out, non_blocking=True)
        spin_sync()
        e2e_each.append((time.perf_counter() - w0) * 1e3)
        e2e_ms += e2e_each[-1]
    t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item()) / args.steps

    # ------------------------------------------------------------ per-launch profile (live, CUDA events)
    prof = ss.profile_slice(block[0] if block else 0)
    launches_per_slice = len(prof)
    by_kind = {}
    for p in prof:
        k = p["kind"]
        d = by_kind.setdefault(k, {"ms": 0.0, "launches": 0, "bytes": 0.0, "cmac": 0.0})
        d["ms"] += p["ms"]
        d["launches"] += 1
        d["bytes"] += p["bytes"]
        d["cmac"] += p["cmac"]
    slice_ms = sum(p["ms"] for p in prof)
    dom = max(by_kind.items(), key=lambda kv: kv[1]["ms"])
    pk = peaks()
    tp = os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else []
    traffic = traffic if isinstance(traffic, list) else [traffic]

    def roofline(kind, d):
        if kind == "gemm_tcgen05":
            # algorithmic work of the 3xTF32 tensor-core GEMM: 3 real GEMMs [Mp x 2K] x [2K x 2N] = 24 flops
            # per complex MAC; peak = TF32 dense = measured bf16 x nominal tf32/bf16 ratio (1.1/2.25)
            achieved = 24.0 * d["cmac"] / (d["ms"] * 1e-3) / 1e12
            peak = pk["bf16"] * (1.1 / 2.25)
            r = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                 "traffic": None, "kernel": "k_gemm_tf32x3", "peak_src": pk["src"] + " bf16 x 1.1/2.25 (tf32)",
                 "useful_complex_tflops": 8.0 * d["cmac"] / (d["ms"] * 1e-3) / 1e12}
        else:
            # SIMT kernels: bound by HBM or by FP32 FMA issue, whichever roofline time is longer.  FP32 peak
            # for register-operand FFMA: 148 SMs x 4 SMSPs x 32 lanes / 2 cycles (reciprocal
            # throughput 2, B300_MICROARCH.md) x 2 flop x 1.965 GHz = 37.2 TFLOP/s; 8 flop per complex MAC
            alu_peak = 148 * 4 * 32 / 2 * 2 * 1.965e9 / 1e12
            bw = d["bytes"] / (d["ms"] * 1e-3) / 1e9
            fl = 8.0 * d["cmac"] / (d["ms"] * 1e-3) / 1e12
            if 8.0 * d["cmac"] / (alu_peak * 1e12) > d["bytes"] / (pk["hbm_gbs"] * 1e9):
                r = {"bound": "alu", "achieved": fl, "peak": alu_peak, "unit": "TFLOP/s", "frac": fl / alu_peak,
                     "traffic": None, "kernel": kind,
                     "peak_src": "derived: 148 SMs x 128 FP32 lanes x 2 flop x 1.965 GHz / 2 (FFMA reciprocal "
                                 "throughput 2 cycles per SMSP, B300_MICROARCH.md)",
                     "hbm_frac": bw / pk["hbm_gbs"]}
            else:
                r = {"bound": "hbm", "achieved": bw, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": bw / pk["hbm_gbs"],
                     "traffic": None, "kernel": kind, "peak_src": pk["src"], "alu_frac": fl / alu_peak}
        r["share_of_slice"] = d["ms"] / slice_ms
        r["launches_per_slice"] = d["launches"]
        r["algorithmic_bytes_per_launch"] = d["bytes"] / max(1, d["launches"])
        # traffic: DRAM bytes per launch of this kernel from the committed ncu capture (one slice)
        for entry in traffic:
            if entry.get("kernel") == r["kernel"]:
                r["traffic"] = entry["dram_bytes_per_launch"]
                r["traffic_src"] = entry["source"]
        return r

    roof = roofline(dom[0], dom[1])
    roof_tensor = roofline("gemm_tcgen05", by_kind["gemm_tcgen05"]) if (
        dom[0] != "gemm_tcgen05" and "gemm_tcgen05" in by_kind) else None
    per_slice_launches, per_contract_launches = ss.launch_counts()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(cfg)

    if rank == 0:
        cmac_total = info["cmac_per_slice"] * nS
        line = {
            "metric": METRIC, "value": slices_per_s, "unit": "slices/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c64", "data": "synthetic",
            "config": {**workload_config(cfg), "parallelism": f"slices/{world}",
                       "l2": "flushed (512 MB write) before every timed step; per-slice working set "
                             f"{info['workspace_bytes'] / 2**30:.2f} GiB > L2",
                       "setup_s": {"build": t_build, "plan": t_plan, "bind": t_bind}},
            "complex_tflops": 8.0 * cmac_total / (ms_per_step * 1e-3) / 1e12,
            "cmac_per_slice": info["cmac_per_slice"], "gemm_cmac_frac": info["gemm_cmac_per_slice"] / max(
                1.0, info["cmac_per_slice"]),
            "bytes_per_slice": info["bytes_per_slice"],
            "time_to_M_amplitudes_s": ms_per_step * 1e-3,
            "e2e": {"value": nS / (e2e_ms * 1e-3), "unit": "slices/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": 8 * len(block), "d2h_bytes_per_step": 8 * M,
                    "ms_each": [round(x, 2) for x in e2e_each]},
            "roofline": roof,
            "roofline_tensor": roof_tensor,
            "kernel_ms_per_slice": {k: round(v["ms"], 4) for k, v in by_kind.items()},
            "clocks": clocks,
            "gpu_launches": args.steps * (len(block) * per_slice_launches + per_contract_launches) * (1 if block else 0),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
