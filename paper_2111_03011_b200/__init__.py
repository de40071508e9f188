"""B200-native sliced sparse-state contraction of arXiv:2111.03011 (Pan, Chen, Zhang).

Thin Python binding of the C ABI in include/tn.h (argument marshalling only; every step of the
hot path runs in libtnb200.so's sm_100a kernels).  There is no CPU fallback: if the library is
missing, importing the binding raises.

    from paper_2111_03011_b200 import SparseState
    ss = SparseState(circuit, bitstrings, open_mask)       # tn_build
    info = ss.plan(max_tensor_size=2**28, n_sliced=8)      # tn_plan
    ss.bind(device=0)                                      # tn_bind_device (torch memory/stream)
    amps = ss.contract(range(2**info["s"]))                # tn_contract
    samples, est = ss.sample(amps.cpu().numpy(), n)        # tn_sample
"""
from __future__ import annotations

import ctypes
import os
from typing import Iterable, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtnb200.so")

TN_OK, TN_EINVAL, TN_EINFEASIBLE, TN_ENUMERIC, TN_ECUDA, TN_ENOMEM = 0, 2, 3, 4, 5, 6
KIND_NAMES = {0: "instantiate", 1: "apply", 2: "prep_a", 3: "prep_b", 4: "gemm_tcgen05", 5: "readout", 6: "permute",
              7: "multi", 8: "accum", 10: "gate_tcgen05"}


class TnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"tn status {status}: {msg}")
        self.status = status


class TnGate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("q0", ctypes.c_int32), ("q1", ctypes.c_int32),
                ("theta", ctypes.c_double), ("phi", ctypes.c_double), ("u", ctypes.c_double * 8)]


class TnCircuit(ctypes.Structure):
    _fields_ = [("n_qubits", ctypes.c_int32), ("n_moments", ctypes.c_int32),
                ("moment_offsets", ctypes.POINTER(ctypes.c_int32)), ("gates", ctypes.POINTER(TnGate)),
                ("qubit_rc", ctypes.POINTER(ctypes.c_int32))]


class TnSlicing(ctypes.Structure):
    _fields_ = [("n_sliced", ctypes.c_int32), ("n_forced", ctypes.c_int32),
                ("forced_wires", ctypes.POINTER(ctypes.c_int32)), ("seed", ctypes.c_uint64),
                ("trials", ctypes.c_int32), ("time_budget_s", ctypes.c_double), ("companions", ctypes.c_int32),
                ("method", ctypes.c_int32), ("max_segments", ctypes.c_int32), ("persist_budget", ctypes.c_double),
                ("plan_path", ctypes.c_char_p)]


class TnPlanInfo(ctypes.Structure):
    _fields_ = [("s", ctypes.c_int32), ("sliced_wires", ctypes.POINTER(ctypes.c_int32)),
                ("n_tensors", ctypes.c_int64), ("n_steps", ctypes.c_int64), ("n_launches", ctypes.c_int64),
                ("peak_elems", ctypes.c_int64), ("workspace_bytes", ctypes.c_int64),
                ("cmac_per_slice", ctypes.c_double), ("bytes_per_slice", ctypes.c_double),
                ("gemm_cmac_per_slice", ctypes.c_double), ("n_invariant_steps", ctypes.c_int64),
                ("invariant_cmac", ctypes.c_double), ("n_companions", ctypes.c_int32),
                ("companion_wires", ctypes.POINTER(ctypes.c_int32)), ("companion_fidelity", ctypes.c_double),
                ("s_local", ctypes.c_int32), ("local_wires", ctypes.POINTER(ctypes.c_int32)),
                ("n_segments", ctypes.c_int32), ("total_cmac", ctypes.c_double), ("persist_bytes", ctypes.c_int64)]


class TnLaunchStat(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("step", ctypes.c_int32), ("cmac", ctypes.c_double),
                ("bytes", ctypes.c_double), ("ms", ctypes.c_double), ("m", ctypes.c_int64),
                ("n", ctypes.c_int64), ("k", ctypes.c_int64), ("rows", ctypes.c_int64), ("seg", ctypes.c_int32),
                ("pad", ctypes.c_int32)]


class TnReport(ctypes.Structure):
    _fields_ = [(name, ctypes.c_double) for name in
                ("f", "F_norm", "xeb", "log_xeb", "entropy_samples", "entropy_state", "pt_ks")]


EXPORTS = ["tn_build", "tn_build_drilled", "tn_plan", "tn_plan_dump", "tn_plan_save", "tn_segment_runs", "tn_bind_device", "tn_contract", "tn_profile_slice",
           "tn_sample", "tn_sample_report", "tn_destroy", "tn_last_error", "tn_version", "tn_debug_gemm_tf32x3",
           "tn_debug_network", "tn_debug_launch_counts"]

_lib = None


def lib():
    """Load libtnb200.so (built by paper_2111_03011_b200.build); raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: run `python -m paper_2111_03011_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, c = ctypes.POINTER, ctypes
    L.tn_build.argtypes = [P(TnCircuit), P(c.c_uint64), c.c_int64, c.c_uint64, P(c.c_void_p)]
    L.tn_build_drilled.argtypes = [P(TnCircuit), P(c.c_uint64), c.c_int64, c.c_uint64, P(c.c_int32), c.c_int32,
                                   P(c.c_void_p)]
    L.tn_plan.argtypes = [c.c_void_p, P(TnSlicing), c.c_int64, P(TnPlanInfo)]
    L.tn_plan_dump.argtypes = [c.c_void_p, c.c_char_p]
    L.tn_plan_save.argtypes = [c.c_void_p, c.c_char_p]
    L.tn_bind_device.argtypes = [c.c_void_p, c.c_int, c.c_void_p, c.c_size_t, c.c_void_p]
    L.tn_contract.argtypes = [c.c_void_p, P(c.c_uint64), c.c_int64, c.c_void_p, c.c_int32, P(c.c_double)]
    L.tn_profile_slice.argtypes = [c.c_void_p, c.c_uint64, P(TnLaunchStat), c.c_int32, P(c.c_int32)]
    L.tn_segment_runs.argtypes = [c.c_void_p, P(c.c_uint64), c.c_int64, P(c.c_int64)]
    L.tn_sample.argtypes = [c.c_void_p, c.c_void_p, c.c_void_p, c.c_int64, c.c_uint64, P(c.c_uint64),
                            P(c.c_double)]
    L.tn_sample_report.argtypes = [c.c_void_p, c.c_void_p, c.c_void_p, c.c_int64, c.c_uint64, c.c_int32, c.c_int32,
                                   P(c.c_uint64), P(c.c_int64), P(TnReport)]
    L.tn_destroy.argtypes = [c.c_void_p]
    L.tn_destroy.restype = None
    L.tn_last_error.argtypes = [c.c_void_p]
    L.tn_last_error.restype = c.c_char_p
    L.tn_version.restype = c.c_char_p
    L.tn_debug_gemm_tf32x3.argtypes = [c.c_void_p, c.c_void_p, c.c_void_p, c.c_int64, c.c_int64, c.c_int64,
                                       c.c_int32, c.c_void_p]
    L.tn_debug_network.argtypes = [c.c_void_p, P(c.c_int64), P(c.c_int64), P(c.c_int64)]
    L.tn_debug_launch_counts.argtypes = [c.c_void_p, P(c.c_int64), P(c.c_int64)]
    for name in ("tn_build", "tn_build_drilled", "tn_plan", "tn_plan_dump", "tn_plan_save", "tn_segment_runs", "tn_bind_device", "tn_contract", "tn_profile_slice",
                 "tn_sample", "tn_sample_report", "tn_debug_gemm_tf32x3", "tn_debug_network", "tn_debug_launch_counts"):
        getattr(L, name).restype = c.c_int
    _lib = L
    return L


def circuit_struct(circuit: dict):
    """Marshal a tn_inputs circuit dict into tn_circuit (keeps the arrays alive on the struct)."""
    moments = circuit["moments"]
    gates = [g for m in moments for g in m]
    arr = (TnGate * max(1, len(gates)))()
    for i, g in enumerate(gates):
        if g["type"] == "single":
            arr[i].kind = 0
            arr[i].q0 = g["target"]
            arr[i].q1 = -1
            m = np.asarray(g["matrix"], dtype=complex).reshape(4)
            for t in range(4):
                arr[i].u[2 * t] = m[t].real
                arr[i].u[2 * t + 1] = m[t].imag
        else:
            arr[i].kind = 1
            arr[i].q0, arr[i].q1 = g["targets"]
            arr[i].theta = g["theta"]
            arr[i].phi = g["phi"]
    offs = (ctypes.c_int32 * (len(moments) + 1))()
    acc = 0
    for i, m in enumerate(moments):
        offs[i] = acc
        acc += len(m)
    offs[len(moments)] = acc
    rc = None
    if circuit.get("qubits"):
        rc = (ctypes.c_int32 * (2 * circuit["n"]))(*[v for p in circuit["qubits"] for v in p])
    cs = TnCircuit(circuit["n"], len(moments), offs, arr, rc)
    cs._keep = (arr, offs, rc)
    return cs


class SparseState:
    """One sparse-state contraction context (tn_ctx).  Single-threaded; one per GPU / rank."""

    def __init__(self, circuit: dict, bitstrings: np.ndarray, open_mask: int = 0, holes: Sequence[int] = ()):
        """tn_build, or tn_build_drilled when `holes` lists fSim gates (indices into the flattened gate
        list, moment by moment) to drill out."""
        L = lib()
        self._circ = circuit_struct(circuit)
        self.bitstrings = np.ascontiguousarray(bitstrings, dtype=np.uint64)
        self.M = len(self.bitstrings)
        self.n = circuit["n"]
        self.open_mask = int(open_mask)
        self.l = 1 << bin(self.open_mask).count("1")
        self.holes = [int(h) for h in holes]
        self._ctx = ctypes.c_void_p()
        harr = (ctypes.c_int32 * max(1, len(self.holes)))(*self.holes)
        rc = L.tn_build_drilled(ctypes.byref(self._circ),
                                self.bitstrings.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), self.M,
                                self.open_mask, harr, len(self.holes), ctypes.byref(self._ctx))
        if rc != TN_OK:
            msg = self.last_error()
            self.close()
            raise TnError(rc, msg)
        self.info = None
        self._work = None
        self._dev = None

    # -------------------------------------------------------------- plumbing
    def last_error(self) -> str:
        if not self._ctx:
            return ""
        return lib().tn_last_error(self._ctx).decode()

    def _check(self, rc):
        if rc != TN_OK:
            raise TnError(rc, self.last_error())

    def close(self):
        if getattr(self, "_ctx", None):
            lib().tn_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- tn_plan
    def plan(self, max_tensor_size: int, n_sliced: int = -1, forced_wires: Sequence = (), seed: int = 1,
             trials: int = 0, time_budget_s: float = 0.0, companions: bool = False, method: int = 0,
             max_segments: int = 0, persist_budget: float = 0.0, plan_path: Optional[str] = None) -> dict:
        """tn_plan.  method 0 auto / 1 flat slicing / 2 loop program (local slices + head reuse);
        plan_path imports a plan file written by save_plan (the search options are then ignored)."""
        fw = (ctypes.c_int32 * max(1, 2 * len(forced_wires)))(*[v for w in forced_wires for v in w])
        sl = TnSlicing(n_sliced, len(forced_wires), fw, seed, trials, time_budget_s, 1 if companions else 0,
                       method, max_segments, persist_budget, plan_path.encode() if plan_path else None)
        info = TnPlanInfo()
        self._check(lib().tn_plan(self._ctx, ctypes.byref(sl), int(max_tensor_size), ctypes.byref(info)))
        self.info = {
            "s": info.s,
            "sliced_wires": [(info.sliced_wires[2 * i], info.sliced_wires[2 * i + 1]) for i in range(info.s)],
            "n_tensors": info.n_tensors, "n_steps": info.n_steps, "n_launches": info.n_launches,
            "peak_elems": info.peak_elems, "workspace_bytes": info.workspace_bytes,
            "cmac_per_slice": info.cmac_per_slice, "bytes_per_slice": info.bytes_per_slice,
            "gemm_cmac_per_slice": info.gemm_cmac_per_slice,
            "n_invariant_steps": info.n_invariant_steps, "invariant_cmac": info.invariant_cmac,
            "companions": [(info.companion_wires[3 * i], info.companion_wires[3 * i + 1],
                            info.companion_wires[3 * i + 2]) for i in range(info.n_companions)],
            "companion_fidelity": info.companion_fidelity,
            "s_local": info.s_local,
            "local_wires": [(info.local_wires[2 * i], info.local_wires[2 * i + 1]) for i in range(info.s_local)],
            "n_segments": info.n_segments, "total_cmac": info.total_cmac, "persist_bytes": info.persist_bytes,
        }
        return self.info

    def save_plan(self, path: str):
        """tn_plan_save: write the current plan as a replayable plan file."""
        self._check(lib().tn_plan_save(self._ctx, path.encode()))

    def dump(self, path: str):
        self._check(lib().tn_plan_dump(self._ctx, path.encode()))

    def network_size(self):
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        self._check(lib().tn_debug_network(self._ctx, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return {"tensors": a.value, "edges": b.value, "internal_edges": c.value}

    def launch_counts(self):
        """(kernels per slice, kernels per tn_contract call) of the bound executor."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        self._check(lib().tn_debug_launch_counts(self._ctx, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    # -------------------------------------------------------------- device
    def bind(self, device: int = 0, workspace=None, stream=None, pipelines: int = 8):
        """tn_bind_device.  workspace: a torch uint8 CUDA tensor (allocated here from torch's caching
        allocator when None, room for `pipelines` concurrent slice pipelines, capped by free memory);
        stream: a torch.cuda.Stream (current stream when None).  The library runs
        floor(workspace bytes / per-pipeline workspace) slice pipelines concurrently (at most 32)."""
        import torch
        if self.info is None:
            raise TnError(TN_EINVAL, "bind before plan")
        dev = torch.device("cuda", device)
        if workspace is None:
            wb = (max(1, self.info["workspace_bytes"]) + 4095) // 4096 * 4096
            free, _ = torch.cuda.mem_get_info(dev)
            p = max(1, min(int(pipelines), int(0.6 * free) // wb))
            workspace = torch.empty(wb * p, dtype=torch.uint8, device=dev)
            self.pipelines = p
        self._work = workspace
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        self._stream = st
        self._dev = device
        self._check(lib().tn_bind_device(self._ctx, device, ctypes.c_void_p(workspace.data_ptr()),
                                         workspace.numel() * workspace.element_size(),
                                         ctypes.c_void_p(st.cuda_stream)))

    def contract(self, slice_ids: Iterable[int], out=None, timed: bool = False):
        """tn_contract on the device: returns a complex64 CUDA tensor of the M amplitudes
        (and the device seconds when timed)."""
        import torch
        ids = np.ascontiguousarray(np.fromiter((int(x) for x in slice_ids), dtype=np.uint64))
        if out is None:
            out = torch.empty(self.M, dtype=torch.complex64, device=torch.device("cuda", self._dev))
        secs = ctypes.c_double(0.0)
        self._check(lib().tn_contract(self._ctx, ids.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(ids),
                                      ctypes.c_void_p(out.data_ptr()), 1, ctypes.byref(secs) if timed else None))
        return (out, secs.value) if timed else out

    def contract_host(self, slice_ids: Iterable[int], out: Optional[np.ndarray] = None) -> np.ndarray:
        """tn_contract with a HOST output buffer (the end-to-end path)."""
        ids = np.ascontiguousarray(np.fromiter((int(x) for x in slice_ids), dtype=np.uint64))
        if out is None:
            out = np.empty(self.M, dtype=np.complex64)
        self._check(lib().tn_contract(self._ctx, ids.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(ids),
                                      ctypes.c_void_p(out.ctypes.data), 0, None))
        return out

    def profile_slice(self, slice_id: int = 0, max_stats: int = 4096) -> List[dict]:
        arr = (TnLaunchStat * max_stats)()
        n = ctypes.c_int32(0)
        self._check(lib().tn_profile_slice(self._ctx, slice_id, arr, max_stats, ctypes.byref(n)))
        return [{"kind": KIND_NAMES.get(a.kind, str(a.kind)), "step": a.step, "cmac": a.cmac, "bytes": a.bytes,
                 "ms": a.ms, "m": a.m, "n": a.n, "k": a.k, "rows": a.rows, "seg": a.seg} for a in arr[:n.value]]

    def segment_runs(self, slice_ids: Iterable[int]) -> List[int]:
        """tn_segment_runs: runs of every loop-program segment for a tn_contract over slice_ids."""
        ids = np.ascontiguousarray(np.fromiter((int(x) for x in slice_ids), dtype=np.uint64))
        runs = np.zeros(max(1, self.info["n_segments"]), dtype=np.int64)
        self._check(lib().tn_segment_runs(self._ctx, ids.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(ids),
                                          runs.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return [int(x) for x in runs]

    # -------------------------------------------------------------- tn_sample
    def sample(self, amps: np.ndarray, n_slices_summed: int, seed: int, ideal: Optional[np.ndarray] = None):
        a = np.ascontiguousarray(amps, dtype=np.complex64)
        idl = None if ideal is None else np.ascontiguousarray(ideal, dtype=np.complex64)
        L = self.M // self.l
        out = np.zeros(L, dtype=np.uint64)
        est = (ctypes.c_double * 3)()
        self._check(lib().tn_sample(self._ctx, ctypes.c_void_p(a.ctypes.data),
                                    None if idl is None else ctypes.c_void_p(idl.ctypes.data),
                                    int(n_slices_summed), int(seed),
                                    out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), est))
        return out, {"fraction": est[0], "F_norm": est[1], "xeb": est[2]}

    def sample_report(self, amps: np.ndarray, n_slices_summed: int, seed: int, sampler: str = "categorical",
                      steps: int = 200, ideal: Optional[np.ndarray] = None):
        """tn_sample_report: (samples, indices j into the request, estimator dict); sampler "categorical"
        (frugal within a group) or "metropolis" (uniform-proposal chain of `steps` steps)."""
        a = np.ascontiguousarray(amps, dtype=np.complex64)
        idl = None if ideal is None else np.ascontiguousarray(ideal, dtype=np.complex64)
        L = self.M // self.l
        out = np.zeros(L, dtype=np.uint64)
        idx = np.zeros(L, dtype=np.int64)
        rep = TnReport()
        self._check(lib().tn_sample_report(self._ctx, ctypes.c_void_p(a.ctypes.data),
                                           None if idl is None else ctypes.c_void_p(idl.ctypes.data),
                                           int(n_slices_summed), int(seed),
                                           {"categorical": 0, "metropolis": 1}[sampler], int(steps),
                                           out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                           idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ctypes.byref(rep)))
        return out, idx, {name: getattr(rep, name) for name, _ in TnReport._fields_}


def debug_gemm(A, B, embed_a: int = 0):
    """C = A @ B (complex64 CUDA tensors) through the tcgen05 3xTF32 path (tn_debug_gemm_tf32x3)."""
    import torch
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    A = A.contiguous()
    B = B.contiguous()
    C = torch.empty((M, N), dtype=torch.complex64, device=A.device)
    rc = lib().tn_debug_gemm_tf32x3(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                   ctypes.c_void_p(C.data_ptr()), M, N, K, int(embed_a),
                                   ctypes.c_void_p(torch.cuda.current_stream(A.device).cuda_stream))
    if rc != TN_OK:
        raise TnError(rc, "debug gemm failed")
    return C
