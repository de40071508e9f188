"""The five BASELINE.json configs as concrete seeded inputs.

Seeds: circuit = 1000 + cfg, bitstrings = 2000 + cfg, sampler = 3000 + cfg.
Open qubits: configs 1-3 the 6 highest ids; 4-5 the paper's ids [11,19,28,29,37,44]
 in our row-major numbering.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

from . import bitstrings as bs
from . import circuits as cc

SUPREMACY = "ABCDCDAB"


@dataclass
class Config:
    cfg: int
    name: str
    layout: str            # "rect:RxC" or "sycamore53"
    cycles: int
    sequence: str
    L: int
    n_open: int
    n_sliced: int          # requested number of sliced wires (planner target)
    log2_tmax: int         # max_tensor_size = 2^log2_tmax complex64 elements
    open_qubits: Optional[List[int]] = None
    final_layer: bool = True
    note: str = ""
    # planner settings (plan search is setup; chosen by measuring candidate plans, tools/plan_sweep.py)
    plan_seed: int = 1
    plan_trials: int = 0
    plan_budget_s: float = 0.0

    def qubits(self):
        if self.layout == "sycamore53":
            return cc.sycamore53_layout()
        r, c = self.layout.split(":")[1].split("x")
        return cc.rect_layout(int(r), int(c))

    def circuit(self, seed: Optional[int] = None) -> dict:
        return cc.generate_circuit(self.qubits(), self.cycles, self.sequence,
                                   1000 + self.cfg if seed is None else seed, self.final_layer)

    def open_ids(self, n: int) -> List[int]:
        if self.open_qubits is not None:
            return list(self.open_qubits)
        return list(range(n - self.n_open, n))

    def bitstrings(self, n: int, seed: Optional[int] = None):
        return bs.generate_groups(n, self.open_ids(n), self.L, 2000 + self.cfg if seed is None else seed)

    def plan_kwargs(self) -> dict:
        return {"n_sliced": self.n_sliced, "seed": self.plan_seed, "trials": self.plan_trials,
                "time_budget_s": self.plan_budget_s}

    def open_mask(self, n: int) -> int:
        return bs.qubit_mask(n, self.open_ids(n))

    @property
    def sampler_seed(self) -> int:
        return 3000 + self.cfg


CONFIGS = {
    1: Config(1, "12q-m4-ABCD", "rect:3x4", 4, "ABCD", L=4, n_open=6, n_sliced=0, log2_tmax=20,
              note="unsliced, full fidelity"),
    2: Config(2, "20q-m8", "rect:4x5", 8, SUPREMACY, L=64, n_open=6, n_sliced=4, log2_tmax=20,
              note="2^4 slices all contracted"),
    3: Config(3, "30q-m12", "rect:5x6", 12, SUPREMACY, L=1024, n_open=6, n_sliced=8, log2_tmax=28,
              note="2^8 slices, fraction sweep", plan_seed=53, plan_trials=96, plan_budget_s=120.0),
    4: Config(4, "53q-m14", "sycamore53", 14, SUPREMACY, L=1 << 14, n_open=6, n_sliced=12, log2_tmax=32,
              open_qubits=[11, 19, 28, 29, 37, 44], note="2^12 slices over 1/2/4/8 GPUs"),
    5: Config(5, "53q-m20", "sycamore53", 20, SUPREMACY, L=1 << 20, n_open=6, n_sliced=-1, log2_tmax=32,
              open_qubits=[11, 19, 28, 29, 37, 44], note="slice subset targeting F~0.002-0.004"),
}


def get(cfg: int) -> Config:
    return CONFIGS[cfg]
