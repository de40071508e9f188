"""Seeded synthetic inputs (circuits, bitstring requests, config table).

Shared by the product tests/bench and by the oracle; contains none of the method's
arithmetic (no gate matrices from parameters, no contraction, no slicing logic).
"""
from . import rng, circuits, bitstrings, configs  # noqa: F401
