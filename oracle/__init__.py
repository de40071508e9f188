"""ORACLE — plain, slow, obviously-correct CPU reference for arXiv:2111.03011's hot path.

THIS PACKAGE IS TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import, call, link or execute anything here.
The product (paper_2111_03011_b200/) never imports it and shares no code, header, table or
constant generator with it; both only read the seeded inputs of tn_inputs/.

Contents
  sv.c / sv.py   fp64 state vector with projector / sigma_z insertion on wires (O1-O5)
  tn_brute.py    brute-force enumeration of the tensor network for tiny circuits (O6)
  rows.py        sparse-state row tables and parent maps (O7)
  metrics.py     F_exact, F_norm, F_sparse, linear XEB, within-group sampler (O5, a9)
  tn_einsum.py   closed-network contraction of single amplitudes (numpy tensordot, own greedy order),
                 for the 53-qubit spot checks (SURVEY §8(c) "53q amplitudes")

Parity status (DESIGN.md §Oracle pins): every function above is pinned by a
`-m "not gpu"` test against a closed form, a printed paper example, an invariant, a
textbook construction or brute force -- none is "parity unpinned".
"""
