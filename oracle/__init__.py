"""Korch oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (numpy, float64) of what
the hot path computes, written from the paper (arXiv 2406.09465,
/root/reference/PAPER.md, cited as P:<line>) and the readings in DESIGN.md
("Readings of the paper").  It shares no code with the CUDA path
(`paper_2406_09465_b200/`) and never imports it; the only shared module is
`korch_workloads` (graph descriptions + seeded input generators, no method
arithmetic).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import anything under `oracle/`.

Modules
  operators      unfissioned operator interpreter (Eq. 1; A10-A12)
  primitives     primitive interpreter, the four categories
  fission        operator -> primitive graph, canonical table
  enumeration    execution states / convex sets / candidates (Thm 1)
  orchestration  Eq. 2-4 feasibility, exhaustive 2^M search, producer-assignment
                 exact search
  evaluate       primitive-graph and orchestration-aware evaluation (A25)

Parity status: every function is pinned by tests/test_oracle_*.py except the
measured kernel costs c_i, which are "parity unpinned" (they are measurements,
P:383 "c_i is the measured run time of kernel K_i"); see DESIGN.md.
"""
