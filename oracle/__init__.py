"""CPU ORACLE for the deferred-compression LoRaSp hot path — TEST INFRASTRUCTURE ONLY.

Plain, slow, sequential NumPy/SciPy code written from PAPER.md (arXiv
1811.11248) and the readings Q1-Q20 of SURVEY.md §8(c) / DESIGN.md.
It shares NO code with the CUDA path (`paper_1811_11248_b200/`), and neither
imports the other.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / --impl reference legs may import it; the product
path never routes through it.

Modules
  dense    — Cholesky, triangular solve, Householder (dlarfg), column-pivoted QR
  analyze  — O2: units, RCB cluster tree, permutation, H_0, per-level schedule
  factor   — O3: Algorithm 1 with the scaled low-rank elimination
  solve    — O4: Algorithm 2; O5: PCG; GMRES(200)
  dist     — the subdomain-distributed factor, apply and PCG, gloo-tested

Parity status: every function is pinned by tests/test_oracle_*.py (P1-P9, the R-floor, the
decision-flag window, PCG beyond iteration 1, the R-coarse neighbour closed form);
the ranks/iterations on C2-C5 are "parity unpinned" beyond oracle-vs-GPU
(no published values exist for these synthetic inputs).
"""
