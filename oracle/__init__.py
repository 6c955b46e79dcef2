"""ORACLE — test infrastructure only (never on the product path).

A plain, slow, obviously-correct CPU implementation of what the gpu-let hot
path computes, written from PAPER.md (arXiv 2109.01611) and the readings of
SURVEY.md §8(c) / DESIGN.md §2.  It shares NO code with the CUDA path
(`paper_2109_01611_b200/`); the only shared module is `synthgen/` (seeded
inputs, no arithmetic of the method).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import anything under `oracle/`.

Parts:
  nn.py, models.py  C1  forward passes (numpy, fp64 accumulation, bf16 rounding
                        at the C1.4 points)
  sched.py          C2  ElasticPartitioning / FindBestFit / SBP / ideal (Alg. 1)
  interf.py         C3  linear interference model fit + predict
  profiles.py       C4  min-envelope, SLO rule, rate scaling, scenarios
  des.py            C5  discrete-event simulator (duty-cycle dispatch)
Parity status of each function is stated in its docstring; "parity unpinned"
items are listed in DESIGN.md §2.
"""
