"""oracle -- the CPU parity oracle.  TEST INFRASTRUCTURE, NOT THE PRODUCT.

Plain, slow, obviously-correct CPU implementation of what the server-side
encrypted embedding lookup of HE-LRM (arxiv 2506.18150) computes, written from
PAPER.md plus the ring-level readings D1-D23 of SURVEY.md section 8(c) (the
paper fixes none of them; DESIGN.md lists every reading).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
`--impl reference` legs may import this package.  It shares no code with the
CUDA path (paper_2506_18150_b200/) and neither imports the other; the only
common module is synth/, the seeded input generator.

Parity status: every function is pinned by tests/test_oracle_*.py against
closed forms, brute force, big-integer definitions or invariants, except the
low-order ciphertext bits of the composite lookup, which only the D1-D23
definitions fix ("parity unpinned by the paper": pinned only by the
invariants listed in DESIGN.md and by oracle <-> GPU agreement).
"""
from .core import *  # noqa: F401,F403
