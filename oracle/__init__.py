"""CPU FP64 oracle for the BAL inexact Newton-PCG hot path of arXiv 2407.00046.

THIS PACKAGE IS TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import or execute it.  The product
path (``paper_2407_00046_b200``) never imports it and shares no code with it; the only shared
module is the seeded input generator ``scenes`` (no method arithmetic).

It is deliberately plain and slow: numpy/scipy in float64, derivatives by forward-mode
second-order AD (``oracle.ad``), projection by LAPACK eigh, map/COO assembly, textbook PCG.
Every function cites the PAPER.md passage (P:line) or SURVEY.md reading (Qn) it follows; the
readings are listed in DESIGN.md.  Parity pins live in ``tests/test_oracle_*.py``.

Parity status: every function is pinned by at least one closed form, invariant, library
special case or brute-force check, except the full multi-step trajectory (oracle.bal.Oracle.step
over many steps), which the paper pins only through invariants -- "parity unpinned" for the
trajectory as a whole (SURVEY c.3 last row).
"""
