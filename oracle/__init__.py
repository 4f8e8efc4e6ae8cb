"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the PMBS hot path.

* ``oracle.ref``  — the unmodified reference library (oracle/_ref, built by
  oracle/Makefile from /root/reference sources) behind a flat C shim.
* ``oracle.port`` — the plain-C restatement (oracle/pmbs_oracle.c), pinned
  bit-for-bit to ``oracle.ref`` and to tests/golden/.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package; the product (paper_2207_06649_b200) never does.
"""
