"""The oracle: a plain, slow, obviously-correct CPU implementation of the
distributed SpMV y = A x of arXiv 2203.02530 (§III-A).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import, call,
link or execute anything under ``oracle/``.  The product path
(``paper_2203_02530_b200``) never imports it, and the two share no code:
only the seeded input generators in ``gen/`` serve both.

Modules
-------
spmv       O1: the serial CSR product (C, ``o1.c``) + dense brute force.
plan       O2: partition, local/remote split, halo lists, pack maps, and a
           lock-step simulation of one schedule over all ranks.
schedules  The program DAG, tab:sync insertion, a happens-before validator
           and a brute-force schedule enumerator.

Every function's docstring cites the PAPER.md passage (``P:n`` = line n) it
follows.  Pins (tests/test_oracle_*.py) tie each part to something other than
itself: brute force, scipy, closed forms, Appendix-B counts, paper sequences.
"""
