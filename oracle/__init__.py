"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously correct CPU implementation of what the FFS hot path computes
(arXiv 2109.07358), written from PAPER.md and used ONLY by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / `--impl reference` leg. The product path
(paper_2109_07358_b200) never imports, links or executes anything under oracle/, and the two
share no code: the only common module is paper_2109_07358_b200.inputs (seeded inputs, none of
the method's arithmetic).

Contents
  ffs_ref.c / ffs_ref_core.h : the paper's algorithm (Supp S1 eager elimination, Eq. 3 weights,
                               inverse-CDF draw) in C, fp64, OpenMP across samples.
  ref.py                     : ctypes binding + build of libffs_ref.so.
  exact.py                   : closed forms / definitions used to PIN the oracle (Eq. 1 brute
                               force, Eq. 2 mixture enumeration, marginal determinant formula,
                               the null-vector definition of h via SVD).

Parity status per function: every exported function is pinned by a
`-m "not gpu"` test in tests/test_oracle.py against something other than itself; none is
"parity unpinned".
"""
