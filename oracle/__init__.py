"""oracle/ -- TEST INFRASTRUCTURE for the B200 PSD-projection path. NOT PRODUCT CODE.

A plain, slow, obviously-correct CPU implementation of what the hot path computes
(arXiv:1912.02767, Rontsis/Goulart/Nakatsukasa, PAPER.md):

  exact.py    Pi_{S+}(A) by its definition: cyclic Jacobi (jacobi.c,
              GvL Alg. 8.5.3) then both closed forms V+L+V+^T and A - V-L-V-^T.
  lobpcg.py   Rayleigh-Ritz (Alg. 2) and LOBPCG for the positive
              eigenpairs (Alg. 3) step by step, with the side rule
              (PAPER.md:505), negation and the Theorem-3 bound.
  philox.py   Philox4x32-10 counter-based RNG + Box-Muller (the random expansion/cold
              block of Alg. 3 line 8; generator reading R11 in DESIGN.md).
  admm.py     Alg. 1 for diagonal SDPs (MaxCut, f1) and the Theorem-1
              infeasibility certificates (f3).

The Moreau/KKT certificate and Theorem 3's exact right-hand side (perp term by Jacobi) are
test-side checks in tests/test_oracle_*.py, not oracle functions. Library primitives used as
single steps (SURVEY §8.c allows them; stated in DESIGN.md §10): numpy matmul (BLAS dgemm),
numpy Householder QR (LAPACK geqrf, the paper's own fallback) and triangular /
linear solves. Every eigendecomposition is the cyclic Jacobi of jacobi.c (no LAPACK eig).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package. It shares no code with paper_1912_02767_b200/ and never imports it.
Parity unpinned: none (every function is pinned in tests/test_oracle_*.py).
"""
