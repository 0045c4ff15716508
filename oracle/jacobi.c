/*
 * oracle/jacobi.c -- TEST INFRASTRUCTURE ONLY (never linked into the product path).
 *
 * Plain cyclic Jacobi eigendecomposition of a dense symmetric fp64 matrix.
 * This is the "full eigendecomposition" the paper replaces (PAPER.md:24-33,
 * Eq. (admm:eqn:eigendecomposition) at PAPER.md:310-318, citing Golub & Van Loan
 * [Golub2013] for the eigendecomposition); the algorithm is GvL 4th ed. Alg. 8.5.2
 * (sym.schur2) + Alg. 8.5.3 (cyclic-by-row Jacobi), written out literally:
 * no blocking, no parallel ordering, no BLAS.
 *
 * Shares no code with paper_1912_02767_b200/ (the CUDA path).
 *
 * Threshold reading (DESIGN.md R-J1): a rotation (p,q) is skipped when
 *   |a_pq| <= u * sqrt(|a_pp| * |a_qq|)  or  |a_pq| <= u * ||A0||_F / n
 * and the iteration stops after the first sweep that performs no rotation.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define AT(M, i, j, ld) (M)[(size_t)(i) + (size_t)(j) * (size_t)(ld)]

/* sym.schur2 (GvL Alg. 8.5.2): c, s such that the (p,q) 2x2 block of J^T A J is diagonal. */
static void sym_schur2(double app, double apq, double aqq, double *c, double *s) {
  if (apq != 0.0) {
    double tau = (aqq - app) / (2.0 * apq);
    double t;
    if (tau >= 0.0)
      t = 1.0 / (tau + sqrt(1.0 + tau * tau));
    else
      t = -1.0 / (-tau + sqrt(1.0 + tau * tau));
    *c = 1.0 / sqrt(1.0 + t * t);
    *s = t * (*c);
  } else {
    *c = 1.0;
    *s = 0.0;
  }
}

/*
 * oracle_jacobi_eig: A (n x n, column-major, leading dim lda) is copied; on return
 *   w[0..n-1]  eigenvalues in ascending order,
 *   V (n x n, column-major, leading dim n) orthonormal eigenvectors, V[:,i] <-> w[i].
 * Returns the number of sweeps performed (>= 1), or -1 if max_sweeps was reached
 * without a rotation-free sweep, -2 on allocation failure, -3 on non-finite input.
 */
int oracle_jacobi_eig(int n, const double *A, int lda, double *w, double *V, int max_sweeps) {
  if (n <= 0) return 1;
  double *M = (double *)malloc(sizeof(double) * (size_t)n * (size_t)n);
  if (!M) return -2;
  double fro = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      double a = AT(A, i, j, lda);
      if (!isfinite(a)) { free(M); return -3; }
      AT(M, i, j, n) = a;
      fro += a * a;
    }
  fro = sqrt(fro);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) AT(V, i, j, n) = (i == j) ? 1.0 : 0.0;

  const double u = 1.1102230246251565e-16; /* unit roundoff 2^-53 */
  const double abs_floor = u * fro / (double)n;
  int sweeps = 0, done = 0;
  while (!done && sweeps < max_sweeps) {
    int rotations = 0;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        double apq = AT(M, p, q, n);
        double app = AT(M, p, p, n), aqq = AT(M, q, q, n);
        if (fabs(apq) <= u * sqrt(fabs(app) * fabs(aqq)) || fabs(apq) <= abs_floor) {
          continue;
        }
        double c, s;
        sym_schur2(app, apq, aqq, &c, &s);
        double t = s / c;
        ++rotations;
        /* A <- J^T A J (GvL Alg. 8.5.2/8.5.3). The annihilated (p,q) block is set
         * exactly: a_pp - t a_pq, a_qq + t a_pq, a_pq = 0 (GvL §8.5.2); the other
         * entries of rows/columns p, q are rotated and mirrored (A stays symmetric). */
        for (int i = 0; i < n; ++i) {
          if (i == p || i == q) continue;
          double aip = AT(M, i, p, n), aiq = AT(M, i, q, n);
          double nip = c * aip - s * aiq, niq = s * aip + c * aiq;
          AT(M, i, p, n) = nip; AT(M, p, i, n) = nip;
          AT(M, i, q, n) = niq; AT(M, q, i, n) = niq;
        }
        AT(M, p, p, n) = app - t * apq;
        AT(M, q, q, n) = aqq + t * apq;
        AT(M, p, q, n) = 0.0; AT(M, q, p, n) = 0.0;
        /* V <- V J */
        for (int i = 0; i < n; ++i) {
          double vip = AT(V, i, p, n), viq = AT(V, i, q, n);
          AT(V, i, p, n) = c * vip - s * viq;
          AT(V, i, q, n) = s * vip + c * viq;
        }
      }
    }
    ++sweeps;
    if (rotations == 0) done = 1;
  }
  /* sort ascending (selection sort on the diagonal, permuting V's columns) */
  for (int i = 0; i < n; ++i) w[i] = AT(M, i, i, n);
  for (int i = 0; i < n - 1; ++i) {
    int k = i;
    for (int j = i + 1; j < n; ++j)
      if (w[j] < w[k]) k = j;
    if (k != i) {
      double t = w[i]; w[i] = w[k]; w[k] = t;
      for (int r = 0; r < n; ++r) {
        double v = AT(V, r, i, n); AT(V, r, i, n) = AT(V, r, k, n); AT(V, r, k, n) = v;
      }
    }
  }
  free(M);
  return done ? sweeps : -1;
}

/*
 * oracle_cholesky: plain right-looking Cholesky of a symmetric matrix (lower factor,
 * column-major, in place on a copy). Returns 0 on success or (j+1) if pivot j is
 * <= pivot_floor (not positive definite to that threshold). Used by the Moreau
 * certificate (membership test of the PSD cone via Cholesky) and by
 * the Cholesky-QR reference.
 */
int oracle_cholesky(int n, const double *G, int ldg, double *L, double pivot_floor) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) AT(L, i, j, n) = (i >= j) ? AT(G, i, j, ldg) : 0.0;
  for (int j = 0; j < n; ++j) {
    double d = AT(L, j, j, n);
    for (int k = 0; k < j; ++k) d -= AT(L, j, k, n) * AT(L, j, k, n);
    if (!(d > pivot_floor)) return j + 1;
    double ljj = sqrt(d);
    AT(L, j, j, n) = ljj;
    for (int i = j + 1; i < n; ++i) {
      double v = AT(L, i, j, n);
      for (int k = 0; k < j; ++k) v -= AT(L, i, k, n) * AT(L, j, k, n);
      AT(L, i, j, n) = v / ljj;
    }
  }
  return 0;
}
