/*
 * oracle.c — the serial CPU oracle for the EbV LU factor + solve hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1907_05767_b200/, libebv.so) never links, loads or
 * calls it, and this file shares no code, header or constant with the CUDA
 * path.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, line numbers there):
 *   - AX = B  <=>  (LU)X = B  <=>  LY = B, then UX = Y          (Eq 1)
 *   - A = LU without pivoting, Doolittle form: L unit lower triangular,
 *     U upper triangular with the pivots A_rr on its diagonal      (Eq 3, P:43-45;
 *     reading R1 in DESIGN.md: Eq 3 draws U unit-diagonal too, Eq 6 divides by
 *     A_rr; the pivots are kept in U)
 *   - step r (0-based k here):
 *       L_(k) column scale   l_ik = a_ik / a_kk,  i > k             (Eq 6-a)
 *       U_(k) row            u_kj = a_kj (post-update row k), j >= k (Eq 6-b)
 *       rank-1 update        a_ij <- a_ij - l_ik * u_kj,  i,j > k   (Eq 6-c, P:71;
 *                            Eq 5-c trailing matrix A^(r))
 *     reading R3: the multiplier is formed first (l = a/a_kk) and the update
 *     is one fused multiply-add fma(-l, u, a) — equal to Eq 6-c's
 *     A - L*U/A_rr in exact arithmetic, with one rounding per update.
 *   - forward substitution  y_i <- y_i - l_ik y_k  for k ascending  (Eq 1)
 *   - backward substitution x_k = y_k / u_kk, then y_i <- y_i - u_ik x_k
 *     for k descending ("UX = B" read as UX = Y, reading R6)      (Eq 1)
 *
 * Canonical evaluation order: every entry's
 * value is the fma chain over ascending k starting from its input value,
 * followed, for an entry of L, by one correctly rounded division.  This is
 * the plain textbook loop nest below, compiled with -ffp-contract=off so the
 * compiler cannot fuse or reorder anything, and with explicit fma().
 *
 * Storage: column-major, a(i,j) = A[i + j*lda], packed in place (strict lower
 * triangle = L multipliers, diagonal and upper = U).
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

/* Pivot check (reading R9): info = first 1-based step r with |u_rr| <= tau;
 * the factorization continues after a failing pivot (LAPACK getrf
 * convention).  Returns info. */
int64_t oracle_lu_factor(int64_t n, double* A, int64_t lda, double tau) {
  int64_t info = 0;
  for (int64_t k = 0; k < n; k++) {
    double piv = A[k + k * lda];
    if (fabs(piv) <= tau && info == 0) info = k + 1;
    /* Eq 6-a: the L_(k) vector (column k below the diagonal) */
    for (int64_t i = k + 1; i < n; i++) A[i + k * lda] = A[i + k * lda] / piv;
    /* Eq 6-c: rank-1 update of the trailing matrix with L_(k) and U_(k) */
    for (int64_t j = k + 1; j < n; j++) {
      double u = A[k + j * lda];
      double* col = A + j * lda;
      const double* l = A + k * lda;
      for (int64_t i = k + 1; i < n; i++) col[i] = fma(-l[i], u, col[i]);
    }
  }
  return info;
}

/* Eq 1: LY = B (unit lower, forward) then UX = Y (upper, backward), for each
 * of the nrhs columns of B (column-major, ldb); B is overwritten with X. */
void oracle_lu_solve(int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb, int64_t nrhs) {
  for (int64_t r = 0; r < nrhs; r++) {
    double* y = B + r * ldb;
    for (int64_t k = 0; k < n; k++) {            /* forward: LY = B */
      double yk = y[k];
      const double* l = LU + k * lda;
      for (int64_t i = k + 1; i < n; i++) y[i] = fma(-l[i], yk, y[i]);
    }
    for (int64_t k = n - 1; k >= 0; k--) {       /* backward: UX = Y */
      double xk = y[k] / LU[k + k * lda];
      y[k] = xk;
      const double* u = LU + k * lda;
      for (int64_t i = 0; i < k; i++) y[i] = fma(-u[i], xk, y[i]);
    }
  }
}

/* Batched independent systems (BASELINE.json configs[4]; reading R16): each
 * system is factored and (if B != NULL) solved by the two functions above. */
void oracle_lu_factor_batched(int64_t n, double* A, int64_t lda, int64_t strideA, int64_t batch,
                              double* B, int64_t ldb, int64_t strideB, int64_t nrhs, double tau,
                              int32_t* info) {
  for (int64_t b = 0; b < batch; b++) {
    int64_t inf = oracle_lu_factor(n, A + b * strideA, lda, tau);
    info[b] = (int32_t)inf;
    if (B) oracle_lu_solve(n, A + b * strideA, lda, B + b * strideB, ldb, nrhs);
  }
}

/* Unit-diagonal normalization (Eq 2: the coefficient matrix drawn
 * with 1 on its diagonal; SPEC S:81-89 normalize_unit_diagonal; SURVEY §8f
 * f3): row i of A and of B divided by a_ii (one correctly rounded division
 * per entry, so the diagonal becomes exactly 1), scales[i] = 1 / a_ii.  A row
 * with a_ii == 0 is left unchanged (scale 0) and reported: returns the first
 * such 1-based row, else 0. */
int64_t oracle_normalize_unit_diagonal(int64_t n, double* A, int64_t lda, double* B, int64_t ldb, int64_t nrhs,
                                       double* scales) {
  int64_t info = 0;
  for (int64_t i = 0; i < n; i++) {
    double d = A[i + i * lda];
    if (d == 0.0) {
      if (info == 0) info = i + 1;
      scales[i] = 0.0;
      continue;
    }
    for (int64_t j = 0; j < n; j++) A[i + j * lda] = A[i + j * lda] / d;
    for (int64_t r = 0; r < nrhs; r++) B[i + r * ldb] = B[i + r * ldb] / d;
    scales[i] = 1.0 / d;
  }
  return info;
}

/* LDU form of a packed Doolittle LU (Eq 3, where U is drawn with a
 * unit diagonal; Eq 6-b's U_(k) row divided by its pivot; reading R1):
 * A = L D U' with D = diag(U) and U'_kj = u_kj / u_kk (j > k, one correctly
 * rounded division).  In place: the strict upper triangle becomes U', the
 * diagonal keeps D (U' has an implicit unit diagonal, like L); D is also
 * copied to d. */
void oracle_lu_to_ldu(int64_t n, double* LU, int64_t lda, double* d) {
  for (int64_t k = 0; k < n; k++) {
    double p = LU[k + k * lda];
    d[k] = p;
    for (int64_t j = k + 1; j < n; j++) LU[k + j * lda] = LU[k + j * lda] / p;
  }
}
