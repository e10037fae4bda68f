"""Exact rational pins for the oracle (TEST INFRASTRUCTURE ONLY).

The no-pivot Doolittle factorization of a strictly diagonally dominant matrix
exists and is unique (every leading principal minor is nonzero), and X = A^-1 B
is unique; so on the exact rational value of the fp64 input both are fixed by
mathematics, independent of any evaluation order.  These routines compute them
in ``fractions.Fraction`` with a textbook Gaussian elimination written
differently from oracle.c (row-oriented, Crout-style dot products for L/U, and
Gauss-Jordan for the solve), so a dropped term, a wrong sign or index or a
transposed operand in oracle.c fails the comparison.

Paper: Eq 1, Eq 3, Eq 6.
"""
from __future__ import annotations

from fractions import Fraction


def to_fractions(a):
    return [[Fraction(float(v)) for v in row] for row in a]


def lu_exact(a):
    """Doolittle via the Crout/Banachiewicz formulas, row by row:
        u_ij = a_ij - sum_{p<i} l_ip u_pj        (j >= i)
        l_ji = (a_ji - sum_{p<i} l_jp u_pi)/u_ii  (j > i)
    Returns (L, U) as lists of Fractions (L unit lower, U upper)."""
    n = len(a)
    A = [[v if isinstance(v, Fraction) else Fraction(float(v)) for v in row] for row in a]
    L = [[Fraction(int(i == j)) for j in range(n)] for i in range(n)]
    U = [[Fraction(0) for _ in range(n)] for _ in range(n)]
    for i in range(n):
        for j in range(i, n):
            U[i][j] = A[i][j] - sum((L[i][p] * U[p][j] for p in range(i)), Fraction(0))
        if U[i][i] == 0:
            raise ZeroDivisionError(f"zero pivot at step {i + 1}")
        for j in range(i + 1, n):
            L[j][i] = (A[j][i] - sum((L[j][p] * U[p][i] for p in range(i)), Fraction(0))) / U[i][i]
    return L, U


def solve_exact(a, b):
    """x = A^-1 b by Gauss-Jordan elimination with exact arithmetic
    (independent of the LU route).  b: list of n values."""
    n = len(a)
    M = [[Fraction(float(v)) for v in row] + [Fraction(float(b[i]))] for i, row in enumerate(a)]
    for c in range(n):
        piv = next(r for r in range(c, n) if M[r][c] != 0)
        M[c], M[piv] = M[piv], M[c]
        inv = 1 / M[c][c]
        M[c] = [v * inv for v in M[c]]
        for r in range(n):
            if r != c and M[r][c] != 0:
                f = M[r][c]
                M[r] = [vr - f * vc for vr, vc in zip(M[r], M[c])]
    return [M[i][n] for i in range(n)]


def det_exact(a):
    """det(A) by exact fraction-free Bareiss elimination (for log-det pins)."""
    n = len(a)
    M = [[Fraction(float(v)) for v in row] for row in a]
    sign, prev = 1, Fraction(1)
    for k in range(n - 1):
        if M[k][k] == 0:
            sw = next((r for r in range(k + 1, n) if M[r][k] != 0), None)
            if sw is None:
                return Fraction(0)
            M[k], M[sw] = M[sw], M[k]
            sign = -sign
        for i in range(k + 1, n):
            for j in range(k + 1, n):
                M[i][j] = (M[i][j] * M[k][k] - M[i][k] * M[k][j]) / prev
        prev = M[k][k]
    return sign * M[n - 1][n - 1]


def brute_force_gauss(a, b):
    """Textbook Gaussian elimination with partial pivoting in float64 (the
    SPEC's GEPP comparison oracle) — a different algorithm whose result
    agrees with the no-pivot solve to ~1e-10 on diagonally dominant input."""
    n = len(a)
    M = [[float(v) for v in row] + [float(b[i])] for i, row in enumerate(a)]
    for c in range(n):
        piv = max(range(c, n), key=lambda r: abs(M[r][c]))
        M[c], M[piv] = M[piv], M[c]
        for r in range(c + 1, n):
            f = M[r][c] / M[c][c]
            for k in range(c, n + 1):
                M[r][k] -= f * M[c][k]
    x = [0.0] * n
    for i in range(n - 1, -1, -1):
        s = M[i][n]
        for k in range(i + 1, n):
            s -= M[i][k] * x[k]
        x[i] = s / M[i][i]
    return x
