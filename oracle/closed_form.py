"""Closed-form LU of A = alpha*I + beta*s s^T (TEST INFRASTRUCTURE ONLY).

For s in {+1,-1}^n and 1-based indices k (SURVEY.md §8c "closed form"), the
no-pivot Doolittle factors are
    d_k  = u_kk = alpha (alpha + k beta) / (alpha + (k-1) beta)
    l_ik = beta s_i s_k / (alpha + k beta)                 (i > k)
    u_kj = alpha beta s_k s_j / (alpha + (k-1) beta)       (j > k)
Derivation: the Schur complement after k steps is alpha*I + beta_k s s^T with
beta_k = alpha beta / (alpha + k beta) (Sherman-Morrison on the rank-one
part), so the pivot at step k+1 is alpha + beta_k, the multipliers are
beta_k s_i s_k / (alpha + beta_k) ... which simplify to the formulas above.
Strictly row diagonally dominant when alpha > (n-2) beta > 0 (e.g. alpha = n,
beta = 1).  Inverse by Sherman-Morrison:
    A^-1 = (1/alpha) (I - beta s s^T / (alpha + n beta)),
    det A = alpha^(n-1) (alpha + n beta) = prod_k d_k.
The paper's method must reach exactly this factorization (unique LU, Eq 3,
P:41-45), so it pins the oracle and the GPU at any n.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np


def matrix(n: int, alpha: float, beta: float, s: np.ndarray) -> np.ndarray:
    s = np.asarray(s, dtype=np.float64)
    return alpha * np.eye(n) + beta * np.outer(s, s)


def factors_exact(n: int, alpha, beta, s):
    """Exact (Fraction) diagonal d_k, and the two per-k scalars from which
    every l_ik, u_kj follows: cl_k = beta/(alpha+k beta), cu_k = alpha beta/(alpha+(k-1)beta)."""
    a, b = Fraction(alpha), Fraction(beta)
    d, cl, cu = [], [], []
    for k in range(1, n + 1):
        d.append(a * (a + k * b) / (a + (k - 1) * b))
        cl.append(b / (a + k * b))
        cu.append(a * b / (a + (k - 1) * b))
    return d, cl, cu


def packed(n: int, alpha, beta, s) -> np.ndarray:
    """The packed LU as float64 (each entry correctly rounded from exact)."""
    s = np.asarray(s, dtype=np.int64)
    d, cl, cu = factors_exact(n, alpha, beta, s)
    dv = np.array([float(x) for x in d])
    clv = np.array([float(x) for x in cl])
    cuv = np.array([float(x) for x in cu])
    out = np.zeros((n, n))
    ss = np.outer(s, s).astype(np.float64)
    il = np.tril_indices(n, -1)
    iu = np.triu_indices(n, 1)
    out[il] = ss[il] * clv[il[1]]       # l_ik, k = column
    out[iu] = ss[iu] * cuv[iu[0]]       # u_kj, k = row
    out[np.diag_indices(n)] = dv
    return out


def solve(n: int, alpha, beta, s, b: np.ndarray) -> np.ndarray:
    """x = A^-1 b via Sherman-Morrison (float64)."""
    s = np.asarray(s, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return (b - beta * s * (s @ b) / (alpha + n * beta)) / alpha
