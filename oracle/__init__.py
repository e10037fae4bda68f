"""Serial CPU oracle for the EbV LU factor + solve hot path (arXiv 1907.05767).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py — never by the product
package ``paper_1907_05767_b200`` (which fails loudly without its CUDA library
instead).  Shares no code with the CUDA path.

Modules
  oracle.c      plain C Doolittle LU + forward/backward substitution in fp64,
                explicit fma, -ffp-contract=off (Eq 1, Eq 6-a..c; see its header)
  exact.py      exact rational LU / solve (fractions.Fraction) and brute-force
                Gaussian elimination — the pins the C oracle is checked against
  closed_form.py closed-form LU of alpha*I + beta*s s^T (any n)
  ebv_plan.py   the paper's bi-vectorization and first-with-last equalization
                (Eq 5, Eq 7) as plain Python

Every function states the PAPER.md line it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

# -ffp-contract=off: no compiler-introduced fma; the only fused operations are
# the explicit fma() calls.  -mfma makes fma() a single instruction (it is
# correctly rounded either way).  No -ffast-math, no -march=native.
CFLAGS = ["-O2", "-mfma", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64, dp, vp = ctypes.c_int64, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p
        lib.oracle_lu_factor.argtypes = [i64, vp, i64, ctypes.c_double]
        lib.oracle_lu_factor.restype = i64
        lib.oracle_lu_solve.argtypes = [i64, vp, i64, vp, i64, i64]
        lib.oracle_lu_solve.restype = None
        lib.oracle_lu_factor_batched.argtypes = [i64, vp, i64, i64, i64, vp, i64, i64, i64,
                                                 ctypes.c_double, vp]
        lib.oracle_lu_factor_batched.restype = None
        lib.oracle_normalize_unit_diagonal.argtypes = [i64, vp, i64, vp, i64, i64, vp]
        lib.oracle_normalize_unit_diagonal.restype = i64
        lib.oracle_lu_to_ldu.argtypes = [i64, vp, i64, vp]
        lib.oracle_lu_to_ldu.restype = None
        del dp
        _lib = lib
    return _lib


def _colmajor(a: np.ndarray) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    return np.array(a, dtype=np.float64, order="F", copy=True)


def lu_factor(a: np.ndarray, tau: float = 0.0):
    """Packed Doolittle LU of a (n x n) without pivoting (Eq 6-a..c).

    Returns (lu, info): lu is a new Fortran-ordered array holding L (strict
    lower, unit diagonal implicit) and U (diagonal + upper); info is 0 or the
    first 1-based step whose pivot satisfies |u_rr| <= tau."""
    lu = _colmajor(a)
    n = lu.shape[0]
    assert lu.shape == (n, n)
    info = _load().oracle_lu_factor(n, lu.ctypes.data, n, float(tau))
    return lu, int(info)


def lu_solve(lu: np.ndarray, b: np.ndarray) -> np.ndarray:
    """X from LY = B (forward) then UX = Y (backward) (Eq 1).
    b may be (n,) or (n, nrhs); returns the same shape."""
    lu = np.asarray(lu, dtype=np.float64, order="F")
    n = lu.shape[0]
    vec = np.ndim(b) == 1
    x = _colmajor(np.reshape(b, (n, -1)))
    _load().oracle_lu_solve(n, lu.ctypes.data, n, x.ctypes.data, n, x.shape[1])
    return x[:, 0].copy() if vec else x


def solve(a: np.ndarray, b: np.ndarray, tau: float = 0.0):
    """AX = B <=> (LU)X = B <=> LY = B, UX = Y (Eq 1). Returns (x, lu, info)."""
    lu, info = lu_factor(a, tau)
    return lu_solve(lu, b), lu, info


def lu_factor_batched(a: np.ndarray, b: np.ndarray | None = None, tau: float = 0.0):
    """Independent systems a[s] (batch, n, n) — each by lu_factor / lu_solve.

    Returns (lu, x, info) with lu (batch, n, n) in logical [i, j] indexing
    (stored column-major per system), x (batch, n, nrhs) or None, info int32."""
    a = np.asarray(a, dtype=np.float64)
    batch, n, _ = a.shape
    # per-system column-major: store transposes contiguously
    at = np.array(np.transpose(a, (0, 2, 1)), order="C", copy=True)
    info = np.zeros(batch, dtype=np.int32)
    if b is not None:
        b = np.asarray(b, dtype=np.float64)
        if b.ndim == 2:
            b = b[:, :, None]
        nrhs = b.shape[2]
        bt = np.array(np.transpose(b, (0, 2, 1)), order="C", copy=True)
        _load().oracle_lu_factor_batched(n, at.ctypes.data, n, n * n, batch, bt.ctypes.data, n, n * nrhs,
                                         nrhs, float(tau), info.ctypes.data)
        x = np.transpose(bt, (0, 2, 1))
    else:
        _load().oracle_lu_factor_batched(n, at.ctypes.data, n, n * n, batch, None, n, 0, 0, float(tau),
                                         info.ctypes.data)
        x = None
    return np.transpose(at, (0, 2, 1)), x, info


def normalize_unit_diagonal(a: np.ndarray, b: np.ndarray | None = None):
    """Row i of a (and of b) divided by a_ii (Eq 2).

    Returns (a', b' or None, scales, info): a' has an exactly-1 diagonal,
    scales[i] = 1/a_ii; info = first 1-based row with a_ii == 0 (left
    unchanged, scale 0), else 0."""
    an = _colmajor(a)
    n = an.shape[0]
    if b is None:
        bn, nrhs, bptr = None, 0, None
    else:
        vec = np.ndim(b) == 1
        bn = _colmajor(np.reshape(b, (n, -1)))
        nrhs, bptr = bn.shape[1], bn.ctypes.data
    scales = np.zeros(n)
    info = _load().oracle_normalize_unit_diagonal(n, an.ctypes.data, n, bptr, n, nrhs, scales.ctypes.data)
    if bn is not None and vec:
        bn = bn[:, 0].copy()
    return an, bn, scales, int(info)


def lu_to_ldu(lu: np.ndarray):
    """LDU form of a packed LU (Eq 3): returns (ldu, d) where ldu
    keeps L (strict lower) and D (diagonal) and holds U' = D^-1 U (strict
    upper, unit diagonal implicit)."""
    ldu = _colmajor(lu)
    n = ldu.shape[0]
    d = np.zeros(n)
    _load().oracle_lu_to_ldu(n, ldu.ctypes.data, n, d.ctypes.data)
    return ldu, d


def unpack(lu: np.ndarray):
    """Split packed LU into (L unit lower, U upper) (Eq 3)."""
    lu = np.asarray(lu)
    n = lu.shape[-1]
    L = np.tril(lu, -1) + np.eye(n)
    U = np.triu(lu)
    return L, U
