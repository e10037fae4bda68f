"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no factorization, no
substitution): only the counter-based generator of the test matrices, which
both sides call on identical seeds.  It is implemented with torch integer ops
so that it produces bit-identical output on the CPU and on a CUDA device.

Generator (the paper never specifies its matrices,
P:37-39 only asks for a "diagonal dominant shape" (Eq 2); distribution per
SPEC S:107, placed on an exact dyadic grid):
  * off-diagonal a_ij = k_ij * 2^-30 with k_ij uniform in [-2^30, 2^30) from a
    32-bit counter hash of (seed, system, i, j)  ->  values uniform in [-1, 1)
  * diagonal a_ii = (sum_{j != i} |k_ij| + 2^30) * 2^-30 = row abs-sum + 1,
    computed in int64 so it is exact and order independent (strict row
    diagonal dominance with margin 1)
  * x_true entries are integers in [-4, 4] from the same hash
  * B = A x_true computed exactly in int64 units of 2^-30 (|B| < 2^48 units,
    so the fp64 value is exact)
Storage: column-major, returned as a torch tensor ``At`` of shape (n, n) whose
row j is column j of A (so At.T is the logical matrix A, and the raw pointer
satisfies a(i, j) = ptr[i + j*n]).
"""
from __future__ import annotations

import torch

M32 = 0xFFFFFFFF
SCALE = 2.0 ** -30
ONE_UNITS = 1 << 30


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for x in [0, 2^32) without int64 overflow."""
    lo, hi = c & 0xFFFF, c >> 16
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & M32


def hash32(x: torch.Tensor) -> torch.Tensor:
    """lowbias32 integer hash on values in [0, 2^32) held in int64."""
    x = x & M32
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def _h(v: int) -> int:
    return int(hash32(torch.tensor([v & M32], dtype=torch.int64))[0])


def system_base(seed: int, system: int) -> int:
    return _h(_h(seed) ^ (system & M32))


def _base_tensor(seed: int, systems: torch.Tensor) -> torch.Tensor:
    return hash32(torch.full_like(systems, _h(seed)) ^ (systems & M32))


def offdiag_units(base, rows: torch.Tensor, cols: torch.Tensor) -> torch.Tensor:
    """k_ij in [-2^30, 2^30) for broadcastable row / column index tensors."""
    h = hash32(hash32(base ^ rows) ^ cols)
    return (h & 0x7FFFFFFF) - ONE_UNITS


def xtrue_units(base, rows: torch.Tensor, rhs: torch.Tensor, n: int) -> torch.Tensor:
    h = hash32(hash32(base ^ 0x68E31DA4) ^ (rhs * n + rows))
    return (h % 9) - 4


def generate(n: int, seed: int = 1, nrhs: int = 1, device="cpu", system: int = 0,
             cols: torch.Tensor | None = None, chunk: int = 2048, with_b: bool = True,
             kl: int | None = None, ku: int | None = None, stencil_m: int | None = None):
    """Strictly row-diagonally-dominant system on the 2^-30 grid.

    Returns dict(At=(ncols, n) float64 column-major storage of A[:, cols],
    X=(n, nrhs) float64 exact solution, B=(n, nrhs) float64 = A X exactly).
    ``cols`` selects a subset of columns (a rank's local slab); row sums are
    always taken over all n columns.  Sparsity (the paper's
    banded / sparse workload, synthetic): ``kl`` / ``ku`` keep only
    the entries with i - j <= kl and j - i <= ku (a band); ``stencil_m``
    keeps the 2D five-point pattern of an m x m grid (n = m^2: neighbours
    i +- 1 within a grid row and i +- m).  Zeros are exact; the diagonal
    stays row abs-sum + 1."""
    dev = torch.device(device)
    base = system_base(seed, system)
    rows = torch.arange(n, dtype=torch.int64, device=dev)
    rr = torch.arange(nrhs, dtype=torch.int64, device=dev)
    X_u = xtrue_units(base, rows[:, None], rr[None, :], n)            # (n, nrhs) int
    rowsum = torch.zeros(n, dtype=torch.int64, device=dev)
    rowdot = torch.zeros(n, nrhs, dtype=torch.int64, device=dev)
    if cols is None:
        cols = torch.arange(n, dtype=torch.int64, device=dev)
    cols = cols.to(dev)
    At = torch.empty(cols.numel(), n, dtype=torch.float64, device=dev)
    pos = torch.full((n,), -1, dtype=torch.int64, device=dev)
    pos[cols] = torch.arange(cols.numel(), dtype=torch.int64, device=dev)
    for j0 in range(0, n, chunk):
        j1 = min(n, j0 + chunk)
        jj = torch.arange(j0, j1, dtype=torch.int64, device=dev)
        K = offdiag_units(base, rows[None, :], jj[:, None])            # (cj, n): K[c, i] = k_{i, j0+c}
        diag = (rows[None, :] == jj[:, None])
        K = torch.where(diag, torch.zeros_like(K), K)
        if kl is not None or ku is not None:
            d = jj[:, None] - rows[None, :]                              # j - i
            keep_b = torch.ones_like(diag)
            if kl is not None:
                keep_b &= (-d) <= kl
            if ku is not None:
                keep_b &= d <= ku
            K = torch.where(keep_b, K, torch.zeros_like(K))
        if stencil_m is not None:
            m = stencil_m
            d = (jj[:, None] - rows[None, :]).abs()
            same_row = (jj[:, None] // m) == (rows[None, :] // m)
            keep_s = ((d == 1) & same_row) | (d == m)
            K = torch.where(keep_s, K, torch.zeros_like(K))
        rowsum += K.abs().sum(0)
        if with_b:
            rowdot += K.t() @ X_u[j0:j1] if dev.type == "cpu" else _int_matmul(K.t(), X_u[j0:j1])
        sel = pos[j0:j1]
        keep = sel >= 0
        if keep.any():
            At[sel[keep]] = K[keep].to(torch.float64) * SCALE
        del K, diag
    dunits = rowsum + ONE_UNITS
    # diagonal entries of the stored columns
    lc = torch.arange(cols.numel(), device=dev)
    At[lc, cols] = dunits[cols].to(torch.float64) * SCALE
    out = {"At": At, "X": X_u.to(torch.float64), "n": n, "seed": seed, "system": system}
    if with_b:
        B_u = rowdot + dunits[:, None] * X_u
        out["B"] = B_u.to(torch.float64) * SCALE
    return out


def _int_matmul(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """int64 (m, k) @ (k, r) on CUDA (no int GEMM there): exact via a
    broadcast multiply + sum over k in slices."""
    out = torch.zeros(a.shape[0], b.shape[1], dtype=torch.int64, device=a.device)
    for r in range(b.shape[1]):
        out[:, r] = (a * b[:, r][None, :]).sum(1)
    return out


def generate_batched(batch: int, n: int = 32, seed: int = 1, nrhs: int = 1, device="cpu",
                     first_system: int = 0):
    """Independent systems (BASELINE.json configs[4]): system s uses
    system_base(seed, first_system + s).  Returns At (batch, n, n) with
    At[s, j, i] = a^(s)_ij (per-system column-major), X and B (batch, n, nrhs)."""
    dev = torch.device(device)
    sys_ids = torch.arange(first_system, first_system + batch, dtype=torch.int64, device=dev)
    base = _base_tensor(seed, sys_ids)[:, None, None]                  # (b,1,1)
    rows = torch.arange(n, dtype=torch.int64, device=dev)
    K = offdiag_units(base, rows[None, None, :], rows[None, :, None])  # (b, j, i) = k_ij
    eye = torch.eye(n, dtype=torch.bool, device=dev)[None]
    K = torch.where(eye, torch.zeros_like(K), K)
    rowsum = K.abs().sum(1)                                           # (b, i)
    dunits = rowsum + ONE_UNITS
    rr = torch.arange(nrhs, dtype=torch.int64, device=dev)
    X_u = xtrue_units(base, rows[None, :, None], rr[None, None, :], n)  # (b, n, nrhs)
    # B_i = sum_j k_ij x_j + d_i x_i   (exact int64)
    B_u = torch.zeros(batch, n, nrhs, dtype=torch.int64, device=dev)
    for r in range(nrhs):
        B_u[:, :, r] = (K * X_u[:, :, r][:, :, None]).sum(1)
    B_u += dunits[:, :, None] * X_u
    At = K.to(torch.float64) * SCALE
    At[:, rows, rows] = dunits.to(torch.float64) * SCALE
    return {"At": At, "X": X_u.to(torch.float64), "B": B_u.to(torch.float64) * SCALE, "n": n}


def closed_form_inputs(n: int, seed: int = 1, alpha: float | None = None, beta: float = 1.0, device="cpu"):
    """A = alpha I + beta s s^T with s_i = +-1 from the hash (oracle/closed_form.py
    gives its LU in closed form).  Returns (At column-major, s int64)."""
    dev = torch.device(device)
    alpha = float(n) if alpha is None else alpha
    rows = torch.arange(n, dtype=torch.int64, device=dev)
    s = (hash32(hash32(torch.full_like(rows, _h(seed) ^ 0x51ED270B)) ^ rows) & 1) * 2 - 1
    sf = s.to(torch.float64)
    At = beta * torch.outer(sf, sf)
    At[rows, rows] += alpha
    return At, s


def generate_leading(n: int, m: int, seed: int = 1, nrhs: int = 1, device="cpu", system: int = 0):
    """The leading m x m principal submatrix of generate(n, seed) (same
    entries bit for bit: the diagonal uses the full-row sums over all n
    columns), plus an exact right-hand side B_m = A_m X_m for the first m
    entries of x_true.  Cost O(m n) hashes — a bounded sample of the
    n x n workload for the CPU baseline."""
    dev = torch.device(device)
    base = system_base(seed, system)
    rows = torch.arange(m, dtype=torch.int64, device=dev)
    rowsum = torch.zeros(m, dtype=torch.int64, device=dev)
    chunk = max(1, (1 << 24) // max(m, 1))
    for j0 in range(0, n, chunk):
        j1 = min(n, j0 + chunk)
        jj = torch.arange(j0, j1, dtype=torch.int64, device=dev)
        K = offdiag_units(base, rows[None, :], jj[:, None])
        K = torch.where(rows[None, :] == jj[:, None], torch.zeros_like(K), K)
        rowsum += K.abs().sum(0)
    jj = torch.arange(m, dtype=torch.int64, device=dev)
    K = offdiag_units(base, rows[None, :], jj[:, None])
    K = torch.where(rows[None, :] == jj[:, None], torch.zeros_like(K), K)
    dunits = rowsum + ONE_UNITS
    rr = torch.arange(nrhs, dtype=torch.int64, device=dev)
    X_u = xtrue_units(base, rows[:, None], rr[None, :], n)
    B_u = (K.t() @ X_u if dev.type == "cpu" else _int_matmul(K.t(), X_u)) + dunits[:, None] * X_u
    At = K.to(torch.float64) * SCALE
    At[jj, jj] = dunits.to(torch.float64) * SCALE
    return {"At": At, "X": X_u.to(torch.float64), "B": B_u.to(torch.float64) * SCALE, "n": m}


def generate_band(n: int, kl: int, ku: int, pad: int, ldab: int, seed: int = 1, nrhs: int = 1, device="cpu",
                  system: int = 0):
    """The banded matrix of ``generate(n, seed, kl=kl, ku=ku)`` (the same
    entries bit for bit) written directly in compact band storage, so orders
    whose dense storage would not fit can be generated: returns dict(AB=(n,
    ldab) float64 whose row j is column j of the ldab x n column-major band
    storage, a_ij at AB[j, pad + ku + i - j] — the layout of include/ebv.h —
    X, B as generate).  Layout only; no arithmetic of the method."""
    dev = torch.device(device)
    base = system_base(seed, system)
    j = torch.arange(n, dtype=torch.int64, device=dev)
    rr = torch.arange(nrhs, dtype=torch.int64, device=dev)
    X_u = xtrue_units(base, j[:, None], rr[None, :], n)                 # (n, nrhs)
    AB = torch.zeros(n, ldab, dtype=torch.float64, device=dev)
    rowsum = torch.zeros(n, dtype=torch.int64, device=dev)
    rowdot = torch.zeros(n, nrhs, dtype=torch.int64, device=dev)
    for d in range(-ku, kl + 1):                                         # diagonal d = i - j
        if d == 0:
            continue
        jj = j[(j + d >= 0) & (j + d < n)]
        ii = jj + d
        K = offdiag_units(base, ii, jj)
        AB[jj, pad + ku + d] = K.to(torch.float64) * SCALE
        rowsum.index_add_(0, ii, K.abs())
        rowdot.index_add_(0, ii, K[:, None] * X_u[jj])
    dunits = rowsum + ONE_UNITS
    AB[j, pad + ku] = dunits.to(torch.float64) * SCALE
    B_u = rowdot + dunits[:, None] * X_u
    return {"AB": AB, "X": X_u.to(torch.float64), "B": B_u.to(torch.float64) * SCALE, "n": n, "seed": seed}


# ---------------------------------------------------------------- edge-case flavours
EDGE_FLAVOURS = ("neg", "rowsign", "colsign", "scaled", "rhs_tiny", "rhs_huge")


def _signs(n: int, seed: int, salt: int, device) -> torch.Tensor:
    rows = torch.arange(n, dtype=torch.int64, device=device)
    return ((hash32(hash32(torch.full_like(rows, _h(seed) ^ salt)) ^ rows) & 1) * 2 - 1).to(torch.float64)


def _pow2(n: int, seed: int, salt: int, emax: int, device) -> torch.Tensor:
    rows = torch.arange(n, dtype=torch.int64, device=device)
    e = (hash32(hash32(torch.full_like(rows, _h(seed) ^ salt)) ^ rows) % (2 * emax + 1)) - emax
    return torch.ldexp(torch.ones(n, dtype=torch.float64, device=device), e)


def edge_flavour(A: torch.Tensor, B: torch.Tensor, flavour: str, seed: int = 1, emax: int = 500):
    """Sign / scale variants of a generated system (A logical (..., n, n), B
    (..., n, nrhs)) that exercise the division edge cases: negative and
    mixed-sign pivots, multipliers and quotients far outside [2^-54, 2^54]
    (subnormal / tiny ones, which the kernels' verified-quotient tests send to
    their true-division branches).  Every transform multiplies rows / columns
    by signs and powers of two, so it is exact (no method arithmetic):
      neg       A' = -A, B' = -B                       (x unchanged)
      rowsign   A' = S1 A, B' = S1 B                   (row signs: mixed pivots)
      colsign   A' = A S2                              (x' = S2 x; B unchanged)
      scaled    A' = D1 S1 A S2 D2, B' = D1 S1 B       (D = 2^e, |e| <= emax)
      rhs_tiny  A' = 2^530 A, B' = 2^-530 B            (x' = 2^-1060 x: subnormal quotients)
      rhs_huge  A' = 2^-500 A, B' = 2^500 B            (x' = 2^1000 x)
    Returns (A', B') as new tensors of A's / B's dtype and device."""
    n = A.shape[-1]
    dev = A.device
    if flavour == "neg":
        return -A, -B
    if flavour == "rowsign":
        s = _signs(n, seed, 0x1B873593, dev)
        return A * s[:, None], B * s[:, None]
    if flavour == "colsign":
        s = _signs(n, seed, 0x2F7A1C3D, dev)
        return A * s[None, :], B.clone()
    if flavour == "scaled":
        s1 = _signs(n, seed, 0x1B873593, dev) * _pow2(n, seed, 0x3C6EF372, emax, dev)
        s2 = _signs(n, seed, 0x2F7A1C3D, dev) * _pow2(n, seed, 0x5BD1E995, emax, dev)
        return A * s1[:, None] * s2[None, :], B * s1[:, None]
    if flavour == "rhs_tiny":
        return torch.ldexp(A, torch.tensor(530, device=dev)), torch.ldexp(B, torch.tensor(-530, device=dev))
    if flavour == "rhs_huge":
        return torch.ldexp(A, torch.tensor(-500, device=dev)), torch.ldexp(B, torch.tensor(500, device=dev))
    raise ValueError(flavour)
