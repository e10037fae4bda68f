"""The paper's bi-vectorization and equalization as plain Python (TEST
INFRASTRUCTURE ONLY) — the integer oracle the product's owner maps are
checked against, bit-exactly.

Bi-vectorization (Eq 5-a/b): L and U are split into the
per-index vectors L_(k) (column k of L strictly below the diagonal) and U_(k)
(row k of U strictly right of the diagonal), k = 1..n-1 (1-based), each of
length n-k (reading R5).

Equalization ("for equalizing vectors of first and end of L matrix and
first and end of U matrix combine together"; Eq 7-a..e; counting
claim P:85 "(n-1)/2 vectors ... (n-1) separated vectors"): within each
triangle pair k with n-k, so every unit has length (n-k)+k = n.  For even n
the two middle vectors L_(n/2), U_(n/2) (length n/2 each) are merged into one
cross-triangle unit (reading R12).  Result: exactly n-1 units, all of length n.

Assignment: units dealt round-robin to W workers in unit order ("fit this
measure with number of thread"; the rule itself is unspecified —
reading R12).
"""
from __future__ import annotations


def bivectorize(n: int):
    """2(n-1) descriptors (triangle, k, length): L ascending k, then U."""
    if n < 2:
        raise ValueError("n must be >= 2")
    return [("L", k, n - k) for k in range(1, n)] + [("U", k, n - k) for k in range(1, n)]


def equalize(desc, n: int):
    """List of units; each unit is a tuple of 1 or 2 descriptors."""
    byk = {(t, k): (t, k, ln) for (t, k, ln) in desc}
    if len(byk) != 2 * (n - 1):
        raise ValueError("descriptor list inconsistent with n")
    units = []
    for t in ("L", "U"):
        for k in range(1, (n - 1) // 2 + 1):
            if k != n - k:
                units.append((byk[(t, k)], byk[(t, n - k)]))
    if n % 2 == 0:
        units.append((byk[("L", n // 2)], byk[("U", n // 2)]))
    return units


def assign(units, workers: int):
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return [u % workers for u in range(len(units))]


def unit_positions(unit, n: int):
    """Expand a unit to its (row, col) 0-based matrix positions."""
    pos = []
    for (t, k, _ln) in unit:
        c = k - 1  # 0-based index of the vector
        if t == "L":
            pos += [(i, c) for i in range(c + 1, n)]
        else:
            pos += [(c, j) for j in range(c + 1, n)]
    return pos


def plan_stats(units, owner, workers: int):
    lengths = [0] * workers
    counts = [0] * workers
    for u, w in zip(units, owner):
        lengths[w] += sum(d[2] for d in u)
        counts[w] += 1
    return lengths, counts


def column_pair_owner(n: int, workers: int):
    """Owner map over n column (or row / block) indices used by the GPU
    kernels (reading R12): index j is paired with n-1-j (first with last,
    so each pair's L-vector lengths sum to n-1 and its on-or-below-diagonal
    column lengths to n+1), pairs p = 0,1,.. in order are dealt round-robin,
    and the middle singleton of odd n is the last pair."""
    return [min(j, n - 1 - j) % workers for j in range(n)]
