"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: the SPEC's worked examples
(tests/golden, cited per entry), exact rational arithmetic, closed forms,
LAPACK special cases, metamorphic invariants and brute force.
"""
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg

import ebv_inputs
import oracle
from oracle import closed_form, exact


def gen(n, seed=1, nrhs=1):
    d = ebv_inputs.generate(n, seed=seed, nrhs=nrhs)
    return d["At"].T.numpy().copy(), d["X"].numpy(), d["B"].numpy()


def fma(a, b, c):
    """Correctly rounded a*b + c via exact rationals (int true division in
    CPython rounds correctly)."""
    from fractions import Fraction
    return float(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


# ---------------------------------------------------------------- worked values
def test_spec_factor_examples(golden):
    for ex in golden["factor"]:
        lu, info = oracle.lu_factor(np.array(ex["a"], dtype=float))
        assert info == ex["info"], ex["cite"]
        if "packed" in ex:
            assert np.array_equal(lu, np.array(ex["packed"], dtype=float)), ex["cite"]


def test_spec_substitution_examples(golden):
    for ex in golden["forward"]:
        # forward only: U = I keeps backward an identity (pack L with unit U)
        packed = np.array(ex["packed"], dtype=float)
        lu = np.tril(packed, -1) + np.eye(len(packed))
        y = oracle.lu_solve(lu, np.array(ex["b"], dtype=float))
        assert np.array_equal(y, np.array(ex["y"])), ex["cite"]
    for ex in golden["backward"]:
        packed = np.array(ex["packed"], dtype=float)
        lu = np.triu(packed)  # L = I: forward is the identity
        x = oracle.lu_solve(lu, np.array(ex["y"], dtype=float))
        assert np.array_equal(x, np.array(ex["x"])), ex["cite"]
    for ex in golden["solve"]:
        x, _, info = oracle.solve(np.array(ex["a"], dtype=float), np.array(ex["b"], dtype=float))
        assert info == 0
        assert np.max(np.abs(x - np.array(ex["x"]))) <= ex["tol"], ex["cite"]


def test_spec_residual_examples(golden):
    for ex in golden["residual_inf"]:
        a, x, b = (np.array(ex[k], dtype=float) for k in ("a", "x", "b"))
        assert np.max(np.abs(a @ x - b)) == ex["r"], ex["cite"]


# ---------------------------------------------------------------- exact rational
@pytest.mark.parametrize("n,seed", [(2, 1), (3, 2), (5, 3), (8, 4), (16, 5), (33, 6), (64, 7)])
def test_exact_rational_lu_and_solve(n, seed):
    """The unique no-pivot LU of the exact input, computed with Crout formulas
    in rationals; the fp64 oracle must agree normwise to ~1e-14, and the exact
    Gauss-Jordan solution of A x = b must be x_true (b = A x_true exactly)."""
    a, x_true, b = gen(n, seed)
    L, U = exact.lu_exact(a)
    lu, info = oracle.lu_factor(a)
    assert info == 0
    Lf = np.array([[float(v) for v in r] for r in L])
    Uf = np.array([[float(v) for v in r] for r in U])
    Lo, Uo = oracle.unpack(lu)
    assert np.max(np.abs(Lo - Lf)) <= 1e-14 * max(1.0, np.max(np.abs(Lf)))
    assert np.max(np.abs(Uo - Uf)) <= 1e-14 * np.max(np.abs(Uf))
    xs = exact.solve_exact(a, b[:, 0])
    assert [float(v) for v in xs] == list(x_true[:, 0])
    x = oracle.lu_solve(lu, b)
    assert np.max(np.abs(x - x_true)) <= 1e-13


def test_exact_first_step_bitwise():
    """After step 1 the multipliers are single correctly rounded divisions
    a_i0 / a_00 (Eq 6-a) and row 0 is untouched (Eq 6-b): bitwise."""
    a, _, _ = gen(12, 7)
    lu, _ = oracle.lu_factor(a)
    assert np.array_equal(lu[1:, 0], a[1:, 0] / a[0, 0])
    assert np.array_equal(lu[0, :], a[0, :])


def test_second_step_bitwise_against_handwritten():
    """Entries of step 2 written out by hand: u_11 = fma(-l10, u01, a11),
    l_21 = fma(-l20, u01, a21) / u11 — a transposed operand or a wrong
    index in the oracle fails this."""
    a, _, _ = gen(6, 11)
    lu, _ = oracle.lu_factor(a)
    l10, l20, u01 = a[1, 0] / a[0, 0], a[2, 0] / a[0, 0], a[0, 1]
    u11 = fma(-l10, u01, a[1, 1])
    assert lu[1, 1] == u11
    assert lu[2, 1] == fma(-l20, u01, a[2, 1]) / u11
    assert lu[1, 2] == fma(-l10, a[0, 2], a[1, 2])


# ---------------------------------------------------------------- closed form
@pytest.mark.parametrize("n", [7, 64, 300])
def test_closed_form_family(n):
    s = np.where(np.arange(n) % 3 == 0, -1, 1)
    a = closed_form.matrix(n, float(n), 1.0, s)
    lu, info = oracle.lu_factor(a)
    assert info == 0
    ref = closed_form.packed(n, n, 1, s)
    rel = np.abs(lu - ref) / np.maximum(np.abs(ref), 1e-300)
    assert np.max(rel) <= 64 * np.finfo(float).eps * n ** 0.5
    b = a @ np.arange(1.0, n + 1.0)
    x = oracle.lu_solve(lu, b)
    assert np.max(np.abs(x - closed_form.solve(n, n, 1.0, s, b))) <= 1e-12 * np.max(np.abs(x))
    # det A = alpha^(n-1) (alpha + n beta) = prod d_k
    logdet = np.sum(np.log(np.abs(np.diag(lu))))
    assert abs(logdet - ((n - 1) * np.log(n) + np.log(2 * n))) <= 1e-12 * abs(logdet)


def test_closed_form_exact_small():
    """Closed form vs exact rational LU: the formulas themselves are pinned."""
    n = 9
    s = np.array([1, -1, 1, 1, -1, -1, 1, -1, 1])
    a = closed_form.matrix(n, 9.0, 1.0, s)
    L, U = exact.lu_exact(a)
    d, cl, cu = closed_form.factors_exact(n, 9, 1, s)
    for k in range(n):
        assert U[k][k] == d[k]
        for i in range(k + 1, n):
            assert L[i][k] == cl[k] * int(s[i]) * int(s[k])
            assert U[k][i] == cu[k] * int(s[k]) * int(s[i])


# ---------------------------------------------------------------- metamorphic
def test_power_of_two_scaling_bitwise():
    a, _, _ = gen(40, 3)
    lu1, _ = oracle.lu_factor(a)
    lu2, _ = oracle.lu_factor(a * 8.0)
    L1, U1 = np.tril(lu1, -1), np.triu(lu1)
    assert np.array_equal(np.tril(lu2, -1), L1)
    assert np.array_equal(np.triu(lu2), 8.0 * U1)


def test_triangular_and_diagonal_inputs():
    rng = np.random.default_rng(5)
    n = 17
    up = np.triu(rng.uniform(-1, 1, (n, n))) + 20 * np.eye(n)
    assert np.array_equal(oracle.lu_factor(up)[0], up)
    lo = np.tril(rng.uniform(-1, 1, (n, n))) + 20 * np.eye(n)
    lu, _ = oracle.lu_factor(lo)
    assert np.array_equal(np.triu(lu), np.diag(np.diag(lo)))
    assert np.array_equal(np.tril(lu, -1), np.tril(lo, -1) / np.diag(lo)[None, :])
    dg = np.diag(rng.uniform(1, 2, n))
    assert np.array_equal(oracle.lu_factor(dg)[0], dg)


def test_block_diagonal_is_blockwise():
    a1, _, _ = gen(10, 1)
    a2, _, _ = gen(7, 2)
    a = scipy.linalg.block_diag(a1, a2)
    lu, _ = oracle.lu_factor(a)
    assert np.array_equal(lu[:10, :10], oracle.lu_factor(a1)[0])
    assert np.array_equal(lu[10:, 10:], oracle.lu_factor(a2)[0])
    assert not lu[10:, :10].any() and not lu[:10, 10:].any()


def test_leading_principal_submatrix_bitwise():
    a, _, _ = gen(64, 9)
    lu, _ = oracle.lu_factor(a)
    for m in (1, 17, 40):
        assert np.array_equal(oracle.lu_factor(a[:m, :m])[0], lu[:m, :m])


# ---------------------------------------------------------------- library special case
@pytest.mark.parametrize("n", [50, 256])
def test_lapack_no_swaps_special_case(n):
    """On these inputs LAPACK getrf makes no interchanges (piv = identity), so
    it computes the same factorization (different summation order)."""
    a, x_true, b = gen(n, 4)
    lu_l, piv = scipy.linalg.lu_factor(a)
    assert np.array_equal(piv, np.arange(n))
    lu, _ = oracle.lu_factor(a)
    assert np.max(np.abs(lu - lu_l)) <= 1e-13 * np.max(np.abs(lu_l))
    x = oracle.lu_solve(lu, b)
    assert np.max(np.abs(x - scipy.linalg.lu_solve((lu_l, piv), b))) <= 1e-12


def test_brute_force_gepp_agreement():
    for seed in range(5):
        a, _, b = gen(12, seed)
        x, _, _ = oracle.solve(a, b[:, 0])
        xb = exact.brute_force_gauss(a, b[:, 0])
        assert np.max(np.abs(x - xb)) <= 1e-12


# ---------------------------------------------------------------- invariants
@pytest.mark.parametrize("n", [64, 512])
def test_reconstruction_and_backward_error(n):
    a, x_true, b = gen(n, 2, nrhs=3)
    lu, info = oracle.lu_factor(a)
    L, U = oracle.unpack(lu)
    assert info == 0
    assert np.max(np.abs(L @ U - a)) / np.max(np.abs(a)) <= 1e-13
    x = oracle.lu_solve(lu, b)
    r = np.max(np.abs(a @ x - b)) / (np.max(np.sum(np.abs(a), 1)) * np.max(np.abs(x)))
    assert r <= 1e-12
    # growth factor <= 2 for diagonally dominant (Wilkinson)
    assert np.max(np.abs(U)) <= 2 * np.max(np.abs(a))


def test_pivot_threshold_semantics():
    a = np.array([[1e-20, 1.0], [1.0, 1.0]])
    assert oracle.lu_factor(a, tau=0.0)[1] == 0
    assert oracle.lu_factor(a, tau=1e-10)[1] == 1
    z = np.eye(4)
    z[2, 2] = 0.0
    lu, info = oracle.lu_factor(z)
    assert info == 3
    # factorization continues past a failing step (LAPACK convention)
    z = np.eye(4)
    z[1, 1] = 0.0
    z[3, 3] = 0.0
    assert oracle.lu_factor(z)[1] == 2


def test_batched_equals_per_system():
    d = ebv_inputs.generate_batched(7, 32, seed=3, nrhs=2)
    a = d["At"].transpose(1, 2).numpy()
    b = d["B"].numpy()
    lu, x, info = oracle.lu_factor_batched(a, b)
    assert not info.any()
    for s in range(7):
        lus, _ = oracle.lu_factor(a[s])
        assert np.array_equal(lu[s], lus)
        assert np.array_equal(x[s], oracle.lu_solve(lus, b[s]))
        assert np.max(np.abs(x[s] - d["X"][s].numpy())) <= 1e-13


def test_no_pivot_failure_over_seeds():
    """no singular-pivot error on strictly DD input (100 seeds)."""
    for seed in range(100):
        a, _, _ = gen(24, seed)
        assert oracle.lu_factor(a)[1] == 0


# ---------------------------------------------------------------- f3: unit diagonal / LDU
def test_spec_normalize_examples(golden):
    for ex in golden["normalize_unit_diagonal"]:
        a = np.array(ex["a"], dtype=np.float64)
        out, _, scales, info = oracle.normalize_unit_diagonal(a)
        assert info == ex["info"], ex["cite"]
        if info == 0:
            assert np.array_equal(out, np.array(ex["out"], dtype=np.float64)), ex["cite"]
            assert np.array_equal(scales, np.array(ex["scales"], dtype=np.float64)), ex["cite"]


def _ulp(x):
    return np.spacing(np.abs(x))


@pytest.mark.parametrize("n,seed", [(7, 1), (40, 2)])
def test_normalize_is_correctly_rounded_and_preserves_dominance(n, seed):
    """Each entry is within half an ulp of the exact quotient a_ij / a_ii
    (exact rationals), the diagonal is exactly 1, strict row dominance
    survives (Eq 2's shape), and the scaled right-hand side keeps the
    solution up to rounding."""
    d = ebv_inputs.generate(n, seed=seed, nrhs=1)
    a = d["At"].T.numpy().copy()
    b = d["B"].numpy().copy()
    out, bn, scales, info = oracle.normalize_unit_diagonal(a, b)
    assert info == 0
    assert np.all(np.diag(out) == 1.0)
    for i in range(n):
        for j in range(n):
            exact = Fraction(a[i, j]) / Fraction(a[i, i])
            assert abs(Fraction(out[i, j]) - exact) <= Fraction(_ulp(out[i, j])) / 2
        assert abs(Fraction(scales[i]) - 1 / Fraction(a[i, i])) <= Fraction(_ulp(scales[i])) / 2
    off = np.abs(out).sum(axis=1) - 1.0
    assert np.all(off < 1.0)
    x = oracle.solve(out, bn)[0]
    assert np.max(np.abs(x - d["X"].numpy())) <= 1e-12


def test_ldu_of_symmetric_matrix_has_u_prime_equal_l_transpose():
    """For symmetric A, A = L D U' = L D L^T, so U' = L^T (a property of the
    factorization, not of the code): checked on the closed-form family
    alpha I + beta s s^T to a few ulps, with D = diag(U) bitwise and L
    untouched bitwise."""
    n = 60
    s_ = np.where(np.random.default_rng(3).random(n) < 0.5, -1.0, 1.0)
    a = closed_form.matrix(n, float(n), 1.0, s_)
    lu, _ = oracle.lu_factor(a)
    ldu, dvec = oracle.lu_to_ldu(lu)
    assert np.array_equal(dvec, np.diag(lu))
    assert np.array_equal(np.tril(ldu), np.tril(lu))
    L = np.tril(lu, -1)
    up = np.triu(ldu, 1)
    assert np.max(np.abs(up - L.T)) <= 4 * np.finfo(float).eps * np.max(np.abs(L))
    # and every U' entry is the correctly rounded quotient u_kj / u_kk
    for k in range(n):
        for j in range(k + 1, n):
            exact = Fraction(lu[k, j]) / Fraction(lu[k, k])
            assert abs(Fraction(ldu[k, j]) - exact) <= Fraction(_ulp(ldu[k, j])) / 2


# ---------------------------------------------------------------- f4: banded / stencil inputs
@pytest.mark.parametrize("n,kl,ku", [(40, 3, 5), (33, 0, 4), (30, 6, 0), (25, 24, 1)])
def test_banded_lu_keeps_the_band(n, kl, ku):
    """No-pivot LU of a (kl, ku)-banded matrix has L of lower bandwidth kl and
    U of upper bandwidth ku (Golub & Van Loan Thm 4.3.1): every entry of the
    oracle's packed factors outside the band is exactly zero, and inside it
    the factors equal the exact rational LU to ~1e-14."""
    d = ebv_inputs.generate(n, seed=n + kl, kl=kl, ku=ku)
    a = d["At"].T.numpy().copy()
    i, j = np.indices((n, n))
    assert np.all(a[(i - j > kl) | (j - i > ku)] == 0.0)
    lu, info = oracle.lu_factor(a)
    assert info == 0
    assert np.all(lu[(i - j > kl) | (j - i > ku)] == 0.0)
    L, U = exact.lu_exact(a)
    Lf = np.array([[float(v) for v in r] for r in L])
    Uf = np.array([[float(v) for v in r] for r in U])
    Lo, Uo = oracle.unpack(lu)
    assert np.max(np.abs(Lo - Lf)) <= 1e-14 * max(1.0, np.max(np.abs(Lf)))
    assert np.max(np.abs(Uo - Uf)) <= 1e-14 * np.max(np.abs(Uf))


def test_stencil_fill_stays_in_the_band():
    """The 2D five-point pattern on an m x m grid: the LU fills in only within
    the bandwidth m (the profile of the outermost nonzeros), exactly zero
    outside; the solution is x_true to rounding."""
    m = 6
    n = m * m
    d = ebv_inputs.generate(n, seed=4, stencil_m=m)
    a = d["At"].T.numpy().copy()
    lu, info = oracle.lu_factor(a)
    i, j = np.indices((n, n))
    assert info == 0 and np.all(lu[np.abs(i - j) > m] == 0.0)
    x = oracle.lu_solve(lu, d["B"].numpy())
    assert np.max(np.abs(x - d["X"].numpy())) <= 1e-13
