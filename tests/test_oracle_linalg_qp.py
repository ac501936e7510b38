"""Oracle sparse linear algebra and ADMM pinned to /root/reference/proj/tests/test_linalg.cpp and
test_qp.cpp (dense numpy oracles as in tests/oracles.hpp).  CPU only."""
import itertools

import numpy as np
import pytest


def random_quasi_definite(r, n, m, density=0.4):
    """oracles.hpp:203-219."""
    B = np.where(r.uniform(size=(n, n)) < density, r.uniform(-1, 1, (n, n)), 0.0)
    A = np.where(r.uniform(size=(m, n)) < density, r.uniform(-1, 1, (m, n)), 0.0)
    K = np.zeros((n + m, n + m))
    K[:n, :n] = B.T @ B + 1e-6 * np.eye(n)
    K[:n, n:] = A.T
    K[n:, :n] = A
    K[n:, n:] = -10.0 * np.eye(m)
    return K


def random_strictly_convex_qp(r, n, m):
    """oracles.hpp:245-266."""
    B = r.uniform(-1, 1, (n, n))
    P = B.T @ B + 0.5 * np.eye(n)
    q = r.uniform(-1, 1, n)
    A = r.uniform(-1, 1, (m, n))
    x0 = r.uniform(-0.5, 0.5, n)
    ax = A @ x0
    lo = ax - 0.1 - r.uniform(0, 1, m)
    hi = ax + 0.1 + r.uniform(0, 1, m)
    return P, q, A, lo, hi


def active_set_enumerate(P, q, A, lo, hi, tol=1e-9):
    """oracles.hpp:281-339: global optimum by enumerating all 3^m active sets."""
    n, m = P.shape[0], A.shape[0]
    best, best_x = np.inf, None
    for assign in itertools.product((0, 1, 2), repeat=m):
        act = [i for i in range(m) if assign[i]]
        na = len(act)
        K = np.zeros((n + na, n + na))
        rhs = np.zeros(n + na)
        K[:n, :n] = P
        rhs[:n] = -q
        for r_, i in enumerate(act):
            K[n + r_, :n] = A[i]
            K[:n, n + r_] = A[i]
            rhs[n + r_] = lo[i] if assign[i] == 1 else hi[i]
        if np.linalg.matrix_rank(K) < n + na:
            continue
        sol = np.linalg.solve(K, rhs)
        x = sol[:n]
        ax = A @ x
        if np.any(ax < lo - tol) or np.any(ax > hi + tol):
            continue
        ok = True
        for r_, i in enumerate(act):
            y = sol[n + r_]
            if (assign[i] == 1 and y > tol) or (assign[i] == 2 and y < -tol):
                ok = False
        if not ok:
            continue
        obj = 0.5 * x @ P @ x + q @ x
        if obj < best - 1e-12:
            best, best_x = obj, x
    return best_x


# ---------------------------------------------------------------- CSC (test_linalg.cpp:14-56)
def test_csc_duplicates_summed(oracle):
    colptr, rowidx, v = oracle.csc_from_triplets([0, 0], [0, 0], [1.0, 2.0], 1, 1)
    assert len(v) == 1 and v[0] == 3.0


def test_csc_random_triplets_match_dense(oracle):
    r = np.random.default_rng(7)
    rows, cols, vals = r.integers(0, 10, 60), r.integers(0, 10, 60), r.uniform(-2, 2, 60)
    dense = np.zeros((10, 10))
    np.add.at(dense, (rows, cols), vals)
    colptr, rowidx, v = oracle.csc_from_triplets(rows, cols, vals, 10, 10)
    rec = np.zeros((10, 10))
    for j in range(10):
        for p in range(colptr[j], colptr[j + 1]):
            rec[rowidx[p], j] = v[p]
        assert np.all(np.diff(rowidx[colptr[j]:colptr[j + 1]]) > 0)
    np.testing.assert_allclose(rec, dense, atol=1e-15)


def test_csc_keeps_explicit_zeros(oracle):
    """csc.cpp:35-91: explicit zeros are kept (build_qp relies on it, mpc.cpp:169-172)."""
    colptr, rowidx, v = oracle.csc_from_triplets([0, 1], [0, 0], [0.0, 1.0], 2, 1)
    assert len(v) == 2 and v[0] == 0.0


def test_csc_out_of_range(oracle):
    with pytest.raises(ValueError):
        oracle.csc_from_triplets([2], [0], [1.0], 2, 2)
    with pytest.raises(ValueError):
        oracle.csc_from_triplets([0], [-1], [1.0], 2, 2)


# ---------------------------------------------------------------- Ruiz (test_linalg.cpp:87-142)
def test_ruiz_identity(oracle):
    K, s = oracle.ruiz(np.eye(4))
    assert np.all(s == 1.0) and np.all(K == np.eye(4))


def test_ruiz_diag_known_answer(oracle):
    K, s = oracle.ruiz(np.diag([1.0, 10000.0]))
    assert s[0] == pytest.approx(1.0, rel=1e-12) and s[1] == pytest.approx(0.01, rel=1e-12)
    np.testing.assert_allclose(np.diag(K), [1.0, 1.0], rtol=1e-12)


def test_ruiz_random_norms_in_range(oracle):
    r = np.random.default_rng(13)
    K = np.tril(r.uniform(-5, 5, (20, 20)) * 10 ** r.uniform(-3, 3, (20, 20)))
    K = K + np.tril(K, -1).T
    S, _ = oracle.ruiz(K)
    norms = np.max(np.abs(S), axis=1)
    assert np.all(norms >= 0.5) and np.all(norms <= 2.0)


def test_ruiz_idempotent(oracle):
    r = np.random.default_rng(17)
    K = random_quasi_definite(r, 8, 5)
    S, _ = oracle.ruiz(K)
    _, s2 = oracle.ruiz(S)
    assert np.max(np.abs(s2 - 1)) < 1e-6


def test_ruiz_zero_row_keeps_scale_one(oracle):
    _, s = oracle.ruiz(np.diag([4.0, 0.0, 9.0]))
    assert s[1] == 1.0 and np.isfinite(s[0])


# ---------------------------------------------------------------- LDL (test_linalg.cpp:144-274)
def test_ldl_identity(oracle):
    perm, D, L, _ = oracle.ldl(np.eye(4))
    assert np.all(L == np.eye(4)) and np.all(D == 1)


def test_ldl_hand_checked_2x2(oracle):
    A = np.array([[2.0, 1.0], [1.0, -1.0]])
    perm, D, L, _ = oracle.ldl(A, use_ordering=False)
    assert L[1, 0] == pytest.approx(0.5, rel=1e-15)
    assert D[0] == pytest.approx(2.0) and D[1] == pytest.approx(-1.5)
    x = oracle.ldl_solve(A, [1.0, 0.0], use_ordering=False)
    np.testing.assert_allclose(x, np.linalg.solve(A, [1.0, 0.0]), atol=1e-14)


def test_ldl_quasi_definite_inertia(oracle):
    r = np.random.default_rng(23)
    for _ in range(20):
        n, m = 2 + r.integers(10), 1 + r.integers(8)
        _, D, _, _ = oracle.ldl(random_quasi_definite(r, n, m))
        assert (D > 0).sum() == n and (D < 0).sum() == m


def test_ldl_reconstruction(oracle):
    r = np.random.default_rng(29)
    for _ in range(100):
        n, m = 2 + r.integers(20), 1 + r.integers(20)
        K = random_quasi_definite(r, n, m)
        perm, D, L, _ = oracle.ldl(K)
        Kp = K[np.ix_(perm, perm)]
        assert np.max(np.abs(Kp - L @ np.diag(D) @ L.T)) <= 1e-10 * np.max(np.abs(K).sum(1))


def test_ldl_solve_residual(oracle):
    r = np.random.default_rng(31)
    for _ in range(20):
        K = random_quasi_definite(r, 30, 20)
        b = r.normal(size=50)
        x = oracle.ldl_solve(K, b)
        bound = 1e-8 * (np.max(np.abs(K).sum(1)) * np.max(np.abs(x)) + np.max(np.abs(b)))
        assert np.max(np.abs(K @ x - b)) <= bound


def test_ldl_zero_pivot_names_column(oracle):
    A = np.array([[1.0, 1.0], [1.0, 1.0]])
    with pytest.raises(ArithmeticError, match="column 1"):
        oracle.ldl(A, use_ordering=False)


def test_ordering_reduces_arrow_fill(oracle):
    """test_linalg.cpp:262-274 (the AMD stand-in reduces fill on an arrow matrix)."""
    n = 40
    A = np.diag(np.full(n, 10.0))
    A[0, 1:] = 1.0
    A[1:, 0] = 1.0
    _, _, _, nat = oracle.ldl(A, use_ordering=False)
    _, _, _, amd = oracle.ldl(A, use_ordering=True)
    assert amd < nat
    x = oracle.ldl_solve(A, np.ones(n))
    assert np.max(np.abs(A @ x - 1)) < 1e-10


# ---------------------------------------------------------------- ADMM (test_qp.cpp)
def test_admm_one_sided_bound(oracle):
    """test_qp.cpp:114-127."""
    r = oracle.admm(np.eye(1), [0.0], np.eye(1), [1.0], [1e30], iters=200)
    assert abs(r["x"][0] - 1.0) < 1e-4 and r["z"][0] >= 1.0 - 1e-6


def test_admm_unconstrained(oracle):
    """test_qp.cpp:129-145."""
    q = np.random.default_rng(11).uniform(-1, 1, 6)
    r = oracle.admm(np.eye(6), q, np.zeros((0, 6)), np.zeros(0), np.zeros(0), iters=100)
    assert np.max(np.abs(r["x"] + q)) < 1e-6


def test_admm_matches_active_set_enumeration(oracle):
    """test_qp.cpp:147-163 / SPEC acceptance #1: 2000 iterations within 1e-4 of the global
    optimum (m <= 6 here to keep the 3^m enumeration fast)."""
    r = np.random.default_rng(2024)
    checked = 0
    for _ in range(40):
        n, m = 2 + r.integers(7), 1 + r.integers(6)
        P, q, A, lo, hi = random_strictly_convex_qp(r, n, m)
        xs = active_set_enumerate(P, q, A, lo, hi)
        if xs is None:
            continue
        checked += 1
        res = oracle.admm(P, q, A, lo, hi, iters=2000)
        assert np.max(np.abs(res["x"] - xs)) <= 1e-4
    assert checked >= 30


def test_admm_residual_shrinks(oracle):
    """test_qp.cpp:165-185 (residual at 2000 iterations <= at 10)."""
    r = np.random.default_rng(77)
    for _ in range(10):
        P, q, A, lo, hi = random_strictly_convex_qp(r, 5, 6)
        a = oracle.admm(P, q, A, lo, hi, iters=11)
        b = oracle.admm(P, q, A, lo, hi, iters=2000)
        assert b["prim"] <= a["prim"] + 1e-15


def test_admm_warm_start_barely_moves(oracle):
    """test_qp.cpp:187-206."""
    r = np.random.default_rng(99)
    P, q, A, lo, hi = random_strictly_convex_qp(r, 4, 4)
    conv = oracle.admm(P, q, A, lo, hi, iters=20000)
    again = oracle.admm(P, q, A, lo, hi, iters=10, x0=conv["x"], y0=conv["y"])
    assert np.max(np.abs(again["x"] - conv["x"])) <= 1e-9


def test_admm_projection_within_bounds(oracle):
    """test_qp.cpp:208-226 (final projected iterate)."""
    r = np.random.default_rng(123)
    P, q, A, lo, hi = random_strictly_convex_qp(r, 5, 5)
    res = oracle.admm(P, q, A, lo, hi, iters=300)
    assert np.all(res["z"] >= lo - 1e-6) and np.all(res["z"] <= hi + 1e-6)


def test_admm_ruiz_on_off_agree(oracle):
    """test_qp.cpp:228-241."""
    r = np.random.default_rng(321)
    for _ in range(10):
        P, q, A, lo, hi = random_strictly_convex_qp(r, 5, 5)
        a = oracle.admm(P, q, A, lo, hi, iters=3000)
        b = oracle.admm(P, q, A, lo, hi, iters=3000, ruiz_iters=0)
        assert np.max(np.abs(a["x"] - b["x"])) <= 1e-6


def test_admm_tolerance_exit(oracle):
    """test_qp.cpp:243-253."""
    r = np.random.default_rng(55)
    P, q, A, lo, hi = random_strictly_convex_qp(r, 4, 3)
    res = oracle.admm(P, q, A, lo, hi, iters=5000, eps_exit=1e-9)
    assert res["iters"] < 5000 and res["prim"] < 1e-8


def test_admm_nan_diverges_at_iteration_zero(oracle):
    """test_qp.cpp:255-270."""
    with pytest.raises(oracle.DivergenceError) as e:
        oracle.admm(np.eye(1), [np.nan], np.eye(1), [-1.0], [1.0], iters=10)
    assert e.value.iteration == 0
