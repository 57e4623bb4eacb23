"""CPU: pin the oracle (oracle/gls_ref.py) against the reference's own outputs (golden vectors made
by tests/golden/make_golden.py) and the reference's known-answer cases."""

import numpy as np
import pytest

from conftest import golden, make_spd, maxnorm
from oracle import gls_ref as O


def test_known_answers_cholesky_and_trsolve():
    # reference tests/test_kernel.py:21-26, 62-69
    assert np.allclose(O.cholesky_spd(np.array([[4.0, 2.0], [2.0, 5.0]])), [[2, 0], [1, 2]])
    assert np.array_equal(O.cholesky_spd(np.eye(3)), np.eye(3))
    L = np.array([[2.0, 0.0], [1.0, 2.0]])
    assert np.array_equal(O.trsolve_lower(L, np.array([2.0, 3.0])), np.array([1.0, 1.0]))
    B = np.arange(12.0).reshape(4, 3)
    assert np.array_equal(O.trsolve_lower(np.eye(4), B), B)
    assert np.array_equal(O.gram(np.ones((3, 1))), [[3.0]])


def test_not_pd_pivot_index():
    M = np.eye(4)
    M[2, 2] = -1.0
    with pytest.raises(O.OracleNotPD) as e:
        O.cholesky_spd(M)
    assert e.value.pivot_index == 2
    g = golden("dense_ops")
    Mb = np.eye(300)
    Mb[211, 211] = -1.0
    with pytest.raises(O.OracleNotPD) as e:
        O.cholesky_spd(Mb)
    assert e.value.pivot_index == int(g["notpd_pivot"])


def test_dense_ops_match_reference():
    # same LAPACK/BLAS calls as the reference; 1e-14 leaves room for another CPU's BLAS kernels
    g = golden("dense_ops")
    for n in (16, 96, 200, 300):
        L = O.cholesky_spd(g[f"M{n}"])
        assert maxnorm(L - g[f"L{n}"]) <= 1e-14 * maxnorm(g[f"L{n}"])
        assert np.all(np.triu(L, 1) == 0)
        X = O.trsolve_lower(g[f"L{n}"], g[f"B{n}"])
        assert maxnorm(X - g[f"X{n}"]) <= 1e-14 * maxnorm(g[f"X{n}"])
        C = O.gram(g[f"B{n}"])
        assert maxnorm(C - g[f"G{n}"]) <= 1e-14 * maxnorm(g[f"G{n}"])
        assert np.array_equal(C, C.T)


def test_small_batch_matches_reference_bitwise():
    g = golden("dense_ops")
    x, ok, bad, packed = O.cholesky_solve_batch(g["S"], g["rhs"], want_inverse=True)
    assert np.array_equal(ok, g["ok"])
    assert np.array_equal(x, g["x"], equal_nan=True)
    assert np.array_equal(packed, g["packed"], equal_nan=True)
    assert bad[5] >= 0 and np.all(bad[np.arange(64) != 5] == -1)


@pytest.mark.parametrize("case", ["seed42", "degenerate", "baseline_p4", "baseline_p8"])
def test_block_solve_matches_reference(case):
    g = golden(case)
    ctx = O.gls_prepare(g["M"], g["XL"], g["y"])
    beta, ok, packed = O.gls_solve_block(ctx, g["G"].astype(float), emit_s_inv=True)
    assert np.array_equal(~ok, g["status"].astype(bool))
    rel, mism = O.compare(beta, g["beta"])
    assert mism == 0 and rel <= 1e-13, rel
    assert maxnorm(np.nan_to_num(packed - g["sinv"])) <= 1e-12 * maxnorm(np.nan_to_num(g["sinv"]))


def test_p_extremes_match_reference():
    g = golden("p_extremes")
    for p in (2, 4, 20):
        ctx = O.gls_prepare(g[f"M{p}"], g[f"XL{p}"], g[f"y{p}"])
        beta, ok = O.gls_solve_block(ctx, g[f"X{p}"])
        rel, mism = O.compare(beta, g[f"beta{p}"])
        assert mism == 0 and rel <= 1e-12


def test_oracle_vs_literal_eq1_seed42():
    # reference tests/test_kernel.py:195-207 and the per-SNP oracle of datagen.py:185-211
    g = golden("seed42")
    ctx = O.gls_prepare(g["M"], g["XL"], g["y"])
    beta, ok = O.gls_solve_block(ctx, g["G"].astype(float))
    rel, mism = O.compare(beta, g["beta_eq1"])
    assert mism == 0 and rel <= 1e-8
    X = g["G"].astype(float)
    for i in range(0, 500, 97):
        e = O.gls_eq1(g["M"], np.hstack([g["XL"], X[:, i:i + 1]]), g["y"])
        assert maxnorm(beta[i] - e) <= 1e-8 * max(maxnorm(e), 1.0)


def test_identity_covariance_is_ols():
    rng = np.random.default_rng(3)
    n = 30
    XL = np.hstack([np.ones((n, 1)), rng.standard_normal((n, 1))])
    y = rng.standard_normal(n)
    X = rng.standard_normal((n, 4))
    ctx = O.gls_prepare(np.eye(n), XL, y)
    beta, ok = O.gls_solve_block(ctx, X)
    for i in range(4):
        Xi = np.hstack([XL, X[:, i:i + 1]])
        e = np.linalg.solve(Xi.T @ Xi, Xi.T @ y)
        assert maxnorm(beta[i] - e) <= 1e-10 * max(maxnorm(e), 1.0)


def test_make_spd_symmetric():
    M = make_spd(20, 1)
    assert np.array_equal(M, M.T)
