"""GPU parity of the drop-in kernel module against the oracle, the reference's golden outputs and
the reference's own test cases (pkg/tests/test_kernel.py).  Tolerances are the reference's;
the north-star bar is <= 1e-9 relative per SNP with zero status mismatches."""

import numpy as np
import pytest

from conftest import golden, make_spd, maxnorm

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K(gpu):
    from paper_1304_2272_b200 import kernel

    return kernel


def betas(rb):
    return np.array([r.beta for r in rb.results])


# ---- Cholesky (reference tests/test_kernel.py:20-58) -----------------------------------------

def test_cholesky_known_answers(K):
    L = K.cholesky_spd(np.array([[4.0, 2.0], [2.0, 5.0]]))
    assert np.allclose(L, [[2.0, 0.0], [1.0, 2.0]])
    assert np.array_equal(K.cholesky_spd(np.eye(3)), np.eye(3))


@pytest.mark.parametrize("n", [16, 96, 200, 300])
def test_cholesky_vs_reference_factor(K, n):
    g = golden("dense_ops")
    L = K.cholesky_spd(g[f"M{n}"])
    assert L.flags.f_contiguous
    assert np.all(np.triu(L, 1) == 0) and np.all(np.diag(L) > 0)
    assert maxnorm(L - g[f"L{n}"]) <= 1e-13 * maxnorm(g[f"L{n}"])
    assert maxnorm(L @ L.T - g[f"M{n}"]) <= 1e-13 * maxnorm(g[f"M{n}"])


def test_cholesky_genotype_style_residual(K):
    rng = np.random.default_rng(42)
    G = rng.integers(0, 3, size=(50, 200)).astype(float)
    M = G @ G.T / 200 + np.eye(50)
    L = K.cholesky_spd(M)
    assert maxnorm(L @ L.T - M) <= 1e-10 * maxnorm(M)


def test_cholesky_input_unmodified_and_errors(K):
    from paper_1304_2272_b200.errors import DimensionMismatch, NotPositiveDefinite

    M = make_spd(10, 0)
    M0 = M.copy()
    K.cholesky_spd(M)
    assert np.array_equal(M, M0)
    bad = np.eye(4)
    bad[2, 2] = -1.0
    with pytest.raises(NotPositiveDefinite) as e:
        K.cholesky_spd(bad)
    assert e.value.pivot_index == 2
    big = np.eye(300)
    big[211, 211] = -1.0          # pivot in the second 128-block: global index reported
    with pytest.raises(NotPositiveDefinite) as e:
        K.cholesky_spd(big)
    assert e.value.pivot_index == int(golden("dense_ops")["notpd_pivot"])
    nanm = np.eye(3)
    nanm[1, 1] = np.nan
    with pytest.raises(NotPositiveDefinite) as e:
        K.cholesky_spd(nanm)
    assert e.value.pivot_index == 1
    with pytest.raises(DimensionMismatch):
        K.cholesky_spd(np.ones((2, 3)))


# ---- triangular solve (reference tests/test_kernel.py:61-88) ---------------------------------

def test_trsolve_known_answers(K):
    L = np.array([[2.0, 0.0], [1.0, 2.0]])
    assert np.array_equal(K.trsolve_lower(L, np.array([2.0, 3.0])), np.array([1.0, 1.0]))
    B = np.arange(12.0).reshape(4, 3)
    assert np.array_equal(K.trsolve_lower(np.eye(4), B), B)


def test_trsolve_residual_random(K):
    rng = np.random.default_rng(1)
    L = np.tril(rng.standard_normal((64, 64))) + 8 * np.eye(64)
    B = rng.standard_normal((64, 8))
    X = K.trsolve_lower(L, B)
    assert maxnorm(L @ X - B) / maxnorm(B) <= 1e-12


def test_trsolve_column_independence(K):
    rng = np.random.default_rng(2)
    L = np.tril(rng.standard_normal((32, 32))) + 6 * np.eye(32)
    B = rng.standard_normal((32, 5))
    full = K.trsolve_lower(L, B)
    one = K.trsolve_lower(L, B[:, 2])
    assert np.array_equal(full[:, 2], one)          # identical per-column arithmetic


@pytest.mark.parametrize("n", [16, 96, 200, 300])
def test_trsolve_vs_reference(K, n):
    g = golden("dense_ops")
    X = K.trsolve_lower(g[f"L{n}"], g[f"B{n}"])
    assert maxnorm(X - g[f"X{n}"]) <= 1e-13 * maxnorm(g[f"X{n}"])


def test_trsolve_dimension_mismatch(K):
    from paper_1304_2272_b200.errors import DimensionMismatch

    with pytest.raises(DimensionMismatch):
        K.trsolve_lower(np.eye(3), np.ones((4, 2)))


# ---- gram and small systems (reference tests/test_kernel.py:91-166) --------------------------

def test_gram(K):
    assert np.array_equal(K.gram(np.ones((3, 1))), np.array([[3.0]]))
    assert np.array_equal(K.gram(np.eye(2)), np.eye(2))
    rng = np.random.default_rng(3)
    A = rng.standard_normal((10, 3))
    assert maxnorm(K.gram(A) - A.T @ A) <= 1e-13
    C = K.gram(rng.standard_normal((50, 7)))
    assert np.array_equal(C, C.T)


def test_small_batch_vs_reference(K):
    g = golden("dense_ops")
    x, ok, packed = K.cholesky_solve_batch(g["S"], g["rhs"], want_inverse=True)
    assert np.array_equal(ok, g["ok"])
    assert np.all(np.isnan(x[~ok])) and np.all(np.isnan(packed[~ok]))
    assert maxnorm(x[ok] - g["x"][ok]) <= 1e-12 * maxnorm(g["x"][ok])
    assert maxnorm(packed[ok] - g["packed"][ok]) <= 1e-12 * maxnorm(g["packed"][ok])


def test_solve_small_spd(K):
    from paper_1304_2272_b200.errors import NotPositiveDefinite

    assert np.array_equal(K.solve_small_spd(np.eye(4), np.array([1.0, 2.0, 3.0, 4.0])),
                          np.array([1.0, 2.0, 3.0, 4.0]))
    S = np.array([[4.0, 2.0], [2.0, 5.0]])
    got = K.solve_small_spd(S, np.array([8.0, 9.0]))
    assert np.allclose(got, [(5 * 8 - 2 * 9) / 16, (4 * 9 - 2 * 8) / 16], rtol=1e-12)
    with pytest.raises(NotPositiveDefinite) as e:
        K.solve_small_spd(np.ones((2, 2)), np.ones(2))
    assert e.value.pivot_index == 1


# ---- prepare (reference tests/test_kernel.py:115-146) ----------------------------------------

def test_prepare_identity_and_scalar(K):
    ctx = K.gls_prepare(np.eye(3), np.ones((3, 1)), np.array([1.0, 2.0, 3.0]))
    assert np.array_equal(ctx.XLbar, np.ones((3, 1)))
    assert np.array_equal(ctx.ybar, np.array([1.0, 2.0, 3.0]))
    assert np.allclose(ctx.S_TL, [[3.0]]) and np.allclose(ctx.b_T, [6.0])
    ctx = K.gls_prepare(2.0 * np.eye(3), np.ones((3, 1)), np.array([1.0, 2.0, 3.0]))
    assert np.allclose(ctx.XLbar, np.ones((3, 1)) / np.sqrt(2))
    assert np.allclose(ctx.S_TL, [[1.5]]) and np.allclose(ctx.b_T, [3.0])


def test_prepare_residuals_and_reference(K):
    g = golden("seed42")
    ctx = K.gls_prepare(g["M"], g["XL"], g["y"])
    assert maxnorm(ctx.L @ ctx.XLbar - g["XL"]) <= 1e-10 * maxnorm(g["XL"])
    assert maxnorm(ctx.L @ ctx.ybar - g["y"]) <= 1e-10 * maxnorm(g["y"])
    assert np.array_equal(ctx.S_TL, ctx.S_TL.T)
    assert np.allclose(ctx.b_T, ctx.XLbar.T @ ctx.ybar)
    assert maxnorm(ctx.L - g["L"]) <= 1e-13 * maxnorm(g["L"])
    assert maxnorm(ctx.S_TL - g["S_TL"]) <= 1e-12 * maxnorm(g["S_TL"])
    assert maxnorm(ctx.b_T - g["b_T"]) <= 1e-12 * maxnorm(g["b_T"])


def test_prepare_rank_deficient(K):
    from paper_1304_2272_b200.errors import RankDeficientCovariates

    with pytest.raises(RankDeficientCovariates):
        K.gls_prepare(np.eye(10), np.ones((10, 2)), np.zeros(10))


# ---- block solve (reference tests/test_kernel.py:169-276) ------------------------------------

def test_block_hand_checkable_and_degenerate(K):
    ctx = K.gls_prepare(np.eye(3), np.ones((3, 1)), np.array([1.0, 2.0, 3.0]))
    res = K.gls_solve_block(ctx, K.SnpBlock(0, np.array([[0.0], [1.0], [2.0]]))).results[0]
    assert res.status == "ok" and np.allclose(res.beta, [1.0, 1.0])
    res = K.gls_solve_block(ctx, K.SnpBlock(0, np.ones((3, 1)))).results[0]
    assert res.status == "degenerate" and np.all(np.isnan(res.beta)) and res.s_inv is None
    data = np.column_stack([np.ones(3), [0.0, 1.0, 2.0]])
    rb = K.gls_solve_block(ctx, K.SnpBlock(0, data))
    assert rb.results[0].status == "degenerate" and rb.results[1].status == "ok"
    assert np.allclose(rb.results[1].beta, [1.0, 1.0])


@pytest.mark.parametrize("case", ["seed42", "degenerate", "baseline_p4", "baseline_p8"])
def test_block_parity_with_reference(K, case):
    from oracle import gls_ref as O

    g = golden(case)
    ctx = K.gls_prepare(g["M"], g["XL"], g["y"])
    rb = K.gls_solve_block(ctx, K.SnpBlock(0, g["G"].astype(float)), emit_s_inv=True)
    beta = betas(rb)
    rel, mism = O.compare(beta, g["beta"])
    assert mism == 0, "status mismatch vs reference"
    assert rel <= 1e-9, rel
    st = np.array([r.status != "ok" for r in rb.results])
    assert np.array_equal(st, g["status"].astype(bool))
    sinv = np.array([r.s_inv for r in rb.results if r.status == "ok"])
    ref = g["sinv"][~g["status"].astype(bool)]
    assert maxnorm(sinv - ref) <= 1e-9 * maxnorm(ref)


def test_seed42_vs_literal_eq1(K):
    from oracle import gls_ref as O

    g = golden("seed42")
    ctx = K.gls_prepare(g["M"], g["XL"], g["y"])
    rb = K.gls_solve_block(ctx, K.SnpBlock(0, g["G"].astype(float)))
    rel, mism = O.compare(betas(rb), g["beta_eq1"])
    assert mism == 0 and rel <= 1e-8


def test_p_extremes(K):
    from oracle import gls_ref as O

    g = golden("p_extremes")
    for p in (2, 4, 20):
        ctx = K.gls_prepare(g[f"M{p}"], g[f"XL{p}"], g[f"y{p}"])
        rb = K.gls_solve_block(ctx, K.SnpBlock(0, g[f"X{p}"]), emit_s_inv=True)
        rel, mism = O.compare(betas(rb), g[f"beta{p}"])
        assert mism == 0 and rel <= 1e-9, (p, rel)


def test_block_size_independence_and_permutation_bitwise(K):
    rng = np.random.default_rng(5)
    n, m = 60, 40
    ctx = K.gls_prepare(make_spd(n, 6), np.hstack([np.ones((n, 1)), rng.standard_normal((n, 2))]),
                        rng.standard_normal(n))
    X = rng.standard_normal((n, m))
    ref = betas(K.gls_solve_block(ctx, K.SnpBlock(0, X)))
    for m_blk in (1, 7, 64):
        parts = []
        for first in range(0, m, m_blk):
            parts.append(betas(K.gls_solve_block(ctx, K.SnpBlock(first, X[:, first:first + m_blk]))))
        assert np.array_equal(np.vstack(parts), ref)          # bitwise, stronger than 1e-12
    perm = rng.permutation(m)
    got = betas(K.gls_solve_block(ctx, K.SnpBlock(0, np.asfortranarray(X[:, perm]))))
    assert np.array_equal(ref[perm], got)
    got4 = betas(K.gls_solve_block(ctx, K.SnpBlock(0, X), threads=4))
    assert np.array_equal(got4, ref)


def test_emit_s_inv_inverse(K):
    rng = np.random.default_rng(11)
    n = 30
    ctx = K.gls_prepare(make_spd(n, 12), np.hstack([np.ones((n, 1)), rng.standard_normal((n, 2))]),
                        rng.standard_normal(n))
    X = rng.standard_normal((n, 4))
    rb = K.gls_solve_block(ctx, K.SnpBlock(0, X), emit_s_inv=True)
    p = ctx.p
    il, jl = np.tril_indices(p)
    for i, r in enumerate(rb.results):
        xb = K.trsolve_lower(ctx.L, X[:, i])
        S = np.empty((p, p))
        S[:p - 1, :p - 1] = ctx.S_TL
        S[p - 1, :p - 1] = S[:p - 1, p - 1] = ctx.XLbar.T @ xb
        S[p - 1, p - 1] = xb @ xb
        Sinv = np.linalg.inv(S)
        assert maxnorm(r.s_inv - Sinv[il, jl]) <= 1e-8 * maxnorm(Sinv)


def test_int8_block_equals_fp64_block_bitwise(K):
    g = golden("baseline_p4")
    ctx = K.gls_prepare(g["M"], g["XL"], g["y"])
    b64 = betas(K.gls_solve_block(ctx, K.SnpBlock(0, g["G"].astype(float))))
    b8 = betas(K.gls_solve_block(ctx, K.SnpBlock(0, np.asfortranarray(g["G"]))))
    assert np.array_equal(b64, b8, equal_nan=True)


def test_solve_whitened_block_matches_fused(K):
    g = golden("seed42")
    ctx = K.gls_prepare(g["M"], g["XL"], g["y"])
    X = g["G"][:, :50].astype(float)
    fused = betas(K.gls_solve_block(ctx, K.SnpBlock(7, X)))
    Xbar = K.trsolve_lower(ctx.L, X)
    res = K.solve_whitened_block(ctx, Xbar, 7, global_indices=np.arange(100, 150))
    assert [r.snp_index for r in res[:2]] == [100, 101]
    assert maxnorm(np.array([r.beta for r in res]) - fused) <= 1e-12 * maxnorm(fused)
    # a context built from host fields only (as the reference's run_dist does)
    host_ctx = K.PreparedContext(L=np.empty((ctx.n, 0)), XLbar=ctx.XLbar, ybar=ctx.ybar,
                                 S_TL=ctx.S_TL, b_T=ctx.b_T)
    res2 = K.solve_whitened_block(host_ctx, Xbar, 7)
    assert np.array_equal(np.array([r.beta for r in res2]), np.array([r.beta for r in res]))


def test_gls_oracle_route(K):
    Xi = np.column_stack([np.ones(3), [0.0, 1.0, 2.0]])
    assert np.allclose(K.gls_oracle(np.eye(3), Xi, np.array([1.0, 2.0, 3.0])), [1.0, 1.0])
    rng = np.random.default_rng(13)
    n = 40
    M = make_spd(n, 14)
    Xi = np.column_stack([np.ones(n), rng.standard_normal((n, 3))])
    y = rng.standard_normal(n)
    b1 = K.gls_oracle(M, Xi, y)
    for c in (0.5, 3.0, 1000.0):
        assert maxnorm(b1 - K.gls_oracle(c * M, Xi, y)) <= 1e-9 * maxnorm(b1)


def test_structured_vs_naive_random(K):
    # reference hypothesis property (tests/test_kernel.py:309-322), fixed seeds
    from oracle import gls_ref as O

    for seed in range(12):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(8, 41))
        q = int(rng.integers(1, 5))
        M = make_spd(n, seed)
        XL = np.hstack([np.ones((n, 1)), rng.standard_normal((n, q - 1))]) if q > 1 else np.ones((n, 1))
        y = rng.standard_normal(n)
        X = rng.standard_normal((n, 5))
        rb = K.gls_solve_block(K.gls_prepare(M, XL, y), K.SnpBlock(0, X))
        for i in range(5):
            e = O.gls_eq1(M, np.hstack([XL, X[:, i:i + 1]]), y)
            assert maxnorm(rb.results[i].beta - e) <= 1e-8 * max(maxnorm(e), 1.0)


def test_tma_trsm_bitwise_equals_cpasync_trsm(K):
    """The persistent TMA/DMMA TRSM (production) and the cp.async DMMA GEMM give identical bits."""
    import torch

    from paper_1304_2272_b200 import _capi
    from paper_1304_2272_b200._capi import ptr, stream_handle
    from paper_1304_2272_b200._device import alloc_cols, transpose_square, upload_cols

    for n, nrhs in ((300, 257), (1000, 1), (129, 700)):
        M = make_spd(n, n)
        _, L, LinvP, Linv = K._potrf_device(M, keep_square_inverse=True)
        np_ = _capi.pad(n)
        LinvT = transpose_square(Linv)
        B = upload_cols(np.random.default_rng(n).standard_normal((n, nrhs)), ld=np_)
        X1 = alloc_cols(nrhs, np_)
        X2 = alloc_cols(nrhs, np_)
        assert _capi.lib().gg_trsm_lower_f64(n, nrhs, ptr(Linv), np_, ptr(B), np_, ptr(X1), np_,
                                             stream_handle()) == 0
        assert _capi.lib().gg_trsm_lower_rm_f64(n, nrhs, ptr(LinvT), np_, ptr(B), np_, ptr(X2),
                                                np_, stream_handle()) == 0
        X3 = alloc_cols(nrhs, np_)
        assert _capi.lib().gg_trsm_lower_packed_f64(n, nrhs, ptr(LinvP), ptr(B), np_, ptr(X3),
                                                    np_, stream_handle()) == 0
        torch.cuda.synchronize()
        assert torch.equal(X1, X2)
        assert torch.equal(X1, X3)
        assert LinvP.numel() * 8 == _capi.lib().gg_packed_lower_bytes(n)


@pytest.mark.parametrize("n", [300, 4100])
def test_skinny_trsm_bitwise_equal_to_tiled(K, n):
    """gg_trsm_lower_packed_f64 with <= 16 right-hand sides (the prepare's [X_L | y]) runs the
    skinny kernel; every column equals, bitwise, the same column whitened by the tiled TMA/DMMA
    kernel inside a wider call (so a SNP equal to a covariate still gives an exactly singular S)."""
    import torch

    from paper_1304_2272_b200 import _capi
    from paper_1304_2272_b200._capi import ptr, stream_handle
    from paper_1304_2272_b200._device import alloc_cols, upload_cols

    M = make_spd(n, n + 1)
    _, L, LinvP, Linv = K._potrf_device(M, keep_square_inverse=True)
    np_ = _capi.pad(n)
    B = upload_cols(np.random.default_rng(n).standard_normal((n, 40)), ld=np_)
    wide = alloc_cols(40, np_)
    assert _capi.lib().gg_trsm_lower_packed_f64(n, 40, ptr(LinvP), ptr(B), np_, ptr(wide), np_,
                                                stream_handle()) == 0
    for c0, cnt in ((0, 1), (3, 9), (24, 16)):
        X = alloc_cols(cnt, np_)
        assert _capi.lib().gg_trsm_lower_packed_f64(n, cnt, ptr(LinvP), ptr(B[c0:]), np_, ptr(X),
                                                    np_, stream_handle()) == 0
        torch.cuda.synchronize()
        assert torch.equal(X[:, :n], wide[c0:c0 + cnt, :n])


def test_cholesky_reads_lower_triangle_and_checks_all_entries(K):
    from paper_1304_2272_b200.errors import NotPositiveDefinite

    M = make_spd(40, 3)
    A = M.copy()
    A[np.triu_indices(40, 1)] = 7.0          # garbage above the diagonal: dpotrf(lower) ignores it
    assert np.array_equal(K.cholesky_spd(A), K.cholesky_spd(M))
    A[3, 30] = np.inf                        # but a non-finite entry anywhere is refused
    with pytest.raises(NotPositiveDefinite) as e:
        K.cholesky_spd(A)
    assert e.value.pivot_index == 3


def test_concurrent_calls_from_threads(K):
    """Threading contract (run_spmd(transport="inproc") calls the kernel module from
    several threads of one process): concurrent gls_solve_block calls on two contexts, from
    threads on the default stream and on their own streams, give the sequential results bitwise
    (per-call workspaces; the int8 kernel's tile counters are per launch)."""
    import threading

    import torch

    rng = np.random.default_rng(21)
    n1, n2, m = 300, 170, 600
    ctx1 = K.gls_prepare(make_spd(n1, 3), np.hstack([np.ones((n1, 1)),
                                                     rng.standard_normal((n1, 2))]),
                         rng.standard_normal(n1))
    ctx2 = K.gls_prepare(make_spd(n2, 4), np.hstack([np.ones((n2, 1)),
                                                     rng.standard_normal((n2, 3))]),
                         rng.standard_normal(n2))
    X1 = np.asfortranarray(rng.integers(0, 3, (n1, m)).astype(np.int8))
    X2 = rng.standard_normal((n2, m))                 # FP64 path
    ref1 = betas(K.gls_solve_block(ctx1, K.SnpBlock(0, X1)))
    ref2 = betas(K.gls_solve_block(ctx2, K.SnpBlock(0, X2)))
    errors = []

    def work(ctx, X, ref, own_stream):
        try:
            s = torch.cuda.Stream() if own_stream else None
            for _ in range(6):
                if s is not None:
                    with torch.cuda.stream(s):
                        got = betas(K.gls_solve_block(ctx, K.SnpBlock(0, X)))
                else:
                    got = betas(K.gls_solve_block(ctx, K.SnpBlock(0, X)))
                if not np.array_equal(got, ref):
                    errors.append("mismatch")
        except Exception as e:        # noqa: BLE001 -- reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=work, args=a) for a in
               [(ctx1, X1, ref1, False), (ctx1, X1, ref1, True), (ctx2, X2, ref2, False),
                (ctx2, X2, ref2, True)]]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
