"""CPU oracle for the GLS hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / reference arm may
import this module, and only as the checker or the timed CPU baseline — never as part of the
product path (paper_1304_2272_b200 has no CPU fallback).

A numpy/scipy restatement of the reference's numerical core (pkg/src/gwasgls/kernel.py), which
itself runs on LAPACK/BLAS (scipy dpotrf / dtrtrs->dtrsm, numpy sums; OpenBLAS, third-party,
not under /root/reference; versions in DESIGN.md).  Each function cites the reference lines it
follows.  Results are returned as arrays (beta, ok, packed S^-1) rather than per-SNP objects.

Pinned: tests/test_oracle_golden.py checks every function against golden vectors produced by
the reference itself (tests/golden/make_golden.py imports /root/reference/pkg/src) and against
the reference's own known-answer cases (tests/test_kernel.py:21-179 in the reference).
"""

from __future__ import annotations

import numpy as np
from scipy.linalg import solve_triangular
from scipy.linalg.lapack import dpotrf

EPS = 2.0 ** -52                                   # kernel.py:28


class OracleNotPD(Exception):
    def __init__(self, pivot_index):
        self.pivot_index = pivot_index
        super().__init__(f"not positive definite (pivot {pivot_index})")


def cholesky_spd(M):
    """kernel.py:92-109 — LAPACK dpotrf(lower=1, clean=1); non-finite -> row of first bad entry."""
    M = np.ascontiguousarray(M, dtype=np.float64)
    bad = np.argwhere(~np.isfinite(M))
    if bad.size:
        raise OracleNotPD(int(bad[0][0]))
    c, info = dpotrf(M, lower=1, clean=1, overwrite_a=0)
    if info > 0:
        raise OracleNotPD(info - 1)
    return c


def trsolve_lower(L, B):
    """kernel.py:112-121 — scipy solve_triangular (dtrtrs -> dtrsm), B copied."""
    B = np.asarray(B, dtype=np.float64)
    one = B.ndim == 1
    X = solve_triangular(L, B[:, None] if one else B, lower=True, check_finite=False)
    return X[:, 0] if one else X


def gram(A):
    """kernel.py:124-131 — A^T A, lower triangle mirrored."""
    C = np.asarray(A, dtype=np.float64).T @ np.asarray(A, dtype=np.float64)
    return np.tril(C) + np.tril(C, -1).T


def cholesky_solve_batch(S, rhs, want_inverse=False):
    """kernel.py:134-208 — batched p x p Cholesky with pivot rule d > p*eps*max|S| and finite,
    placeholder pivot 1.0, NaN solutions for failed systems, optional packed S^-1.

    Returns (x, ok, first_bad[, packed]); first_bad is the first failing pivot or -1."""
    S = np.asarray(S, dtype=np.float64)
    rhs = np.asarray(rhs, dtype=np.float64)
    B, p, _ = S.shape
    thresh = p * EPS * np.max(np.abs(S), axis=(-2, -1))
    ok = np.ones(B, dtype=bool)
    first_bad = np.full(B, -1)
    L = np.zeros_like(S)
    for j in range(p):
        d = S[:, j, j] - np.einsum("bk,bk->b", L[:, j, :j], L[:, j, :j]) if j else S[:, j, j].copy()
        good = np.isfinite(d) & (d > thresh)
        first_bad[(~good) & ok] = j
        ok &= good
        L[:, j, j] = np.sqrt(np.where(good, d, 1.0))
        for i in range(j + 1, p):
            s = S[:, i, j] - np.einsum("bk,bk->b", L[:, i, :j], L[:, j, :j]) if j else S[:, i, j]
            L[:, i, j] = s / L[:, j, j]

    def substitute(b):                  # b: (B, p, r); forward then back substitution
        z = np.empty_like(b)
        for i in range(p):
            acc = b[:, i, :].copy()
            for k in range(i):
                acc -= L[:, i, k][:, None] * z[:, k, :]
            z[:, i, :] = acc / L[:, i, i][:, None]
        x = np.empty_like(b)
        for i in range(p - 1, -1, -1):
            acc = z[:, i, :].copy()
            for k in range(i + 1, p):
                acc -= L[:, k, i][:, None] * x[:, k, :]
            x[:, i, :] = acc / L[:, i, i][:, None]
        return x

    x = substitute(rhs[:, :, None])[:, :, 0]
    x[~ok] = np.nan
    if not want_inverse:
        return x, ok, first_bad
    inv = substitute(np.broadcast_to(np.eye(p), (B, p, p)).copy())
    il, jl = np.tril_indices(p)
    packed = inv[:, il, jl]
    packed[~ok] = np.nan
    return x, ok, first_bad, packed


class Prepared:
    """kernel.py:68-89 (PreparedContext) as plain arrays."""

    def __init__(self, L, XLbar, ybar, S_TL, b_T):
        self.L, self.XLbar, self.ybar, self.S_TL, self.b_T = L, XLbar, ybar, S_TL, b_T

    @property
    def p(self):
        return self.XLbar.shape[1] + 1


def gls_prepare(M, XL, y):
    """kernel.py:233-257 — factor, whiten X_L and y, S_TL = gram, SPD check, b_T."""
    M = np.asarray(M, dtype=np.float64)
    XL = np.asarray(XL, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64).ravel()
    L = cholesky_spd(M)
    XLbar = trsolve_lower(L, XL)
    ybar = trsolve_lower(L, y)
    S_TL = gram(XLbar)
    _, ok, bad = cholesky_solve_batch(S_TL[None], np.zeros((1, S_TL.shape[0])))
    if not ok[0]:
        raise ValueError(f"rank deficient covariates (pivot {int(bad[0])})")
    return Prepared(L, XLbar, ybar, S_TL, XLbar.T @ ybar)


def column_sums(Xbar, XLbar, ybar):
    """kernel.py:260-270 — per-column reductions with np.sum."""
    S_BL = np.stack([np.sum(Xbar * XLbar[:, k][:, None], axis=0)
                     for k in range(XLbar.shape[1])], axis=1)
    return S_BL, np.sum(Xbar * Xbar, axis=0), np.sum(Xbar * ybar[:, None], axis=0)


def solve_whitened(ctx, Xbar, emit_s_inv=False):
    """kernel.py:273-312 — assemble S, rhs per SNP and solve; returns (beta, ok[, packed]).
    Degenerate SNPs get all-NaN beta (kernel.py:305-311)."""
    q = ctx.XLbar.shape[1]
    p = q + 1
    cnt = Xbar.shape[1]
    S_BL, S_BR, b_B = column_sums(Xbar, ctx.XLbar, ctx.ybar)
    S = np.empty((cnt, p, p))
    S[:, :q, :q] = ctx.S_TL
    S[:, q, :q] = S_BL
    S[:, :q, q] = S_BL
    S[:, q, q] = S_BR
    rhs = np.empty((cnt, p))
    rhs[:, :q] = ctx.b_T
    rhs[:, q] = b_B
    out = cholesky_solve_batch(S, rhs, want_inverse=emit_s_inv)
    beta, ok = out[0], out[1]
    beta[~ok] = np.nan
    return (beta, ok, out[3]) if emit_s_inv else (beta, ok)


def gls_solve_block(ctx, X, emit_s_inv=False, threads=1):
    """kernel.py:315-342 — whiten the block (dtrsm, BLAS-threaded) then solve_whitened; with
    threads > 1 and at least 2*threads columns the per-SNP epilogue runs data-parallel over the
    same disjoint column ranges as the reference (np.linspace bounds, a ThreadPoolExecutor,
    kernel.py:326-341; numpy releases the GIL inside its reductions).  Results do not depend on
    the split (per-column arithmetic)."""
    Xbar = trsolve_lower(ctx.L, np.asarray(X, dtype=np.float64))
    cnt = Xbar.shape[1]
    if threads <= 1 or cnt < 2 * threads:
        return solve_whitened(ctx, Xbar, emit_s_inv)
    from concurrent.futures import ThreadPoolExecutor

    bounds = np.linspace(0, cnt, threads + 1, dtype=int)
    ranges = [(bounds[i], bounds[i + 1]) for i in range(threads) if bounds[i] < bounds[i + 1]]
    with ThreadPoolExecutor(max_workers=threads) as pool:
        parts = list(pool.map(lambda se: solve_whitened(ctx, Xbar[:, se[0]:se[1]], emit_s_inv),
                              ranges))
    return tuple(np.concatenate([p[k] for p in parts]) for k in range(len(parts[0])))


def gls_eq1(M, Xi, y):
    """kernel.py:345-355 — literal Eq. 1 through general solves (no structure)."""
    MinvX = np.linalg.solve(M, Xi)
    Minvy = np.linalg.solve(M, np.asarray(y, dtype=np.float64).ravel())
    return np.linalg.solve(Xi.T @ MinvX, Xi.T @ Minvy)


def compare(beta_a, beta_b):
    """datagen.py:230-247 — max relative inf-norm discrepancy over SNPs ok in both, plus the
    number of status disagreements (a SNP is degenerate iff its beta row is all-NaN)."""
    da = np.all(np.isnan(beta_a), axis=1)
    db = np.all(np.isnan(beta_b), axis=1)
    mism = int(np.sum(da != db))
    both = ~da & ~db
    if not np.any(both):
        return 0.0, mism
    diff = np.max(np.abs(beta_a[both] - beta_b[both]), axis=1)
    scale = np.maximum(np.max(np.abs(beta_a[both]), axis=1), 1e-300)
    return float(np.max(diff / scale)), mism
