"""GPU: the FP64 GEMM on the int8 tensor cores (Ozaki scheme, csrc/ozaki_i8.cu) against an
extended-precision product, and the factorisation that uses it (gg_potrf_f64 with
GG_FACTOR_OZAKI=1) against the DMMA factorisation and the CPU oracle."""

import numpy as np
import pytest

from conftest import make_spd

pytestmark = pytest.mark.gpu


def _ozaki(A, B, C0, alpha, beta, flags, a_rowmajor=False, b_rowmajor=False, same=False):
    """C = beta C0 + alpha A B^T through gg_gemm_ozaki_f64; A (m x k), B (ncols x k) host arrays
    uploaded column-major (or row-major when asked)."""
    import torch

    from paper_1304_2272_b200 import _capi
    from paper_1304_2272_b200._capi import check, ptr, stream_handle

    dev = _capi.device()
    m, k = A.shape
    nc = B.shape[0]

    def up(X, rowmajor):
        if rowmajor:   # X[i, k] at i * k_dim + k
            return torch.from_numpy(np.ascontiguousarray(X)).to(dev), X.shape[1], 1
        return torch.from_numpy(np.ascontiguousarray(X.T)).to(dev), 1, X.shape[0]

    Ad, a_rs, a_cs = up(A, a_rowmajor)
    if same:
        Bd, b_rs, b_cs = None, 0, 0
    else:
        Bd, b_rs, b_cs = up(B, b_rowmajor)
    Cd = torch.from_numpy(np.ascontiguousarray(C0.T)).to(dev)          # column-major m x nc
    lib = _capi.lib()
    wsb = int(lib.gg_gemm_ozaki_workspace_bytes(m, nc, k, int(same)))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    rc = lib.gg_gemm_ozaki_f64(m, nc, k, ptr(Ad), a_rs, a_cs, None if same else ptr(Bd), b_rs,
                               b_cs, ptr(Cd), m, alpha, beta, flags, ptr(ws), wsb,
                               stream_handle())
    check(rc, "gg_gemm_ozaki_f64")
    return Cd.cpu().numpy().T


def _scale(X):
    """2^e per row with max|X[i,:]| < 2^e (the slicing exponents)."""
    mx = np.max(np.abs(X), axis=1)
    e = np.where(mx > 0, np.frexp(mx)[1], 0)
    return np.ldexp(1.0, e)


@pytest.mark.parametrize("m,nc,k,a_rm,b_rm", [
    (128, 64, 32, False, False),       # one tile, one stage
    (300, 130, 1000, False, True),     # ragged tiles, k not a multiple of 32, mixed layouts
    (77, 200, 9000, True, False),      # two k chunks (8192 + 808)
])
def test_ozaki_gemm_accuracy(gpu, m, nc, k, a_rm, b_rm):
    rng = np.random.default_rng(m * 7 + k)
    A = rng.standard_normal((m, k)) * np.ldexp(1.0, rng.integers(-20, 20, (m, 1)))
    B = rng.standard_normal((nc, k)) * np.ldexp(1.0, rng.integers(-20, 20, (nc, 1)))
    A[3, :] = 0.0                                     # an all-zero row
    C0 = rng.standard_normal((m, nc))
    got = _ozaki(A, B, C0, -1.5, 0.75, 0, a_rm, b_rm)
    ref = (0.75 * C0.astype(np.longdouble)
           - 1.5 * (A.astype(np.longdouble) @ B.astype(np.longdouble).T))
    scale = 1.5 * np.outer(_scale(A), _scale(B)) * np.sqrt(k) + 0.75 * np.abs(C0)
    err = np.abs(got - ref.astype(np.float64)) / scale
    assert float(err.max()) <= 2.0 ** -50, float(err.max())
    # the FP64 GEMM itself: the same order of error
    f64 = 0.75 * C0 - 1.5 * (A @ B.T)
    err64 = np.abs(f64 - ref.astype(np.float64)) / scale
    assert float(err.max()) <= 16 * max(float(err64.max()), 2.0 ** -53)


def test_ozaki_gemm_bitwise_deterministic_and_beta_zero(gpu):
    rng = np.random.default_rng(3)
    A = rng.standard_normal((257, 700))
    B = rng.standard_normal((65, 700))
    C0 = np.full((257, 65), np.nan)                   # beta = 0 must not read C
    g1 = _ozaki(A, B, C0, 1.0, 0.0, 0)
    g2 = _ozaki(A, B, C0, 1.0, 0.0, 0)
    assert np.all(np.isfinite(g1))
    assert np.array_equal(g1, g2)


def test_ozaki_syrk_lower(gpu):
    """B = A (one set of slices), only tiles on/below the diagonal: the Cholesky trailing update."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((600, 1024))
    C0 = rng.standard_normal((600, 600))
    got = _ozaki(A, A, C0, -1.0, 1.0, 4, same=True)
    ref = C0 - A @ A.T
    low = np.tril(np.ones((600, 600), bool))
    assert float(np.max(np.abs(got - ref)[low])) <= 1e-12 * 1024
    # tiles strictly above the diagonal (128-row x 64-column tiles) are untouched
    assert np.array_equal(got[:128, 128:], C0[:128, 128:])


def test_ozaki_syrk_leading_columns(gpu):
    """B = A with ncols < m: B~ is the first ncols rows of A~ (the factorisation's update of the
    next outer block only, before the deferred far-column SYRK)."""
    rng = np.random.default_rng(6)
    A = rng.standard_normal((700, 1536))
    C0 = rng.standard_normal((700, 300))
    got = _ozaki(A, A[:300], C0, -1.0, 1.0, 4, same=True)
    ref = C0 - A @ A[:300].T
    low = np.tril(np.ones((700, 300), bool))
    assert float(np.max(np.abs(got - ref)[low])) <= 1e-12 * 1536
    # equal to the two-operand form bit for bit (same slices, same products)
    two = _ozaki(A, A[:300], C0, -1.0, 1.0, 4)
    assert np.array_equal(got[low], two[low])


@pytest.mark.parametrize("agg", ["1", "2", "3"])
def test_potrf_syrk_aggregation(gpu, agg, monkeypatch):
    """Deferred trailing SYRKs (GG_SYRK_AGG outer blocks stacked along k; n = 4500 is 4.5 outer
    blocks: partial next-block updates, full updates of depth 2048 / 3072 and the ragged end)
    give the factor and inverse of the one-SYRK-per-block schedule to FP64 working accuracy."""
    n = 4500
    M = make_spd(n, n)
    monkeypatch.setenv("GG_SYRK_AGG", agg)
    Lo, Io = _factor(M, True, monkeypatch)
    Ld, Id = _factor(M, False, monkeypatch)
    assert float(np.max(np.abs(Lo - Ld))) <= 1e-13 * float(np.max(np.abs(Ld)))
    assert float(np.max(np.abs(Io - Id))) <= 1e-13 * float(np.max(np.abs(Id)))
    res = np.abs(np.tril(Lo) @ np.tril(Lo).T - M).max() / np.abs(M).max()
    assert res <= 1e-14, res


def test_ozaki_triangular_operands(gpu):
    """The trtri GEMMs: B~(j,k) = 0 for k < j (flag 2) and A~ lower triangular (flag 1), with a k
    range longer than one launch's chunk (8192) so the triangle's offsets move with the chunk."""
    rng = np.random.default_rng(11)
    n = 9000
    A = rng.standard_normal((640, n))
    Bt = rng.standard_normal((n, 520))
    Bl = np.tril(Bt)                                         # Bl[k, j] = 0 for k < j
    got = _ozaki(A, Bl.T.copy(), np.zeros((640, 520)), 1.0, 0.0, 2, b_rowmajor=True)
    ref = A @ Bl
    assert float(np.max(np.abs(got - ref))) <= 1e-12 * np.sqrt(n) * 8
    Al = np.tril(rng.standard_normal((700, 700)))
    T = rng.standard_normal((700, 300))
    got = _ozaki(Al, T.T.copy(), np.zeros((700, 300)), -1.0, 0.0, 1, b_rowmajor=True)
    assert float(np.max(np.abs(got + Al @ T))) <= 1e-12 * 700


def test_ozaki_triangle_flags_ignore_memory_outside_the_triangle(gpu):
    """flags 1 / 2 declare A~ lower (A~(i,k) = 0 for k > i) and B~(j,k) = 0 for k < j: whatever
    memory holds there is sliced as zeros (the clustered kernel runs each cluster over the union
    of its tiles' k ranges), so garbage outside the triangle changes nothing."""
    rng = np.random.default_rng(13)
    n = 1100
    A = rng.standard_normal((640, n))
    Bt = rng.standard_normal((n, 520))
    Bl = np.tril(Bt)
    Bg = Bl + np.triu(rng.standard_normal((n, 520)), 1) * 1e6       # garbage above the diagonal
    got = _ozaki(A, Bg.T.copy(), np.zeros((640, 520)), 1.0, 0.0, 2, b_rowmajor=True)
    ref = _ozaki(A, Bl.T.copy(), np.zeros((640, 520)), 1.0, 0.0, 2, b_rowmajor=True)
    assert np.array_equal(got, ref)
    Al = np.tril(rng.standard_normal((700, 700)))
    Ag = Al + np.triu(rng.standard_normal((700, 700)), 1) * 1e6
    T = rng.standard_normal((700, 300))
    got = _ozaki(Ag, T.T.copy(), np.zeros((700, 300)), -1.0, 0.0, 1, b_rowmajor=True)
    ref = _ozaki(Al, T.T.copy(), np.zeros((700, 300)), -1.0, 0.0, 1, b_rowmajor=True)
    assert np.array_equal(got, ref)


def _factor(M, ozaki, monkeypatch):
    from paper_1304_2272_b200 import kernel

    monkeypatch.setenv("GG_FACTOR_OZAKI", "1" if ozaki else "0")
    n, L, LinvP, Linv = kernel._potrf_device(M, keep_square_inverse=True)
    return L[:n, :n].cpu().numpy().T, Linv[:n, :n].cpu().numpy().T


@pytest.mark.parametrize("n", [1500, 3000])
def test_potrf_ozaki_matches_dmma(gpu, n, monkeypatch):
    """Cholesky + inverse with the int8 Ozaki updates vs the DMMA updates (and the factor's
    residual): same factor to FP64 working accuracy."""
    M = make_spd(n, n)
    Lo, Io = _factor(M, True, monkeypatch)
    Ld, Id = _factor(M, False, monkeypatch)
    assert float(np.max(np.abs(Lo - Ld))) <= 1e-13 * float(np.max(np.abs(Ld)))
    assert float(np.max(np.abs(Io - Id))) <= 1e-13 * float(np.max(np.abs(Id)))
    res = np.abs(np.tril(Lo) @ np.tril(Lo).T - M).max() / np.abs(M).max()
    assert res <= 1e-14, res
    ires = np.abs(np.tril(Io) @ np.tril(Lo) - np.eye(n)).max()
    assert ires <= 1e-13, ires


def test_potrf_ozaki_not_pd_pivot(gpu, monkeypatch):
    """A not-PD pivot past the first Ozaki update is still reported at the right global index."""
    from paper_1304_2272_b200 import kernel
    from paper_1304_2272_b200.errors import NotPositiveDefinite

    n = 3000
    M = make_spd(n, 1)
    M[2500, 2500] = -1.0
    monkeypatch.setenv("GG_FACTOR_OZAKI", "1")
    with pytest.raises(NotPositiveDefinite) as ei:
        kernel._potrf_device(M)
    assert ei.value.pivot_index == 2500


def test_gls_parity_with_ozaki_factor(gpu, monkeypatch):
    """The whole GLS block on the BASELINE generator at n = 2500 with the Ozaki factorisation,
    against the CPU oracle (north-star tolerance 1e-9; observed ~1e-13)."""
    from oracle import gls_ref as O
    from paper_1304_2272_b200 import datagen, kernel

    monkeypatch.setenv("GG_FACTOR_OZAKI", "1")
    spec = datagen.BaselineSpec(n=2500, m=700, p=4, m_kin=1500, a=0.6, seed=42)
    M = datagen.kinship_covariance_host(spec)
    XL, y = datagen.covariates_host(spec)
    G = datagen.genotypes_host(spec.seed, spec.n, spec.m, 0, spec.m).astype(np.float64)
    ctx = kernel.gls_prepare(M, XL, y)
    rb = kernel.gls_solve_block(ctx, kernel.SnpBlock(0, G))
    beta = np.array([r.beta for r in rb.results])
    ob, ok = O.gls_solve_block(O.gls_prepare(M, XL, y), G)
    rel, mism = O.compare(beta, ob)
    assert mism == 0 and rel <= 1e-11, (rel, mism)


def test_ozaki_gemm_extreme_exponents(gpu):
    """Rows scaled near the ends of the FP64 range: products that overflow give inf, products
    deep in the subnormal range round like IEEE, normal ones stay accurate."""
    rng = np.random.default_rng(17)
    A = rng.standard_normal((130, 96))
    B = rng.standard_normal((70, 96))
    A[0] *= 2.0 ** 600
    B[0] *= 2.0 ** 600                   # (0, 0) overflows
    A[1] *= 2.0 ** -540
    B[1] *= 2.0 ** -540                  # (1, 1) ~2^-1080: subnormal
    A[2] *= 2.0 ** 500
    B[2] *= 2.0 ** -500                  # (2, 2) normal after huge and tiny scales
    got = _ozaki(A, B, np.zeros((130, 70)), 1.0, 0.0, 0)
    with np.errstate(over="ignore", under="ignore", invalid="ignore"):
        ref = A.astype(np.longdouble) @ B.astype(np.longdouble).T
    assert np.isinf(got[0, 0])
    assert abs(got[1, 1] - float(ref[1, 1])) <= 2.0 ** -1074 * 4 + 1e-15 * abs(float(ref[1, 1]))
    assert abs(got[2, 2] - float(ref[2, 2])) <= 1e-14 * float(np.abs(A[2]) @ np.abs(B[2]))
    mask = np.ones_like(got, bool)
    mask[:3, :] = False
    mask[:, :3] = False
    with np.errstate(over="ignore", invalid="ignore"):
        assert float(np.max(np.abs(got - ref.astype(np.float64))[mask])) <= 1e-13
