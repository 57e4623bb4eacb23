"""GPU: the int8 tensor-core TRSM path (inverse split into int8 slices, exact int32 products,
FP64 recombination) against the FP64 DMMA path and the oracle; its fused reductions against the
standalone ones; device-side fallback for non-integer FP64 blocks."""

import numpy as np
import pytest

from conftest import golden, make_spd, maxnorm

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K(gpu):
    from paper_1304_2272_b200 import kernel

    return kernel


def _betas(rb):
    return np.array([r.beta for r in rb.results])


@pytest.mark.parametrize("n,cnt", [(37, 5), (300, 257), (1000, 129), (1001, 300)])
def test_i8_trsm_matches_dmma(K, n, cnt):
    import torch

    from paper_1304_2272_b200 import _capi
    from paper_1304_2272_b200._capi import ptr, stream_handle
    from paper_1304_2272_b200._device import alloc_cols, upload_cols

    M = make_spd(n, n)
    _, L, LinvP, Linv = K._potrf_device(M, keep_square_inverse=True)
    sl, expo = K._slice_inverse(Linv, n)
    G = np.random.default_rng(n).integers(0, 3, (n, cnt))
    np_ = _capi.pad(n)
    Xd = K._trsm_device(LinvP, n, upload_cols(G.astype(float), ld=np_), cnt)
    Xi = K._trsm_i8_device(sl, expo, n, G)
    torch.cuda.synchronize()
    ref = Xd[:, :n].cpu().numpy()
    got = Xi[:, :n].cpu().numpy()
    colrel = np.max(np.abs(got - ref), axis=1) / np.max(np.abs(ref), axis=1)
    assert colrel.max() <= 1e-13, colrel.max()
    assert bool((Xi[:, n:] == 0).all())
    # bitwise column-permutation invariance of the tensor-core path
    perm = np.random.default_rng(1).permutation(cnt)
    Xp = K._trsm_i8_device(sl, expo, n, G[:, perm]).cpu().numpy()
    assert np.array_equal(Xp, Xi.cpu().numpy()[perm])


def test_i8_trsm_small_and_ragged_shapes(K):
    """Edge shapes of the int8 TRSM (n below / at / above the 32-row block and 128-row tile
    boundaries, 1 .. 300 columns, partial SNP pairs) against the FP64 DMMA TRSM."""
    import torch

    from paper_1304_2272_b200 import _capi
    from paper_1304_2272_b200._device import upload_cols

    for n in (1, 2, 5, 31, 32, 33, 127, 128, 129, 257):
        M = make_spd(n, 3 * n + 1)
        _, L, LinvP, Linv = K._potrf_device(M, keep_square_inverse=True)
        sl, expo = K._slice_inverse(Linv, n)
        np_ = _capi.pad(n)
        for cnt in (1, 3, 130, 300):
            G = np.random.default_rng(n * 1000 + cnt).integers(0, 3, (n, cnt))
            Xd = K._trsm_device(LinvP, n, upload_cols(G.astype(float), ld=np_), cnt)
            Xi = K._trsm_i8_device(sl, expo, n, G)
            torch.cuda.synchronize()
            ref = Xd[:, :n].cpu().numpy()
            got = Xi[:, :n].cpu().numpy()
            scale = np.maximum(np.max(np.abs(ref), axis=1), 1e-300)
            colrel = np.max(np.abs(got - ref), axis=1) / scale
            assert colrel.max() <= 1e-13, (n, cnt, colrel.max())
            assert bool((Xi[:, n:] == 0).all()), (n, cnt)


def test_i8_trsm_accuracy_vs_extended_precision(K):
    """Accuracy of the sliced inverse on a kinship covariance (the BASELINE workload's M): the
    int8 path's Xbar = Linv G against Linv G in extended precision for the same FP64 inverse.
    7 slices + head with a round-to-nearest last slice: ~2e-15 of the column maximum (the FP64
    DMMA TRSM's own rounding is ~1e-15); all-truncated slices were 5e-15, 6 slices 3e-13."""
    import torch

    from paper_1304_2272_b200 import datagen

    n, cnt = 1500, 48
    spec = datagen.BaselineSpec(n=n, m=cnt, p=4)
    M = datagen.kinship_covariance_host(spec)
    _, L, LinvP, Linv = K._potrf_device(M, keep_square_inverse=True)
    sl, expo = K._slice_inverse(Linv, n)
    G = np.random.default_rng(5).integers(0, 3, (n, cnt))
    Xi = K._trsm_i8_device(sl, expo, n, G)[:, :n].cpu().numpy().T      # (n, cnt)
    Li = Linv[:n, :n].cpu().numpy().T                                   # row-major Linv
    ref = (Li.astype(np.longdouble) @ G.astype(np.longdouble)).astype(np.float64)
    err = np.max(np.abs(Xi - ref) / np.max(np.abs(ref), axis=0))
    assert err <= 4e-15, err
    torch.cuda.synchronize()


@pytest.mark.parametrize("case", ["seed42", "baseline_p4", "baseline_p8", "degenerate"])
def test_i8_and_dmma_paths_agree_with_reference(K, case):
    from oracle import gls_ref as O

    g = golden(case)
    X = g["G"].astype(float)
    ctx8 = K.gls_prepare(g["M"], g["XL"], g["y"])
    ctx64 = K.gls_prepare(g["M"], g["XL"], g["y"], int8_split=False)
    assert ctx8._dev.slices is not None and ctx64._dev.slices is None
    b8 = _betas(K.gls_solve_block(ctx8, K.SnpBlock(0, X)))
    b64 = _betas(K.gls_solve_block(ctx64, K.SnpBlock(0, X)))
    for b in (b8, b64):
        rel, mism = O.compare(b, g["beta"])
        assert mism == 0 and rel <= 1e-9, rel
    rel, mism = O.compare(b8, b64)
    assert mism == 0 and rel <= 1e-12


def test_fused_reductions_equal_standalone(K):
    """The TRSM epilogue's fused partial dots give the same bits as the standalone reductions
    applied to the same Xbar (one canonical order)."""
    g = golden("baseline_p4")
    ctx = K.gls_prepare(g["M"], g["XL"], g["y"])
    G = g["G"][:, :300]
    fused = _betas(K.gls_solve_block(ctx, K.SnpBlock(0, np.asfortranarray(G))))
    n = g["M"].shape[0]
    Xbar = K._trsm_i8_device(ctx._dev.slices, ctx._dev.expo, n, G)[:, :n].cpu().numpy().T
    res = K.solve_whitened_block(ctx, Xbar, 0)
    assert np.array_equal(np.array([r.beta for r in res]), fused)


def test_non_integer_block_falls_back_to_dmma(K):
    """FP64 blocks are narrowed on the device; any non-integer value routes the block through
    the FP64 DMMA TRSM (chosen on the device, no host sync).  Results match the oracle."""
    from oracle import gls_ref as O

    rng = np.random.default_rng(3)
    n = 200
    M = make_spd(n, 5)
    XL = np.hstack([np.ones((n, 1)), rng.standard_normal((n, 2))])
    y = rng.standard_normal(n)
    Xint = rng.integers(0, 3, (n, 40)).astype(float)
    Xmix = Xint.copy()
    Xmix[7, 3] = 0.5                              # one non-integer dosage
    Xbig = Xint.copy()
    Xbig[0, 0] = 300.0                            # out of int8 range
    ctx = K.gls_prepare(M, XL, y)
    octx = O.gls_prepare(M, XL, y)
    for X in (Xint, Xmix, Xbig):
        got = _betas(K.gls_solve_block(ctx, K.SnpBlock(0, X)))
        ref, ok = O.gls_solve_block(octx, X)
        rel, mism = O.compare(got, ref)
        assert mism == 0 and rel <= 1e-11, rel


@pytest.mark.parametrize("m_blk", [1, 7, 40, 64])
def test_path_selection_is_per_column(K, m_blk):
    """Integer and fractional dosages in one block: every column takes its path (int8 tensor
    cores or FP64 DMMA) from its own values, so an integer column's result is bitwise the same
    whatever its neighbours, the block size or its position (a block-wide gate made it
    depend on them).  Fractional columns still match the oracle; the same holds for int8 blocks
    with values past the exact bound (simulated by a large value in a FP64 block)."""
    from oracle import gls_ref as O

    rng = np.random.default_rng(31)
    n = 300
    M = make_spd(n, 8)
    XL = np.hstack([np.ones((n, 1)), rng.standard_normal((n, 2))])
    y = rng.standard_normal(n)
    X = rng.integers(0, 3, (n, 64)).astype(float)
    frac = [3, 10, 11, 40, 63]
    X[:, frac] += rng.uniform(0.05, 0.95, (n, len(frac)))      # imputed (fractional) dosages
    X[5, 20] = 300.0                                           # out of int8 range
    ctx = K.gls_prepare(M, XL, y)
    alone = _betas(K.gls_solve_block(ctx, K.SnpBlock(0, np.delete(X, frac + [20], axis=1))))
    got = np.concatenate([_betas(K.gls_solve_block(ctx, K.SnpBlock(f, X[:, f:f + m_blk])))
                          for f in range(0, 64, m_blk)])
    ints = [j for j in range(64) if j not in frac + [20]]
    assert np.array_equal(got[ints], alone, equal_nan=True)
    octx = O.gls_prepare(M, XL, y)
    ref, _ = O.gls_solve_block(octx, X)
    rel, mism = O.compare(got, ref)
    assert mism == 0 and rel <= 1e-11, rel


def test_pending_result_blocks_pipeline(K):
    """gls_solve_block returns once the block's copy is done; results resolve on first access.
    Many unresolved blocks (more than the stream's device regions), a reused host buffer and
    out-of-order resolution give exactly the results of resolving each call at once."""
    rng = np.random.default_rng(12)
    n = 257
    M = make_spd(n, 4)
    XL = np.hstack([np.ones((n, 1)), rng.standard_normal((n, 1))])
    ctx = K.gls_prepare(M, XL, rng.standard_normal(n))
    blocks = [rng.integers(0, 3, (n, 33)).astype(np.int8, order="F") for _ in range(7)]
    eager = [_betas(K.gls_solve_block(ctx, K.SnpBlock(33 * i, b))) for i, b in enumerate(blocks)]
    buf = np.empty((n, 33), dtype=np.int8, order="F")
    pend = []
    for i, b in enumerate(blocks):
        buf[...] = b                                   # the caller's reused double buffer
        pend.append(K.gls_solve_block(ctx, K.SnpBlock(33 * i, buf)))
    assert not all(p.done for p in pend)
    for i in (6, 0, 3, 1, 2, 5, 4):
        assert pend[i].first_index == 33 * i
        assert np.array_equal(_betas(pend[i]), eager[i], equal_nan=True)


def test_intercept_duplicate_exactly_singular(K):
    """A SNP equal to the intercept: whitened by the same tensor-core kernel as X_L[:,0] and
    reduced in the same order, S is exactly singular and the SNP is flagged degenerate."""
    rng = np.random.default_rng(9)
    n = 150
    M = make_spd(n, 2)
    XL = np.hstack([np.ones((n, 1)), rng.standard_normal((n, 2))])
    ctx = K.gls_prepare(M, XL, rng.standard_normal(n))
    X = rng.integers(0, 3, (n, 10)).astype(np.int8)
    X[:, 4] = 1
    rb = K.gls_solve_block(ctx, K.SnpBlock(0, np.asfortranarray(X)))
    st = [r.status for r in rb.results]
    assert st[4] == "degenerate" and st.count("degenerate") == 1


@pytest.mark.parametrize("n", [300, 1001])
def test_slices_from_packed_and_block_cyclic_sources(K, n):
    """The tile-packed slices are identical whether cut from the row-major inverse, the packed
    FP64 inverse, or assembled from a 2x2 block-cyclic distribution (row exponents MAX-reduced,
    per-rank slices with zeros elsewhere SUM-reduced) -- the config-4 construction."""
    import torch

    from paper_1304_2272_b200 import _capi
    from paper_1304_2272_b200._capi import ptr, stream_handle

    lib = _capi.lib()
    s = stream_handle()
    M = make_spd(n, n + 1)
    _, L, LinvP, Linv = K._potrf_device(M, keep_square_inverse=True)
    sl_ref, ex_ref = K._slice_inverse(Linv, n)
    np_ = _capi.pad(n)
    sl = torch.empty_like(sl_ref)
    ex = torch.empty_like(ex_ref)
    assert lib.gg_slice_packed_inverse_i8(n, ptr(LinvP), ptr(sl), ptr(ex), s) == 0
    torch.cuda.synchronize()
    assert torch.equal(ex, ex_ref) and torch.equal(sl, sl_ref)
    # 2x2 block-cyclic, nb = 128: local blocks of each "rank" from the full column-major inverse
    nb, gr, gc = 128, 2, 2
    Linv_h = Linv[:np_, :np_].cpu().numpy()          # (cols, rows): Linv_h[k, i] = Linv[i, k]
    nbk = np_ // nb
    exps, slcs = [], []
    for pr in range(gr):
        for pc in range(gc):
            rows = [I for I in range(nbk) if I % gr == pr]
            cols = [J for J in range(nbk) if J % gc == pc]
            loc = np.zeros((len(cols) * nb, len(rows) * nb))   # column-major local (cols, rows)
            for a_, I in enumerate(rows):
                for b_, J in enumerate(cols):
                    loc[b_ * nb:(b_ + 1) * nb, a_ * nb:(a_ + 1) * nb] = \
                        Linv_h[J * nb:(J + 1) * nb, I * nb:(I + 1) * nb]
            B = torch.from_numpy(loc).cuda()
            e = torch.empty_like(ex)
            assert lib.gg_row_exponents_blockcyclic(n, nb, gr, gc, pr, pc, ptr(B),
                                                    len(rows) * nb, ptr(e), s) == 0
            exps.append(e)
            slcs.append((B, rows))
    emax = torch.stack(exps).max(dim=0).values
    meta = torch.empty_like(ex)
    assert lib.gg_slice_meta_i8(n, ptr(emax), ptr(meta), s) == 0
    torch.cuda.synchronize()
    assert torch.equal(meta[:np_], ex_ref[:np_]) and not meta[np_:].any()
    total = torch.zeros(sl_ref.numel(), dtype=torch.int32, device="cuda")
    heads = torch.zeros(np_, dtype=torch.int32, device="cuda")
    for (B, rows), (pr, pc) in zip(slcs, [(0, 0), (0, 1), (1, 0), (1, 1)]):
        part = torch.full_like(sl_ref, 7)
        m = meta.clone()
        assert lib.gg_slice_blockcyclic_i8(n, nb, gr, gc, pr, pc, ptr(B), len(rows) * nb,
                                           ptr(m), ptr(part), s) == 0
        total += part.to(torch.int32)
        heads += m[np_:]
    torch.cuda.synchronize()
    assert torch.equal(total.to(torch.int8), sl_ref) and int(total.abs().max()) <= 128
    assert torch.equal(heads, ex_ref[np_:])


def test_dynamic_scheduler_stress_deterministic(K):
    """Many launches of the tile-queue kernel with ragged shapes (1 .. 2 SNP tiles, partial row
    blocks): every repeat is bitwise identical to the first (no scheduling race, no hang)."""
    import torch

    from paper_1304_2272_b200 import _capi
    from paper_1304_2272_b200._capi import ptr, stream_handle

    lib = _capi.lib()
    s = stream_handle()
    rng = np.random.default_rng(11)
    for n, cnts in ((130, (1, 7, 255, 256, 257, 513)), (1000, (33, 300))):
        M = make_spd(n, n + 3)
        XL = np.hstack([np.ones((n, 1)), rng.standard_normal((n, 2))])
        ctx = K.gls_prepare(M, XL, rng.standard_normal(n))
        d = ctx._dev
        n16 = -(-n // 16) * 16
        for cnt in cnts:
            G = torch.zeros((cnt, n16), dtype=torch.int8)
            G[:, :n] = torch.from_numpy(rng.integers(0, 3, (cnt, n)).astype(np.int8))
            G = G.cuda()
            P = torch.empty(int(lib.gg_partials_bytes(n, cnt, d.q)) // 8, dtype=torch.float64,
                            device="cuda")
            ref = None
            W = _capi.i8_work()
            for rep in range(40):
                assert lib.gg_trsm_lower_i8_partials(n, cnt, ptr(d.slices), ptr(d.expo), ptr(G),
                                                     n16, d.q, ptr(d.XLy), ptr(d.ybar), ptr(P),
                                                     None, 0, None, 0, ptr(W), s) == 0
                if rep == 0:
                    ref = P.clone()
            torch.cuda.synchronize()
            assert torch.equal(P, ref), (n, cnt)


@pytest.mark.parametrize("p", [2, 8, 20])
def test_i8_path_all_covariate_counts(K, p):
    """The fused epilogue's partial dots for p = 2, 8, 20 (q = 1, 7, 19: the
    three reduction variants) against the oracle."""
    from oracle import gls_ref as O

    rng = np.random.default_rng(50 + p)
    n = 333
    M = make_spd(n, p)
    XL = np.hstack([np.ones((n, 1)), rng.standard_normal((n, p - 2))]) if p >= 2 \
        else np.zeros((n, 0))
    y = rng.standard_normal(n)
    G = rng.integers(0, 3, (n, 70)).astype(np.int8)
    ctx = K.gls_prepare(M, XL, y)
    assert ctx._dev.slices is not None
    rb = K.gls_solve_block(ctx, K.SnpBlock(0, np.asfortranarray(G)), emit_s_inv=True)
    got = _betas(rb)
    ref, ok = O.gls_solve_block(O.gls_prepare(M, XL, y), G.astype(float))
    rel, mism = O.compare(got, ref)
    assert mism == 0 and rel <= 1e-10, rel


@pytest.mark.parametrize("grp", ["1", "3", "7", "1000"])
def test_i8_trsm_snp_group_order_is_bitwise_invariant(K, grp, monkeypatch):
    """The SNP-group tile order (GG_I8_SNP_GROUP pairs per group, default sqrt-scaled in n) only
    changes which cluster computes a tile when: every column is bitwise the same, including the
    ragged last group and the partial last pair."""
    import torch

    n, cnt = 700, 8 * 256 + 77                   # 9 pairs: groups of 1, 3 (3x3), 7 (7+2), all
    M = make_spd(n, 2 * n)
    _, L, LinvP, Linv = K._potrf_device(M, keep_square_inverse=True)
    sl, expo = K._slice_inverse(Linv, n)
    G = np.random.default_rng(7).integers(0, 3, (n, cnt))
    monkeypatch.delenv("GG_I8_SNP_GROUP", raising=False)
    ref = K._trsm_i8_device(sl, expo, n, G).cpu().numpy()
    monkeypatch.setenv("GG_I8_SNP_GROUP", grp)
    got = K._trsm_i8_device(sl, expo, n, G).cpu().numpy()
    torch.cuda.synchronize()
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("env", [{"GG_I8_ORDER": "1"}, {"GG_I8_QUAD": "1"},
                                 {"GG_I8_QUAD": "1", "GG_I8_QUAD_ILV": "0"}])
def test_i8_trsm_tile_variants_are_bitwise_invariant(K, env, monkeypatch):
    """The measured tile variants -- zigzag tile order, QUAD tiles (one row block x two SNP pairs)
    in B- and A-stationary MMA order -- change only when and where a tile is computed: every
    column (X-bar and the fused partial dots through the block solve) is bitwise the default's."""
    import torch

    from oracle import gls_ref as O

    n, cnt = 900, 6 * 256 + 33
    M = make_spd(n, 3 * n)
    XL = np.column_stack([np.ones(n), np.random.default_rng(1).standard_normal((n, 2))])
    y = np.random.default_rng(2).standard_normal(n)
    G = np.random.default_rng(8).integers(0, 3, (n, cnt)).astype(np.int8)
    ctx = K.gls_prepare(M, XL, y)
    for k in ("GG_I8_ORDER", "GG_I8_QUAD", "GG_I8_QUAD_ILV"):
        monkeypatch.delenv(k, raising=False)
    ref = np.array([r.beta for r in K.gls_solve_block(ctx, K.SnpBlock(0, np.asfortranarray(G))).results])
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    got = np.array([r.beta for r in K.gls_solve_block(ctx, K.SnpBlock(0, np.asfortranarray(G))).results])
    torch.cuda.synchronize()
    assert np.array_equal(got, ref, equal_nan=True)
    octx = O.gls_prepare(M, XL, y)
    ob, _ = O.gls_solve_block(octx, G.astype(np.float64))
    rel, mism = O.compare(got, ob)
    assert mism == 0 and rel <= 1e-9
