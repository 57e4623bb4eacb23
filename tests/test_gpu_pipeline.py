"""GPU: streaming engines (reference tests/test_pipeline.py / test_acceptance.py behaviour), the
device generator, the raw DMMA GEMM, and full-size (BASELINE config 1) properties."""

import numpy as np
import pytest

from conftest import golden, maxnorm, write_golden_dataset

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods(gpu):
    from paper_1304_2272_b200 import datagen, fileio, kernel, pipeline

    return kernel, pipeline, fileio, datagen


def read_betas(path):
    from paper_1304_2272_b200 import fileio

    return fileio.read_matrix(path, "GWAB")


def test_engines_match_reference_and_each_other(mods, tmp_path):
    from oracle import gls_ref as O

    K, P, F, _ = mods
    g = golden("seed42")
    paths = write_golden_dataset(tmp_path, g)
    P.run_incore(paths)
    inc = read_betas(paths.out).betas
    rel, mism = O.compare(inc, g["beta"])
    assert mism == 0 and rel <= 1e-9
    rel, mism = O.compare(inc, g["beta_eq1"])
    assert mism == 0 and rel <= 1e-8
    for m_blk in (1, 7, 64, 500):
        paths.out = str(tmp_path / f"ooc{m_blk}.gwab")
        s = P.run_ooc(paths, P.SolveConfig(m_blk=m_blk))
        assert s.buffer_regions == 2 and s.m_blk == m_blk
        assert np.array_equal(read_betas(paths.out).betas, inc)     # bitwise across block sizes
    assert s.bytes_written == 500 * 32 and s.bytes_read >= 8 * 100 * 500
    assert s.t_prepare >= 0 and s.t_compute >= 0 and s.t_io_wait >= 0
    assert s.t_prepare + s.t_compute + s.t_io_wait <= s.t_total * 1.05


def test_int8_stream_equals_fp64_stream(mods, tmp_path):
    K, P, F, _ = mods
    g = golden("baseline_p4")
    p64 = write_golden_dataset(tmp_path, g, int8=False, name="f64")
    p8 = write_golden_dataset(tmp_path, g, int8=True, name="i8")
    P.run_ooc(p64, P.SolveConfig(m_blk=300))
    P.run_ooc(p8, P.SolveConfig(m_blk=512))
    a, b = read_betas(p64.out).betas, read_betas(p8.out).betas
    assert np.array_equal(a, b, equal_nan=True)
    from oracle import gls_ref as O

    rel, mism = O.compare(a, g["beta"])
    assert mism == 0 and rel <= 1e-9


def test_degenerate_markers_flagged(mods, tmp_path):
    K, P, F, _ = mods
    g = golden("degenerate")
    paths = write_golden_dataset(tmp_path, g)
    P.run_ooc(paths, P.SolveConfig(m_blk=16))
    st = read_betas(paths.out).statuses
    assert set(np.nonzero(st == "degenerate")[0]) == {10, 20}
    paths.out = str(tmp_path / "inc.gwab")
    P.run_incore(paths)
    assert set(np.nonzero(read_betas(paths.out).statuses == "degenerate")[0]) == {10, 20}


def test_emit_sinv_flows_to_file(mods, tmp_path):
    K, P, F, _ = mods
    g = golden("seed42")
    paths = write_golden_dataset(tmp_path, g)
    P.run_ooc(paths, P.SolveConfig(m_blk=200, emit_s_inv=True))
    pay = read_betas(paths.out)
    assert pay.sinv.shape == (500, 10) and np.all(np.isfinite(pay.sinv))
    ok = ~g["status"].astype(bool)
    assert maxnorm(pay.sinv[ok] - g["sinv"][ok]) <= 1e-9 * maxnorm(g["sinv"][ok])


def test_memory_budget(mods, tmp_path, monkeypatch):
    from paper_1304_2272_b200.errors import ConfigError

    K, P, F, _ = mods
    g = golden("seed42")
    paths = write_golden_dataset(tmp_path, g)
    with pytest.raises(ConfigError):
        P.run_incore(paths, P.SolveConfig(mem_budget_bytes=8 * 100 * 500))
    s = P.run_ooc(paths, P.SolveConfig(m_blk=32, mem_budget_bytes=8 * 100 * 500))
    assert s.buffer_regions == 2
    with pytest.raises(ConfigError):
        P.run_ooc(paths, P.SolveConfig(m_blk=500, mem_budget_bytes=1000))
    monkeypatch.setenv("GWAS_GLS_MEM_BUDGET_BYTES", "1000")
    with pytest.raises(ConfigError):
        P.run_incore(paths)


def test_scale_invariance_and_identity(mods, tmp_path):
    # reference acceptance criterion 9 (tests/test_acceptance.py:282-334)
    K, P, F, _ = mods
    g = golden("seed42")
    ctx = K.gls_prepare(g["M"], g["XL"], g["y"])
    X = g["G"][:, :120].astype(float)
    b = np.array([r.beta for r in K.gls_solve_block(ctx, K.SnpBlock(0, X)).results])
    ctx_c = K.gls_prepare(7.5 * g["M"], g["XL"], g["y"])
    bc = np.array([r.beta for r in K.gls_solve_block(ctx_c, K.SnpBlock(0, X)).results])
    assert np.max(np.abs(bc - b) / np.maximum(np.abs(b), 1.0)) <= 1e-9
    ctx_i = K.gls_prepare(np.eye(100), g["XL"], g["y"])
    bi = np.array([r.beta for r in K.gls_solve_block(ctx_i, K.SnpBlock(0, X)).results])
    for i in range(120):
        Xi = np.hstack([g["XL"], X[:, i:i + 1]])
        e, *_ = np.linalg.lstsq(Xi, g["y"], rcond=None)
        assert maxnorm(bi[i] - e) <= 1e-10 * max(maxnorm(e), 1.0)


def test_solve_array_pinned(mods):
    import torch

    K, P, F, _ = mods
    g = golden("baseline_p8")
    ctx = K.gls_prepare(g["M"], g["XL"], g["y"])
    G = torch.from_numpy(np.ascontiguousarray(g["G"].T)).pin_memory().numpy().T
    res = P.solve_array(ctx, G, m_blk=128, emit_s_inv=True)
    from oracle import gls_ref as O

    rel, mism = O.compare(np.where(res.ok[:, None], res.beta, np.nan), g["beta"])
    assert mism == 0 and rel <= 1e-9


def test_device_generator_matches_host(mods):
    K, P, F, D = mods
    spec = D.BaselineSpec(n=777, m=5000, p=4)
    dev = D.genotypes_device(spec, 1234, 300).cpu().numpy()      # (cnt, n)
    host = D.genotypes_host(spec.seed, spec.n, spec.m, 1234, 300)
    assert np.array_equal(dev.T, host)
    small = D.BaselineSpec(n=300, m=10, p=4, m_kin=500, a=0.6)
    Md = D.kinship_covariance_device(small).cpu().numpy()
    Mh = D.kinship_covariance_host(small)
    assert np.array_equal(Md, Md.T)
    assert maxnorm(Md - Mh) <= 1e-13 * maxnorm(Mh)


@pytest.mark.parametrize("m,ncols,k,trans", [(128, 1, 16, 0), (256, 300, 128, 0), (384, 256, 512, 1),
                                              (128, 129, 48, 0)])
def test_raw_dgemm(mods, m, ncols, k, trans):
    import torch

    from paper_1304_2272_b200 import _capi
    from paper_1304_2272_b200._capi import ptr, stream_handle

    rng = np.random.default_rng(m + ncols)
    A = rng.standard_normal((m, k))
    B = rng.standard_normal((ncols, k)) if trans else rng.standard_normal((k, ncols))
    C0 = rng.standard_normal((m, ncols))
    dev = torch.device("cuda")
    Ad = torch.from_numpy(np.asfortranarray(A).T.copy()).to(dev)
    Bd = torch.from_numpy(np.asfortranarray(B).T.copy()).to(dev)
    Cd = torch.from_numpy(np.asfortranarray(C0).T.copy()).to(dev)
    rc = _capi.lib().gg_dgemm_f64(m, ncols, k, -1.5, ptr(Ad), m, ptr(Bd), B.shape[0], trans, 0.5,
                                  ptr(Cd), m, stream_handle())
    assert rc == 0
    got = Cd.cpu().numpy().T
    expect = -1.5 * A @ (B.T if trans else B) + 0.5 * C0
    assert maxnorm(got - expect) <= 1e-13 * maxnorm(expect)


def test_config1_full_size_block(mods):
    """BASELINE config 1 at full n = 10,000 (one 8,192-SNP block): sampled parity against the
    CPU oracle, column-permutation bitwise invariance, int8 == FP64 bitwise."""
    import torch

    from oracle import gls_ref as O

    K, P, F, D = mods
    spec = D.CONFIGS[1]
    Mt = D.kinship_covariance_device(spec)
    M = Mt.cpu().numpy()
    XL, y = D.covariates_host(spec)
    ctx = K.gls_prepare(M, XL, y)
    G = D.genotypes_device(spec, 0, 8192).cpu().numpy().T          # n x 8192 int8, F-order
    res = P.solve_array(ctx, np.asfortranarray(G), m_blk=8192)
    assert np.all(res.ok)
    # sampled oracle parity (CPU dpotrf at n = 1e4 takes a few seconds)
    octx = O.gls_prepare(M, XL, y)
    sample = np.r_[0:8, 4000:4004, 8188:8192]
    ob, ok = O.gls_solve_block(octx, G[:, sample].astype(float))
    rel, mism = O.compare(res.beta[sample], ob)
    assert mism == 0 and rel <= 1e-9, rel
    perm = np.random.default_rng(0).permutation(8192)
    res_p = P.solve_array(ctx, np.asfortranarray(G[:, perm].astype(float)), m_blk=8192)
    assert np.array_equal(res_p.beta, res.beta[perm])
    torch.cuda.empty_cache()


def test_config3_full_size_sample(mods):
    """BASELINE config 3 at full n = 40,000, p = 8 (M = 0.5 K + 0.5 I): the Ozaki-factorised,
    int8-swept path against the CPU oracle on a sample of SNPs from an 8,192-SNP block, plus
    bitwise equality of the int8 and FP64 host inputs on that sample."""
    import torch

    from oracle import gls_ref as O

    K, P, F, D = mods
    spec = D.CONFIGS[3]
    Mt = D.kinship_covariance_device(spec)
    XL, y = D.covariates_host(spec)
    ctx = K.gls_prepare(Mt, XL, y)
    M = Mt.cpu().numpy()
    del Mt
    G = D.genotypes_device(spec, 0, 8192).cpu().numpy().T          # n x 8192 int8
    res = P.solve_array(ctx, np.asfortranarray(G), m_blk=8192)
    assert np.all(res.ok)
    sample = np.r_[0:6, 5000:5003, 8189:8192]
    octx = O.gls_prepare(M, XL, y)                                  # CPU dpotrf at n = 4e4
    ob, ok = O.gls_solve_block(octx, G[:, sample].astype(float))
    rel, mism = O.compare(res.beta[sample], ob)
    assert mism == 0 and rel <= 1e-9, rel
    res_f = P.solve_array(ctx, np.asfortranarray(G[:, sample].astype(float)), m_blk=8192)
    assert np.array_equal(res_f.beta, res.beta[sample])
    del ctx
    torch.cuda.empty_cache()
