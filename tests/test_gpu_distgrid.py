"""GPU: the distributed (config-4) engine with the sm_100a kernels -- one rank, and several ranks
sharing this one B200 (threads with a reference-contract transport, or processes over gloo
through transport.run_spmd): world 2 and 4 on grids 1x2 / 2x2, against the CPU oracle.  The
ranks' kernels never wait on one another on the device (every exchange is a host-mediated
transport or gloo collective), so co-locating them on one GPU is safe."""

import numpy as np
import pytest

from conftest import golden, make_spd, write_golden_dataset

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,nb", [(1000, 256), (2100, 512)])   # nb = 512: Ozaki updates
def test_device_dist_factor_inverse_pack(gpu, n, nb):
    from scipy.linalg import cholesky, solve_triangular

    from paper_1304_2272_b200 import distgrid, kernel

    M = make_spd(n, 3)
    ops = distgrid.DeviceOps()
    lay = distgrid.BlockCyclic(n, nb, distgrid.grid_create(1), 0)
    A, B = distgrid.local_from_global(M, lay, ops)
    distgrid.dist_potrf_inv(A, B, lay, ops)
    L = distgrid.gather_matrix(A, lay, ops)
    Li = distgrid.gather_matrix(B, lay, ops)
    Lr = cholesky(M, lower=True)
    Lir = solve_triangular(Lr, np.eye(n), lower=True)
    assert np.max(np.abs(L - Lr)) <= 1e-13 * np.max(np.abs(Lr))
    assert np.max(np.abs(Li - Lir)) <= 1e-12 * np.max(np.abs(Lir))
    P = distgrid.assemble_packed_inverse(B, lay, ops)
    _, _, P1 = kernel._potrf_device(M)
    assert P.shape == P1.shape
    assert float((P - P1).abs().max()) <= 1e-12 * float(P1.abs().max())


def test_device_dist_not_pd(gpu):
    from paper_1304_2272_b200 import distgrid
    from paper_1304_2272_b200.errors import NotPositiveDefinite

    M = make_spd(600, 4)
    M[450, 450] = -1.0
    ops = distgrid.DeviceOps()
    lay = distgrid.BlockCyclic(600, 128, distgrid.grid_create(1), 0)
    A, B = distgrid.local_from_global(M, lay, ops)
    with pytest.raises(NotPositiveDefinite) as e:
        distgrid.dist_potrf_inv(A, B, lay, ops)
    assert e.value.pivot_index == 450


@pytest.mark.parametrize("fp64_inverse", [None, False])
@pytest.mark.parametrize("case", ["baseline_p4", "degenerate"])
def test_run_dist_end_to_end(gpu, tmp_path, case, fp64_inverse):
    """Both forms of the distributed prepare: replicated packed FP64 inverse + slices, and the
    config-4 form (slices only, [X_L | y] whitened from the block-cyclic inverse)."""
    from oracle import gls_ref as O
    from paper_1304_2272_b200 import distgrid, fileio

    g = golden(case)
    paths = write_golden_dataset(tmp_path, g)
    s = distgrid.run_dist_engine(paths, distgrid.DistConfig(m_blk=257, nb=128,
                                                           fp64_inverse=fp64_inverse))
    assert s.mode == "dist" and s.np_ == 1
    pay = fileio.read_matrix(paths.out, "GWAB")
    rel, mism = O.compare(pay.betas, g["beta"])
    assert mism == 0 and rel <= 1e-9


def test_slices_only_context_rejects_non_integer_blocks(gpu):
    """Without an FP64 inverse a non-integer column cannot be computed: it is marked invalid on
    the device and the host raises (no silent wrong numbers)."""
    from paper_1304_2272_b200 import kernel
    from paper_1304_2272_b200.errors import DeviceError

    rng = np.random.default_rng(2)
    n = 200
    M = make_spd(n, 5)
    XL = np.hstack([np.ones((n, 1)), rng.standard_normal((n, 2))])
    ctx = kernel.gls_prepare(M, XL, rng.standard_normal(n))
    ctx._dev.LinvP = None
    X = rng.integers(0, 3, (n, 20)).astype(float)
    ok = kernel.gls_solve_block(ctx, kernel.SnpBlock(0, X))
    assert all(r.status in ("ok", "degenerate") for r in ok.results)
    X[5, 3] = 0.25
    with pytest.raises(DeviceError):       # raised when the (asynchronous) block resolves
        kernel.gls_solve_block(ctx, kernel.SnpBlock(0, X)).results


def _ref_cfg(m_blk):
    """A reference-style DistConfig (distgrid.py:322-328 fields) for the reference signature."""
    from types import SimpleNamespace

    return SimpleNamespace(m_blk=m_blk, emit_s_inv=False, nb=64, threads=1)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", ["baseline_p4", "degenerate"])
def test_reference_signature_run_dist_multi_rank(gpu, tmp_path, world, case):
    """run_dist(t, paths, cfg) -- the reference's SPMD signature -- on `world` ranks sharing this
    GPU (threads driving a reference-contract transport): the fused block-cyclic factorisation
    with row/column broadcasts, replicated slices, SNP-sharded sweep; golden results."""
    from oracle import gls_ref as O
    from paper_1304_2272_b200 import distgrid, fileio
    from spmd_inproc import run_spmd

    g = golden(case)
    paths = write_golden_dataset(tmp_path, g)
    res = run_spmd(world, distgrid.run_dist, paths, _ref_cfg(16 * world))
    assert all(r.mode == "dist" and r.np_ == world for r in res)
    assert res[0].combine_bytes == 0 and res[0].localpart_bytes == 0
    pay = fileio.read_matrix(paths.out, "GWAB")
    rel, mism = O.compare(pay.betas, g["beta"])
    assert mism == 0 and rel <= 1e-9


def test_reference_signature_rejects_indivisible_block(gpu, tmp_path):
    from paper_1304_2272_b200 import distgrid
    from paper_1304_2272_b200.errors import ConfigError
    from spmd_inproc import run_spmd

    paths = write_golden_dataset(tmp_path, golden("seed42"))
    with pytest.raises(ConfigError):
        run_spmd(3, distgrid.run_dist, paths, _ref_cfg(128))


@pytest.mark.parametrize("world", [2, 4])
def test_dist_cholesky_and_trsolve_reference_signatures_on_device(gpu, world):
    """dist_cholesky(M, t, nb) / dist_trsolve(L, B, t, nb) with element-cyclic operands on the
    device ops (reference tests/test_distgrid.py:140-238 tolerances)."""
    from scipy.linalg import cholesky, solve_triangular

    from paper_1304_2272_b200 import distgrid
    from spmd_inproc import EC, gather_ec, run_spmd

    n = 300
    M = make_spd(n, 42)
    rng = np.random.default_rng(5)
    B = rng.standard_normal((n, 20))

    def body(t):
        g = distgrid.grid_create(t.size)
        Ld = distgrid.dist_cholesky(EC.of(M, g, t.rank), t, nb=8)
        X = distgrid.dist_trsolve(Ld, EC.of(B, g, t.rank), t, nb=16)
        return gather_ec(Ld, t), gather_ec(X, t)

    Lr = cholesky(M, lower=True)
    Xr = solve_triangular(Lr, B, lower=True)
    for L, X in run_spmd(world, body):
        assert np.max(np.abs(L - Lr)) <= 1e-10 * np.max(np.abs(M))
        assert np.max(np.abs(Lr @ X - B)) / np.max(np.abs(B)) <= 1e-12
        assert np.max(np.abs(X - Xr)) <= 1e-10 * np.max(np.abs(Xr))


def test_config4_form_at_n10k_grid_2x2_against_the_oracle(gpu):
    """BASELINE.md §3's smaller-n 2D run of the config-4 path: n = 10,000, nb = 512, grid 2x2
    (four ranks on this GPU), M generated per rank on the device (local_from_spec), fused
    Cholesky + inverse with row/column broadcasts, int8 slices assembled without any replicated
    FP64 inverse, [X_L | y] whitened from the block-cyclic inverse, then a 1,024-SNP sample
    through the slices-only context -- against the CPU oracle on the gathered M."""
    import torch

    from oracle import gls_ref as O
    from paper_1304_2272_b200 import datagen, distgrid, kernel
    from spmd_inproc import run_spmd

    spec = datagen.BaselineSpec(n=10_000, m=1024, p=4, m_kin=5000, a=0.6)
    XL, y = datagen.covariates_host(spec)

    def body(t):
        ops = distgrid.DeviceOps()
        lay = distgrid.BlockCyclic(spec.n, 512, distgrid.grid_create(t.size), t.rank)
        A, B = distgrid.local_from_spec(spec, lay, ops)
        blocks = (lay.global_rows(lay.row_blocks), lay.global_rows(lay.col_blocks),
                  ops.to_host(A).copy())
        distgrid.dist_potrf_inv(A, B, lay, ops, t)
        S, e = distgrid.assemble_slices(B, lay, ops, t)
        XLy = distgrid.whiten_blockcyclic(B, lay, ops, np.column_stack([XL, y]), t)
        ctx = kernel.prepare_from_inverse(None, spec.n, XL, y, slices=S, expo=e, XLy=XLy)
        G = datagen.genotypes_host(spec.seed, spec.n, spec.m, 0, spec.m)
        beta = np.array([r.beta for r in kernel.gls_solve_block(ctx, kernel.SnpBlock(0, G)).results])
        torch.cuda.synchronize()
        return blocks, beta

    res = run_spmd(4, body)
    Md = datagen.kinship_covariance_device(spec).cpu().numpy()
    n = spec.n
    for (rows, cols, A), _ in res:        # per-rank blocks == the dense device construction
        rv, cv = rows < n, cols < n
        sub, ref = A[np.ix_(rv, cv)], Md[np.ix_(rows[rv], cols[cv])]
        low = rows[rv][:, None] >= cols[cv][None, :]
        assert np.array_equal(sub[low], ref[low])
    octx = O.gls_prepare(Md, XL, y)
    G = datagen.genotypes_host(spec.seed, spec.n, spec.m, 0, spec.m).astype(np.float64)
    ob, _ = O.gls_solve_block(octx, G)
    for _, beta in res:
        rel, mism = O.compare(beta, ob)
        assert mism == 0 and rel <= 1e-9, rel
        assert np.array_equal(beta, res[0][1], equal_nan=True)     # identical on every rank


def _nccl_transport_run_dist(t, paths):
    from paper_1304_2272_b200 import distgrid

    return distgrid.run_dist(t, paths, None)


def test_run_spmd_nccl_transport_processes(gpu, tmp_path, monkeypatch):
    """transport.run_spmd(2, run_dist, ..., transport="nccl") as two processes on this GPU (the
    collectives on gloo: NCCL refuses two ranks on one device) -- the launcher, NcclTransport and
    the engine end to end."""
    from oracle import gls_ref as O
    from paper_1304_2272_b200 import fileio, transport

    monkeypatch.setenv("GG_SPMD_BACKEND", "gloo")
    monkeypatch.setenv("GG_SPMD_TIMEOUT", "600")
    g = golden("seed42")
    paths = write_golden_dataset(tmp_path, g)
    res = transport.run_spmd(2, _nccl_transport_run_dist, paths, transport="nccl")
    assert [r.np_ for r in res] == [2, 2]
    pay = fileio.read_matrix(paths.out, "GWAB")
    rel, mism = O.compare(pay.betas, g["beta"])
    assert mism == 0 and rel <= 1e-9


def test_config4_form_at_n40k_world2_on_one_gpu(gpu):
    """VERDICT r1 item 4's bar: the distributed config-4 form at n = 40,000 on two ranks sharing
    this GPU (tools/dist_n40k.py): per-rank generation, fused Cholesky + inverse with row/column
    broadcasts, slices without a replicated FP64 inverse -- equal to the single-GPU prepare."""
    import re
    import subprocess
    import sys

    from conftest import REPO

    out = subprocess.run([sys.executable, f"{REPO}/tools/dist_n40k.py"], capture_output=True,
                         text=True, timeout=1500)
    assert out.returncode == 0, out.stderr[-3000:]
    rels = [float(x) for x in re.findall(r"max rel ([0-9.e+-]+)", out.stdout)]
    assert len(rels) == 2 and max(rels) <= 1e-9, out.stdout
    assert "status mismatches 0" in out.stdout and "identical results on every rank: True" in \
        out.stdout, out.stdout


def _gather_LLi(A, B, lay, ops, t=None):
    from paper_1304_2272_b200 import distgrid

    return distgrid.gather_matrix(A, lay, ops, t), distgrid.gather_matrix(B, lay, ops, t)


@pytest.mark.parametrize("world", [1, 2, 4])
def test_native_driver_matches_python_driver_bitwise(gpu, world):
    """gg_dist_potrf_f64 (C++ loop, collectives through callbacks into the transport) against the
    Python driver of the same engine: the same kernels in the same order -> bitwise the same
    factor and inverse on every rank (n = 2,100, nb = 512: Ozaki and DMMA updates, ragged
    last block)."""
    from paper_1304_2272_b200 import distgrid
    from spmd_inproc import run_spmd

    n, nb = 2100, 512
    M = make_spd(n, 8)

    def body(t):
        ops = distgrid.DeviceOps()
        lay = distgrid.BlockCyclic(n, nb, distgrid.grid_create(t.size), t.rank)
        out = []
        for native in (True, False):
            A, B = distgrid.local_from_global(M, lay, ops)
            distgrid.dist_potrf_inv(A, B, lay, ops, t, native=native)
            out.append((ops.to_host(A).copy(), ops.to_host(B).copy()))
        return out

    for (An, Bn), (Ap, Bp) in run_spmd(world, body):
        assert np.array_equal(An, Ap) and np.array_equal(Bn, Bp)


def test_native_driver_nccl_world1(gpu):
    """The NCCL backend of gg_dist_potrf_f64 (communicators from a unique id, row / column split,
    ncclBroadcast / ncclAllReduce issued even on groups of one) at world 1 -- bitwise the
    single-rank Python driver.  (NCCL refuses two ranks on one GPU; world > 1 runs the same loop
    over the callback backend above.)"""
    import ctypes as C

    import torch

    from paper_1304_2272_b200 import _capi, distgrid

    n, nb = 1500, 512
    M = make_spd(n, 9)
    ops = distgrid.DeviceOps()
    lay = distgrid.BlockCyclic(n, nb, distgrid.grid_create(1), 0)
    lib = _capi.lib()
    uid = (C.c_ubyte * 128)()
    _capi.check(lib.gg_dist_nccl_unique_id(uid), "gg_dist_nccl_unique_id")
    h = C.c_void_p()
    _capi.check(lib.gg_dist_comms_nccl(0, 1, 1, 1, uid, C.byref(h)), "gg_dist_comms_nccl")
    try:
        A, B = distgrid.local_from_global(M, lay, ops)
        ws = torch.empty(int(lib.gg_dist_potrf_workspace_bytes(n, nb, h)), dtype=torch.uint8,
                         device="cuda")
        info = C.c_int(-1)
        _capi.check(lib.gg_dist_potrf_f64(n, nb, _capi.ptr(A), lay.m_loc, _capi.ptr(B), lay.m_loc,
                                          h, _capi.ptr(ws), ws.numel(), C.byref(info),
                                          _capi.stream_handle()), "gg_dist_potrf_f64")
        A2, B2 = distgrid.local_from_global(M, lay, ops)
        distgrid.dist_potrf_inv(A2, B2, lay, ops, native=False)
        assert torch.equal(A, A2) and torch.equal(B, B2)
    finally:
        lib.gg_dist_comms_free(h)


@pytest.mark.parametrize("world", [2, 4])
def test_native_driver_not_pd_global_pivot_every_rank(gpu, world):
    from paper_1304_2272_b200 import distgrid
    from paper_1304_2272_b200.errors import NotPositiveDefinite
    from spmd_inproc import run_spmd

    n = 1300
    M = make_spd(n, 10)
    M[777, 777] = -5.0

    def body(t):
        ops = distgrid.DeviceOps()
        lay = distgrid.BlockCyclic(n, 256, distgrid.grid_create(t.size), t.rank)
        A, B = distgrid.local_from_global(M, lay, ops)
        try:
            distgrid.dist_potrf_inv(A, B, lay, ops, t)
        except NotPositiveDefinite as e:
            return e.pivot_index
        return None

    assert run_spmd(world, body) == [777] * world


@pytest.mark.parametrize("world", [1, 2, 4])
def test_native_trsolve_matches_python_driver_bitwise(gpu, world):
    """gg_dist_trsm_f64 (the distributed blocked substitution in C++) against the Python driver:
    bitwise the same replicated solution on every rank, and dtrsm-accurate."""
    from scipy.linalg import cholesky, solve_triangular

    from paper_1304_2272_b200 import distgrid
    from spmd_inproc import run_spmd

    n, nb = 1700, 256
    M = make_spd(n, 12)
    R = np.random.default_rng(3).standard_normal((n, 7))

    def body(t):
        ops = distgrid.DeviceOps()
        lay = distgrid.BlockCyclic(n, nb, distgrid.grid_create(t.size), t.rank)
        A, B = distgrid.local_from_global(M, lay, ops)
        distgrid.dist_potrf_inv(A, B, lay, ops, t)
        Xn = distgrid.dist_trsolve_bc(A, lay, ops, R, t, native=True)
        Xp = distgrid.dist_trsolve_bc(A, lay, ops, R, t, native=False)
        return Xn, Xp

    Lr = cholesky(M, lower=True)
    Xr = solve_triangular(Lr, R, lower=True)
    for Xn, Xp in run_spmd(world, body):
        assert np.array_equal(Xn, Xp)
        assert np.max(np.abs(Xn - Xr)) <= 1e-12 * np.max(np.abs(Xr))
