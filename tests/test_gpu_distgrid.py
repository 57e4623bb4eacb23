"""GPU: the distributed (config-4) engine with the sm_100a kernels on one rank (grid 1x1; the
multi-rank communication logic is covered over gloo in tests/test_distgrid_gloo.py)."""

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
    s = distgrid.run_dist(paths, distgrid.DistConfig(m_blk=257, nb=128, fp64_inverse=fp64_inverse))
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
