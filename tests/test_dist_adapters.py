"""CPU: the reference-signature distributed entry points (distgrid.dist_cholesky, dist_trsolve,
the element-cyclic <-> block-cyclic redistribution, the row/column sub-communicators of
comm.TransportComm) driven by a reference-contract transport (tests/spmd_inproc.py), with the
numpy ops of tests/dist_cpu_ops.py; and the per-rank generation of the config-4 covariance.
The cases mirror the reference's tests/test_distgrid.py:140-238."""

import numpy as np
import pytest

from conftest import make_spd
from dist_cpu_ops import CpuOps
from spmd_inproc import EC, gather_ec, run_spmd


def _grid(np_):
    from paper_1304_2272_b200 import distgrid

    return distgrid.grid_create(np_)


@pytest.mark.parametrize("np_", [2, 4, 6])
@pytest.mark.parametrize("n", [16, 96, 200, 300])
def test_dist_cholesky_matches_replicated(np_, n):
    from scipy.linalg import cholesky

    from paper_1304_2272_b200 import distgrid

    M = make_spd(n, 42)
    Lref = cholesky(M, lower=True)

    def body(t):
        D = EC.of(M, _grid(t.size), t.rank)
        Ld = distgrid.dist_cholesky(D, t, nb=8, ops=CpuOps())
        assert isinstance(Ld, EC) and Ld.local.shape == D.local.shape
        return gather_ec(Ld, t)

    for L in run_spmd(np_, body):
        assert np.max(np.abs(L - Lref)) <= 1e-12 * np.max(np.abs(M))
        assert np.all(np.triu(L, 1) == 0)


def test_dist_cholesky_identity_and_global_pivot():
    from paper_1304_2272_b200 import distgrid
    from paper_1304_2272_b200.errors import NotPositiveDefinite

    def ident(t):
        return gather_ec(distgrid.dist_cholesky(EC.of(np.eye(16), _grid(4), t.rank), t, nb=4,
                                                ops=CpuOps()), t)

    assert all(np.array_equal(L, np.eye(16)) for L in run_spmd(4, ident))
    M = np.eye(300)
    M[209, 209] = -1.0

    def bad(t):
        with pytest.raises(NotPositiveDefinite) as e:
            distgrid.dist_cholesky(EC.of(M, _grid(6), t.rank), t, ops=CpuOps())
        return e.value.pivot_index

    assert run_spmd(6, bad) == [209] * 6


@pytest.mark.parametrize("np_", [2, 4])
def test_dist_trsolve_identity_and_residual(np_):
    from scipy.linalg import solve_triangular

    from paper_1304_2272_b200 import distgrid

    rng = np.random.default_rng(5)
    B0 = rng.standard_normal((12, 5))

    def ident(t):
        g = _grid(t.size)
        X = distgrid.dist_trsolve(EC.of(np.eye(12), g, t.rank), EC.of(B0, g, t.rank), t, nb=4,
                                  ops=CpuOps())
        return gather_ec(X, t)

    assert all(np.allclose(X, B0) for X in run_spmd(np_, ident))
    n = 300                                   # three 128-blocks: the blocked substitution runs
    L = np.tril(rng.standard_normal((n, n))) + 10 * np.eye(n)
    B = rng.standard_normal((n, 64))

    def solve(t):
        g = _grid(t.size)
        return gather_ec(distgrid.dist_trsolve(EC.of(L, g, t.rank), EC.of(B, g, t.rank), t,
                                               nb=16, ops=CpuOps()), t)

    Xref = solve_triangular(L, B, lower=True)
    for X in run_spmd(np_, solve):
        assert np.max(np.abs(L @ X - B)) / np.max(np.abs(B)) <= 1e-12
        assert np.max(np.abs(X - Xref)) <= 1e-10 * np.max(np.abs(Xref))


@pytest.mark.parametrize("np_", [3, 6, 8])
def test_block_cyclic_factor_with_sub_communicators_on_transport(np_):
    """dist_potrf_inv's row / column broadcasts over TransportComm sub-groups (point-to-point
    messages of a reference-contract transport) on 1x3, 2x3 and 2x4 grids, with ranks that own
    no block at all (n = 300, nb = 128: 3 x 3 blocks)."""
    from scipy.linalg import cholesky, solve_triangular

    from paper_1304_2272_b200 import distgrid

    n, nb = 300, 128
    M = make_spd(n, 11)

    def body(t):
        ops = CpuOps()
        lay = distgrid.BlockCyclic(n, nb, _grid(t.size), t.rank)
        A, B = distgrid.local_from_global(M, lay, ops)
        distgrid.dist_potrf_inv(A, B, lay, ops, t)
        return (distgrid.gather_matrix(A, lay, ops, t), distgrid.gather_matrix(B, lay, ops, t))

    Lr = cholesky(M, lower=True)
    Lir = solve_triangular(Lr, np.eye(n), lower=True)
    for L, Li in run_spmd(np_, body):
        assert np.max(np.abs(L - Lr)) <= 1e-13 * np.max(np.abs(Lr))
        assert np.max(np.abs(Li - Lir)) <= 1e-12 * np.max(np.abs(Lir))


def test_element_cyclic_block_cyclic_round_trip():
    from paper_1304_2272_b200 import distgrid

    A = np.random.default_rng(3).standard_normal((301, 301))

    def body(t):
        g = _grid(t.size)
        ops = CpuOps()
        comm = distgrid.as_comm(t)
        lay = distgrid.BlockCyclic(301, 128, g, t.rank)
        D = EC.of(A, g, t.rank)
        Ab = distgrid.ec_to_bc(D.local, 301, 301, g, t.rank, lay, comm, ops, pad_identity=False)
        full = distgrid.gather_matrix(Ab, lay, ops, t)
        back = distgrid.bc_to_ec(Ab, 301, 301, g, t.rank, lay, comm, ops)
        return full, np.array_equal(back, D.local)

    for full, ok in run_spmd(6, body):
        assert np.array_equal(full, A) and ok


def test_config4_blocks_generated_per_rank_match_the_host_construction():
    """local_from_spec: each rank's M_IJ from the counter-based kinship markers equals the
    corresponding blocks of datagen's dense construction (no n x n array on any rank)."""
    from paper_1304_2272_b200 import datagen, distgrid

    spec = datagen.BaselineSpec(n=300, m=10, p=4, m_kin=200, a=0.6)
    Mh = datagen.kinship_covariance_host(spec)

    def body(t):
        ops = CpuOps()
        lay = distgrid.BlockCyclic(spec.n, 128, _grid(t.size), t.rank)
        A, _ = distgrid.local_from_spec(spec, lay, ops)
        return distgrid.gather_matrix(A, lay, ops, t)

    for M in run_spmd(4, body):
        assert np.max(np.abs(np.tril(M) - np.tril(Mh))) <= 1e-14 * np.max(np.abs(Mh))
