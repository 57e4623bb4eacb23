"""CPU: the distributed (config-4) engine's communication logic over gloo at world sizes 1, 2, 4
(grids 1x1, 1x2, 2x2): block-cyclic layout maps, the fused Cholesky + inverse, the not-PD pivot,
and the all-reduce assembly of the packed inverse.  Local numerics come from tests/dist_cpu_ops.py;
the same code path runs with the sm_100a kernels in tests/test_gpu_distgrid.py."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import REPO, make_spd


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, nb, bad_pivot, q):
    import sys

    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, n, nb, bad_pivot, q, dist)
    except Exception as e:     # report instead of leaving the parent waiting on the queue
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def _body(rank, world, n, nb, bad_pivot, q, dist):
    from dist_cpu_ops import CpuOps
    from paper_1304_2272_b200 import distgrid
    from paper_1304_2272_b200.errors import NotPositiveDefinite

    M = make_spd(n, 7)
    if bad_pivot is not None:
        M[bad_pivot, bad_pivot] = -5.0
    ops = CpuOps()
    grid = distgrid.grid_create(world)
    lay = distgrid.BlockCyclic(n, nb, grid, rank)
    A, B = distgrid.local_from_global(M, lay, ops)
    try:
        distgrid.dist_potrf_inv(A, B, lay, ops, dist)
    except NotPositiveDefinite as e:
        q.put((rank, "notpd", e.pivot_index))
        return
    L = distgrid.gather_matrix(A, lay, ops, dist)
    Li = distgrid.gather_matrix(B, lay, ops, dist)
    P = distgrid.assemble_packed_inverse(B, lay, ops, dist).numpy()
    S, e = distgrid.assemble_slices(B, lay, ops, dist)
    RHS = np.random.default_rng(3).standard_normal((n, 3))
    W = distgrid.whiten_blockcyclic(B, lay, ops, RHS, dist)
    q.put((rank, "ok", (L, Li, P, S.numpy(), e.numpy(), ops.to_host(W), RHS)))


def _run(world, n, nb, bad_pivot=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, nb, bad_pivot, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    errs = [o for o in out if o[1] == "error"]
    assert not errs, errs
    for p in procs:
        assert p.exitcode == 0
    return sorted(out, key=lambda x: x[0])


def test_grid_and_layout_maps():
    from paper_1304_2272_b200 import distgrid

    assert [(g.r, g.c) for g in map(distgrid.grid_create, (1, 2, 4, 6, 8))] == \
        [(1, 1), (1, 2), (2, 2), (2, 3), (2, 4)]
    grid = distgrid.grid_create(8)
    seen = {}
    for rank in range(8):
        lay = distgrid.BlockCyclic(1000, 64, grid, rank)
        for I in lay.row_blocks:
            for J in lay.col_blocks:
                assert lay.owner(I, J) == rank
                seen[(I, J)] = rank
        # owned block-rows after K start at rows_through(K)
        for K in range(lay.nblk):
            assert lay.rows_through(K) == 64 * sum(1 for I in lay.row_blocks if I <= K)
    assert len(seen) == lay.nblk ** 2


@pytest.mark.parametrize("world", [1, 2, 4])
def test_dist_cholesky_inverse_and_packed_assembly(world):
    from dist_cpu_ops import pack_lower_dense
    from scipy.linalg import cholesky, solve_triangular

    n, nb = 700, 128
    out = _run(world, n, nb)
    M = make_spd(n, 7)
    Lr = cholesky(M, lower=True)
    Lir = solve_triangular(Lr, np.eye(n), lower=True)
    Pr = pack_lower_dense(Lir, n)
    from dist_cpu_ops import row_exponents_dense, slice_meta_dense, slices_dense

    np_ = -(-n // 128) * 128
    for rank, kind, (L, Li, P, S, e, W, RHS) in out:
        assert kind == "ok"
        assert np.max(np.abs(L - Lr)) <= 1e-13 * np.max(np.abs(Lr))
        assert np.all(np.triu(L, 1) == 0)
        assert np.max(np.abs(Li - Lir)) <= 1e-12 * np.max(np.abs(Lir))
        assert np.max(np.abs(P - Pr)) <= 1e-12 * np.max(np.abs(Pr))
        assert np.array_equal(P, out[0][2][2])          # identical replica on every rank
        # int8 slices: MAX-reduced exponents, SUM-reduced per-rank slices and heads equal what
        # one GPU would cut from the gathered inverse, identical on every rank
        Lg = np.eye(np_)
        Lg[:n, :n] = np.tril(Li)
        meta = slice_meta_dense(row_exponents_dense(Lg))
        Sx = slices_dense(lambda i, kend: Lg[i, :kend], meta, np_)
        assert np.array_equal(e, meta)
        assert np.array_equal(S, Sx)
        assert np.array_equal(S, out[0][2][3])
        # whitening from the block-cyclic inverse
        Wr = Lir @ RHS
        assert np.max(np.abs(W[:n] - Wr)) <= 1e-12 * np.max(np.abs(Wr)) and not W[n:].any()


def test_dist_not_positive_definite_global_pivot():
    out = _run(2, 500, 128, bad_pivot=300)
    assert all(kind == "notpd" and piv == 300 for _, kind, piv in out)
