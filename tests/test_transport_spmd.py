"""CPU: transport.run_spmd(..., transport="nccl") -- the reference's SPMD launcher contract
(transport.py:267-327) on spawned processes over torch.distributed (gloo here via
GG_SPMD_BACKEND; NCCL on the B200 box): the Transport byte API, results in rank order, failures
re-raised, and the fused distributed factorisation driven through ``t`` (its TorchComm with
row / column sub-communicators)."""

import os

import numpy as np
import pytest

from conftest import REPO, make_spd


@pytest.fixture(autouse=True)
def _gloo(monkeypatch):
    monkeypatch.setenv("GG_SPMD_BACKEND", "gloo")
    monkeypatch.setenv("GG_SPMD_TIMEOUT", "300")


def _api_body(t):
    import torch

    out = {}
    if t.rank == 0:
        t.send(1, b"hello")
    if t.rank == 1:
        out["p2p"] = t.recv(0)
    out["bcast"] = t.broadcast(2, b"root2" if t.rank == 2 else b"")
    out["gather"] = t.allgather(bytes([t.rank]))
    out["a2a"] = t.alltoall([bytes([t.rank, d]) for d in range(t.size)])
    out["obj"] = t.allgather_obj({"r": t.rank})
    x = torch.full((3,), float(t.rank + 1), dtype=torch.float64)
    t.comm.all_reduce(x)
    out["sum"] = x.tolist()
    t.barrier()
    return out


def _factor_body(t, n, nb):
    import sys

    sys.path.insert(0, os.path.join(REPO, "tests"))
    from dist_cpu_ops import CpuOps
    from paper_1304_2272_b200 import distgrid

    M = make_spd(n, 5)
    ops = CpuOps()
    lay = distgrid.BlockCyclic(n, nb, distgrid.grid_create(t.size), t.rank)
    A, B = distgrid.local_from_global(M, lay, ops)
    distgrid.dist_potrf_inv(A, B, lay, ops, t)
    return distgrid.gather_matrix(B, lay, ops, t)


def _fail_body(t):
    if t.rank == 1:
        raise ValueError("rank 1 failed")
    return t.rank


def test_transport_contract_and_rank_order():
    from paper_1304_2272_b200 import transport

    res = transport.run_spmd(4, _api_body, transport="nccl")
    assert res[1]["p2p"] == b"hello"
    for r, o in enumerate(res):
        assert o["bcast"] == b"root2"
        assert o["gather"] == [bytes([s]) for s in range(4)]
        assert o["a2a"] == [bytes([s, r]) for s in range(4)]
        assert o["obj"] == [{"r": s} for s in range(4)]
        assert o["sum"] == [10.0] * 3


def test_factorisation_through_the_transport():
    from scipy.linalg import cholesky, solve_triangular

    from paper_1304_2272_b200 import transport

    n, nb = 600, 128
    res = transport.run_spmd(6, _factor_body, n, nb, transport="nccl")
    Lir = solve_triangular(cholesky(make_spd(n, 5), lower=True), np.eye(n), lower=True)
    for Li in res:
        assert np.max(np.abs(Li - Lir)) <= 1e-12 * np.max(np.abs(Lir))


def test_failure_is_reraised_and_unknown_transport_rejected():
    from paper_1304_2272_b200 import transport

    with pytest.raises(ValueError, match="rank 1 failed"):
        transport.run_spmd(2, _fail_body, transport="nccl")
    with pytest.raises(ValueError):
        transport.run_spmd(2, _fail_body, transport="carrier-pigeon")
