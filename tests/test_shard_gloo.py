"""CPU: the multi-GPU sharding logic at world_size 2 over gloo (file creation protocol, round-robin
block ownership, offset-addressed writes, totals).  The per-block arithmetic is injected from the
CPU oracle here; the GPU engine behind the same code path is covered by the gpu tests."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import REPO, golden, write_golden_dataset


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _prepare(paths):
    from oracle import gls_ref as O
    from paper_1304_2272_b200 import fileio

    ctx = O.gls_prepare(fileio.read_matrix(paths.cov, "GWAM"),
                        fileio.read_matrix(paths.covariates, "GWAC"),
                        fileio.read_matrix(paths.pheno, "GWAY"))
    return ctx


def _solve(ctx, data, first):
    from oracle import gls_ref as O
    from paper_1304_2272_b200 import kernel

    beta, ok, packed = O.gls_solve_block(ctx, np.asarray(data, dtype=float), emit_s_inv=True)
    status = np.where(ok, -1, 0).astype(np.int32)
    return kernel.ResultArrays(first_index=first, beta=beta, status=status, sinv=packed)


def _worker(rank, world, port, paths, m_blk, out_q):
    import sys

    sys.path.insert(0, REPO)
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1304_2272_b200 import shard

        s = shard.run_sharded(paths, shard.ShardConfig(m_blk=m_blk, emit_s_inv=True),
                              prepare_fn=_prepare, solve_fn=_solve)
        out_q.put((rank, s.np_, s.m, s.bytes_written))
    finally:
        dist.destroy_process_group()


def test_shard_blocks_partition():
    from paper_1304_2272_b200.shard import shard_blocks

    for m, m_blk, world in ((200_000, 8192, 8), (17, 3, 2), (5, 8, 4)):
        allb = sorted(b for r in range(world) for b in shard_blocks(m, m_blk, r, world))
        assert sum(c for _, c in allb) == m
        assert [f for f, _ in allb] == list(range(0, m, m_blk))
        sizes = [sum(c for _, c in shard_blocks(m, m_blk, r, world)) for r in range(world)]
        assert max(sizes) - min(sizes) <= m_blk


@pytest.mark.parametrize("world", [2])
def test_sharded_run_gloo(tmp_path, world):
    from oracle import gls_ref as O
    from paper_1304_2272_b200 import fileio

    g = golden("seed42")
    paths = write_golden_dataset(tmp_path, g)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, paths, 64, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got = sorted(q.get(timeout=10) for _ in range(world))
    assert [r for r, *_ in got] == list(range(world))
    assert all(npr == world and m == 500 for _, npr, m, _ in got)
    assert got[0][3] == 500 * fileio.record_size(4, 1)      # totals over ranks
    pay = fileio.read_matrix(paths.out, "GWAB")
    rel, mism = O.compare(pay.betas, g["beta"])
    assert mism == 0 and rel <= 1e-12
    ok = ~g["status"].astype(bool)
    assert np.max(np.abs(pay.sinv[ok] - g["sinv"][ok])) <= 1e-12 * np.max(np.abs(g["sinv"]))
