"""SNP-sharded multi-GPU engine (BASELINE configs 2-3).

One process per GPU (torch.distributed; NCCL on the B200 box, gloo in the CPU tests).  Every b_i
depends only on its own marker column, so the markers shard with NO data-path
collective:
  * L is replicated by redundant factorisation on every rank — the kernels are deterministic,
    so every GPU holds a bitwise-identical L (no broadcast of n x n needed);
  * the 8192-marker blocks of the plan are dealt round-robin (balanced; the partial last block
    lands on one rank);
  * each rank streams its blocks through its own double-buffered engine and writes its GWAB
    records at their global offsets (the reference's ranks do the same, distgrid.py:390-446);
  * the only synchronisation is a host barrier around file creation and completion.
The same ``stream_shard`` runs the sweep of the distributed engine (distgrid.run_dist), whose
ranks share a replicated packed inverse.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import fileio, kernel
from .comm import as_comm
from .pipeline import RunSummary, _load_prepare, block_plan, stream_file_blocks


@dataclass
class ShardConfig:
    m_blk: int = 8192
    emit_s_inv: bool = False


@dataclass
class ShardStats:
    m: int
    m_blk: int
    t_compute: float
    t_io_wait: float
    t_loop: float
    t_device: float
    bytes_read: int
    bytes_written: int
    snps_per_s: float


def shard_blocks(m, m_blk, rank, world):
    """Round-robin assignment of the plan's blocks; the union over ranks is the full plan."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return [b for i, b in enumerate(block_plan(m, m_blk).blocks) if i % world == rank]


def _dist():
    try:
        import torch.distributed as dist
    except ImportError:   # pragma: no cover
        return None
    return dist if dist.is_available() and dist.is_initialized() else None


def _barrier(dist):
    if dist is not None:
        dist.barrier()


def stream_shard(paths, ctx, cfg=None, solve_fn=None, comm=None):
    """Stream this rank's share of the marker blocks of ``paths.geno`` against ``ctx`` and write
    their records at global offsets of ``paths.out`` (rank 0 creates the file).  Collective over
    ``comm`` (default: the initialised torch.distributed group; any communicator of comm.py, e.g.
    a reference transport); returns job-level ShardStats on every rank.

    solve_fn(ctx, data, first) -> kernel.ResultArrays replaces the device stream in the CPU
    tests of the sharding logic."""
    cfg = cfg or ShardConfig()
    dist = as_comm(comm) if comm is not None else as_comm(_dist())
    rank = dist.rank if dist else 0
    world = dist.size if dist else 1
    _, n, m = fileio.total_genotype_bytes(paths.geno)
    m_blk = min(cfg.m_blk, m)
    p = ctx.p
    flags = 1 if cfg.emit_s_inv else 0
    if rank == 0:
        writer = fileio.BlockWriter(paths.out, m, p, flags, create=True)
    _barrier(dist)
    if rank != 0:
        writer = fileio.BlockWriter(paths.out, m, p, flags, create=False)
    mine = shard_blocks(m, m_blk, rank, world)
    reader = fileio.BlockReader(paths.geno)
    t_dev = 0.0
    try:
        if solve_fn is None:
            if mine:
                engine, t_io, _, t_loop = stream_file_blocks(ctx, reader, writer, mine, m_blk,
                                                             cfg.emit_s_inv)
                t_dev = engine.device_ms / 1e3
            else:
                t_io, t_loop = 0.0, 0.0
        else:
            t0 = time.perf_counter()
            t_io = 0.0
            buf = np.empty((n, m_blk), dtype=reader.dtype, order="F")
            for first, cnt in mine:
                t1 = time.perf_counter()
                blk = reader.wait(reader.start(first, cnt, buf))
                t_io += time.perf_counter() - t1
                arr = solve_fn(ctx, blk.data, first)
                writer.wait(writer.start(kernel.ResultBlock.from_arrays(arr)))
            t_loop = time.perf_counter() - t0
    finally:
        reader.close()
        writer.close()
    _barrier(dist)
    stats = dict(bytes_read=reader.bytes_read, bytes_written=writer.bytes_written,
                 t_loop=t_loop, t_dev=t_dev)
    allst = dist.allgather_obj(stats) if dist is not None else [stats]
    t_max = max(s["t_loop"] for s in allst)
    return ShardStats(m=m, m_blk=m_blk, t_compute=max(t_loop - t_io, 0.0), t_io_wait=t_io,
                      t_loop=t_loop, t_device=max(s["t_dev"] for s in allst),
                      bytes_read=sum(s["bytes_read"] for s in allst),
                      bytes_written=sum(s["bytes_written"] for s in allst),
                      snps_per_s=m / t_max if t_max > 0 else 0.0)


def run_sharded(paths, cfg=None, prepare_fn=None, solve_fn=None):
    """SPMD body: call on every rank.  Redundant gls_prepare on the rank's GPU, then
    ``stream_shard``.  Returns a RunSummary carrying the job totals.

    prepare_fn(paths) -> ctx and solve_fn are injection points for the CPU tests."""
    cfg = cfg or ShardConfig()
    dist = _dist()
    world = dist.get_world_size() if dist else 1
    t_start = time.perf_counter()
    _, n, m = fileio.total_genotype_bytes(paths.geno)
    if prepare_fn is None:
        ctx, t_prep, _ = _load_prepare(paths)
    else:
        t0 = time.perf_counter()
        ctx = prepare_fn(paths)
        t_prep = time.perf_counter() - t0
    s = stream_shard(paths, ctx, cfg, solve_fn=solve_fn)
    return RunSummary(
        mode="sharded", n=n, m=m, p=ctx.p, m_blk=s.m_blk, np_=world, threads=1,
        t_prepare=t_prep, t_compute=s.t_compute, t_io_wait=s.t_io_wait,
        t_total=time.perf_counter() - t_start, bytes_read=s.bytes_read,
        bytes_written=s.bytes_written, buffer_regions=2, gpus=world, t_device=s.t_device,
        snps_per_s=s.snps_per_s)
