"""Streaming drivers on the B200: the paper's double-buffered out-of-core loop (PAPER.md:259-295,
reference pipeline.py:1-238) recast for a GPU.

    load_start(first)                          host thread: file -> pinned region
    for each block:
        load_wait(current); load_start(next)   (region reuse gated by its H2D event)
        H2D current on the copy stream         (pitched copy into the np-padded device block)
        whiten + solve on the compute stream   (DMMA TRSM + fused epilogue, one launch each)
        D2H results into the region's pinned result buffer
        collect previous block; store_start(previous records)
    store_wait(last)

Two regions alternate; a region under in-flight transfer is never touched (rendezvous through
CUDA events on the device side and tickets on the host side).  Per-column arithmetic does not
depend on the block size, so incore, ooc at any m_blk, and the sharded engine agree bitwise.
"""

from __future__ import annotations

import collections
import os
import time
from dataclasses import dataclass, field, fields

import numpy as np

from . import _capi, fileio, kernel
from ._capi import check, ptr
from ._device import BlockWorkspace, alloc_cols
from .errors import ConfigError

DEFAULT_M_BLK = 5000          # pipeline.py:30
GPU_M_BLK = 8192              # BASELINE configs 1-3
MEM_BUDGET_ENV = "GWAS_GLS_MEM_BUDGET_BYTES"


@dataclass
class BlockPlan:
    m: int
    m_blk: int
    blocks: list


def block_plan(m, m_blk):
    """Contiguous disjoint blocks of at most m_blk columns covering [0, m) (pipeline.py:41-46)."""
    if m < 1 or m_blk < 1:
        raise ConfigError("m and m_blk must be >= 1")
    return BlockPlan(m=m, m_blk=m_blk,
                     blocks=[(f, min(m_blk, m - f)) for f in range(0, m, m_blk)])


@dataclass
class RunSummary:
    """Single-record run report; serialises to one key=value line (pipeline.py:49-99).
    GPU runs add ``gpus``, ``t_device`` (device seconds of the stream) and ``snps_per_s``."""

    mode: str = ""
    n: int = 0
    m: int = 0
    p: int = 0
    m_blk: int = 0
    np_: int = 1
    threads: int = 1
    t_prepare: float = 0.0
    t_compute: float = 0.0
    t_io_wait: float = 0.0
    t_redistribute: float = 0.0
    t_total: float = 0.0
    bytes_read: int = 0
    bytes_written: int = 0
    peak_resident_est: int = 0
    buffer_regions: int = 0
    combine_bytes: int = 0
    localpart_bytes: int = 0
    seed: int = -1
    gpus: int = 1
    t_device: float = 0.0
    snps_per_s: float = 0.0
    block_cpu_times: list = field(default_factory=list)   # the driving thread's CPU seconds per
                                                          # block (time.thread_time: the I/O
                                                          # agents' and the driver's spin threads
                                                          # excluded -- reference pipeline.py:206)

    def to_record(self):
        parts = []
        for f in fields(self):
            v = getattr(self, f.name)
            if isinstance(v, list):
                continue
            parts.append(f"{f.name}={v:.6f}" if isinstance(v, float) else f"{f.name}={v}")
        return " ".join(parts)

    @classmethod
    def from_record(cls, line):
        typed = {f.name: f.type for f in fields(cls)}
        kw = {}
        for tok in line.split():
            k, v = tok.split("=", 1)
            t = typed.get(k)
            if t is None:
                continue
            kw[k] = v if t in (str, "str") else float(v) if t in (float, "float") else int(v)
        return cls(**kw)


@dataclass
class SolvePaths:
    cov: str
    covariates: str
    pheno: str
    geno: str
    out: str


@dataclass
class SolveConfig:
    m_blk: int = DEFAULT_M_BLK
    threads: int = 1
    emit_s_inv: bool = False
    mem_budget_bytes: int | None = None

    def budget(self):
        if self.mem_budget_bytes is not None:
            return self.mem_budget_bytes
        env = os.environ.get(MEM_BUDGET_ENV)
        return int(env) if env else None


def _read_cov_device(path):
    """GWAM -> device: parallel preads into pinned memory, one H2D copy, and the reader's
    symmetry / finiteness checks (fileio.py:153-157) done on the device."""
    import torch

    from .errors import AsymmetricCovariance

    n = fileio.read_dims(path, "GWAM")[0]
    host = torch.empty(8 * n * n, dtype=torch.uint8).pin_memory()
    got = fileio.pread_into(path, fileio.header_size("GWAM"), memoryview(host.numpy()))
    if got < 8 * n * n:
        raise fileio.TruncatedFile(f"expected {8 * n * n} payload bytes, got {got}")
    Md = host.view(torch.float64).reshape(n, n).to(_capi.device(), non_blocking=True)
    if not bool(torch.equal(Md, Md.T)):
        raise AsymmetricCovariance("covariance file is not exactly symmetric")
    if not bool(torch.isfinite(Md).all()):
        raise AsymmetricCovariance("covariance file has non-finite entries")
    return Md


def _load_prepare(paths):
    t0 = time.perf_counter()
    Md = _read_cov_device(paths.cov)
    XL = fileio.read_matrix(paths.covariates, "GWAC")
    y = fileio.read_matrix(paths.pheno, "GWAY")
    ctx = kernel.gls_prepare(Md, XL, y)
    return ctx, time.perf_counter() - t0, Md.numel() * 8


# ---------------------------------------------------------------------------------------------
# the device stream
# ---------------------------------------------------------------------------------------------

class StreamEngine:
    """Two-region host->device genotype stream with asynchronous result return.

    ``submit(slot, host_block, first, cnt)`` enqueues H2D (copy stream) -> TRSM + epilogue
    (compute stream) -> D2H of the results into pinned buffers and returns a ticket;
    ``collect(ticket)`` waits for that block and returns its ResultArrays.  ``slot`` names the
    caller's host input region (REGIONS = 2, the reference's double buffer): ``wait_h2d(slot)``
    returns once the region's last H2D is done, so it may be refilled.  On the device the
    blocks rotate through DEV_REGIONS input/workspace/result regions, so the H2D of block i+1
    is ordered only after the compute of block i+1-DEV_REGIONS -- the copy engine runs back to
    back instead of waiting for the host to collect block i-1.  host_block is an n x >= cnt
    Fortran-ordered (ideally pinned) array of float64 or int8."""

    REGIONS = 2
    DEV_REGIONS = 3

    def __init__(self, ctx, m_blk, int8=False, emit_s_inv=False):
        import torch

        self.torch = torch
        self.d = ctx._dev
        if self.d is None or (self.d.LinvP is None and self.d.slices is None):
            raise ConfigError("StreamEngine needs a device-prepared context")
        self.m_blk = int(m_blk)
        self.int8 = bool(int8)
        self.emit_s_inv = bool(emit_s_inv)
        d = self.d
        # int8 dosage rows pitched to 16 bytes (TMA operand of the tensor-core TRSM)
        self.ld_in = (-(-d.n // 16) * 16) if self.int8 else d.np_
        dt = torch.int8 if self.int8 else torch.float64
        R = self.DEV_REGIONS
        self.ws = [BlockWorkspace(d, self.m_blk, emit_s_inv, self.int8) for _ in range(R)]
        self.dev_in = [alloc_cols(self.m_blk, self.ld_in, dtype=dt) for _ in range(R)]
        p = d.p
        self.h_beta = [torch.empty((self.m_blk, p), dtype=torch.float64).pin_memory()
                       for _ in range(R)]
        self.h_status = [torch.empty((self.m_blk,), dtype=torch.int32).pin_memory()
                         for _ in range(R)]
        self.h_sinv = [torch.empty((self.m_blk, p * (p + 1) // 2), dtype=torch.float64)
                       .pin_memory() if emit_s_inv else None for _ in range(R)]
        self.copy_stream = torch.cuda.Stream()
        self.compute_stream = torch.cuda.Stream()
        # the regions above were allocated (and zero-filled: the padding rows the TRSM reads)
        # on the current stream; order both engine streams after that work
        self.copy_stream.wait_stream(torch.cuda.current_stream())
        self.compute_stream.wait_stream(torch.cuda.current_stream())
        self.h2d_start = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
        self.h2d_done = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
        self.done = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
        self.start_ev = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
        self.meta = [None] * R
        self.busy = [False] * R
        self.host_ev = {}                  # host region -> event after its last H2D
        self._h2d_open = [False] * R
        self._next = 0
        self.device_ms = 0.0
        self.h2d_ms = 0.0
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def wait_h2d(self, slot):
        """Host rendezvous: the host input region ``slot`` may be refilled after this."""
        ev = self.host_ev.get(slot)
        if ev is not None:
            ev.synchronize()

    def begin(self, first, cnt, global_indices=None):
        """Open the next device region for a block of ``cnt`` markers; returns its ticket."""
        r = self._next % self.DEV_REGIONS
        if self.busy[r]:
            raise ConfigError(f"device region {r} still in flight (collect it first)")
        if not 0 < cnt <= self.m_blk:
            raise ConfigError(f"block of {cnt} markers does not fit m_blk={self.m_blk}")
        self._next += 1
        self.busy[r] = True
        self.meta[r] = (first, cnt, global_indices)
        self._h2d_open[r] = False
        return r

    def h2d(self, r, host_part, col0, cols, slot):
        """Copy host columns (n x >= cols, Fortran-ordered, ideally pinned) into columns
        col0 .. col0+cols of region r on the copy stream; ``slot`` names the host region the
        columns came from (see wait_h2d)."""
        torch = self.torch
        d = self.d
        item = 1 if self.int8 else 8
        hb = host_part
        if hb.shape[0] != d.n or hb.shape[1] < cols or not hb.flags.f_contiguous:
            raise ConfigError("host block must be n x >= cnt and Fortran-ordered")
        if hb.dtype != (np.int8 if self.int8 else np.float64):
            raise ConfigError(f"host block dtype {hb.dtype} does not match the stream")
        if col0 < 0 or col0 + cols > self.meta[r][1]:
            raise ConfigError("host part outside the block")
        dst = self.dev_in[r]
        with torch.cuda.stream(self.copy_stream):
            if not self._h2d_open[r]:
                # the device input region is free once the previous compute on it is done
                self.copy_stream.wait_event(self.done[r])
                self.h2d_start[r].record(self.copy_stream)
                self._h2d_open[r] = True
            rc = _capi.lib().gg_memcpy2d_async(
                _capi.C.c_void_p(dst.data_ptr() + col0 * self.ld_in * item), self.ld_in * item,
                _capi.C.c_void_p(hb.ctypes.data), d.n * item, d.n * item, int(cols), 1,
                _capi.C.c_void_p(self.copy_stream.cuda_stream))
            check(rc, "gg_memcpy2d_async")
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        self.host_ev[slot] = ev
        self.h2d_bytes += d.n * item * cols

    def launch(self, r):
        """All of region r's columns are queued: TRSM + epilogue + D2H of the results."""
        torch = self.torch
        d = self.d
        first, cnt, gi = self.meta[r]
        dst = self.dev_in[r]
        self.h2d_done[r].record(self.copy_stream)
        ws = self.ws[r]
        with torch.cuda.stream(self.compute_stream):
            self.compute_stream.wait_event(self.h2d_done[r])
            self.start_ev[r].record(self.compute_stream)
            s = _capi.C.c_void_p(self.compute_stream.cuda_stream)
            if self.int8:
                ws.run(cnt, G8=dst, ldg=self.ld_in, stream=s)
            else:
                ws.run(cnt, X64=dst, ldx=self.ld_in, stream=s)
            self.h_beta[r][:cnt].copy_(ws.beta[:cnt], non_blocking=True)
            self.h_status[r][:cnt].copy_(ws.status[:cnt], non_blocking=True)
            if self.emit_s_inv:
                self.h_sinv[r][:cnt].copy_(ws.sinv[:cnt], non_blocking=True)
            self.done[r].record(self.compute_stream)
        self.d2h_bytes += cnt * (8 * d.p + 4 + (8 * d.p * (d.p + 1) // 2 if self.emit_s_inv else 0))

    def submit(self, slot, host_block, first, cnt, global_indices=None):
        """begin + one H2D of the whole block from host region ``slot`` + launch."""
        r = self.begin(first, cnt, global_indices)
        try:
            self.h2d(r, host_block, 0, cnt, slot)
        except Exception:
            self.busy[r] = False
            raise
        self.launch(r)
        return r

    def collect(self, ticket):
        r = ticket
        if not self.busy[r]:
            raise ConfigError(f"device region {r} has nothing in flight")
        self.done[r].synchronize()
        self.device_ms += self.start_ev[r].elapsed_time(self.done[r])
        self.h2d_ms += self.h2d_start[r].elapsed_time(self.h2d_done[r])
        first, cnt, gi = self.meta[r]
        self.busy[r] = False
        return kernel.ResultArrays(
            first_index=first,
            beta=self.h_beta[r][:cnt].numpy().copy(),
            status=self.h_status[r][:cnt].numpy().copy(),
            sinv=self.h_sinv[r][:cnt].numpy().copy() if self.emit_s_inv else None,
            global_indices=gi)


def pinned_empty(n, cols, dtype):
    """Pinned, Fortran-ordered n x cols host buffer (numpy view of pinned torch storage)."""
    import torch

    tdt = torch.int8 if np.dtype(dtype) == np.int8 else torch.float64
    t = torch.empty((cols, n), dtype=tdt).pin_memory()
    return t.numpy().T, t       # keep the torch tensor alive alongside the view


def stream_blocks(engine, blocks, fill, on_result):
    """Generic double-buffered loop.

    blocks   : [(first, count)] in order
    fill     : fill(slot, first, count) -> host block (n x >= count, F-order) ready to copy;
               may return a ticket-like callable for asynchronous loads (see run_ooc)
    on_result: on_result(ResultArrays) for each block, in order
    Returns (t_io_wait, block_cpu_times)."""
    t_wait = 0.0
    cpu_times = []
    nb = len(blocks)
    pending = collections.deque()     # tickets of blocks whose results are not yet collected
    for bi, (first, cnt) in enumerate(blocks):
        slot = bi % StreamEngine.REGIONS
        cpu0 = time.thread_time()
        t0 = time.perf_counter()
        host_block = fill(slot, first, cnt, bi, nb)
        t_wait += time.perf_counter() - t0
        if len(pending) == engine.DEV_REGIONS:     # its device region is needed again
            on_result(engine.collect(pending.popleft()))
        pending.append(engine.submit(slot, host_block, first, cnt))
        cpu_times.append(time.thread_time() - cpu0)
    while pending:
        on_result(engine.collect(pending.popleft()))
    return t_wait, cpu_times


def stream_file_blocks(ctx, reader, writer, blocks, m_blk, emit_s_inv=False, parts=2):
    """Double-buffered file -> GPU -> file loop over ``blocks`` (any subset of the plan, e.g.
    one rank's shard).  Returns (engine, t_io_wait, block_cpu_times, t_loop).

    The two host regions (the reference's double buffer, pipeline.py:174-238) are each read
    and copied in ``parts`` column pieces: the read of piece j+2 reuses the host memory of piece
    j+2-2*parts as soon as that piece's H2D is done, so file reads run back to back beside the
    H2D copies and the compute instead of alternating with them."""
    n = reader.n
    int8 = reader.kind == "GWAI"
    engine = StreamEngine(ctx, m_blk, int8=int8, emit_s_inv=emit_s_inv)
    dtype = np.int8 if int8 else np.float64
    regions = [pinned_empty(n, m_blk, dtype) for _ in range(StreamEngine.REGIONS)]
    in_bufs = [r[0] for r in regions]
    width = writer.record_bytes // 8
    rec_bufs = [np.empty((m_blk, width)) for _ in range(2)]
    state = {"store": None, "rec": 0, "io": 0.0}
    P = max(1, int(os.environ.get("GG_STREAM_PARTS", parts)))
    pieces = []                    # (block index, piece k, col0, col1, first, cnt)
    for bi, (first, cnt) in enumerate(blocks):
        edges = [(k * cnt) // P for k in range(P + 1)]
        for k in range(P):
            if edges[k + 1] > edges[k]:
                pieces.append((bi, k, edges[k], edges[k + 1], first, cnt))
    tickets = {}
    # reads kept in flight: up to 2 P - 1 pieces fit the two regions beside the piece being copied
    # (GG_STREAM_AHEAD / GG_STREAM_PARTS: measurement knobs)
    AHEAD = max(1, min(2 * P - 1, int(os.environ.get("GG_STREAM_AHEAD", "2"))))

    def host_slot(piece):
        bi, k = piece[0], piece[1]
        return (bi % StreamEngine.REGIONS) * P + k

    def start_read(j):
        pc = pieces[j]
        bi, k, c0, c1, first, cnt = pc
        engine.wait_h2d(host_slot(pc))       # the piece that used this memory is copied
        view = in_bufs[bi % StreamEngine.REGIONS][:, c0:c1]
        tickets[j] = (reader.start(first + c0, c1 - c0, view), view)   # view kept alive

    def on_result(arr):
        t0 = time.perf_counter()
        if state["store"] is not None:
            writer.wait(state["store"])
        state["io"] += time.perf_counter() - t0
        k = state["rec"] % 2                  # the store of the other record buffer is done
        state["rec"] += 1
        rec = writer.encode(kernel.ResultBlock.from_arrays(arr))
        buf = rec_bufs[k][:rec.shape[0]]
        buf[...] = rec
        state["store"] = writer.start_records(arr.first_index, buf, key=id(rec_bufs[k]))

    t0 = time.perf_counter()
    t_wait = 0.0
    cpu_times = []
    pending = collections.deque()
    cur = None
    for j in range(min(AHEAD, len(pieces))):
        start_read(j)
    cpu0 = time.thread_time()
    for j, pc in enumerate(pieces):
        bi, k, c0, c1, first, cnt = pc
        tw = time.perf_counter()
        blk = reader.wait(tickets.pop(j)[0])
        t_wait += time.perf_counter() - tw
        if cur is None:
            if len(pending) == engine.DEV_REGIONS:     # its device region is needed again
                on_result(engine.collect(pending.popleft()))
            cur = engine.begin(first, cnt)
        engine.h2d(cur, blk.data, c0, c1 - c0, host_slot(pc))
        if j + AHEAD < len(pieces):
            start_read(j + AHEAD)
        if j + 1 == len(pieces) or pieces[j + 1][0] != bi:
            engine.launch(cur)
            pending.append(cur)
            cur = None
            cpu_times.append(time.thread_time() - cpu0)
            cpu0 = time.thread_time()
    while pending:
        on_result(engine.collect(pending.popleft()))
    t1 = time.perf_counter()
    if state["store"] is not None:
        writer.wait(state["store"])
    t_end = time.perf_counter()
    state["io"] += t_end - t1
    return engine, t_wait + state["io"], cpu_times, t_end - t0


def _run_stream(paths, cfg, mode, m_blk_override=None):
    cfg = cfg or SolveConfig()
    t_start = time.perf_counter()
    geno_bytes, n, m = fileio.total_genotype_bytes(paths.geno)
    item = 1 if fileio.genotype_kind(paths.geno) == "GWAI" else 8
    ctx, t_prep, m_bytes = _load_prepare(paths)
    p = ctx.p
    flags = 1 if cfg.emit_s_inv else 0
    rsz = fileio.record_size(p, flags)
    m_blk = min(m_blk_override or cfg.m_blk, m)
    plan = block_plan(m, m_blk)
    reader = fileio.BlockReader(paths.geno)
    writer = fileio.BlockWriter(paths.out, m, p, flags)
    try:
        engine, t_io, cpu_times, t_loop = stream_file_blocks(ctx, reader, writer, plan.blocks,
                                                             m_blk, cfg.emit_s_inv)
    finally:
        reader.close()
        writer.close()
    return RunSummary(
        mode=mode, n=n, m=m, p=p, m_blk=m_blk, np_=1, threads=cfg.threads,
        t_prepare=t_prep, t_compute=max(t_loop - t_io, 0.0), t_io_wait=t_io,
        t_total=time.perf_counter() - t_start,
        bytes_read=reader.bytes_read + m_bytes, bytes_written=writer.bytes_written,
        peak_resident_est=8 * n * n + 2 * (item * n * m_blk + m_blk * rsz) + 8 * n * p,
        buffer_regions=StreamEngine.REGIONS, gpus=1, t_device=engine.device_ms / 1e3,
        snps_per_s=m / t_loop if t_loop > 0 else 0.0, block_cpu_times=cpu_times)


def run_incore(paths, cfg=None):
    """Whole-genotype engine (pipeline.py:134-171).  The genotypes must fit the memory budget
    (ConfigError otherwise); on the GPU they are solved in device-sized slices of the same
    per-column arithmetic, so the result equals a single block bitwise."""
    cfg = cfg or SolveConfig()
    geno_bytes, n, m = fileio.total_genotype_bytes(paths.geno)
    budget = cfg.budget()
    need = geno_bytes + 8 * n * n
    if budget is not None and need > budget:
        raise ConfigError(f"in-core run needs {need} bytes (genotypes + covariance), "
                          f"budget is {budget}")
    s = _run_stream(paths, cfg, "incore", m_blk_override=min(m, GPU_M_BLK))
    s.buffer_regions = 1
    s.m_blk = m
    return s


def run_ooc(paths, cfg=None):
    """Out-of-core engine (pipeline.py:174-238): two buffer regions, asynchronous file loads,
    H2D on a copy stream, compute on a compute stream, asynchronous result stores."""
    cfg = cfg or SolveConfig()
    geno_bytes, n, m = fileio.total_genotype_bytes(paths.geno)
    item = 1 if fileio.genotype_kind(paths.geno) == "GWAI" else 8
    m_blk = min(cfg.m_blk, m)
    p = fileio.read_dims(paths.covariates, "GWAC")[1] + 1
    rsz = fileio.record_size(p, 1 if cfg.emit_s_inv else 0)
    budget = cfg.budget()
    region = item * n * m_blk + m_blk * rsz
    if budget is not None and 2 * region > budget:
        raise ConfigError(f"two buffer regions need {2 * region} bytes, budget is {budget}")
    return _run_stream(paths, cfg, "ooc")


def solve_array(ctx, X, m_blk=GPU_M_BLK, emit_s_inv=False, first_index=0, engine=None):
    """Public array entry point of the stream: solve every column of the host genotype matrix
    X (n x m, FP64 or int8, Fortran-ordered; pinned memory gives overlapped H2D) against a
    device-prepared context.  Returns ResultArrays for all m markers."""
    X = np.asarray(X)
    if not X.flags.f_contiguous:
        X = np.asfortranarray(X)
    n, m = X.shape
    int8 = X.dtype == np.int8
    if engine is None:
        engine = StreamEngine(ctx, min(m_blk, m), int8=int8, emit_s_inv=emit_s_inv)
    m_blk = engine.m_blk
    plan = block_plan(m, m_blk)
    p = ctx.p
    beta = np.empty((m, p))
    status = np.empty(m, dtype=np.int32)
    sinv = np.empty((m, p * (p + 1) // 2)) if emit_s_inv else None

    def fill(slot, first, cnt, bi, nb):
        return X[:, first:first + cnt]

    def on_result(arr):
        f = arr.first_index - first_index
        beta[f:f + arr.count] = arr.beta
        status[f:f + arr.count] = arr.status
        if sinv is not None:
            sinv[f:f + arr.count] = arr.sinv

    blocks = [(first_index + f, c) for f, c in plan.blocks]

    def fill_off(slot, first, cnt, bi, nb):
        return fill(slot, first - first_index, cnt, bi, nb)

    stream_blocks(engine, blocks, fill_off, on_result)
    return kernel.ResultArrays(first_index=first_index, beta=beta, status=status, sinv=sinv)
