"""Distributed engine for covariances larger than one GPU (BASELINE config 4).

Replaces the reference's distributed engine (distgrid.py:1-469: element-cyclic M on a 2D grid,
replicated panels gathered with Python all-gathers, 1D<->2D all-to-all redistribution of every
SNP block) with a B200 design:

* M and L live 2D BLOCK-cyclic (block nb = 512 by default; nb = 1 would be the reference's
  element-cyclic map) on the r x c grid of ``grid_create`` (same rule as distgrid.py:43-52);
  every rank reads or generates only its own blocks — there is no root scatter.
* ``dist_potrf_inv``: right-looking blocked Cholesky FUSED with the triangular inverse (a
  right-looking TRSM of the identity, X = L^-1), one pass over the block columns K:
    1. the owner of (K, K) factors and inverts the diagonal block on its GPU (gg_potrf_f64);
       the inverse is broadcast to all ranks;
    2. process column K%c forms the panel L_IK = A_IK L_KK^-T, process row K%r forms the
       inverse's block row X_KJ = L_KK^-1 B_KJ (DMMA GEMMs);
    3. panel and block row are made global with one NCCL all-reduce each over disjoint
       supports (exact: every element has exactly one non-zero contributor);
    4. every rank updates its own blocks: A_IJ -= L_IK L_JK^T and B_IJ -= L_IK X_KJ.
  NCCL carries ~2 n nb doubles per step (n = 150,000, nb = 512: 1.2 GB, < 2 ms on NVLink 5)
  against (n - K nb)^2 nb / (r c) FMAs of local GEMM.
* ``assemble_packed_inverse``: each rank writes its blocks of L^-1 into the packed tile-major
  layout of the TRSM (zeros elsewhere, gg_pack_lower_blockcyclic_f64) and one all-reduce makes
  the packed inverse replicated: 90 GB at n = 150,000, which fits one B200's 180 GB although M
  (180 GB) does not.  From there the SNP sweep is the single-GPU stream, sharded over ranks with
  no per-block communication (the reference redistributes every block twice,
  distgrid.py:422-428).

Local matrices are column-major torch tensors of shape (local_cols, local_rows).  The numerical
work goes through an ``ops`` object: ``DeviceOps`` (the sm_100a library) in production; the CPU
tests inject a numpy implementation to check the distributed logic over gloo.
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass

import numpy as np

from . import fileio
from .errors import ConfigError, DimensionMismatch, NotPositiveDefinite

DEFAULT_NB = 512


@dataclass(frozen=True)
class GridLayout:
    np_: int
    r: int
    c: int

    def coord(self, rank):
        return rank // self.c, rank % self.c

    def rank_of(self, prow, pcol):
        return prow * self.c + pcol


def grid_create(np_):
    """Process grid as close to square as possible: r = largest divisor of np with r <= sqrt(np)
    (the reference's rule, distgrid.py:43-52)."""
    if np_ < 1:
        raise ConfigError("need at least one rank")
    r = max(d for d in range(1, int(math.isqrt(np_)) + 1) if np_ % d == 0)
    return GridLayout(np_=np_, r=r, c=np_ // r)


class BlockCyclic:
    """nb x nb block-cyclic layout of an n x n matrix over ``grid``, as seen by ``rank``."""

    def __init__(self, n, nb, grid, rank):
        if nb < 1:
            raise ConfigError("block size must be positive")
        self.n, self.nb, self.grid, self.rank = n, nb, grid, rank
        self.pr, self.pc = grid.coord(rank)
        self.nblk = -(-n // nb)
        self.n_pad = self.nblk * nb
        self.row_blocks = list(range(self.pr, self.nblk, grid.r))
        self.col_blocks = list(range(self.pc, self.nblk, grid.c))
        self.m_loc = len(self.row_blocks) * nb
        self.n_loc = len(self.col_blocks) * nb

    def owner(self, I, J):
        return self.grid.rank_of(I % self.grid.r, J % self.grid.c)

    def lrow(self, I):
        return (I // self.grid.r) * self.nb

    def lcol(self, J):
        return (J // self.grid.c) * self.nb

    def rows_through(self, K):
        """Local rows of the owned block-rows I <= K (the owned I > K start there)."""
        return 0 if K < self.pr else ((K - self.pr) // self.grid.r + 1) * self.nb

    def cols_through(self, K):
        return 0 if K < self.pc else ((K - self.pc) // self.grid.c + 1) * self.nb

    def global_rows(self, blocks):
        nb = self.nb
        return np.concatenate([np.arange(I * nb, (I + 1) * nb) for I in blocks]) \
            if blocks else np.zeros(0, dtype=np.int64)

    def rows_after_global(self, K):
        return self.global_rows([I for I in self.row_blocks if I > K])

    def cols_after_global(self, K):
        return self.global_rows([J for J in self.col_blocks if J > K])

    def cols_through_global(self, K):
        return self.global_rows([J for J in self.col_blocks if J <= K])


def local_from_global(M, layout, ops):
    """This rank's blocks of the (host) n x n matrix M, identity on the padding; A_loc and the
    identity's share B_loc (column-major local tensors)."""
    n, nb = layout.n, layout.nb
    rows = layout.global_rows(layout.row_blocks)
    cols = layout.global_rows(layout.col_blocks)
    Mp = np.zeros((len(rows), len(cols)))
    rv, cv = rows < n, cols < n
    if rv.any() and cv.any():
        Mp[np.ix_(rv, cv)] = np.asarray(M)[np.ix_(rows[rv], cols[cv])]
    eye = (rows[:, None] == cols[None, :])
    pad = eye & (rows[:, None] >= n)
    Mp[pad] = 1.0
    A = ops.from_host(Mp)
    B = ops.from_host(eye.astype(np.float64))
    return A, B


def local_from_gwam(path, layout, ops):
    """Read only this rank's blocks of a GWAM file (memory-mapped), identity on the padding."""
    n = fileio.read_dims(path, "GWAM")[0]
    if n != layout.n:
        raise DimensionMismatch("covariance file does not match the layout")
    mm = np.memmap(path, dtype="<f8", mode="r", offset=fileio.header_size("GWAM"),
                   shape=(n, n), order="F")
    return local_from_global(mm, layout, ops)


def _allreduce(t, dist):
    if dist is not None:
        dist.all_reduce(t)
    return t


def _allreduce_max(t, dist):
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t


def _broadcast(t, src, dist):
    if dist is not None:
        dist.broadcast(t, src)
    return t


def dist_potrf_inv(A, B, layout, ops, dist=None):
    """Fused distributed Cholesky + inverse (see module doc).  A (this rank's blocks of M) is
    overwritten with L, B (this rank's blocks of I) with L^-1.  Raises NotPositiveDefinite with
    the global pivot on every rank."""
    nb, g = layout.nb, layout.grid
    rank = layout.rank
    for K in range(layout.nblk):
        owner = layout.owner(K, K)
        Dinv = ops.empty(nb, nb)
        status = ops.int_tensor(-1)
        if rank == owner:
            st, Lkk, Linvkk = ops.potrf_inv(A, layout.lrow(K), layout.lcol(K), nb)
            status.fill_(st)
            if st < 0:
                ops.copy_block(A, layout.lrow(K), layout.lcol(K), Lkk)
                Dinv.copy_(Linvkk)
        _broadcast(status, owner, dist)
        st = int(status.item())
        if st >= 0:
            raise NotPositiveDefinite(K * nb + st)
        _broadcast(Dinv, owner, dist)
        r0 = layout.rows_through(K)
        m_below = layout.m_loc - r0
        grows = layout.rows_after_global(K)
        # panel L_IK = A_IK Dinv^T on process column K % c; made global by an exact all-reduce
        Pfull = ops.zeros(nb, layout.n_pad)                      # (n_pad x nb) column-major
        if layout.pc == K % g.c and m_below > 0:
            tmp = ops.empty(nb, m_below)
            ops.gemm(tmp, 0, 0, m_below, nb, A, r0, layout.lcol(K), Dinv, 0, 0, nb,
                     1.0, 0.0, trans_b=True)
            ops.copy_block(A, r0, layout.lcol(K), tmp)
            ops.scatter_cols_rows(Pfull, grows, tmp)
        _allreduce(Pfull, dist)
        # block row K of the inverse, X_KJ = Dinv B_KJ on process row K % r
        cl = layout.cols_through(K)
        gcols = layout.cols_through_global(K)
        Xfull = ops.zeros(layout.n_pad, nb)                      # (nb x n_pad) column-major
        if layout.pr == K % g.r and cl > 0:
            tmpx = ops.empty(cl, nb)
            ops.gemm(tmpx, 0, 0, nb, cl, Dinv, 0, 0, B, layout.lrow(K), 0, nb, 1.0, 0.0,
                     trans_b=False)
            ops.copy_block(B, layout.lrow(K), 0, tmpx)
            ops.scatter_cols(Xfull, gcols, tmpx)
        _allreduce(Xfull, dist)
        if m_below == 0:
            continue
        P_rows = ops.gather_rows(Pfull, grows)                   # (m_below x nb)
        c0 = layout.cols_through(K)
        n_right = layout.n_loc - c0
        if n_right > 0:
            P_cols = ops.gather_rows(Pfull, layout.cols_after_global(K))   # (n_right x nb)
            ops.gemm(A, r0, c0, m_below, n_right, P_rows, 0, 0, P_cols, 0, 0, nb, -1.0, 1.0,
                     trans_b=True)
        if cl > 0:
            X_cols = ops.gather_cols(Xfull, gcols)               # (nb x cl)
            ops.gemm(B, r0, 0, m_below, cl, P_rows, 0, 0, X_cols, 0, 0, nb, -1.0, 1.0,
                     trans_b=False)
    ops.zero_upper_blocks(A, layout)
    return A, B


def assemble_packed_inverse(B, layout, ops, dist=None):
    """Replicate the packed tile-major inverse on every rank from the block-cyclic shares."""
    P = ops.pack_blockcyclic(B, layout)
    return _allreduce(P, dist)


def assemble_slices(B, layout, ops, dist=None):
    """Replicated int8 slices + slice metadata of the inverse from the block-cyclic shares: each
    rank takes its rows' off-diagonal / diagonal exponents over its blocks (MAX all-reduce), turns
    them into the row exponents, then cuts the slices of the elements it owns (zeros elsewhere)
    and the heads of the diagonals it owns; SUM all-reduces of both over disjoint supports are
    exact.  Needs 3.5 np^2 bytes per rank (79 GB at n = 1.5e5) and no replicated FP64 inverse."""
    ex2 = ops.row_exponents(B, layout)
    _allreduce_max(ex2, dist)
    meta = ops.slice_meta(ex2, layout)
    S = ops.slice_blockcyclic(B, layout, meta)
    _allreduce(meta[meta.numel() // 2:], dist)
    return _allreduce(S, dist), meta


def whiten_blockcyclic(B, layout, ops, RHS, dist=None):
    """[X_L | y] bar = L^-1 [X_L | y] from the block-cyclic inverse: one local GEMM of this
    rank's blocks against the rows of RHS it needs, scattered to global rows and summed over
    ranks (FP64 all-reduce).  RHS: host (n x k).  Returns a replicated (k, n_pad) tensor."""
    n, k = RHS.shape
    full = np.zeros((layout.n_pad, k))
    full[:n] = RHS                       # padding rows zero (the inverse is identity there)
    cols = layout.global_rows(layout.col_blocks)
    rows = layout.global_rows(layout.row_blocks)
    Y = ops.zeros(k, layout.n_pad)
    if len(rows) and len(cols):
        Xloc = ops.from_host(full[cols])                     # (n_loc x k)
        Yloc = ops.empty(k, layout.m_loc)
        ops.gemm(Yloc, 0, 0, layout.m_loc, k, B, 0, 0, Xloc, 0, 0, layout.n_loc, 1.0, 0.0,
                 trans_b=False)
        ops.scatter_cols_rows(Y, rows, Yloc)
    return _allreduce(Y, dist)


def gather_matrix(D, layout, ops, dist=None):
    """Full n x n host copy of a block-cyclic matrix on every rank (tests / small n only)."""
    full = np.zeros((layout.n_pad, layout.n_pad))
    rows = layout.global_rows(layout.row_blocks)
    cols = layout.global_rows(layout.col_blocks)
    if len(rows) and len(cols):
        full[np.ix_(rows, cols)] = ops.to_host(D)
    t = ops.from_host(full)
    _allreduce(t, dist)
    return ops.to_host(t)[:layout.n, :layout.n]


# ---------------------------------------------------------------------------------------------
# the production ops: sm_100a kernels through the C-ABI
# ---------------------------------------------------------------------------------------------

class DeviceOps:
    """Local numerics of the distributed engine on this rank's GPU."""

    def __init__(self):
        import torch

        from . import _capi

        self.torch = torch
        self.capi = _capi
        self.dev = _capi.device()
        self._oz_ws = None      # Ozaki GEMM workspace, grown on demand

    # -- buffers (column-major (rows x cols) matrix = torch tensor (cols, rows)) --------------
    def empty(self, ncols, nrows):
        return self.torch.empty((ncols, nrows), dtype=self.torch.float64, device=self.dev)

    def zeros(self, ncols, nrows):
        return self.torch.zeros((ncols, nrows), dtype=self.torch.float64, device=self.dev)

    def int_tensor(self, v):
        return self.torch.tensor([v], dtype=self.torch.int64, device=self.dev)

    def from_host(self, A):
        A = np.asarray(A, dtype=np.float64)
        return self.torch.from_numpy(np.ascontiguousarray(A.T)).to(self.dev)

    def to_host(self, T):
        return T.cpu().numpy().T

    def _p(self, T, r0, c0):
        return self.capi.C.c_void_p(T.data_ptr() + (c0 * T.shape[1] + r0) * 8)

    # -- numerics ------------------------------------------------------------------------------
    def potrf_inv(self, A, r0, c0, nb):
        """Factor + invert the nb x nb diagonal block at (r0, c0); (status, L, Linv)."""
        torch, capi = self.torch, self.capi
        L = self.empty(nb, nb)
        Li = self.empty(nb, nb)
        ws = torch.empty(int(capi.lib().gg_potrf_workspace_bytes(nb)), dtype=torch.uint8,
                         device=self.dev)
        info = (capi.C.c_int * 2)()
        rc = capi.lib().gg_potrf_f64(nb, self._p(A, r0, c0), A.shape[1], 0, capi.ptr(L),
                                     capi.ptr(Li), nb, capi.ptr(ws), info, capi.stream_handle())
        if rc == capi.GG_ENOTPD:
            return int(info[0]), L, Li
        capi.check(rc, "gg_potrf_f64")
        return -1, L, Li

    def gemm(self, C, cr, cc, m, n, A, ar, ac, B, br, bc, k, alpha, beta, trans_b):
        """C[cr:cr+m, cc:cc+n] = beta C + alpha A op(B).  Large updates (every dimension >= 512:
        the trailing updates of dist_potrf_inv) run on the int8 tensor cores through the
        Ozaki-scheme GEMM (gg_gemm_ozaki_f64, FP64-GEMM accuracy) unless GG_FACTOR_OZAKI=0;
        the rest on the DMMA GEMM."""
        capi = self.capi
        if min(m, n, k) >= 512 and os.environ.get("GG_FACTOR_OZAKI", "1") != "0":
            lib = capi.lib()
            need = int(lib.gg_gemm_ozaki_workspace_bytes(m, n, k, 0))
            if self._oz_ws is None or self._oz_ws.numel() < need:
                self._oz_ws = None
                self._oz_ws = self.torch.empty(need, dtype=self.torch.uint8, device=self.dev)
            ldb = B.shape[1]
            b_rs, b_cs = (1, ldb) if trans_b else (ldb, 1)
            rc = lib.gg_gemm_ozaki_f64(m, n, k, self._p(A, ar, ac), 1, A.shape[1],
                                       self._p(B, br, bc), b_rs, b_cs, self._p(C, cr, cc),
                                       C.shape[1], alpha, beta, 0, capi.ptr(self._oz_ws),
                                       self._oz_ws.numel(), capi.stream_handle())
            capi.check(rc, "gg_gemm_ozaki_f64")
            return
        rc = capi.lib().gg_dgemm_f64(m, n, k, alpha, self._p(A, ar, ac), A.shape[1],
                                     self._p(B, br, bc), B.shape[1], 1 if trans_b else 0, beta,
                                     self._p(C, cr, cc), C.shape[1], capi.stream_handle())
        capi.check(rc, "gg_dgemm_f64")

    def copy_block(self, dst, r0, c0, src):
        ncols, nrows = src.shape
        dst[c0:c0 + ncols, r0:r0 + nrows].copy_(src)

    def scatter_cols_rows(self, full, grows, tmp):
        idx = self.torch.as_tensor(grows, device=self.dev)
        full[:, idx] = tmp

    def scatter_cols(self, full, gcols, tmp):
        idx = self.torch.as_tensor(gcols, device=self.dev)
        full[idx, :] = tmp

    def gather_rows(self, full, grows):
        idx = self.torch.as_tensor(grows, device=self.dev)
        return full[:, idx].contiguous()

    def gather_cols(self, full, gcols):
        idx = self.torch.as_tensor(gcols, device=self.dev)
        return full[idx, :].contiguous()

    def zero_upper_blocks(self, A, layout):
        nb = layout.nb
        for jl, J in enumerate(layout.col_blocks):
            for il, I in enumerate(layout.row_blocks):
                if I < J:
                    A[jl * nb:(jl + 1) * nb, il * nb:(il + 1) * nb].zero_()

    def row_exponents(self, B, layout):
        torch, capi = self.torch, self.capi
        e = torch.empty(int(capi.lib().gg_slice_meta_ints(layout.n)), dtype=torch.int32,
                        device=self.dev)
        ldl = max(B.shape[1], 1)
        rc = capi.lib().gg_row_exponents_blockcyclic(
            layout.n, layout.nb, layout.grid.r, layout.grid.c, layout.pr, layout.pc,
            capi.ptr(B) if B.numel() else capi.ptr(e), ldl, capi.ptr(e), capi.stream_handle())
        capi.check(rc, "gg_row_exponents_blockcyclic")
        return e

    def slice_meta(self, ex2, layout):
        meta = self.torch.empty_like(ex2)
        capi = self.capi
        rc = capi.lib().gg_slice_meta_i8(layout.n, capi.ptr(ex2), capi.ptr(meta),
                                         capi.stream_handle())
        capi.check(rc, "gg_slice_meta_i8")
        return meta

    def slice_blockcyclic(self, B, layout, expo):
        torch, capi = self.torch, self.capi
        S = torch.empty(int(capi.lib().gg_inverse_slices_bytes(layout.n)), dtype=torch.int8,
                        device=self.dev)
        ldl = max(B.shape[1], 1)
        rc = capi.lib().gg_slice_blockcyclic_i8(
            layout.n, layout.nb, layout.grid.r, layout.grid.c, layout.pr, layout.pc,
            capi.ptr(B) if B.numel() else capi.ptr(S), ldl, capi.ptr(expo), capi.ptr(S),
            capi.stream_handle())
        capi.check(rc, "gg_slice_blockcyclic_i8")
        return S

    def pack_blockcyclic(self, B, layout):
        torch, capi = self.torch, self.capi
        P = torch.empty(int(capi.lib().gg_packed_lower_bytes(layout.n)) // 8,
                        dtype=torch.float64, device=self.dev)
        ldl = max(B.shape[1], 1)
        rc = capi.lib().gg_pack_lower_blockcyclic_f64(layout.n, layout.nb, layout.grid.r,
                                                      layout.grid.c, layout.pr, layout.pc,
                                                      capi.ptr(B) if B.numel() else capi.ptr(P),
                                                      ldl, capi.ptr(P), capi.stream_handle())
        capi.check(rc, "gg_pack_lower_blockcyclic_f64")
        return P


# ---------------------------------------------------------------------------------------------
# the SPMD driver
# ---------------------------------------------------------------------------------------------

@dataclass
class DistConfig:
    m_blk: int = 8192
    emit_s_inv: bool = False
    nb: int = DEFAULT_NB
    int8: bool = True                  # replicate the int8 slices (dosage blocks on tcgen05)
    fp64_inverse: bool | None = None   # replicate the packed FP64 inverse (None: if it fits)


def run_dist(paths, cfg=None, ops=None, sweep=True):
    """SPMD body (one process per GPU under torchrun; torch.distributed initialised by the
    caller, NCCL on the B200 box).  Factor + invert M in 2D block-cyclic form, replicate the
    packed inverse, prepare the context, then stream this rank's share of the SNP blocks with
    offset-addressed result writes (no per-block communication).  Returns a RunSummary."""
    import torch.distributed as tdist

    from . import kernel
    from .pipeline import RunSummary
    from .shard import ShardConfig, stream_shard

    cfg = cfg or DistConfig()
    dist = tdist if tdist.is_available() and tdist.is_initialized() else None
    rank = dist.get_rank() if dist else 0
    world = dist.get_world_size() if dist else 1
    ops = ops or DeviceOps()
    t_start = time.perf_counter()
    n = fileio.read_dims(paths.cov, "GWAM")[0]
    grid = grid_create(world)
    layout = BlockCyclic(n, cfg.nb, grid, rank)
    A, B = local_from_gwam(paths.cov, layout, ops)
    dist_potrf_inv(A, B, layout, ops, dist)
    if sweep:
        A = None                           # L itself is not needed by the sweep
    XL = fileio.read_matrix(paths.covariates, "GWAC")
    y = fileio.read_matrix(paths.pheno, "GWAY")
    slices, expo = assemble_slices(B, layout, ops, dist) if cfg.int8 else (None, None)
    fp64 = cfg.fp64_inverse
    if fp64 is None:   # the same decision on every rank (same n, same device class)
        fp64 = _packed_inverse_fits(layout.n, ops)
    if fp64 or slices is None:
        LinvP = assemble_packed_inverse(B, layout, ops, dist)
        del B
        ctx = kernel.prepare_from_inverse(LinvP, n, XL, y, slices=slices, expo=expo)
    else:   # config-4 sizes: no replicated FP64 inverse; whiten from the block-cyclic one
        LinvP = None
        XLy = whiten_blockcyclic(B, layout, ops, np.column_stack([XL, np.ravel(y)]), dist)
        del B
        ctx = kernel.prepare_from_inverse(None, n, XL, y, slices=slices, expo=expo, XLy=XLy)
    t_prepare = time.perf_counter() - t_start
    if not sweep:
        return ctx, (A, layout)
    s = stream_shard(paths, ctx, ShardConfig(m_blk=cfg.m_blk, emit_s_inv=cfg.emit_s_inv))
    return RunSummary(
        mode="dist", n=n, m=s.m, p=ctx.p, m_blk=s.m_blk, np_=world, threads=1,
        t_prepare=t_prepare, t_compute=s.t_compute, t_io_wait=s.t_io_wait,
        t_total=time.perf_counter() - t_start, bytes_read=s.bytes_read,
        bytes_written=s.bytes_written, buffer_regions=2, gpus=world, t_device=s.t_device,
        snps_per_s=s.snps_per_s,
        peak_resident_est=8 * layout.m_loc * layout.n_loc * 2
        + (8 * LinvP.numel() if LinvP is not None else 0)
        + (slices.numel() if slices is not None else 0))


def _packed_inverse_fits(n, ops):
    """Room for the replicated packed FP64 inverse (4 np^2 doubles) next to the slices."""
    torch = getattr(ops, "torch", None)
    if torch is None or not torch.cuda.is_available():
        return True
    from . import _capi
    free, _ = torch.cuda.mem_get_info(_capi.device())
    return int(_capi.lib().gg_packed_lower_bytes(n)) < 0.6 * free


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
