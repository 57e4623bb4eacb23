"""Test-only CPU implementation of the distributed engine's local numerics (numpy/scipy on torch
CPU tensors), used to check paper_1304_2272_b200.distgrid's communication logic over gloo.  The
production path uses distgrid.DeviceOps (sm_100a kernels)."""

import numpy as np
import torch
from scipy.linalg import solve_triangular
from scipy.linalg.lapack import dpotrf


INT_MIN = -2 ** 31


def slice_offsets(i, k, np_):
    """Byte offsets of element (i, k) in the tile-packed slice layout, one per slice."""
    mt, kt = i // 128, k // 128
    base = (mt * (mt + 1) // 2 + kt) * 131072 + (i % 128) * 128 + (k % 128)
    return base[..., None] + 16384 * np.arange(8)


def slices_dense(Linv_rows, expo, np_):
    """Tile-packed int8 slices of a dense lower-triangular inverse given row exponents (the
    restatement of slice_rows_kernel, used as the CPU ops' implementation and the check)."""
    nt = np_ // 128
    out = np.zeros(nt * (nt + 1) // 2 * 131072, dtype=np.int8)
    for i in range(np_):
        kend = (i // 128 + 1) * 128
        k = np.arange(kend)
        v = np.where(k <= i, Linv_rows(i, kend), 0.0)
        v = np.where(v != 0.0, np.ldexp(v, -int(expo[i])), 0.0)
        q = np.empty((kend, 8))
        for s in range(8):
            t = v * 128.0
            q[:, s] = np.trunc(t)
            v = t - q[:, s]
        out[slice_offsets(i, k, np_)] = q.astype(np.int8)
    return out


def row_exponents_dense(rows_abs_max):
    e = np.full(rows_abs_max.shape, INT_MIN, dtype=np.int32)
    nz = rows_abs_max > 0
    e[nz] = np.frexp(rows_abs_max[nz])[1]
    return e


def pack_lower_dense(Dense, n):
    """Packed tile-major layout of the lower triangle of a dense (>= np x np) matrix."""
    np_ = -(-n // 128) * 128
    nmt = np_ // 128
    P = np.zeros(4 * nmt * (nmt + 1) * 2048)
    D = np.zeros((np_, np_))
    k = min(Dense.shape[0], np_)
    D[:k, :k] = Dense[:k, :k]
    for i in range(np_ - k):
        D[k + i, k + i] = 1.0
    D = np.tril(D)
    for mt in range(nmt):
        rows = D[mt * 128:(mt + 1) * 128, :(mt + 1) * 128]          # 128 x 128(mt+1)
        tiles = rows.reshape(128, 8 * (mt + 1), 16).transpose(1, 0, 2)
        t0 = 4 * mt * (mt + 1)
        P[t0 * 2048:(t0 + 8 * (mt + 1)) * 2048] = tiles.ravel()
    return P


class CpuOps:
    def empty(self, ncols, nrows):
        return torch.empty((ncols, nrows), dtype=torch.float64)

    def zeros(self, ncols, nrows):
        return torch.zeros((ncols, nrows), dtype=torch.float64)

    def int_tensor(self, v):
        return torch.tensor([v], dtype=torch.int64)

    def from_host(self, A):
        return torch.from_numpy(np.ascontiguousarray(np.asarray(A, dtype=np.float64).T))

    def to_host(self, T):
        return T.numpy().T

    def potrf_inv(self, A, r0, c0, nb):
        blk = A[c0:c0 + nb, r0:r0 + nb].numpy().T
        L, info = dpotrf(np.ascontiguousarray(blk), lower=1, clean=1)
        if info > 0:
            return info - 1, self.zeros(nb, nb), self.zeros(nb, nb)
        Li = solve_triangular(L, np.eye(nb), lower=True)
        return -1, self.from_host(L), self.from_host(np.tril(Li))

    def gemm(self, C, cr, cc, m, n, A, ar, ac, B, br, bc, k, alpha, beta, trans_b):
        Am = A[ac:ac + k, ar:ar + m].T
        Bm = B[bc:bc + k, br:br + n] if trans_b else B[bc:bc + n, br:br + k].T
        Cv = C[cc:cc + n, cr:cr + m]
        res = alpha * (Am @ Bm)
        if beta != 0.0:              # beta == 0 must not read C (may be uninitialised)
            res = res + beta * Cv.T
        Cv.copy_(res.T)

    def copy_block(self, dst, r0, c0, src):
        ncols, nrows = src.shape
        dst[c0:c0 + ncols, r0:r0 + nrows].copy_(src)

    def scatter_cols_rows(self, full, grows, tmp):
        full[:, torch.as_tensor(grows)] = tmp

    def scatter_cols(self, full, gcols, tmp):
        full[torch.as_tensor(gcols), :] = tmp

    def gather_rows(self, full, grows):
        return full[:, torch.as_tensor(grows)].contiguous()

    def gather_cols(self, full, gcols):
        return full[torch.as_tensor(gcols), :].contiguous()

    def zero_upper_blocks(self, A, layout):
        nb = layout.nb
        for jl, J in enumerate(layout.col_blocks):
            for il, I in enumerate(layout.row_blocks):
                if I < J:
                    A[jl * nb:(jl + 1) * nb, il * nb:(il + 1) * nb].zero_()

    def _full_share(self, B, layout):
        full = np.zeros((layout.n_pad, layout.n_pad))
        rows = layout.global_rows(layout.row_blocks)
        cols = layout.global_rows(layout.col_blocks)
        if len(rows) and len(cols):
            full[np.ix_(rows, cols)] = self.to_host(B)
        return full

    def row_exponents(self, B, layout):
        full = np.tril(self._full_share(B, layout))
        return torch.from_numpy(row_exponents_dense(np.abs(full).max(axis=1)))

    def slice_blockcyclic(self, B, layout, expo):
        full = np.tril(self._full_share(B, layout))
        S = slices_dense(lambda i, kend: full[i, :kend], expo.numpy(), layout.n_pad)
        return torch.from_numpy(S)

    def pack_blockcyclic(self, B, layout):
        full = np.zeros((layout.n_pad, layout.n_pad))
        rows = layout.global_rows(layout.row_blocks)
        cols = layout.global_rows(layout.col_blocks)
        if len(rows) and len(cols):
            full[np.ix_(rows, cols)] = self.to_host(B)
        # padding diagonal is carried by exactly one owner; pack without adding it again
        np_ = -(-layout.n // 128) * 128
        P = pack_lower_dense(full, np_)
        return torch.from_numpy(P)
