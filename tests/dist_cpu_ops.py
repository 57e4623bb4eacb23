"""Test-only CPU implementation of the distributed engine's local numerics (numpy/scipy on torch
CPU tensors), used to check paper_1304_2272_b200.distgrid's communication logic over gloo.  The
production path uses distgrid.DeviceOps (sm_100a kernels)."""

import numpy as np
import torch
from scipy.linalg import solve_triangular
from scipy.linalg.lapack import dpotrf


INT_MIN = -2 ** 31


S = 7              # int8 slices (trsm_i8.cu)
HEAD_BITS = 20     # diagonal head width (trsm_i8.cu)
TILE = S * 128 * 128


def slice_offsets(i, k, np_):
    """Byte offsets of element (i, k) in the tile-packed slice layout, one per slice."""
    mt, kt = i // 128, k // 128
    base = (mt * (mt + 1) // 2 + kt) * TILE + (i % 128) * 128 + (k % 128)
    return base[..., None] + 16384 * np.arange(S)


def _exp_of(x):
    e = np.full(x.shape, INT_MIN, dtype=np.int64)
    nz = x > 0
    e[nz] = np.frexp(x[nz])[1]
    return e


def row_exponents_dense(full_tril):
    """[e_off | e_diag] of a dense lower-triangular (np x np) matrix (row_exponent_kernel)."""
    off = np.abs(np.tril(full_tril, -1)).max(axis=1)
    return np.concatenate([_exp_of(off), _exp_of(np.abs(np.diag(full_tril)))]).astype(np.int32)


def slice_meta_dense(ex2):
    """Row exponents e' = max(e_off, e_diag - HEAD_BITS), heads zeroed (slice_meta_kernel)."""
    np_ = len(ex2) // 2
    eo, ed = ex2[:np_].astype(np.int64), ex2[np_:].astype(np.int64)
    e = np.where(ed == INT_MIN, eo,
                 np.where(eo == INT_MIN, ed - HEAD_BITS, np.maximum(eo, ed - HEAD_BITS)))
    e = np.where(e == INT_MIN, 0, e)
    return np.concatenate([e, np.zeros(np_, dtype=np.int64)]).astype(np.int32)


def slices_dense(Linv_rows, meta, np_):
    """Tile-packed int8 slices of a dense lower-triangular inverse given the metadata (the
    restatement of slice_rows_kernel, used as the CPU ops' implementation and the check); the
    heads of rows with a nonzero diagonal are written into meta[np_:] in place."""
    nt = np_ // 128
    out = np.zeros(nt * (nt + 1) // 2 * TILE, dtype=np.int8)
    for i in range(np_):
        kend = (i // 128 + 1) * 128
        k = np.arange(kend)
        v = np.where(k <= i, Linv_rows(i, kend), 0.0)
        v = np.where(v != 0.0, np.ldexp(v, -int(meta[i])), 0.0)
        if v[i] != 0.0:
            h = np.trunc(v[i])
            meta[np_ + i] = int(h)
            v[i] -= h
        V = np.zeros(kend, dtype=np.int64)      # the truncated digits' exact value
        for s in range(S):
            t = v * 128.0
            qs = np.trunc(t) if s < S - 1 else np.clip(np.rint(t), -127.0, 127.0)
            V = V * 128 + qs.astype(np.int64)
            v = t - qs
        q = np.empty((kend, S), dtype=np.int64)  # re-encoded with floor digits
        q[:, 0] = V >> (7 * (S - 1))
        for s in range(1, S):
            q[:, s] = (V >> (7 * (S - 1 - s))) & 127
        out[slice_offsets(i, k, np_)] = q.astype(np.int8)
    return out


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

    def identity_share(self, layout):
        B = self.zeros(layout.n_loc, layout.m_loc)
        for I in layout.row_blocks:
            if I in layout.col_blocks:
                self.set_diag(B, layout.lrow(I), layout.lcol(I), 0, layout.nb, 1.0, add=False)
        return B

    def set_diag(self, A, r0, c0, lo, hi, value, add):
        if hi <= lo:
            return
        idx = torch.arange(lo, hi)
        if add:
            A[c0 + idx, r0 + idx] += value
        else:
            A[c0 + idx, r0 + idx] = value

    def potrf_inv(self, A, r0, c0, nb):
        blk = A[c0:c0 + nb, r0:r0 + nb].numpy().T
        L, info = dpotrf(np.ascontiguousarray(blk), lower=1, clean=1)
        if info > 0:
            return info - 1, self.zeros(nb, nb), self.zeros(nb, nb)
        Li = solve_triangular(L, np.eye(nb), lower=True)
        return -1, self.from_host(L), self.from_host(np.tril(Li))

    def trtri(self, A, r0, c0, nb):
        blk = np.tril(A[c0:c0 + nb, r0:r0 + nb].numpy().T)
        return self.from_host(solve_triangular(blk, np.eye(nb), lower=True))

    def kinship_blocks(self, spec, layout):
        """Host restatement of DeviceOps.kinship_blocks (datagen's construction per block)."""
        from paper_1304_2272_b200 import datagen

        Z = np.zeros((layout.n_pad, spec.m_kin))
        Z[:spec.n] = datagen.standardized_host(spec.seed, spec.n, spec.m_kin, spec.maf)
        rows = layout.global_rows(layout.row_blocks)
        cols = layout.global_rows(layout.col_blocks)
        A = (Z[rows] @ Z[cols].T) / spec.m_kin * spec.a
        d = rows[:, None] == cols[None, :]
        A[d & (rows[:, None] < spec.n)] += 1.0 - spec.a
        return self.from_host(A)

    def gemm(self, C, cr, cc, m, n, A, ar, ac, B, br, bc, k, alpha, beta, trans_b):
        if m == 0 or n == 0:
            return
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

    def copy_rows(self, dst, dst_rows, src, src_rows):
        dst[:, torch.as_tensor(dst_rows)] = src[:, torch.as_tensor(src_rows)]

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

    def _tril_share(self, B, layout):
        np_ = -(-layout.n // 128) * 128
        full = self._full_share(B, layout)
        out = np.zeros((np_, np_))
        m = min(np_, full.shape[0])
        out[:m, :m] = full[:m, :m]
        return np.tril(out), np_

    def row_exponents(self, B, layout):
        full, _ = self._tril_share(B, layout)
        return torch.from_numpy(row_exponents_dense(full))

    def slice_meta(self, ex2, layout):
        return torch.from_numpy(slice_meta_dense(ex2.numpy()))

    def slice_blockcyclic(self, B, layout, meta):
        full, np_ = self._tril_share(B, layout)
        S = slices_dense(lambda i, kend: full[i, :kend], meta.numpy(), np_)
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
