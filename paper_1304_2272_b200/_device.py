"""Device-side data layout and the resident context of the GLS sweep.

Layout in HBM: every matrix whose rows run over the n individuals is column-major
FP64 with its rows padded to np = pad(n) (multiple of 128).  A torch tensor of shape
(ncols, ld) (row-major) holds such a matrix: column j is the contiguous row ``t[j, :]``.
Padding rows of right-hand sides are zero; L and Linv carry the identity on the padding block.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import check, pad, ptr, stream_handle


def _torch():
    import torch

    return torch


_TORCH_DTYPES = {
    np.float64: lambda: _torch().float64,
    np.int8: lambda: _torch().int8,
    np.int32: lambda: _torch().int32,
}


def alloc_cols(ncols, ld, dtype=None, zero=True):
    """Column-major (ld x ncols) device buffer as a (ncols, ld) torch tensor."""
    torch = _torch()
    dtype = dtype or torch.float64
    dev = _capi.device()
    if zero:
        return torch.zeros((max(int(ncols), 0), int(ld)), dtype=dtype, device=dev)
    return torch.empty((max(int(ncols), 0), int(ld)), dtype=dtype, device=dev)


def upload_cols(A, ld=None, out=None, pinned=False):
    """Host (nrows x ncols) array -> column-major device buffer with rows padded to ``ld``.

    Rows beyond ``nrows`` are zero.  A may be any layout; a 1-D array is one column."""
    torch = _torch()
    A = np.asarray(A)
    if A.ndim == 1:
        A = A[:, None]
    nrows, ncols = A.shape
    ld = pad(nrows) if ld is None else ld
    if out is None:
        out = alloc_cols(ncols, ld, dtype=_TORCH_DTYPES[A.dtype.type]())
    host = torch.from_numpy(np.asfortranarray(A).T)   # (ncols, nrows), C-contiguous view
    if pinned:
        host = host.pin_memory()
    out[:ncols, :nrows].copy_(host, non_blocking=pinned)
    return out


def download_cols(t, nrows, ncols=None):
    """Column-major device buffer -> host (nrows x ncols) F-ordered numpy array."""
    ncols = t.shape[0] if ncols is None else ncols
    return t[:ncols, :nrows].cpu().numpy().T


def transpose_square(A):
    """Row-major copy (as a column-major matrix: T = A^T) of a square (np, np) device buffer."""
    T = alloc_cols(A.shape[0], A.shape[1], zero=False)
    check(_capi.lib().gg_transpose_f64(A.shape[1], ptr(A), A.shape[1], ptr(T), T.shape[1],
                                       stream_handle()), "gg_transpose_f64")
    return T


def upload_square_identity_padded(A, n, ld):
    """Host n x n lower-triangular matrix -> (ld x ld) device buffer extended by the identity."""
    torch = _torch()
    out = alloc_cols(ld, ld)
    upload_cols(np.asarray(A, dtype=np.float64), ld=ld, out=out)
    if ld > n:
        idx = torch.arange(n, ld, device=out.device)
        out[idx, idx] = 1.0
    return out


@dataclass
class DeviceContext:
    """Marker-independent state resident on one GPU (the device half of PreparedContext)."""

    n: int
    np_: int
    q: int
    L: object          # (np, np) col-major factor, or None (contexts built from host fields)
    LinvP: object      # packed tile-major lower inverse (TMA TRSM operand), or None
    XLy: object        # (q + 1, np): whitened covariates, then whitened phenotype
    S_TL: object       # (q * q,) row-major
    b_T: object        # (q,)
    slices: object = None   # int8 slices of the inverse (tile-packed) for the tensor-core TRSM
    expo: object = None     # slice metadata: row exponents, diagonal heads (2 np int32)

    @property
    def p(self):
        return self.q + 1

    @property
    def XLbar(self):
        return self.XLy[: self.q]

    @property
    def ybar(self):
        return self.XLy[self.q]

    @classmethod
    def from_host(cls, XLbar, ybar, S_TL, b_T):
        """Device copies of the small prepared fields (for contexts built by callers, e.g. the
        reference's run_dist at distgrid.py:385-386)."""
        torch = _torch()
        XLbar = np.asarray(XLbar, dtype=np.float64)
        ybar = np.asarray(ybar, dtype=np.float64).ravel()
        n, q = XLbar.shape
        np_ = pad(n)
        XLy = upload_cols(np.column_stack([XLbar, ybar]), ld=np_)
        dev = XLy.device
        S = torch.from_numpy(np.ascontiguousarray(S_TL, dtype=np.float64).ravel()).to(dev)
        b = torch.from_numpy(np.ascontiguousarray(b_T, dtype=np.float64).ravel()).to(dev)
        return cls(n=n, np_=np_, q=q, L=None, LinvP=None, XLy=XLy, S_TL=S, b_T=b)


class BlockWorkspace:
    """Reusable device buffers for streamed blocks of up to ``m_blk`` SNPs (no per-block
    allocation on the hot loop)."""

    def __init__(self, dctx, m_blk, emit_s_inv=False, int8_input=False):
        torch = _torch()
        self.dctx = dctx
        self.m_blk = int(m_blk)
        self.int8_input = bool(int8_input)
        p = dctx.p
        dev = _capi.device()
        have_slices = dctx.slices is not None
        nbytes = int(_capi.lib().gg_gls_block_workspace_bytes(
            dctx.n, dctx.q, self.m_blk, 1 if int8_input else 0, 1 if have_slices else 0))
        self.work = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.beta = torch.empty((self.m_blk, p), dtype=torch.float64, device=dev)
        self.status = torch.empty((self.m_blk,), dtype=torch.int32, device=dev)
        self.sinv = (torch.empty((self.m_blk, p * (p + 1) // 2), dtype=torch.float64, device=dev)
                     if emit_s_inv else None)

    def run(self, cnt, X64=None, ldx=0, G8=None, ldg=0, stream=None):
        """TRSM + reductions + small solves for ``cnt`` columns already on the device."""
        d = self.dctx
        if cnt > self.m_blk:
            raise ValueError("block larger than the workspace")
        if d.LinvP is None and d.slices is None:
            raise ValueError("context has no device factor (prepared from host fields only)")
        if (G8 is not None) != self.int8_input:
            raise ValueError("input kind does not match the workspace")
        s = stream_handle() if stream is None else stream
        rc = _capi.lib().gg_gls_block_f64(
            d.n, d.q, int(cnt), ptr(d.LinvP), ptr(d.slices), ptr(d.expo), ptr(d.XLy),
            ptr(d.ybar), ptr(d.S_TL), ptr(d.b_T), ptr(X64), int(ldx), ptr(G8), int(ldg),
            ptr(self.work), ptr(self.beta), ptr(self.status), ptr(self.sinv), s)
        check(rc, "gg_gls_block_f64")
