"""Drop-in for ``gwasgls.kernel`` (reference pkg/src/gwasgls/kernel.py) on the B200.

Same names, signatures, return types, in-place behaviour and exceptions as the reference; the
arithmetic runs in libgwasgls_b200.so (sm_100a FP64 DMMA kernels) through the C-ABI.  There is
no CPU fallback: without a CUDA device or the native library every entry point raises
``DeviceError``.

    b_i = (X_i^T M^-1 X_i)^-1 X_i^T M^-1 y

``gls_prepare`` factors M once (blocked Cholesky + triangular inverse, kept resident on the
device), whitens X_L and y, and forms S_TL / b_T; ``gls_solve_block`` streams one block of SNP
columns through the TRSM (Linv * X on DMMA tiles) and the fused epilogue (reductions + batched
p x p Cholesky solve).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import check, pad, ptr, stream_handle
from ._device import (
    BlockWorkspace,
    DeviceContext,
    alloc_cols,
    download_cols,
    upload_cols,
    upload_square_identity_padded,
)
from .errors import DeviceError, DimensionMismatch, NotPositiveDefinite, RankDeficientCovariates

EPS = 2.0 ** -52   # kernel.py:28


@dataclass
class SnpBlock:
    """A contiguous run of marker columns (allele dosages), n x count (kernel.py:31-48).

    ``data`` is FP64 as in the reference; int8 dosages are accepted too and widened on the
    device (the BASELINE config-2 genotype stream)."""

    first_index: int
    data: np.ndarray

    def __post_init__(self):
        if self.data.ndim != 2 or self.data.shape[1] < 1:
            raise DimensionMismatch("SnpBlock needs an n x count matrix with count >= 1")

    @property
    def n(self):
        return self.data.shape[0]

    @property
    def count(self):
        return self.data.shape[1]


@dataclass
class SnpResult:
    """Per-marker output (kernel.py:51-59)."""

    snp_index: int
    beta: np.ndarray
    s_inv: np.ndarray | None = None
    status: str = "ok"


class _LazyResults:
    """Read-only sequence of SnpResult views over the block's result arrays.

    The reference builds one Python object per SNP (kernel.py:295-311, ~1.4 us/SNP); here the
    objects are materialised on access, so the streaming engines never pay for them."""

    def __init__(self, arrays):
        self._a = arrays

    def __len__(self):
        return self._a.count

    def _one(self, k):
        a = self._a
        gidx = a.first_index + k if a.global_indices is None else int(a.global_indices[k])
        if a.status[k] == -1:
            return SnpResult(snp_index=gidx, beta=a.beta[k],
                             s_inv=a.sinv[k] if a.sinv is not None else None, status="ok")
        return SnpResult(snp_index=gidx, beta=np.full(a.beta.shape[1], np.nan), s_inv=None,
                         status="degenerate")

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self._one(i) for i in range(*k.indices(len(self)))]
        if k < 0:
            k += len(self)
        if not 0 <= k < len(self):
            raise IndexError(k)
        return self._one(k)

    def __iter__(self):
        for k in range(len(self)):
            yield self._one(k)

    def __eq__(self, other):
        return list(self) == list(other)

    def __add__(self, other):
        return list(self) + list(other)

    def __radd__(self, other):
        return list(other) + list(self)


@dataclass
class ResultArrays:
    """Array form of a block's results: beta (cnt x p, NaN rows for degenerate markers),
    status (cnt; -1 ok, else first failing pivot), optional packed S^-1."""

    first_index: int
    beta: np.ndarray
    status: np.ndarray
    sinv: np.ndarray | None = None
    global_indices: np.ndarray | None = None

    def __post_init__(self):
        if np.any(self.status == STATUS_INVALID):
            raise DeviceError(
                "block holds dosages the int8 tensor-core path cannot compute exactly and the "
                "context has no FP64 inverse to fall back on (distributed engine: use "
                "DistConfig(fp64_inverse=True))")

    @property
    def count(self):
        return self.beta.shape[0]

    @property
    def ok(self):
        return self.status == -1


class ResultBlock:
    """(kernel.py:62-65).  ``results`` is list-like; ``arrays`` (when present) is the array
    form used by the vectorised BlockWriter.

    A block returned by ``gls_solve_block`` may still be computing on the device when the call
    returns (its input has been copied, so the caller may reuse the buffer, as the reference's
    double buffer does, pipeline.py:195-212): the first read of ``results`` or ``arrays`` waits
    for it.  That lets consecutive calls overlap the next block's host->device copy with this
    block's TRSM."""

    def __init__(self, first_index, results=None, arrays=None):
        self.first_index = first_index
        self._results = [] if results is None and arrays is None else results
        self._arrays = arrays
        self._pending = None

    @classmethod
    def from_arrays(cls, arrays):
        return cls(first_index=arrays.first_index, results=_LazyResults(arrays), arrays=arrays)

    @classmethod
    def pending(cls, first_index, resolve):
        """A block whose arrays come from ``resolve()`` on first access."""
        b = cls(first_index)
        b._pending = resolve
        return b

    def _resolve(self):
        if self._pending is not None:
            resolve, self._pending = self._pending, None
            arrays = resolve()
            self._arrays = arrays
            self._results = _LazyResults(arrays)

    @property
    def done(self):
        return self._pending is None

    @property
    def results(self):
        self._resolve()
        return self._results

    @results.setter
    def results(self, value):
        self._pending = None
        self._results = value

    @property
    def arrays(self):
        self._resolve()
        return self._arrays

    @arrays.setter
    def arrays(self, value):
        self._pending = None
        self._arrays = value

    def __eq__(self, other):
        if not isinstance(other, ResultBlock) and not hasattr(other, "results"):
            return NotImplemented
        return self.first_index == other.first_index and list(self.results) == list(other.results)

    def __repr__(self):
        state = "pending" if self._pending is not None else f"{len(self.results)} results"
        return f"ResultBlock(first_index={self.first_index}, {state})"


class PreparedContext:
    """Marker-independent quantities (kernel.py:68-89).

    Host fields L, XLbar, ybar, S_TL, b_T keep the reference's meaning (numpy arrays); the
    factor lives on the device (``_dev``) and ``L`` is downloaded only when read."""

    def __init__(self, L=None, XLbar=None, ybar=None, S_TL=None, b_T=None, _dev=None):
        self._L = L
        self.XLbar = XLbar
        self.ybar = ybar
        self.S_TL = S_TL
        self.b_T = b_T
        self._dev = _dev

    @property
    def L(self):
        if self._L is None and self._dev is not None and self._dev.L is not None:
            self._L = np.asfortranarray(download_cols(self._dev.L, self._dev.n, self._dev.n))
        return self._L

    @L.setter
    def L(self, value):
        self._L = value

    @property
    def n(self):
        if self._dev is not None:
            return self._dev.n
        return self.XLbar.shape[0]

    @property
    def p(self):
        return self.XLbar.shape[1] + 1

    def device(self):
        """Device half of the context, built from the host fields when missing."""
        if self._dev is None:
            self._dev = DeviceContext.from_host(self.XLbar, self.ybar, self.S_TL, self.b_T)
        return self._dev

    def __repr__(self):
        return f"PreparedContext(n={self.n}, p={self.p}, device={self._dev is not None})"


# ---------------------------------------------------------------------------------------------
# factorisation and triangular solves
# ---------------------------------------------------------------------------------------------

def _pack_lower(Linv_colmajor, n):
    """Square column-major inverse -> packed tile-major lower tiles (the TRSM's A operand)."""
    torch = __import__("torch")
    P = torch.empty(int(_capi.lib().gg_packed_lower_bytes(n)) // 8, dtype=torch.float64,
                    device=Linv_colmajor.device)
    check(_capi.lib().gg_pack_lower_f64(n, ptr(Linv_colmajor), Linv_colmajor.shape[1], 0, ptr(P),
                                        stream_handle()), "gg_pack_lower_f64")
    return P


def _slice_inverse(Linv_colmajor, n):
    """int8 slices + metadata (row exponents, diagonal heads) of the inverse: the operands of the
    tensor-core TRSM."""
    torch = __import__("torch")
    from ._device import transpose_square

    LinvT = transpose_square(Linv_colmajor)
    sl = torch.empty(int(_capi.lib().gg_inverse_slices_bytes(n)), dtype=torch.int8,
                     device=LinvT.device)
    expo = torch.empty(int(_capi.lib().gg_slice_meta_ints(n)), dtype=torch.int32,
                       device=LinvT.device)
    check(_capi.lib().gg_slice_inverse_i8(n, ptr(LinvT), LinvT.shape[1], ptr(sl), ptr(expo),
                                          stream_handle()), "gg_slice_inverse_i8")
    del LinvT
    return sl, expo


def _slices_fit(n):
    """Room for the int8 slices (3.5 np^2 bytes) next to what is already resident."""
    torch = __import__("torch")
    free, _ = torch.cuda.mem_get_info(_capi.device())
    return int(_capi.lib().gg_inverse_slices_bytes(n)) < 0.8 * free


def _slice_packed(LinvP, n):
    """int8 slices + metadata from the packed FP64 inverse."""
    torch = __import__("torch")
    sl = torch.empty(int(_capi.lib().gg_inverse_slices_bytes(n)), dtype=torch.int8,
                     device=LinvP.device)
    expo = torch.empty(int(_capi.lib().gg_slice_meta_ints(n)), dtype=torch.int32,
                       device=LinvP.device)
    check(_capi.lib().gg_slice_packed_inverse_i8(n, ptr(LinvP), ptr(sl), ptr(expo),
                                                 stream_handle()), "gg_slice_packed_inverse_i8")
    return sl, expo


STATUS_INVALID = -2   # GG_STATUS_INVALID (include/gwasgls_b200.h)


def _int8_exact(col):
    """Integer values the int8 tensor-core path computes exactly at this n (the int32 bound of
    gg_i8_value_bound: 127 up to n = 132,104)."""
    bound = _capi.lib().gg_i8_value_bound(len(col))
    return bool(np.all(np.isfinite(col)) and np.all(col == np.trunc(col))
                and np.all(np.abs(col) <= bound))


def _trsm_i8_device(slices, expo, n, A):
    """X = L^-1 A for a host matrix of int8-exact columns, on the tensor-core path."""
    torch = __import__("torch")
    n16 = -(-n // 16) * 16
    A = np.asarray(A)
    G = torch.zeros((A.shape[1], n16), dtype=torch.int8)
    G[:, :n] = torch.from_numpy(np.ascontiguousarray(A.T).astype(np.int8))
    G = G.to(slices.device)
    X = alloc_cols(A.shape[1], pad(n))
    work = _capi.i8_work(slices.device)
    check(_capi.lib().gg_trsm_lower_i8(n, A.shape[1], ptr(slices), ptr(expo), ptr(G), n16, ptr(X),
                                       pad(n), ptr(work), stream_handle()), "gg_trsm_lower_i8")
    return X


def _potrf_device(M, keep_square_inverse=False):
    """Device Cholesky + inverse of the n x n matrix M (host array, or CUDA tensor read
    row-major); returns (n, L_dev, LinvP_dev) with the inverse in the packed tile-major layout
    (the A operand of the TMA TRSM), plus the square column-major inverse if asked."""
    torch = __import__("torch")
    n = M.shape[0]
    np_ = pad(n)
    if isinstance(M, np.ndarray):
        # the C-contiguous buffer goes up as is; the kernels read it row-major (no host transpose)
        Md = torch.from_numpy(np.ascontiguousarray(M, dtype=np.float64)).to(_capi.device())
    else:
        Md = M.contiguous()                      # device tensor, row-major (n, n)
    L = alloc_cols(np_, np_, zero=False)
    Linv = alloc_cols(np_, np_, zero=False)
    ws = torch.empty(int(_capi.lib().gg_potrf_workspace_bytes(n)), dtype=torch.uint8,
                     device=Md.device)
    info = (_capi.C.c_int * 2)()
    rc = _capi.lib().gg_potrf_f64(n, ptr(Md), n, 1, ptr(L), ptr(Linv), np_, ptr(ws), info,
                                  stream_handle())
    del Md
    if rc == _capi.GG_ENOTPD:
        if info[1]:
            raise NotPositiveDefinite(int(info[0]), "non-finite entry in covariance")
        raise NotPositiveDefinite(int(info[0]))
    check(rc, "gg_potrf_f64")
    LinvP = _pack_lower(Linv, n)
    if keep_square_inverse:
        return n, L, LinvP, Linv
    del Linv
    return n, L, LinvP


def cholesky_spd(M):
    """Lower Cholesky factor of an SPD matrix (kernel.py:92-109).

    The input is not modified; raises NotPositiveDefinite carrying the 0-based pivot (or, for
    non-finite input, the row of the first non-finite entry in row-major order)."""
    M = np.ascontiguousarray(M, dtype=np.float64)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise DimensionMismatch("covariance must be square")
    n, L, _ = _potrf_device(M)
    return np.asfortranarray(download_cols(L, n, n))


def _trtri_device(L):
    """Device inverse of a host lower-triangular L; returns (n, LinvP_dev) (packed tiles)."""
    torch = __import__("torch")
    n = L.shape[0]
    np_ = pad(n)
    Ld = upload_square_identity_padded(np.tril(L), n, np_)
    Linv = alloc_cols(np_, np_, zero=False)
    ws = torch.empty(int(_capi.lib().gg_trtri_workspace_bytes(n)), dtype=torch.uint8,
                     device=Ld.device)
    check(_capi.lib().gg_trtri_lower_f64(n, ptr(Ld), np_, ptr(Linv), np_, ptr(ws),
                                         stream_handle()), "gg_trtri_lower_f64")
    return n, _pack_lower(Linv, n)


def _trsm_device(dLinvP, n, B_dev, nrhs):
    """X = L^-1 B on the device (TMA/DMMA kernel; LinvP is the packed inverse)."""
    np_ = pad(n)
    X = alloc_cols(nrhs, np_, zero=False)
    check(_capi.lib().gg_trsm_lower_packed_f64(n, nrhs, ptr(dLinvP), ptr(B_dev), B_dev.shape[1],
                                               ptr(X), np_, stream_handle()),
          "gg_trsm_lower_packed_f64")
    return X


def trsolve_lower(L, B):
    """Solve L X = B for X with L lower triangular, column by column (kernel.py:112-121)."""
    L = np.asarray(L, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    squeeze = B.ndim == 1
    if squeeze:
        B = B[:, None]
    if L.ndim != 2 or L.shape[0] != L.shape[1] or L.shape[0] != B.shape[0]:
        raise DimensionMismatch(f"trsolve: L is {L.shape}, B is {B.shape}")
    n, nrhs = B.shape
    if nrhs == 0:
        return np.empty((n, 0)) if not squeeze else np.empty(n)
    # blocked forward substitution on the device (diagonal-block inverses + DMMA GEMM updates):
    # O(n^2 nrhs) and backward-stable like dtrsm, no O(n^3) explicit inverse per call
    torch = __import__("torch")
    np_ = pad(n)
    Ld = upload_square_identity_padded(np.tril(L), n, np_)
    Bd = upload_cols(B, ld=np_)
    ws = torch.empty(int(_capi.lib().gg_trsm_lower_blocked_workspace_bytes(n, nrhs)),
                     dtype=torch.uint8, device=Ld.device)
    check(_capi.lib().gg_trsm_lower_blocked_f64(n, nrhs, ptr(Ld), np_, ptr(Bd), np_, ptr(Bd), np_,
                                                ptr(ws), stream_handle()),
          "gg_trsm_lower_blocked_f64")
    X = np.asfortranarray(download_cols(Bd, n, nrhs))
    return X[:, 0] if squeeze else X


# ---------------------------------------------------------------------------------------------
# reductions and small systems
# ---------------------------------------------------------------------------------------------

def _dots_device(Xd, n, cnt, XLd, q, yd):
    """dots (cnt x (q+2)) of the device columns Xd against XLd (q columns) and yd."""
    torch = __import__("torch")
    out = torch.empty((max(cnt, 1), q + 2), dtype=torch.float64, device=Xd.device)
    work = torch.empty(max(int(_capi.lib().gg_partials_bytes(n, max(cnt, 1), q)), 8),
                       dtype=torch.uint8, device=Xd.device)
    check(_capi.lib().gg_gls_dots_f64(n, cnt, q, ptr(Xd), Xd.shape[1],
                                      ptr(XLd) if q > 0 else None,
                                      XLd.shape[1] if q > 0 else pad(n), ptr(yd), ptr(out),
                                      ptr(work), stream_handle()), "gg_gls_dots_f64")
    return out[:cnt]


def gram(A):
    """A^T A with exact stored symmetry (kernel.py:124-131), on the device with the same
    summation order as the per-SNP reductions."""
    A = np.asarray(A, dtype=np.float64)
    if A.ndim != 2:
        raise DimensionMismatch("gram expects a matrix")
    n, k = A.shape
    if k == 0:
        return np.zeros((0, 0))
    Ad = upload_cols(A)
    zeros = alloc_cols(1, Ad.shape[1])
    C = _dots_device(Ad, n, k, Ad, k, zeros[0]).cpu().numpy()[:, :k]
    return np.tril(C) + np.tril(C, -1).T


def _small_solve_device(S, rhs, want_inverse):
    torch = __import__("torch")
    B, p, _ = S.shape
    dev = _capi.device()
    Sd = torch.from_numpy(np.ascontiguousarray(S)).to(dev)
    rd = torch.from_numpy(np.ascontiguousarray(rhs)).to(dev)
    x = torch.empty((B, p), dtype=torch.float64, device=dev)
    st = torch.empty((B,), dtype=torch.int32, device=dev)
    si = (torch.empty((B, p * (p + 1) // 2), dtype=torch.float64, device=dev)
          if want_inverse else None)
    check(_capi.lib().gg_small_spd_solve_f64(B, p, ptr(Sd), ptr(rd), ptr(x), ptr(st), ptr(si),
                                             stream_handle()), "gg_small_spd_solve_f64")
    return x.cpu().numpy(), st.cpu().numpy(), (si.cpu().numpy() if si is not None else None)


def cholesky_solve_batch(S, rhs, want_inverse=False):
    """Solve S[k] x[k] = rhs[k] for a batch of small SPD systems (kernel.py:138-208).

    Pivot rule d > p * eps * max|S[k]| (kernel.py:134-135); failed systems come back NaN with
    ok[k] = False.  Returns (x, ok) or (x, ok, s_inv_packed) in np.tril_indices order."""
    S = np.asarray(S, dtype=np.float64)
    rhs = np.asarray(rhs, dtype=np.float64)
    if S.ndim != 3 or S.shape[1] != S.shape[2] or rhs.shape != S.shape[:2]:
        raise DimensionMismatch("cholesky_solve_batch: S is (B,p,p), rhs is (B,p)")
    B, p, _ = S.shape
    if B == 0:
        x = np.empty((0, p))
        return (x, np.ones(0, dtype=bool)) if not want_inverse else \
            (x, np.ones(0, dtype=bool), np.empty((0, p * (p + 1) // 2)))
    x, st, packed = _small_solve_device(S, rhs, want_inverse)
    ok = st < 0
    if not want_inverse:
        return x, ok
    return x, ok, packed


def solve_small_spd(S, rhs):
    """Solve one small SPD system S x = rhs via Cholesky (kernel.py:211-230); raises
    NotPositiveDefinite with the first failing pivot."""
    S = np.asarray(S, dtype=np.float64)
    rhs = np.asarray(rhs, dtype=np.float64)
    if S.ndim != 2 or S.shape[0] != S.shape[1] or S.shape[0] != rhs.shape[0]:
        raise DimensionMismatch("solve_small_spd: shapes disagree")
    x, st, _ = _small_solve_device(S[None], rhs[None], False)
    if st[0] >= 0:
        raise NotPositiveDefinite(int(st[0]))
    return x[0]


# ---------------------------------------------------------------------------------------------
# the GLS sweep
# ---------------------------------------------------------------------------------------------

def gls_prepare(M, XL, y, int8_split=True):
    """Hoist all marker-independent work (kernel.py:233-257): factor M (device Cholesky +
    inverse, kept resident), whiten XL and y with the same TRSM kernel as the SNP blocks, and
    form S_TL and b_T with the same reduction kernel as the per-SNP sums.

    M may also be a CUDA float64 tensor (n, n) already resident on the device (row-major, as a
    C-contiguous array would be): the factorisation then reads it in place, no host round trip.

    int8_split (default) also stores the inverse as int8 slices so that dosage blocks run on
    the int8 tensor cores (exact integer products, FP64 recombination); False keeps only the
    FP64 DMMA TRSM."""
    torch = __import__("torch")
    if not (isinstance(M, torch.Tensor) and M.is_cuda and M.dtype == torch.float64):
        M = np.ascontiguousarray(M, dtype=np.float64)
    XL = np.asarray(XL, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64).ravel()
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise DimensionMismatch("covariance must be square")
    n = M.shape[0]
    if XL.ndim != 2 or XL.shape[0] != n or y.shape[0] != n:
        raise DimensionMismatch(f"gls_prepare: n={n} but XL {XL.shape}, y {y.shape}")
    q = XL.shape[1]
    if q + 1 > _capi.GG_PMAX:
        raise DimensionMismatch(f"p = {q + 1} exceeds the supported maximum {_capi.GG_PMAX}")
    torch.cuda.nvtx.range_push("gls_prepare")
    try:
        _, L, LinvP, Linv = _potrf_device(M, keep_square_inverse=True)
        slices, expo = _slice_inverse(Linv, n) if int8_split else (None, None)
        del Linv
        return prepare_from_inverse(LinvP, n, XL, y, L=L, slices=slices, expo=expo,
                                    int8_split=int8_split)
    finally:
        torch.cuda.nvtx.range_pop()


def prepare_from_inverse(LinvP, n, XL, y, L=None, slices=None, expo=None, XLy=None,
                         int8_split=True):
    """The marker-independent tail of gls_prepare (kernel.py:246-257) given the inverse:
    whiten [X_L | y] with the streamed TRSM kernel, S_TL = gram(X_L bar) and b_T with the
    per-SNP reduction kernel, SPD check of S_TL.  Shared by gls_prepare and the distributed
    engine, whose factor exists only block-cyclically (L None); at config-4 sizes that engine
    also has no replicated FP64 inverse (LinvP None) and passes the whitened [X_L | y] (XLy,
    device, (q + 1, gg_pad(n))) it formed itself plus the int8 slices, and without LinvP no
    slices are cut here (slices come from the caller)."""
    torch = __import__("torch")
    XL = np.asarray(XL, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64).ravel()
    q = XL.shape[1]
    np_ = pad(n)
    if XLy is None:
        RHS = upload_cols(np.column_stack([XL, y]), ld=np_)
        XLy = _trsm_device(LinvP, n, RHS, q + 1)
    if int8_split and slices is None and LinvP is not None and _slices_fit(n):
        slices, expo = _slice_packed(LinvP, n)
    if slices is not None:
        # covariate columns that are exact small integers (the intercept) are whitened by the
        # same tensor-core kernel as the dosage blocks, so a SNP equal to such a column gives
        # an exactly singular S (degenerate-SNP fixture)
        ints = [j for j in range(q) if _int8_exact(XL[:, j])]
        if ints:
            Xi = _trsm_i8_device(slices, expo, n, XL[:, ints])
            for c, j in enumerate(ints):
                XLy[j].copy_(Xi[c])
    dev = XLy.device
    dots = _dots_device(XLy, n, q, XLy, q, XLy[q]) if q > 0 else None
    if q > 0:
        C = dots[:, :q]
        S_TL_d = (torch.tril(C) + torch.tril(C, -1).T).contiguous()
        b_T_d = dots[:, q + 1].contiguous()
        x = torch.empty((1, q), dtype=torch.float64, device=dev)
        st = torch.empty((1,), dtype=torch.int32, device=dev)
        zero = torch.zeros((1, q), dtype=torch.float64, device=dev)
        check(_capi.lib().gg_small_spd_solve_f64(1, q, ptr(S_TL_d), ptr(zero), ptr(x), ptr(st),
                                                 None, stream_handle()),
              "gg_small_spd_solve_f64")
        piv = int(st.cpu()[0])
        if piv >= 0:
            raise RankDeficientCovariates(
                f"whitened covariates are rank deficient (pivot {piv})")
        S_TL = S_TL_d.cpu().numpy().reshape(q, q)
        b_T = b_T_d.cpu().numpy()
    else:
        S_TL_d = torch.zeros((0,), dtype=torch.float64, device=dev)
        b_T_d = torch.zeros((0,), dtype=torch.float64, device=dev)
        S_TL, b_T = np.zeros((0, 0)), np.zeros(0)
    host = download_cols(XLy, n, q + 1)
    XLbar = np.asfortranarray(host[:, :q])
    ybar = np.ascontiguousarray(host[:, q])
    dctx = DeviceContext(n=n, np_=np_, q=q, L=L, LinvP=LinvP, XLy=XLy, S_TL=S_TL_d.reshape(-1),
                         b_T=b_T_d, slices=slices, expo=expo)
    return PreparedContext(L=None, XLbar=XLbar, ybar=ybar, S_TL=S_TL, b_T=b_T, _dev=dctx)


def _collect(ws, cnt, first_index, global_indices, emit_s_inv):
    beta = ws.beta[:cnt].cpu().numpy()
    status = ws.status[:cnt].cpu().numpy()
    sinv = ws.sinv[:cnt].cpu().numpy() if emit_s_inv else None
    gi = None if global_indices is None else np.asarray(global_indices)
    return ResultBlock.from_arrays(ResultArrays(first_index=first_index, beta=beta,
                                                status=status, sinv=sinv, global_indices=gi))


def device_context(ctx, need_factor=False):
    """Device half of any PreparedContext-like object (ours, or the reference's dataclass built
    by a caller such as run_dist, distgrid.py:385).  Built from the host fields on first use and
    cached on the object; with ``need_factor`` the inverse is derived from ``ctx.L`` unless the
    context already carries one (packed FP64 or, in the distributed config-4 form, only the int8
    slices: blocks that need FP64 then come back invalid)."""
    d = getattr(ctx, "_dev", None)
    if d is None:
        d = DeviceContext.from_host(ctx.XLbar, ctx.ybar, ctx.S_TL, ctx.b_T)
        ctx._dev = d
    if need_factor and d.LinvP is None and d.slices is None:
        L = np.asarray(ctx.L, dtype=np.float64)
        if L.ndim != 2 or L.shape != (d.n, d.n):
            raise DimensionMismatch("context has no usable Cholesky factor for the TRSM")
        _, d.LinvP = _trtri_device(L)
        if d.slices is None and _slices_fit(d.n):   # dosage blocks then take the int8 path
            d.slices, d.expo = _slice_packed(d.LinvP, d.n)
    return d


def solve_whitened_block(ctx, Xbar, first_index, global_indices=None, emit_s_inv=False):
    """Per-marker assembly and solve for already-whitened columns Xbar (n x count)
    (kernel.py:273-312); the fused device epilogue.  Returns a list of SnpResult."""
    torch = __import__("torch")
    d = device_context(ctx)
    Xbar = np.asarray(Xbar, dtype=np.float64)
    if Xbar.ndim != 2 or Xbar.shape[0] != d.n:
        raise DimensionMismatch(f"Xbar has shape {Xbar.shape}, context has n={d.n}")
    cnt = Xbar.shape[1]
    ws = BlockWorkspace(d, max(cnt, 1), emit_s_inv=emit_s_inv)
    if cnt:
        Xd = upload_cols(Xbar, ld=d.np_)
        work = torch.empty(int(_capi.lib().gg_partials_bytes(d.n, cnt, d.q)), dtype=torch.uint8,
                           device=Xd.device)
        check(_capi.lib().gg_gls_epilogue_f64(
            d.n, cnt, d.q, ptr(Xd), d.np_, ptr(d.XLy), d.np_, ptr(d.ybar), ptr(d.S_TL),
            ptr(d.b_T), ptr(ws.beta), ptr(ws.status), ptr(ws.sinv), ptr(work), stream_handle()),
            "gg_gls_epilogue_f64")
    return list(_collect(ws, cnt, first_index, global_indices, emit_s_inv).results)


class _BlockStream:
    """One calling thread's device stream for gls_solve_block: a pipeline.StreamEngine (pinned
    result buffers, copy + compute streams, DEV_REGIONS device regions) plus the blocks still
    pending in its regions.  A block's region is resolved (results copied to the host) before it
    is reused, so a caller may hold any number of unresolved ResultBlocks."""

    def __init__(self, engine):
        self.engine = engine
        self.owner = {}            # device region -> its pending ResultBlock

    def submit(self, data, first, cnt):
        eng = self.engine
        r = eng._next % eng.DEV_REGIONS
        prev = self.owner.pop(r, None)
        if prev is not None:
            prev._resolve()         # frees region r (collect -> host arrays)
        t = eng.begin(first, cnt)
        try:
            eng.h2d(t, data, 0, cnt, slot=t)
        except Exception:
            eng.busy[t] = False
            raise
        eng.launch(t)
        # the caller may reuse `data` once this returns (the reference's double buffer,
        # pipeline.py:195-212): wait for the copy, not for the compute
        eng.wait_h2d(t)
        blk = ResultBlock.pending(first, lambda: self._collect(t))
        self.owner[t] = blk
        return blk

    def _collect(self, t):
        self.owner.pop(t, None)
        return self.engine.collect(t)


_streams_lock = threading.Lock()


def _block_stream(ctx, d, int8, emit_s_inv, cnt):
    """The calling thread's block stream for this device context and input kind (rebuilt with
    more room when a larger block arrives).  Kept on the context itself, so it lives and dies
    with it; one per thread (run_spmd's inproc ranks call concurrently, transport.py:279-291)."""
    from . import pipeline

    with _streams_lock:
        cache = d.__dict__.setdefault("_block_streams", {})
    key = (threading.get_ident(), bool(int8), bool(emit_s_inv), _capi.device().index)
    bs = cache.get(key)
    if bs is not None and bs.engine.m_blk < cnt:
        for blk in list(bs.owner.values()):
            blk._resolve()
        bs = None
    if bs is None:
        m_blk = int(cnt)           # a stream's blocks share one size (the last may be shorter)
        shim = type("_Ctx", (), {"_dev": d})()
        bs = cache[key] = _BlockStream(pipeline.StreamEngine(shim, m_blk, int8=int8,
                                                             emit_s_inv=emit_s_inv))
    return bs


def gls_solve_block(ctx, blk, emit_s_inv=False, threads=1):
    """Solve every marker in the block against the prepared context (kernel.py:315-342).

    The block is copied to the device on a copy stream and solved on a compute stream (int8
    tensor-core TRSM with the reductions fused into its epilogue, then the batched p x p solves;
    per-column fallback to the FP64 DMMA TRSM for non-integer dosages).  The call returns once
    the copy is done; the ResultBlock resolves on first access, so back-to-back calls overlap the
    next block's copy with this block's compute.  ``threads`` is accepted for signature
    compatibility (results never depend on it, tests/test_kernel.py:243-256)."""
    d = device_context(ctx, need_factor=True)
    if blk.n != d.n:
        raise DimensionMismatch(f"block has n={blk.n}, context has n={d.n}")
    cnt = blk.count
    data = blk.data
    int8 = data.dtype == np.int8
    if not int8:
        data = np.asarray(data, dtype=np.float64)
    if not data.flags.f_contiguous:
        data = np.asfortranarray(data)
    bs = _block_stream(ctx, d, int8, emit_s_inv, cnt)
    return bs.submit(data, blk.first_index, cnt)


def gls_oracle(M, Xi, y):
    """Literal evaluation of the GLS formula through a general linear solve against M
    (kernel.py:345-355) - a test route, evaluated on the device with dense LU."""
    torch = __import__("torch")
    dev = _capi.device()
    M = torch.from_numpy(np.asarray(M, dtype=np.float64)).to(dev)
    Xi = torch.from_numpy(np.asarray(Xi, dtype=np.float64)).to(dev)
    y = torch.from_numpy(np.asarray(y, dtype=np.float64).ravel()).to(dev)
    MinvX = torch.linalg.solve(M, Xi)
    Minvy = torch.linalg.solve(M, y)
    A = Xi.T @ MinvX
    b = Xi.T @ Minvy
    return torch.linalg.solve(A, b).cpu().numpy()
