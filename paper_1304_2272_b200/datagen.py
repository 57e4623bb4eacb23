"""Synthetic BASELINE datasets (BASELINE.json ``configs``).

Randomness comes from counter-based splitmix64 streams keyed by (seed, stream, counter) — the
construction of the reference's datagen.py:35-60 — so host (numpy) and device (CUDA,
``gg_gen_genotypes_i8``) draw bit-identical genotypes.  Genotype stream layout follows the
reference's gen_dataset (datagen.py:139-146): for marker j and individual i,
u1 = U(GENO, j*n + i), u2 = U(GENO, (m + j)*n + i), G = [u1 < f_j] + [u2 < f_j],
f_j = lo + U(MAF, j) * (hi - lo).

BASELINE generator (configs[0]): kinship K = Z Z^T / m_k from m_k extra standardised markers
Z = (G - 2f) / sqrt(2f(1-f)) (true f), M = a K + (1 - a) I mirrored from the lower triangle,
X_L = [1, N(0,1) x (p-2)], y ~ N(0,1).  Normals use Box-Muller on the host only (libm and CUDA
log/cos are not bit-identical).  No public dataset is involved; these seeded synthetic inputs
stand in for the paper's experiments.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import fileio
from .errors import ConfigError

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
STREAM_MAF = 1
STREAM_GENO = 2
STREAM_COV = 3
STREAM_NOISE = 5
STREAM_KIN_MAF = 11
STREAM_KIN_GENO = 12


def mix64(z):
    """splitmix64 finalizer on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def stream_key(seed, stream):
    with np.errstate(over="ignore"):
        return mix64(np.uint64(seed) * GOLDEN + np.uint64(stream))


def stream_u64(seed, stream, counters):
    counters = np.asarray(counters, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64((counters + np.uint64(1)) * GOLDEN + stream_key(seed, stream))


def stream_uniform(seed, stream, start, count):
    idx = np.arange(start, start + count, dtype=np.uint64)
    return (stream_u64(seed, stream, idx) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def stream_normal(seed, stream, start, count):
    u = stream_uniform(seed, stream, 2 * start, 2 * count)
    u1 = u[0::2] + 2.0 ** -54
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u[1::2])


def marker_freqs(seed, stream, first, count, maf=(0.05, 0.5)):
    return maf[0] + stream_uniform(seed, stream, first, count) * (maf[1] - maf[0])


def genotypes_host(seed, n, m, first, count, maf=(0.05, 0.5), stream_maf=STREAM_MAF,
                   stream_geno=STREAM_GENO):
    """int8 dosages of markers [first, first+count) of an m-marker panel, n x count F-order."""
    f = marker_freqs(seed, stream_maf, first, count, maf)
    j = np.arange(first, first + count, dtype=np.uint64)
    i = np.arange(n, dtype=np.uint64)
    c1 = j[None, :] * np.uint64(n) + i[:, None]
    c2 = (j[None, :] + np.uint64(m)) * np.uint64(n) + i[:, None]
    u1 = (stream_u64(seed, stream_geno, c1) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    u2 = (stream_u64(seed, stream_geno, c2) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    g = (u1 < f[None, :]).astype(np.int8) + (u2 < f[None, :]).astype(np.int8)
    return np.asfortranarray(g)


def standardized_host(seed, n, m_k, maf=(0.05, 0.5)):
    """Z = (G - 2f)/sqrt(2f(1-f)) for the m_k kinship markers (n x m_k, FP64)."""
    g = genotypes_host(seed, n, m_k, 0, m_k, maf, STREAM_KIN_MAF, STREAM_KIN_GENO)
    f = marker_freqs(seed, STREAM_KIN_MAF, 0, m_k, maf)
    two_f = 2.0 * f
    return (g.astype(np.float64) - two_f[None, :]) / np.sqrt(two_f * (1.0 - f))[None, :]


@dataclass
class BaselineSpec:
    """One BASELINE.json config: n individuals, m markers, p = q + 1 parameters."""

    n: int
    m: int
    p: int = 4
    seed: int = 42
    m_kin: int = 5000
    a: float = 0.6
    maf: tuple = (0.05, 0.5)

    def __post_init__(self):
        if not (2 <= self.p <= 20):
            raise ConfigError("p must lie in [2, 20]")
        if self.n < 1 or self.m < 1 or self.m_kin < 1:
            raise ConfigError("n, m and m_kin must be >= 1")
        if not (0.0 <= self.a < 1.0):
            raise ConfigError("kinship weight a must lie in [0, 1)")


CONFIGS = {
    0: BaselineSpec(n=1000, m=10_000, p=4, m_kin=5000, a=0.6),
    1: BaselineSpec(n=10_000, m=200_000, p=4, m_kin=5000, a=0.6),
    2: BaselineSpec(n=10_000, m=10_000_000, p=4, m_kin=5000, a=0.6),
    3: BaselineSpec(n=40_000, m=2_000_000, p=8, m_kin=5000, a=0.5),
    4: BaselineSpec(n=150_000, m=1_000_000, p=4, m_kin=20_000, a=0.6),
}


def covariates_host(spec):
    """X_L = [1, N(0,1) x (p-2)] (n x q, F-order) and y ~ N(0,1)."""
    n, q = spec.n, spec.p - 1
    XL = np.empty((n, q), order="F")
    XL[:, 0] = 1.0
    if q > 1:
        XL[:, 1:] = stream_normal(spec.seed, STREAM_COV, 0, n * (q - 1)).reshape(
            (n, q - 1), order="F")
    y = stream_normal(spec.seed, STREAM_NOISE, 0, n)
    return XL, y


def kinship_covariance_host(spec):
    """M = a Z Z^T / m_k + (1 - a) I, exactly symmetric (lower mirrored)."""
    Z = standardized_host(spec.seed, spec.n, spec.m_kin, spec.maf)
    K = (Z @ Z.T) / spec.m_kin
    M = spec.a * K + (1.0 - spec.a) * np.eye(spec.n)
    return np.tril(M) + np.tril(M, -1).T


def kinship_covariance_device(spec):
    """Same construction on the GPU (DMMA SYRK through gg_dgemm_f64); returns a torch tensor
    (n, n) holding M column-major (= M, since M is symmetric).  Used for large n."""
    import torch

    from . import _capi
    from ._capi import check, pad, ptr, stream_handle
    from ._device import alloc_cols

    n, mk = spec.n, spec.m_kin
    np_ = pad(n)
    mk16 = ((mk + 15) // 16) * 16
    Z = alloc_cols(mk16, np_)                      # padded columns stay zero
    for first in range(0, mk, 65535):
        cnt = min(65535, mk - first)
        check(_capi.lib().gg_gen_genotypes_i8(
            spec.seed, STREAM_KIN_MAF, STREAM_KIN_GENO, n, mk, first, cnt, spec.maf[0],
            spec.maf[1], None, 0, ptr(Z[first:]), np_, stream_handle()), "gg_gen_genotypes_i8")
    K = alloc_cols(np_, np_, zero=False)
    check(_capi.lib().gg_dgemm_f64(np_, np_, mk16, 1.0, ptr(Z), np_, ptr(Z), np_, 1, 0.0,
                                   ptr(K), np_, stream_handle()), "gg_dgemm_f64")
    del Z
    Kn = K[:n, :n]                                  # (col, row) view; symmetric by construction
    M = (Kn / mk) * spec.a
    M.diagonal().add_(1.0 - spec.a)
    low = torch.tril(M.T)                          # lower triangle of the column-major matrix
    M = low + torch.tril(low, -1).T
    return M.T.contiguous()                        # (col, row) storage of the symmetric M


def genotypes_device(spec, first, count, out=None, ld=None):
    """int8 dosages for markers [first, first+count) on the device: (count, ld) tensor."""
    import torch

    from . import _capi
    from ._capi import check, ptr, stream_handle

    ld = spec.n if ld is None else ld
    if out is None:
        out = torch.empty((count, ld), dtype=torch.int8, device=_capi.device())
    for off in range(0, count, 65535):
        cnt = min(65535, count - off)
        check(_capi.lib().gg_gen_genotypes_i8(
            spec.seed, STREAM_MAF, STREAM_GENO, spec.n, spec.m, first + off, cnt, spec.maf[0],
            spec.maf[1], ptr(out[off:]), ld, None, 0, stream_handle()), "gg_gen_genotypes_i8")
    return out


@dataclass
class DatasetPaths:
    cov: str
    covariates: str
    pheno: str
    geno: str

    @classmethod
    def in_dir(cls, out_dir, int8=False):
        return cls(cov=os.path.join(out_dir, "covariance.gwam"),
                   covariates=os.path.join(out_dir, "covariates.gwac"),
                   pheno=os.path.join(out_dir, "phenotype.gway"),
                   geno=os.path.join(out_dir, "genotypes.gwai" if int8 else "genotypes.gwax"))


def write_dataset(spec, out_dir, int8=False, M=None, chunk=4096, device=False):
    """Write GWAM/GWAC/GWAY and the genotype file (GWAX FP64 or GWAI int8), streaming the
    genotypes in column chunks so m may exceed host memory (``device``: generate the chunks
    with the bit-identical device generator)."""
    os.makedirs(out_dir, exist_ok=True)
    paths = DatasetPaths.in_dir(out_dir, int8=int8)
    if M is None:
        M = kinship_covariance_host(spec)
    fileio.write_matrix(paths.cov, "GWAM", M)
    XL, y = covariates_host(spec)
    fileio.write_matrix(paths.covariates, "GWAC", XL)
    fileio.write_matrix(paths.pheno, "GWAY", y)
    kind = "GWAI" if int8 else "GWAX"
    with open(paths.geno, "wb") as f:
        f.write(fileio.pack_header(kind, (spec.n, spec.m)))
        for j0 in range(0, spec.m, chunk):
            cnt = min(chunk, spec.m - j0)
            if device:
                g = genotypes_device(spec, j0, cnt).cpu().numpy().T
            else:
                g = genotypes_host(spec.seed, spec.n, spec.m, j0, cnt, spec.maf)
            arr = g if int8 else g.astype(np.float64, order="F")
            f.write(arr.tobytes(order="F"))
    return paths
