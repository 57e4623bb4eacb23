"""Generate the golden fixtures of tests/golden/ by running the REFERENCE implementation.

Run here (the container that mounts /root/reference); the GPU box only reads the committed
.npz files.  Every output below is produced by the reference package itself
(/root/reference/pkg/src/gwasgls: kernel.gls_prepare / gls_solve_block / cholesky_spd /
trsolve_lower / cholesky_solve_batch, datagen.gen_dataset / oracle_solve_all), so the fixtures
pin both our CPU oracle (oracle/gls_ref.py) and the GPU path.

    python tests/golden/make_golden.py
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from gwasgls import datagen as rdatagen  # noqa: E402
from gwasgls import fileio as rfileio  # noqa: E402
from gwasgls import kernel as rkernel  # noqa: E402

from paper_1304_2272_b200 import datagen as ourgen  # noqa: E402  (host generator only)


def ref_block(M, XL, y, X, emit_s_inv=True):
    ctx = rkernel.gls_prepare(M, XL, y)
    rb = rkernel.gls_solve_block(ctx, rkernel.SnpBlock(0, np.asfortranarray(X, dtype=float)),
                                 emit_s_inv=emit_s_inv)
    p = ctx.p
    beta = np.array([r.beta for r in rb.results])
    status = np.array([0 if r.status == "ok" else 1 for r in rb.results], dtype=np.int8)
    sinv = np.array([r.s_inv if r.s_inv is not None else np.full(p * (p + 1) // 2, np.nan)
                     for r in rb.results])
    return ctx, beta, status, sinv


def make_spd_like_ref_tests(n, seed):
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, 2 * n))
    M = G @ G.T / (2 * n) + np.eye(n)
    return np.tril(M) + np.tril(M, -1).T


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def case_dataset(name, spec, mutate=None):
    with tempfile.TemporaryDirectory() as d:
        paths = rdatagen.gen_dataset(spec, d)
        M = rfileio.read_matrix(paths.cov, "GWAM")
        XL = rfileio.read_matrix(paths.covariates, "GWAC")
        y = rfileio.read_matrix(paths.pheno, "GWAY")
        X = rfileio.read_matrix(paths.geno, "GWAX")
        if mutate is not None:
            mutate(X)
        ctx, beta, status, sinv = ref_block(M, XL, y, X)
        extra = {}
        if spec.n <= rdatagen.ORACLE_MAX_N and spec.m <= rdatagen.ORACLE_MAX_M and mutate is None:
            out = os.path.join(d, "oracle.gwab")
            extra["beta_eq1"] = rdatagen.oracle_solve_all(paths, out).betas
    save(name, M=M, XL=XL, y=y, G=X.astype(np.int8), beta=beta, status=status, sinv=sinv,
         L=ctx.L, XLbar=ctx.XLbar, ybar=ctx.ybar, S_TL=ctx.S_TL, b_T=ctx.b_T,
         n=spec.n, m=spec.m, p=spec.p, seed=spec.seed, **extra)


def case_baseline(name, spec):
    """Our BASELINE generator (host numpy) for the inputs, the reference for the outputs."""
    M = ourgen.kinship_covariance_host(spec)
    XL, y = ourgen.covariates_host(spec)
    G = ourgen.genotypes_host(spec.seed, spec.n, spec.m, 0, spec.m, spec.maf)
    ctx, beta, status, sinv = ref_block(M, XL, y, G.astype(float))
    save(name, M=M, XL=XL, y=y, G=G, beta=beta, status=status, sinv=sinv, n=spec.n, m=spec.m,
         p=spec.p, seed=spec.seed, m_kin=spec.m_kin, a=spec.a)


def case_p_extremes():
    rng = np.random.default_rng(16)
    n = 120
    out = {}
    for p in (2, 4, 20):
        M = make_spd_like_ref_tests(n, p)
        XL = np.hstack([np.ones((n, 1)), rng.standard_normal((n, p - 2))]) if p > 2 \
            else np.ones((n, 1))
        y = rng.standard_normal(n)
        X = rng.standard_normal((n, 8))
        _, beta, status, sinv = ref_block(M, XL, y, X)
        out.update({f"M{p}": M, f"XL{p}": XL, f"y{p}": y, f"X{p}": X, f"beta{p}": beta,
                    f"sinv{p}": sinv})
    save("p_extremes", **out)


def case_dense_ops():
    out = {}
    for n in (16, 96, 200, 300):
        M = make_spd_like_ref_tests(n, 42)
        L = rkernel.cholesky_spd(M)
        B = np.random.default_rng(n).standard_normal((n, 9))
        out[f"M{n}"] = M
        out[f"L{n}"] = L
        out[f"B{n}"] = B
        out[f"X{n}"] = rkernel.trsolve_lower(L, B)
        out[f"G{n}"] = rkernel.gram(B)
    rng = np.random.default_rng(7)
    S = rng.standard_normal((64, 6, 6))
    S = S @ S.transpose(0, 2, 1) + 0.1 * np.eye(6)
    S[5] = np.outer(S[5, 0], S[5, 0])   # rank one -> failed system
    rhs = rng.standard_normal((64, 6))
    x, ok, packed = rkernel.cholesky_solve_batch(S, rhs, want_inverse=True)
    out.update(S=S, rhs=rhs, x=x, ok=ok, packed=packed)
    # not-positive-definite pivots
    Mbad = np.eye(300)
    Mbad[211, 211] = -1.0
    try:
        rkernel.cholesky_spd(Mbad)
    except Exception as e:  # NotPositiveDefinite
        out["notpd_pivot"] = np.int64(e.pivot_index)
    save("dense_ops", **out)


def case_streams():
    """splitmix64 counter streams of the reference generator (datagen.py:35-60)."""
    out = {}
    for seed, stream in ((42, 1), (42, 2), (7, 3), (123456789, 5)):
        out[f"u64_{seed}_{stream}"] = rdatagen._stream_u64(seed, stream, 1000, 64)
        out[f"unif_{seed}_{stream}"] = rdatagen._stream_uniform(seed, stream, 0, 64)
    save("streams", **out)


def main():
    case_streams()
    case_dense_ops()
    case_p_extremes()
    case_dataset("seed42", rdatagen.GenSpec(n=100, m=500, p=4, seed=42))

    def degen(X):
        X[:, 10] = 0.0
        X[:, 20] = 1.0
    case_dataset("degenerate", rdatagen.GenSpec(n=60, m=40, p=4, seed=42), mutate=degen)
    case_baseline("baseline_p4", ourgen.BaselineSpec(n=300, m=2000, p=4, m_kin=500, a=0.6))
    case_baseline("baseline_p8", ourgen.BaselineSpec(n=256, m=500, p=8, m_kin=400, a=0.5))


if __name__ == "__main__":
    main()
