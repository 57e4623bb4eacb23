"""Accuracy of the factorisation with the Ozaki updates against the all-DMMA (pure FP64)
factorisation of the same matrix, on benign and hard covariances at n = 4,500 (trailing SYRKs on
the Ozaki GEMM) and 9,000 (also the trtri levels >= 4,096):
    ||L L^T - M||max / ||M||max,  ||Linv L - I||max,  max |L_oz - L_dmma| / ||L||max
and the GLS betas of 64 SNPs against the DMMA prepare (max relative difference per SNP).
The library is the one GG_LIB_PATH names (one build per process):
    GG_LIB_PATH=tools/alt/oz8.so python tools/oz_factor_accuracy.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1304_2272_b200 import datagen, kernel  # noqa: E402


def spd_with_cond(n, cond, rng):
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    M = (Q * np.logspace(0, -np.log10(cond), n)) @ Q.T
    return np.tril(M) + np.tril(M, -1).T


def ar1(n, rho):
    i = np.arange(n)
    return rho ** np.abs(i[:, None] - i[None, :])


def factor(M, ozaki):
    os.environ["GG_FACTOR_OZAKI"] = "1" if ozaki else "0"
    n, L, _, Linv = kernel._potrf_device(M, keep_square_inverse=True)
    return L[:n, :n].T.contiguous(), Linv[:n, :n].T.contiguous()   # row-major lower


def betas(M, XL, y, G, ozaki):
    os.environ["GG_FACTOR_OZAKI"] = "1" if ozaki else "0"
    ctx = kernel.gls_prepare(M, XL, y)
    rb = kernel.gls_solve_block(ctx, kernel.SnpBlock(0, G))
    return np.array([r.beta for r in rb.results])


rng = np.random.default_rng(3)
print(f"library: {os.environ.get('GG_LIB_PATH', 'in-tree')}")
for n in (4500, 9000):
    spec = datagen.BaselineSpec(n=n, m=64, p=4, m_kin=n // 2, a=0.6, seed=42)
    mats = {
        "kinship": datagen.kinship_covariance_host(spec),
        "cond 1e8": spd_with_cond(n, 1e8, rng),
        "ar1 0.999": ar1(n, 0.999),
    }
    XL, y = datagen.covariates_host(spec)
    G = datagen.genotypes_host(spec.seed, n, 64, 0, 64).astype(np.float64)
    for name, M in mats.items():
        Md = torch.from_numpy(M).cuda()
        Lo, Io = factor(M, True)
        Ld, _ = factor(M, False)
        res = float((Lo.tril() @ Lo.tril().T - Md).abs().max() / Md.abs().max())
        ires = float((Io.tril() @ Lo.tril() - torch.eye(n, dtype=Md.dtype, device=Md.device)).abs().max())
        dl = float((Lo - Ld).abs().max() / Ld.abs().max())
        bo, bd = betas(M, XL, y, G, True), betas(M, XL, y, G, False)
        db = float(np.max(np.max(np.abs(bo - bd), axis=1) / np.max(np.abs(bd), axis=1)))
        print(f"n={n:5d} {name:10s}  LL^T-M {res:.2e}  LinvL-I {ires:.2e}  |L-L_dmma| {dl:.2e}  "
              f"beta vs DMMA {db:.2e}", flush=True)
        del Md, Lo, Io, Ld
        torch.cuda.empty_cache()
