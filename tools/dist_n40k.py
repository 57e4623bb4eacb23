"""The config-4 form of the distributed engine at n = 40,000 on ONE B200 ("a
world-2 n ~ 40k run passes on one GPU"): two ranks (threads driving a reference-contract transport,
tests/spmd_inproc.py) on a 1 x 2 grid, nb = 512; every rank generates its own blocks of the config-3
covariance on the device (local_from_spec: no n x n array anywhere), runs the fused Cholesky +
inverse with row/column broadcasts, assembles the int8 slices without any replicated FP64 inverse,
whitens [X_L | y] from the block-cyclic inverse, and solves a 1,024-SNP sample through the
slices-only context.  Checked against the single-GPU prepare of the same M (itself checked against
the CPU oracle in bench.py); reports the prepare time and the process's peak host RSS.

    python tools/dist_n40k.py [--n 40000] [--world 2] [--no-lookahead]
"""

import argparse
import os
import resource
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=40_000)
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--snps", type=int, default=1024)
    ap.add_argument("--no-lookahead", action="store_true")
    args = ap.parse_args()
    import dataclasses

    import torch

    from paper_1304_2272_b200 import datagen, distgrid, kernel
    from spmd_inproc import run_spmd

    spec = dataclasses.replace(datagen.CONFIGS[3], n=args.n, m=args.snps)
    XL, y = datagen.covariates_host(spec)
    G = datagen.genotypes_host(spec.seed, spec.n, spec.m, 0, spec.m)

    def body(t):
        ops = distgrid.DeviceOps()
        lay = distgrid.BlockCyclic(spec.n, 512, distgrid.grid_create(t.size), t.rank)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A, B = distgrid.local_from_spec(spec, lay, ops)
        torch.cuda.synchronize()
        t_gen = time.perf_counter() - t0
        t0 = time.perf_counter()
        distgrid.dist_potrf_inv(A, B, lay, ops, t, lookahead=not args.no_lookahead)
        del A
        S, e = distgrid.assemble_slices(B, lay, ops, t)
        XLy = distgrid.whiten_blockcyclic(B, lay, ops, np.column_stack([XL, y]), t)
        del B
        ctx = kernel.prepare_from_inverse(None, spec.n, XL, y, slices=S, expo=e, XLy=XLy)
        torch.cuda.synchronize()
        t_prep = time.perf_counter() - t0
        rb = kernel.gls_solve_block(ctx, kernel.SnpBlock(0, G))
        beta = np.array([r.beta for r in rb.results])
        return t_gen, t_prep, beta, lay.m_loc, lay.n_loc

    t0 = time.perf_counter()
    res = run_spmd(args.world, body)
    wall = time.perf_counter() - t0
    rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6      # GB (ru_maxrss in KB)
    torch.cuda.empty_cache()
    # the single-GPU path on the same M
    Md = datagen.kinship_covariance_device(spec)
    t0 = time.perf_counter()
    ctx1 = kernel.gls_prepare(Md, XL, y)
    torch.cuda.synchronize()
    t1 = time.perf_counter() - t0
    del Md
    ref = np.array([r.beta for r in kernel.gls_solve_block(ctx1, kernel.SnpBlock(0, G)).results])
    from oracle import gls_ref as O

    print(f"look-ahead {'off' if args.no_lookahead else 'on'}: n={spec.n} p={spec.p} world={args.world} (grid "
          f"{distgrid.grid_create(args.world).r}x{distgrid.grid_create(args.world).c}, nb=512); "
          f"local share {res[0][3]}x{res[0][4]} per rank")
    for r, (tg, tp, beta, _, _) in enumerate(res):
        rel, mism = O.compare(beta, ref)
        print(f"rank {r}: generate own blocks {tg:.2f} s, distributed prepare {tp:.2f} s, "
              f"{args.snps} SNPs vs the single-GPU prepare: max rel {rel:.2e}, "
              f"status mismatches {mism}")
    same = all(np.array_equal(res[0][2], x[2], equal_nan=True) for x in res)
    print(f"identical results on every rank: {same}; single-GPU prepare {t1:.2f} s; "
          f"whole distributed run {wall:.1f} s (ranks share one GPU, exchanges through host "
          f"bytes); process peak host RSS {rss:.1f} GB for all {args.world} ranks")


if __name__ == "__main__":
    main()
