"""One-off calibration of the CPU reference arm (not part of bench.py or the tests): time the
reference package's own `gls_prepare` + `gls_solve_block(threads=T)` (kernel.py:233-342, imported
from a transient, git-ignored copy under baseline/_ref) against the oracle port bench.py times
(oracle/gls_ref.py), on the same inputs and host cores, and check they agree.

    PYTHONPATH=baseline/_ref python tools/ref_vs_port_timing.py [--config 3] [--snps 512]
"""

import argparse
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--snps", type=int, default=512)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import gwasgls.kernel as RK  # the reference itself (baseline/_ref on PYTHONPATH)

    import bench
    from oracle import gls_ref as O
    from paper_1304_2272_b200 import datagen

    spec = datagen.CONFIGS[args.config]
    cores = bench._blas_threads()
    M = bench.kinship_host_lean(spec)
    XL, y = datagen.covariates_host(spec)
    G = datagen.genotypes_host(spec.seed, spec.n, spec.m, 0, args.snps).astype(np.float64,
                                                                             order="F")
    t0 = time.perf_counter()
    rctx = RK.gls_prepare(M, XL, y)
    t_rprep = time.perf_counter() - t0
    t0 = time.perf_counter()
    octx = O.gls_prepare(M, XL, y)
    t_oprep = time.perf_counter() - t0
    del M
    blk = RK.SnpBlock(first_index=0, data=G)
    tr, to = [], []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        rb = RK.gls_solve_block(rctx, blk, threads=cores)
        tr.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        ob, _ = O.gls_solve_block(octx, G, threads=cores)
        to.append(time.perf_counter() - t0)
    rbeta = np.array([r.beta for r in rb.results])
    rel, mism = O.compare(ob, rbeta)
    print(f"config {args.config} (n={spec.n}, p={spec.p}), {args.snps}-SNP block, {cores} threads, "
          f"best of {args.reps}")
    print(f"reference gwasgls: gls_prepare {t_rprep:.1f} s, gls_solve_block "
          f"{min(tr):.3f} s = {args.snps / min(tr):.1f} SNPs/s")
    print(f"oracle port      : gls_prepare {t_oprep:.1f} s, gls_solve_block "
          f"{min(to):.3f} s = {args.snps / min(to):.1f} SNPs/s")
    print(f"port / reference speed {min(tr) / min(to):.3f}; results max rel {rel:.2e}, "
          f"status mismatches {mism}")


if __name__ == "__main__":
    main()
