"""Prepare-phase timing (Cholesky + inverse) at BASELINE sizes; prints the C++ phase split when
GG_POTRF_TIMING=1.   python tools/prof_prepare.py --n 10000 40000"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1304_2272_b200 import datagen, kernel

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="+", default=[10000])
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
for n in args.n:
    spec = datagen.BaselineSpec(n=n, m=1, p=4)
    Md = datagen.kinship_covariance_device(spec)
    XL, y = datagen.covariates_host(spec)
    for rep in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx = kernel.gls_prepare(Md, XL, y)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"n={n} rep={rep} gls_prepare {dt * 1e3:.1f} ms  ({n ** 3 / 3 / dt / 1e12:.2f} TF/s of n^3/3)",
              flush=True)
    del ctx, Md
    torch.cuda.empty_cache()
