"""One gls_prepare at size n (default 40000) after one warm-up prepare at n = 2048: the target of
an ncu capture of the prepare's kernels (leaf, Ozaki GEMM, DMMA GEMMs).
    python tools/prof_prepare_once.py [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1304_2272_b200 import datagen, kernel  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
for nn in (2048, n):
    spec = datagen.BaselineSpec(n=nn, m=1, p=4)
    Md = datagen.kinship_covariance_device(spec)
    XL, y = datagen.covariates_host(spec)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx = kernel.gls_prepare(Md, XL, y)
    torch.cuda.synchronize()
    print(f"n={nn} gls_prepare {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    del ctx, Md
    torch.cuda.empty_cache()
