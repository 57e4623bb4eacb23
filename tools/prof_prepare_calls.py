"""Wall time of consecutive gls_prepare calls at config-1 size (first-call overheads vs steady
state), optionally with GG_FACTOR_OZAKI=0."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1304_2272_b200 import datagen, kernel  # noqa: E402

n = int(os.environ.get("N", "10000"))
spec = datagen.BaselineSpec(n=n, m=1, p=4)
Md = datagen.kinship_covariance_device(spec)
XL, y = datagen.covariates_host(spec)
torch.cuda.synchronize()
for i in range(3):
    t0 = time.perf_counter()
    ctx = kernel.gls_prepare(Md, XL, y)
    torch.cuda.synchronize()
    print(f"n={n} prepare call {i}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    del ctx
