"""One int8 TRSM (+ fused partials) launch at config-1 (or CFG=3) sizes inside NVTX range "hot/", for
ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1304_2272_b200 import _capi, datagen, kernel  # noqa: E402
from paper_1304_2272_b200._capi import check, ptr  # noqa: E402

lib = _capi.lib()
import dataclasses  # noqa: E402

# CFG=3: BASELINE config 3 (n = 4e4, p = 8, a = 0.5); default config 1 (N overrides n)
cfg = int(os.environ.get("CFG", "1"))
cnt = 8192
spec = dataclasses.replace(datagen.CONFIGS[cfg], m=cnt)
if "N" in os.environ:
    spec = dataclasses.replace(spec, n=int(os.environ["N"]))
n = spec.n
ctx = kernel.gls_prepare(datagen.kinship_covariance_device(spec), *datagen.covariates_host(spec))
d = ctx._dev
n16 = -(-n // 16) * 16
G16 = datagen.genotypes_device(spec, 0, cnt, ld=n16)
P = torch.empty(int(lib.gg_partials_bytes(n, cnt, d.q)) // 8, dtype=torch.float64, device="cuda")
s = _capi.stream_handle()
W = _capi.i8_work()
for rep in range(2):
    if rep:
        torch.cuda.nvtx.range_push("hot")
    check(lib.gg_trsm_lower_i8_partials(n, cnt, ptr(d.slices), ptr(d.expo), ptr(G16), n16, d.q,
                                        ptr(d.XLy), ptr(d.ybar), ptr(P), None, 0, None, 0, ptr(W), s), "i8")
    if rep:
        torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
print("ok")
