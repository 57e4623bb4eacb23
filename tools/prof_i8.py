"""One int8 TRSM (+ fused partials) launch at config-1 sizes inside NVTX range "hot/", for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1304_2272_b200 import _capi, datagen, kernel  # noqa: E402
from paper_1304_2272_b200._capi import check, ptr  # noqa: E402

lib = _capi.lib()
n, cnt = int(os.environ.get("N", "10000")), 8192
spec = datagen.BaselineSpec(n=n, m=cnt, p=4)
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
