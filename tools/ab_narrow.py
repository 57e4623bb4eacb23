"""A/B timing of gg_narrow_f64_i8 (FP64 dosages -> int8, config-1 block: n = 1e4, 8192 SNPs)
across library builds on one box, round-robin; outputs are checked equal to the in-tree's.
    python tools/ab_narrow.py tools/alt/lib_a.so [...]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1304_2272_b200 import _capi  # noqa: E402
from paper_1304_2272_b200._capi import ptr  # noqa: E402

n, cnt = 10000, 8192
n16 = -(-n // 16) * 16
X = torch.randint(0, 3, (cnt, n), dtype=torch.float64, device="cuda")
s = _capi.stream_handle()
libs = []
for path in [_capi.LIB_PATH] + sys.argv[1:]:
    lib = C.CDLL(path)
    f = lib.gg_narrow_f64_i8
    f.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_void_p, C.c_longlong,
                  C.c_void_p, C.c_void_p]
    libs.append((os.path.basename(path), f, torch.full((cnt, n16), 5, dtype=torch.int8,
                                                       device="cuda"), []))
bad = torch.zeros(1, dtype=torch.int32, device="cuda")
for rep in range(10):
    for name, f, G, ts in libs:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        assert f(n, cnt, ptr(X), n, ptr(G), n16, ptr(bad), s) == 0
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
ref = libs[0][2]
assert int(bad) == 0 and torch.equal(ref[:, :n].to(torch.float64), X) and not ref[:, n:].any()
for name, f, G, ts in libs:
    t = sorted(ts[1:])
    gbs = (cnt * n * 9) / (t[0] * 1e-3) / 1e9
    print(f"{name}: {t[0]:.4f} ms (median {t[len(t) // 2]:.4f}), {gbs:.0f} GB/s, "
          f"equal to in-tree: {torch.equal(G, ref)}")
