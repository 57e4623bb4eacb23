"""A/B timing of gg_potrf_f64 (Cholesky + inverse) across library builds on one box.
    python tools/ab_potrf.py tools/alt/lib_a.so [...]   (the in-tree library is always included)"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1304_2272_b200 import _capi, datagen  # noqa: E402

for n in (10000, 40000):
    spec = datagen.BaselineSpec(n=n, m=1, p=4)
    Md = datagen.kinship_covariance_device(spec)
    np_ = _capi.pad(n)
    L = torch.empty((np_, np_), dtype=torch.float64, device="cuda")
    Li = torch.empty_like(L)
    for path in [_capi.LIB_PATH] + sys.argv[1:]:
        lib = C.CDLL(path)
        lib.gg_potrf_workspace_bytes.restype = C.c_size_t
        ws = torch.empty(int(lib.gg_potrf_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
        info = (C.c_int * 2)()
        ts = []
        for rep in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rc = lib.gg_potrf_f64(n, C.c_void_p(Md.data_ptr()), n, 1, C.c_void_p(L.data_ptr()),
                                  C.c_void_p(Li.data_ptr()), np_, C.c_void_p(ws.data_ptr()), info,
                                  C.c_void_p(torch.cuda.current_stream().cuda_stream))
            b.record()
            torch.cuda.synchronize()
            assert rc == 0, rc
            ts.append(a.elapsed_time(b))
        print(f"n={n} {os.path.basename(path)}: {min(ts):.1f} ms", flush=True)
    del Md, L, Li
    torch.cuda.empty_cache()
