"""A/B timing of gg_potrf_f64 (Cholesky + inverse) across library builds and environment variants
on one box; also the max difference of L and Linv against the first variant.
    GG_AB_ENVS="GG_FACTOR_OZAKI=0;GG_FACTOR_OZAKI=1" python tools/ab_potrf.py [lib.so ...]
    (GG_AB_SIZES="10000,40000"; GG_POTRF_TIMING=1 prints the phases)"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1304_2272_b200 import _capi, datagen  # noqa: E402

variants = [(p, None) for p in [_capi.LIB_PATH] + sys.argv[1:]]
for spec_ in filter(None, os.environ.get("GG_AB_ENVS", "").split(";")):
    variants.append((_capi.LIB_PATH, tuple(spec_.split("=", 1))))
for n in [int(x) for x in os.environ.get("GG_AB_SIZES", "10000,40000").split(",")]:
    spec = datagen.BaselineSpec(n=n, m=1, p=4)
    Md = datagen.kinship_covariance_device(spec)
    np_ = _capi.pad(n)
    L = torch.empty((np_, np_), dtype=torch.float64, device="cuda")
    Li = torch.empty_like(L)
    ref = None
    for path, env in variants:
        if env:
            os.environ[env[0]] = env[1]
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
        if env:
            del os.environ[env[0]]
        Lc, Ic = torch.tril(L[:n, :n]), torch.tril(Li[:n, :n])
        if ref is None:
            ref = (Lc.clone(), Ic.clone())
            diff = ""
        else:
            dl = float((Lc - ref[0]).abs().max() / ref[0].abs().max())
            di = float((Ic - ref[1]).abs().max() / ref[1].abs().max())
            diff = f"  max rel diff vs first: L {dl:.2e}, Linv {di:.2e}"
        name = os.path.basename(path) + (f" {env[0]}={env[1]}" if env else "")
        print(f"n={n} {name}: {min(ts):.1f} ms (ws {ws.numel() / 1e9:.2f} GB){diff}", flush=True)
        del ws
    del Md, L, Li, ref
    torch.cuda.empty_cache()
