"""Profiling driver for ncu: config-1 sizes (n = 10,000, one 8,192-SNP block).

Runs gls_prepare once, then inside the NVTX range "hot/" one TRSM launch and one fused epilogue
launch, so `ncu --nvtx --nvtx-include "hot/"` captures exactly the hot-path kernels.  Also prints
a CUDA-event breakdown of the prepare phase (no profiler needed).

    python tools/prof_hot.py [--n 10000] [--cnt 8192] [--reps 3]
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1304_2272_b200 import _capi, datagen, kernel  # noqa: E402
from paper_1304_2272_b200._capi import check, ptr  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--cnt", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    lib = _capi.lib()
    spec = datagen.BaselineSpec(n=args.n, m=args.cnt, p=4)
    n = spec.n
    np_ = _capi.pad(n)
    Md = datagen.kinship_covariance_device(spec)
    M = Md.cpu().numpy()
    XL, y = datagen.covariates_host(spec)
    s = _capi.stream_handle()
    W = _capi.i8_work()
    # prepare breakdown
    for rep in range(2):
        t0 = time.perf_counter()
        ctx = kernel.gls_prepare(M, XL, y)
        torch.cuda.synchronize()
        t_api = time.perf_counter() - t0
        L = torch.empty((np_, np_), dtype=torch.float64, device="cuda")
        Li = torch.empty_like(L)
        ws = torch.empty(lib.gg_potrf_workspace_bytes(n), dtype=torch.uint8, device="cuda")
        info = (_capi.C.c_int * 2)()
        Mpad = torch.zeros((n, np_), dtype=torch.float64, device="cuda")
        Mpad[:, :n] = Md
        a, b = ev(), ev()
        a.record()
        check(lib.gg_potrf_f64(n, ptr(Mpad), np_, 0, ptr(L), ptr(Li), np_, ptr(ws), info, s), "potrf")
        b.record()
        torch.cuda.synchronize()
        print(f"prepare api {t_api * 1e3:.1f} ms; gg_potrf_f64 (chol + inverse) {a.elapsed_time(b):.2f} ms")
    d = ctx._dev
    G = datagen.genotypes_device(spec, 0, args.cnt)
    X = torch.zeros((args.cnt, np_), dtype=torch.float64, device="cuda")
    check(lib.gg_widen_i8_f64(n, args.cnt, ptr(G), n, ptr(X), np_, s), "widen")
    xbar = torch.empty_like(X)
    beta = torch.empty((args.cnt, d.p), dtype=torch.float64, device="cuda")
    st = torch.empty((args.cnt,), dtype=torch.int32, device="cuda")
    for _ in range(2):
        check(lib.gg_trsm_lower_packed_f64(n, args.cnt, ptr(d.LinvP), ptr(X), np_, ptr(xbar), np_, s), "trsm")
    torch.cuda.synchronize()
    # int8 tensor-core path (the production path for dosage blocks)
    n16 = -(-n // 16) * 16
    G16 = datagen.genotypes_device(spec, 0, args.cnt, ld=n16)
    P = torch.empty(int(lib.gg_partials_bytes(n, args.cnt, d.q)) // 8, dtype=torch.float64,
                    device="cuda")
    for rep in range(args.reps + 1):
        a, b, c = ev(), ev(), ev()
        if rep > 0:
            torch.cuda.nvtx.range_push("hot")
        a.record()
        check(lib.gg_trsm_lower_i8_partials(n, args.cnt, ptr(d.slices), ptr(d.expo), ptr(G16), n16,
                                            d.q, ptr(d.XLy), ptr(d.ybar), ptr(P), None, 0, None, 0,
                                            ptr(W), s), "trsm_i8")
        b.record()
        check(lib.gg_gls_reduce_solve_f64(n, args.cnt, d.q, ptr(P), ptr(d.S_TL), ptr(d.b_T),
                                          ptr(beta), ptr(st), None, s), "reduce")
        c.record()
        if rep > 0:
            torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        fl = float(n) * n * args.cnt
        print(f"i8 rep {rep}: trsm+partials {a.elapsed_time(b):.3f} ms = "
              f"{fl / a.elapsed_time(b) / 1e9:.1f} TF/s FP64-equivalent; reduce+solve "
              f"{b.elapsed_time(c):.3f} ms")
    for rep in range(args.reps):
        a, b, c = ev(), ev(), ev()
        a.record()
        check(lib.gg_trsm_lower_packed_f64(n, args.cnt, ptr(d.LinvP), ptr(X), np_, ptr(xbar), np_, s), "trsm")
        b.record()
        check(lib.gg_gls_epilogue_f64(n, args.cnt, d.q, ptr(xbar), np_, ptr(d.XLy), np_, ptr(d.ybar),
                                      ptr(d.S_TL), ptr(d.b_T), ptr(beta), ptr(st), None, ptr(P), s), "epi")
        c.record()
        torch.cuda.synchronize()
        t_trsm = a.elapsed_time(b)
        t_epi = b.elapsed_time(c)
        fl = float(n) * n * args.cnt
        print(f"rep {rep}: trsm {t_trsm:.3f} ms = {fl / t_trsm / 1e9:.2f} TF/s; epilogue {t_epi:.3f} ms "
              f"= {8.0 * np_ * args.cnt / t_epi / 1e6:.1f} GB/s (Xbar read)")
    assert int((st >= 0).sum()) == 0


if __name__ == "__main__":
    main()
