"""Check and time the int8 tensor-core TRSM (trsm_i8_kernel) against the FP64 DMMA TRSM.

    python tools/check_i8.py [--n 1000 10000] [--cnt 8192] [--reps 5]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1304_2272_b200 import _capi, datagen, kernel  # noqa: E402
from paper_1304_2272_b200._capi import check, ptr, stream_handle  # noqa: E402
from paper_1304_2272_b200._device import alloc_cols, transpose_square  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[1000, 10000])
    ap.add_argument("--cnt", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    lib = _capi.lib()
    s = stream_handle()
    W = _capi.i8_work()
    for n in args.n:
        spec = datagen.BaselineSpec(n=n, m=args.cnt, p=4)
        Md = datagen.kinship_covariance_device(spec)
        _, L, LinvP, Linv = kernel._potrf_device(Md, keep_square_inverse=True)
        np_ = _capi.pad(n)
        LinvT = transpose_square(Linv)
        del Linv
        S = lib.gg_i8_slices()
        sl = torch.empty(int(lib.gg_inverse_slices_bytes(n)), dtype=torch.int8, device="cuda")
        expo = torch.empty(int(lib.gg_slice_meta_ints(n)), dtype=torch.int32, device="cuda")
        check(lib.gg_slice_inverse_i8(n, ptr(LinvT), np_, ptr(sl), ptr(expo), s), "slice")
        ldg = -(-n // 16) * 16
        G = datagen.genotypes_device(spec, 0, args.cnt, ld=ldg)           # (cnt, ldg) int8
        X64 = alloc_cols(args.cnt, np_)
        check(lib.gg_widen_i8_f64(n, args.cnt, ptr(G), ldg, ptr(X64), np_, s), "widen")
        Xd = alloc_cols(args.cnt, np_)
        Xi = alloc_cols(args.cnt, np_)
        check(lib.gg_trsm_lower_packed_f64(n, args.cnt, ptr(LinvP), ptr(X64), np_, ptr(Xd), np_,
                                           s), "trsm dmma")
        check(lib.gg_trsm_lower_i8(n, args.cnt, ptr(sl), ptr(expo), ptr(G), ldg, ptr(Xi), np_, ptr(W), s),
              "trsm i8")
        torch.cuda.synchronize()
        diff = (Xi[:, :n] - Xd[:, :n]).abs().max().item()
        scale = Xd[:, :n].abs().max().item()
        colrel = ((Xi[:, :n] - Xd[:, :n]).abs().amax(1) / Xd[:, :n].abs().amax(1)).max().item()
        print(f"n={n} S={S}: max|i8 - dmma| = {diff:.3e} (max |Xbar| {scale:.3e}); "
              f"max column-relative {colrel:.3e}; pad rows zero: "
              f"{bool((Xi[:, n:] == 0).all().item())}", flush=True)
        perm = torch.randperm(args.cnt, device="cuda")
        Gp = G[perm].contiguous()
        Xp = alloc_cols(args.cnt, np_)
        check(lib.gg_trsm_lower_i8(n, args.cnt, ptr(sl), ptr(expo), ptr(Gp), ldg, ptr(Xp), np_, ptr(W), s),
              "trsm i8 perm")
        torch.cuda.synchronize()
        print(f"  permutation bitwise: {bool(torch.equal(Xp, Xi[perm]))}", flush=True)
        for name, fn in (("dmma", lambda: lib.gg_trsm_lower_packed_f64(
                n, args.cnt, ptr(LinvP), ptr(X64), np_, ptr(Xd), np_, s)),
                         ("i8", lambda: lib.gg_trsm_lower_i8(
                n, args.cnt, ptr(sl), ptr(expo), ptr(G), ldg, ptr(Xi), np_, ptr(W), s))):
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.reps):
                fn()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / args.reps
            fl = float(n) * n * args.cnt
            print(f"  {name}: {ms:.3f} ms per {args.cnt}-SNP block = {fl / ms / 1e9:.1f} "
                  f"TF/s FP64-equivalent ({args.cnt / ms * 1e3:.0f} SNPs/s)", flush=True)
        del sl, L, LinvP, LinvT, G, X64, Xd, Xi, Xp, Gp, Md
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
