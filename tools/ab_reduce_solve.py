"""Time gg_gls_reduce_solve_f64 alone (config-3 or config-1 sizes, one 8,192-SNP block of random
partials) -- run once per library build (GG_LIB_PATH) for an A/B; prints ms per launch and the
achieved HBM GB/s over the partials it reads.

    [GG_LIB_PATH=tools/alt/x.so] python tools/ab_reduce_solve.py [--n 40000] [--q 7]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1304_2272_b200 import _capi  # noqa: E402
from paper_1304_2272_b200._capi import ptr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=40000)
    ap.add_argument("--q", type=int, default=7)
    ap.add_argument("--cnt", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    lib = _capi.lib()
    dev = torch.device("cuda", 0)
    n, q, cnt, p = a.n, a.q, a.cnt, a.q + 1
    nbytes = int(lib.gg_partials_bytes(n, cnt, q))
    g = torch.Generator(device=dev).manual_seed(0)
    P = torch.rand(nbytes // 8, dtype=torch.float64, device=dev, generator=g)
    S_TL = (torch.eye(q, dtype=torch.float64, device=dev) * 1e6).contiguous()
    b_T = torch.ones(q, dtype=torch.float64, device=dev)
    beta = torch.empty((cnt, p), dtype=torch.float64, device=dev)
    status = torch.empty((cnt,), dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    sh = _capi.stream_handle()
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(a.reps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(a.reps)]
    for i in range(a.reps + 3):
        flush.zero_()                           # cold L2, as inside the sweep (the TRSM ran between)
        j = max(0, i - 3)
        e0[j].record()
        rc = lib.gg_gls_reduce_solve_f64(n, cnt, q, ptr(P), ptr(S_TL), ptr(b_T), ptr(beta),
                                         ptr(status), None, sh)
        e1[j].record()
        assert rc == 0, _capi.last_error()
    torch.cuda.synchronize()
    ms = sorted(x.elapsed_time(y) for x, y in zip(e0, e1))
    med = ms[len(ms) // 2]
    rd = 8.0 * (q + 2) * cnt * (-(-n // 32))
    print(f"{os.environ.get('GG_LIB_PATH', 'in-tree')}: n={n} q={q} cnt={cnt}: median {med:.4f} ms, "
          f"{rd / med / 1e6:.0f} GB/s over {rd / 1e6:.0f} MB of partials; checksum "
          f"{float(beta.sum()):.17g}")


if __name__ == "__main__":
    main()
