"""What-if (timing only, results invalid): how much of the TRSM's power -- its clock under the
board's cap -- follows the dosage operand (A)?  Runs the config-3 sweep of bench.py with the
resident int8 dosages replaced in place by (a) zeros, (b) the dosages recentred on each marker's
most frequent value (more zeros, but -1 appears), (c) presence bits, (d) a sparse panel, and the
real dosages, printing SNPs/s, TOPS, the median SM clock and the zero fraction of each.

    python tools/whatif_genotypes.py [--snps 524288] [--steps 3]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--snps", type=int, default=524_288)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    args = ap.parse_args()
    import torch

    from paper_1304_2272_b200 import _capi

    dev = torch.device("cuda", 0)
    sw = bench.Sweep(args.config, args.snps, 1, 0, dev, 8192, "i8", "i8", keep_host_M=False)
    G = sw.Gres                              # (m, n16) int8, row j = marker j
    n = sw.n
    blk = 65536

    def apply(fn):
        for j0 in range(0, sw.m, blk):
            g = G[j0:j0 + blk, :n]
            g.copy_(fn(g, j0))

    def recentre(g, j0):
        cnt = torch.stack([(g == v).sum(dim=1) for v in (0, 1, 2)], dim=1)
        mode = cnt.argmax(dim=1).to(torch.int8)
        return g - mode[:, None]

    def sparse(g, j0):
        keep = torch.rand(g.shape, device=dev) < 0.2
        return torch.where(keep, g, torch.zeros_like(g))

    real = None
    variants = [("real {0,1,2}", None), ("recentred on the mode", recentre),
                ("presence bits g > 0", lambda g, j0: (g > 0).to(torch.int8)),
                ("80% of entries zeroed", sparse),
                ("all zero", lambda g, j0: torch.zeros_like(g)), ("real {0,1,2}", None)]
    host = G.cpu() if G.numel() < 3e10 else None     # restore between variants
    for name, fn in variants:
        if host is not None:
            G.copy_(host)
        if fn is not None:
            apply(fn)
        zf = sum(float((G[j0:j0 + blk, :n] == 0).sum()) for j0 in range(0, sw.m, blk)) / (
            float(sw.m) * n)
        ms, clk, trsm_ms = bench.timed_sweep(sw, args.steps, 2, False, None, 0, dev)
        tops = int(_capi.lib().gg_i8_slices()) * float(sw.n) ** 2 * sw.m / (trsm_ms / 1e3) / 1e12
        print(f"{name:24s} zeros {zf:5.3f}  {sw.m * args.steps / (ms / 1e3):10.1f} SNPs/s  "
              f"{tops:7.1f} TOPS  {clk.get('sm_mhz')} MHz  {clk.get('power_w_max')} W", flush=True)


if __name__ == "__main__":
    main()
