"""What-if (timing only, results invalid): does the TRSM's power -- and so its clock under the
board's cap -- depend on the bits of the slice operand it streams?  Runs the config-3 sweep of
bench.py with the int8 slices replaced by (a) zeros, (b) random bytes confined to the low k bits,
and (c) the real slices, and prints SNPs/s, TOPS and the median SM clock of each.

    python tools/whatif_operands.py [--snps 262144] [--steps 3]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--snps", type=int, default=2_000_000)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    args = ap.parse_args()
    import torch

    from paper_1304_2272_b200 import _capi

    dev = torch.device("cuda", 0)
    sw = bench.Sweep(args.config, args.snps, 1, 0, dev, 8192, "i8", "i8", keep_host_M=False)
    real = sw.d.slices.clone()
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    # (name, low, high): uniform random digits in [low, high); None = the real slices, 0 = zeros
    variants = [("real slices", None), ("zero slices", 0), ("random [-2, 2)", (-2, 2)),
                ("random [-8, 8)", (-8, 8)), ("random [-128, 128)", (-128, 128)),
                ("random [0, 128)", (0, 128)), ("random [0, 64)", (0, 64)),
                ("random [-64, 64)", (-64, 64)), ("real |slices|", "abs"), ("real slices", None)]
    if os.environ.get("WHATIF_SET") == "first":
        variants = variants[:5] + variants[-1:]
    for name, rng in variants:
        if rng is None:
            sw.d.slices.copy_(real)
        elif rng == 0:
            sw.d.slices.zero_()
        elif rng == "abs":
            sw.d.slices.copy_(real.abs())
        else:
            r = torch.randint(rng[0], rng[1], real.shape, device=dev, dtype=torch.int16,
                              generator=g)
            sw.d.slices.copy_(r.to(torch.int8))
        ms, clk, trsm_ms = bench.timed_sweep(sw, args.steps, 2, False, None, 0, dev)
        tops = int(_capi.lib().gg_i8_slices()) * float(sw.n) ** 2 * sw.m / (trsm_ms / 1e3) / 1e12
        print(f"{name:22s} {sw.m * args.steps / (ms / 1e3):10.1f} SNPs/s  {tops:7.1f} TOPS  "
              f"{clk.get('sm_mhz')} MHz  {clk.get('power_w_max')} W", flush=True)


if __name__ == "__main__":
    main()
