"""What-ifs of the int8 TRSM inside the config-3 sweep (timing only, results invalid): prepare
runs normally, then the sweep is timed with GG_I8_WHATIF set (bits: 1 no genotype loads, 2 no
slice loads, 4 no epilogue work) and with optional tile-order knobs, printing SNPs/s, TOPS and the
median SM clock.

    python tools/whatif_trsm.py [--snps 2000000] [--steps 3] 0 4 ...

Tokens e0..e3 time the (bitwise-equal) epilogue forms instead: GG_I8_EPI bit 1 = I2F.F64.S64
conversions, bit 2 = one dot chain at a time (e0 = the default, e3 = the form before r02's end).
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
    ap.add_argument("whatifs", nargs="*", default=["0", "4"])
    args = ap.parse_args()
    import torch

    from paper_1304_2272_b200 import _capi

    dev = torch.device("cuda", 0)
    sw = bench.Sweep(args.config, args.snps, 1, 0, dev, 8192, "i8", "i8", keep_host_M=False)
    if "split" in args.whatifs:
        # the unfused form: the TRSM writes Xbar (no fused dots), then the standalone partials +
        # reduce/solve (gg_gls_epilogue_f64) read it back -- the same bits (one canonical order)
        from paper_1304_2272_b200._capi import ptr

        lib, d = _capi.lib(), sw.d
        X = torch.empty((sw.m_blk, sw.np_), dtype=torch.float64, device=dev)
        work = torch.empty(int(lib.gg_partials_bytes(sw.n, sw.m_blk, sw.q)), dtype=torch.uint8,
                           device=dev)

        def split_step(record):
            for i, (f, c) in enumerate(sw.plan):
                if record:
                    sw.ev_pairs[i][0].record(sw.stream)
                rc = lib.gg_trsm_lower_i8(sw.n, c, ptr(d.slices), ptr(d.expo), ptr(sw.Gres[f:]),
                                          sw.n16, ptr(X), sw.np_, ptr(sw.W8), sw.sh)
                if record:
                    sw.ev_pairs[i][1].record(sw.stream)
                rc |= lib.gg_gls_epilogue_f64(sw.n, c, sw.q, ptr(X), sw.np_, ptr(d.XLy), sw.np_,
                                              ptr(d.ybar), ptr(d.S_TL), ptr(d.b_T),
                                              ptr(sw.beta[f]), ptr(sw.status[f]), None,
                                              ptr(work), sw.sh)
                assert rc == 0, _capi.last_error()

    for w in args.whatifs + [args.whatifs[0]]:
        if w == "split":
            fused, sw.step = sw.step, split_step
            ms, clk, trsm_ms = bench.timed_sweep(sw, args.steps, 2, False, None, 0, dev)
            sw.step = fused
            print(f"split (TRSM + stores, then partials + solve) {sw.m * args.steps / (ms / 1e3):10.1f}"
                  f" SNPs/s  TRSM share {trsm_ms / (ms / args.steps):.3f}  {clk.get('sm_mhz')} MHz",
                  flush=True)
            continue
        if w.startswith("e"):   # epilogue form A/B (valid results): GG_I8_EPI=<digits after e>
            os.environ["GG_I8_WHATIF"] = "0"
            os.environ["GG_I8_EPI"] = w[1:]
        else:
            os.environ["GG_I8_WHATIF"] = w
            os.environ.pop("GG_I8_EPI", None)
        ms, clk, trsm_ms = bench.timed_sweep(sw, args.steps, 2, False, None, 0, dev)
        tops = int(_capi.lib().gg_i8_slices()) * float(sw.n) ** 2 * sw.m / (trsm_ms / 1e3) / 1e12
        print(f"GG_I8_{'EPI' if w.startswith('e') else 'WHATIF'}={w:3s} {sw.m * args.steps / (ms / 1e3):10.1f} SNPs/s  {tops:7.1f} TOPS"
              f"  {clk.get('sm_mhz')} MHz  {clk.get('power_w_max')} W", flush=True)
    os.environ.pop("GG_I8_WHATIF", None)
    os.environ.pop("GG_I8_EPI", None)


if __name__ == "__main__":
    main()
