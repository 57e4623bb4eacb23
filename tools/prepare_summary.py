"""Summarise an ncu launch list of gls_prepare (several metrics per launch) into profiles/.

    ncu --nvtx --nvtx-include "gls_prepare/" --metrics gpu__time_duration.sum,<pipe metrics>,
        dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file X.csv \
        python tools/prof_prepare.py --n 10000 40000
    python tools/prepare_summary.py X.csv --out profiles/r02_prepare_launches.md

Each prepare run starts at its potrf's input check (nonfinite_kernel); the second run of each n (warm) is
summarised: per kernel the launches, device time, share, time-weighted pipe utilisation and
DRAM bytes.
"""

import argparse
import collections
import csv

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "%": 1.0}
FIRST = "init_factor"           # the first launch of every gls_prepare (potrf's input pass)
PIPES = [("DMMA", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
         ("FP64", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
         ("tensor (all)", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
         ("tcgen05 (tc)", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active")]


def val(v, u):
    try:
        return float(v.replace(",", "")) * SCALE.get(u, 1.0)
    except ValueError:
        return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--out", required=True)
    ap.add_argument("--ns", type=int, nargs="+", default=[10000, 40000])
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ui, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"), h.index("ID"))
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        d = per[int(r[ii])]
        d[r[mi]] = val(r[vi], r[ui])
        d["name"] = r[ki].split("(")[0]
    runs, cur = [], []
    for i in sorted(per):
        if FIRST in per[i]["name"] and cur:
            runs.append(cur)
            cur = []
        cur.append(i)
    runs.append(cur)
    runs = [r for r in runs if any(FIRST in per[i]["name"] for i in r)]
    out = ["# gls_prepare launch list (ncu --clock-control none; cold-cache, serialised: compare "
           "shares)", "",
           "Per kernel: launches, device time, share of the prepare, time-weighted pipe "
           "utilisation (% of peak sustained active), DRAM bytes.  `tcgen05 (tc)` is the int8 "
           "tensor pipe of the Ozaki-scheme GEMMs; DMMA the FP64 tensor pipe.", ""]
    for n, run in zip(args.ns, runs[1::2]):
        agg = collections.defaultdict(lambda: collections.defaultdict(float))
        for i in run:
            d = per[i]
            a = agg[d["name"]]
            t = d.get("gpu__time_duration.sum", 0.0)
            a["n"] += 1
            a["t"] += t
            for _, m in PIPES:
                a[m] += t * d.get(m, 0.0)
            a["dram"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        tot = sum(a["t"] for a in agg.values())
        out += [f"## n = {n:,} (second prepare of the run): {tot * 1e3:.1f} ms of device time", "",
                "| kernel | launches | ms | share | " + " | ".join(p for p, _ in PIPES)
                + " | DRAM GB |", "|---|---|---|---|" + "---|" * len(PIPES) + "---|"]
        for name, a in sorted(agg.items(), key=lambda x: -x[1]["t"]):
            if a["t"] / tot < 0.001:
                continue
            pipes = " | ".join(f"{a[m] / a['t']:.1f}%" if a["t"] else "-" for _, m in PIPES)
            out.append(f"| `{name[:70]}` | {int(a['n'])} | {a['t'] * 1e3:.2f} | "
                       f"{100 * a['t'] / tot:.1f}% | {pipes} | {a['dram'] / 1e9:.2f} |")
        out.append("")
    open(args.out, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
