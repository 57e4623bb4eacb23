"""Summarise ncu outputs into profiles/ (run here, on the CPU box, after gpurun brought them back).

    python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
        --tag r01 [--cnt 8192 --n 10000]

Writes profiles/<tag>_ncu_kernels.json (key metrics per profiled kernel), profiles/<tag>_launches.md
(share of device time per kernel from the launch list) and profiles/ncu_trsm_summary.json
(per-launch DRAM traffic of the TRSM kernel, read by bench.py for roofline.traffic).
"""

import argparse
import collections
import csv
import io
import json
import os
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROFILES = os.path.join(REPO, "profiles")

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "sm__cycles_active.avg",
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_si(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * SCALE.get(unit, 1)


def kernels(rep):
    hdr, units, rows = raw_rows(rep)
    ki = hdr.index("Kernel Name")
    res = []
    for r in rows:
        d = {"kernel": r[ki].split("(")[0]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = to_si(r[i], units[i])
                d[k + ".unit"] = "s" if units[i] in SCALE and "sec" in units[i] else units[i]
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += to_si(r[vi], r[ui])
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--cnt", type=int, default=8192)
    ap.add_argument("--q", type=int, default=3, help="covariates (p - 1) of the workload")
    ap.add_argument("--engine", choices=["dmma", "i8"], default="i8")
    args = ap.parse_args()
    os.makedirs(PROFILES, exist_ok=True)
    if args.rep:
        ks = kernels(args.rep)
        with open(os.path.join(PROFILES, f"{args.tag}_ncu_kernels.json"), "w") as f:
            json.dump({"source": os.path.basename(args.rep), "kernels": ks}, f, indent=1)
        trsm = [k for k in ks if ("trsm_i8" in k["kernel"]) == (args.engine == "i8")
                and ("trsm" in k["kernel"] or "dgemm" in k["kernel"])]
        if trsm:
            k = trsm[0]
            rd, wr = k.get("dram__bytes_read.sum"), k.get("dram__bytes_write.sum")
            if args.engine == "i8":   # int8 dosages in, 7 int8 slices of the triangle, partials out
                algo = (args.n * args.cnt + 7 * args.n * args.n / 2
                        + 8.0 * (args.q + 2) * args.cnt * args.n / 32)
            else:                     # FP64 block in, packed FP64 triangle, FP64 Xbar out
                algo = 8.0 * (args.n * args.cnt * 2 + args.n * args.n / 2)
            summ = {
                "source": f"profiles/{args.tag}_ncu_kernels.json ({os.path.basename(args.rep)}, "
                          "ncu --set full --clock-control none)",
                "kernel": k["kernel"], "n": args.n, "snps_per_launch": args.cnt,
                "dram_bytes_per_launch": (rd or 0) + (wr or 0),
                "dram_read_bytes": rd, "dram_write_bytes": wr,
                "algorithmic_bytes_per_launch": algo,
                "duration_s": k.get("gpu__time_duration.sum"),
                "dmma_pipe_active_pct": k.get(
                    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
            }
            suffix = "" if args.n == 10000 else f"_n{args.n}"
            with open(os.path.join(PROFILES, f"ncu_trsm_{args.engine}_summary{suffix}.json"),
                      "w") as f:
                json.dump(summ, f, indent=1)
            print(json.dumps(summ, indent=1))
    if args.launches:
        agg = launches(args.launches)
        tot = sum(v[1] for v in agg.values())
        lines = [f"# Launch list ({args.tag}): ncu --metrics gpu__time_duration.sum "
                 "--clock-control none (cold-cache, serialised: compare shares)", "",
                 "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for name, (cnt, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| `{name[:90]}` | {cnt} | {t * 1e3:.3f} | {100 * t / tot:.1f}% |")
        with open(os.path.join(PROFILES, f"{args.tag}_launches.md"), "w") as f:
            f.write("\n".join(lines) + "\n")
        print("\n".join(lines[:14]))


if __name__ == "__main__":
    main()
