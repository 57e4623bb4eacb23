#!/usr/bin/env python
"""Benchmark of the GLS hot path on B200 (BASELINE.json configs[1], the metric's config).

Workload: n = 10,000 individuals, p = 4, m = 200,000 SNPs per GPU, FP64, blocks of 8,192 SNPs
(24 full + one 3,392 tail), seeded synthetic BASELINE data.  One STEP is one
full sweep of the rank's 200,000 SNPs: per block one FP64 -> int8 narrow of the dosages (side
stream, one block ahead), one int8 tensor-core TRSM launch (Xbar = Linv * G with the per-SNP
partial dots fused into its epilogue) and one reduce + batched p x p solve launch.  The genotypes
(FP64, 16.2 GB per GPU) are resident in HBM when the timed region starts; they are larger than
L2, so no L2 flush is needed.  gls_prepare (Cholesky + inverse + slicing) runs once, outside the
step, timed apart.  `--trsm dmma` runs the FP64 DMMA TRSM + epilogue instead.

Multi-GPU (torchrun): SNP-sharded weak scaling — rank r owns markers [r*m, (r+1)*m) of an
N*m-marker panel; L is factored redundantly on every rank; no collective in the timed region
except the barriers that bracket it; time = max over ranks of the CUDA-event time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "GLS solves (SNPs/sec) at 1/2/4/8 B200; TRSM FP64 TFLOP/s vs FP64 peak"
UNIT = "SNPs/s"
# FP64 roofline denominator.  MEASURED_PEAKS.json carries no FP64 figure, so the peak is our own
# measurement on this pool's B200s: DMMA m8n8k4 sustained over 200 launches at 1965 MHz
# (tools/fp64_peak.cu, profiles/r01_fp64_peak.log).  cuBLAS DGEMM 8192^3 reached 35.48 there.
FP64_PEAK_TFLOPS = 37.09
FP64_PEAK_SOURCE = ("measured: DMMA m8n8k4 sustained 37.09 TF/s @1965 MHz, tools/fp64_peak.cu "
                    "(profiles/r01_fp64_peak.log); MEASURED_PEAKS.json has no FP64 entry")
# int8 tensor-core peak (the int8 TRSM's roofline): measured with tools/i8_peak.cu on this pool's
# B200 (tcgen05.mma.cta_group::1.kind::i8 M128 N256 K32 back to back on every SM).
I8_PEAK_TOPS = 4428.7
I8_PEAK_SOURCE = ("measured: tcgen05.mma.kind::i8 M128 N256 K32 back to back on 148 SMs, 4428.7 "
                  "TOPS (tools/i8_peak.cu, profiles/r01_i8_peak.log); MEASURED_PEAKS.json has no "
                  "int8 entry")
CPU_SAMPLE_SNPS = 4096
REF_SAMPLE_SNPS = 2048


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--snps", type=int, default=None, help="SNPs per GPU (default: config's m)")
    ap.add_argument("--block-snps", type=int, default=8192)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--trsm", choices=["i8", "dmma"], default="i8",
                    help="TRSM engine: int8 tensor cores with the sliced inverse (default) or "
                         "the FP64 DMMA kernel")
    ap.add_argument("--resident", choices=["f64", "i8"], default=None,
                    help="genotype storage in HBM (default: FP64 if it fits, else int8)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons, power = [], [], set(), []
        names = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "power_w_max": max(power) if power else None, "samples": len(sm),
                "reasons": sorted(reasons)}


def load_traffic(engine):
    """Per-launch DRAM bytes of the TRSM kernel from the committed ncu --set full summary."""
    path = os.path.join(REPO, "profiles", f"ncu_trsm_{engine}_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    except (OSError, ValueError):
        return None, None


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------

def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1304_2272_b200 import _capi, datagen, kernel, pipeline
    from paper_1304_2272_b200._capi import check, ptr
    from paper_1304_2272_b200._device import alloc_cols

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    use_dist = world > 1 or os.environ.get("GG_BENCH_FORCE_DIST") == "1"
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    lib = _capi.lib()
    spec = datagen.CONFIGS[args.config]
    m = args.snps or spec.m
    spec = dataclasses.replace(spec, m=m * world)     # the N*m-marker panel
    n, p = spec.n, spec.p
    q = p - 1
    np_ = _capi.pad(n)
    m_blk = args.block_snps

    # ---- data (identical M on every rank; rank-local marker range) --------------------------
    t0 = time.perf_counter()
    Md = datagen.kinship_covariance_device(spec)          # (n, n) on the device
    XL, y = datagen.covariates_host(spec)
    torch.cuda.synchronize()
    t_gen_m = time.perf_counter() - t0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    ctx = kernel.gls_prepare(Md, XL, y)                  # device-resident M, no host round trip
    e1.record()
    torch.cuda.synchronize()
    t_prepare = time.perf_counter() - t0
    prepare_ms_device = e0.elapsed_time(e1)
    d = ctx._dev
    M = Md.cpu().numpy() if (rank == 0 and world == 1 and not args.no_cpu_baseline) else None
    del Md
    # genotypes resident in HBM: FP64 (config 1) when they fit, else int8 {0,1,2} dosages (the
    # config 2/3 storage format)
    free_b, _ = torch.cuda.mem_get_info(dev)
    resident = args.resident or ("f64" if 8 * m * np_ < 0.6 * free_b else "i8")
    use_i8 = args.trsm == "i8" and d.slices is not None
    n16 = -(-n // 16) * 16
    first_marker = rank * m
    X = Gres = None
    if resident == "f64":
        X = torch.empty((m, np_), dtype=torch.float64, device=dev)
        X[:, n:].zero_()
        G = torch.empty((m_blk, n), dtype=torch.int8, device=dev)
        for j0 in range(0, m, m_blk):
            cnt = min(m_blk, m - j0)
            datagen.genotypes_device(spec, first_marker + j0, cnt, out=G)
            check(lib.gg_widen_i8_f64(n, cnt, ptr(G), n, ptr(X[j0:]), np_,
                                      _capi.stream_handle()), "widen")
        del G
    else:
        Gres = datagen.genotypes_device(spec, first_marker, m, ld=n16)   # (m, n16) int8
    # FP64-resident dosages are narrowed to int8 on a side stream, one block ahead, into a double
    # buffer: the HBM-bound narrow of block i+1 runs beside the tensor-core TRSM of block i
    g8s = [torch.empty((m_blk, n16), dtype=torch.int8, device=dev) for _ in range(2)] \
        if (use_i8 and X is not None) else None
    side = torch.cuda.Stream(device=dev) if g8s is not None else None
    narrow_done = [torch.cuda.Event() for _ in range(2)]
    trsm_done = [torch.cuda.Event() for _ in range(2)]
    trsm_started = [False, False]
    xin = alloc_cols(m_blk, np_) if (not use_i8 and X is None) else None
    xbar = alloc_cols(m_blk, np_, zero=False) if not use_i8 else None
    P = torch.empty(int(lib.gg_partials_bytes(n, m_blk, q)) // 8, dtype=torch.float64, device=dev)
    bad = torch.zeros((1,), dtype=torch.int32, device=dev)
    beta = torch.empty((m, p), dtype=torch.float64, device=dev)
    status = torch.empty((m,), dtype=torch.int32, device=dev)
    plan = pipeline.block_plan(m, m_blk).blocks
    stream = torch.cuda.current_stream()
    sh = _capi.C.c_void_p(stream.cuda_stream)
    ev_pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in plan]
    launches_per_block = 0
    serial_narrow = os.environ.get("GG_BENCH_SERIAL_NARROW") == "1"

    def step(record):
        nonlocal launches_per_block
        for i, (f, c) in enumerate(plan):
            rc = 0
            nl = 0
            if use_i8:
                if X is not None:            # FP64 dosages -> int8 (exactness flag checked after)
                    slot = i % 2
                    if serial_narrow:
                        rc |= lib.gg_narrow_f64_i8(n, c, ptr(X[f]), np_, ptr(g8s[slot]), n16,
                                                   ptr(bad), sh)
                    else:
                        with torch.cuda.stream(side):
                            if trsm_started[slot]:      # buffer free once its last TRSM is done
                                side.wait_event(trsm_done[slot])
                            rc |= lib.gg_narrow_f64_i8(n, c, ptr(X[f]), np_, ptr(g8s[slot]),
                                                       n16, ptr(bad),
                                                       _capi.C.c_void_p(side.cuda_stream))
                            narrow_done[slot].record(side)
                        stream.wait_event(narrow_done[slot])
                    G, ldg, nl = g8s[slot], n16, nl + 1
                else:
                    G, ldg = Gres[f:], n16
                if record:
                    ev_pairs[i][0].record(stream)
                rc |= lib.gg_trsm_lower_i8_partials(n, c, ptr(d.slices), ptr(d.expo), ptr(G), ldg,
                                                    q, ptr(d.XLy), ptr(d.ybar), ptr(P), None, 0,
                                                    None, 0, sh)
                if record:
                    ev_pairs[i][1].record(stream)
                if X is not None:
                    trsm_done[i % 2].record(stream)
                    trsm_started[i % 2] = True
                rc |= lib.gg_gls_reduce_solve_f64(n, c, q, ptr(P), ptr(d.S_TL), ptr(d.b_T),
                                                  ptr(beta[f]), ptr(status[f]), None, sh)
                nl += 2
            else:
                if X is not None:
                    src = X[f]
                else:
                    rc |= lib.gg_widen_i8_f64(n, c, ptr(Gres[f]), n16, ptr(xin), np_, sh)
                    src, nl = xin, nl + 1
                if record:
                    ev_pairs[i][0].record(stream)
                rc |= lib.gg_trsm_lower_packed_f64(n, c, ptr(d.LinvP), ptr(src), np_, ptr(xbar),
                                                   np_, sh)
                if record:
                    ev_pairs[i][1].record(stream)
                rc |= lib.gg_gls_epilogue_f64(n, c, q, ptr(xbar), np_, ptr(d.XLy), np_,
                                              ptr(d.ybar), ptr(d.S_TL), ptr(d.b_T), ptr(beta[f]),
                                              ptr(status[f]), None, ptr(P), sh)
                nl += 3          # TRSM + partials + reduce/solve
            if rc:
                raise RuntimeError(_capi.last_error())
            launches_per_block = nl
        return None

    def barrier():
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(False)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    trsm_ms = 0.0
    t_start.record(stream)
    for k in range(args.steps):
        step(True)
    t_end.record(stream)
    torch.cuda.synchronize()
    for a_ev, b_ev in ev_pairs:
        trsm_ms += a_ev.elapsed_time(b_ev)     # last step's per-launch times
    clk = clocks.stop()
    elapsed_ms = t_start.elapsed_time(t_end)
    barrier()
    if use_dist:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    if int(bad.item()) != 0:
        raise RuntimeError("non-integer dosages reached the int8 path")
    ok_all = bool((status >= 0).sum().item() == 0)
    snps_per_step_total = m * world
    value = snps_per_step_total * args.steps / (elapsed_ms / 1e3)
    traffic_full, ncu = load_traffic("i8" if use_i8 else "dmma")
    if ncu is not None and (ncu.get("n") != n or ncu.get("snps_per_launch") != m_blk):
        traffic_full, ncu = None, None      # the committed capture is of another workload
    flops_per_step = float(n) * n * m
    trsm_tflops = flops_per_step / (trsm_ms / 1e3) / 1e12          # FP64-equivalent rate
    step_tflops = flops_per_step * args.steps / (elapsed_ms / 1e3) / 1e12
    if use_i8:
        slices = int(lib.gg_i8_slices())
        tops = slices * flops_per_step / (trsm_ms / 1e3) / 1e12     # int8 ops: S slices x n^2
        roofline = {
            "bound": "tensor",
            "kernel": "trsm_i8_dual_kernel (persistent CTA-pair TMA + tcgen05.mma.kind::i8 TRSM, "
                      "two row blocks per tile, fused reductions; inverse split into int8 slices)",
            "achieved": round(tops, 1), "peak": I8_PEAK_TOPS, "unit": "TOPS",
            "frac": round(tops / I8_PEAK_TOPS, 4),
            "traffic": traffic_full,
            "algorithmic_unit": f"{slices} slices x n^2 int8 ops per SNP (exact int32 products of "
                                "the sliced inverse with the dosages) x SNPs per launch",
            "peak_source": I8_PEAK_SOURCE,
            "fp64_equivalent_tflops": round(trsm_tflops, 2),
            "fp64_equivalent_vs_dmma_peak": round(trsm_tflops / FP64_PEAK_TFLOPS, 3),
            "trsm_share_of_step": round(trsm_ms / (elapsed_ms / args.steps), 4),
        }
    else:
        roofline = {
            "bound": "tensor",
            "kernel": "trsm_tma_kernel (persistent TMA + DMMA TRSM, Xbar = Linv*X)",
            "achieved": round(trsm_tflops, 3), "peak": FP64_PEAK_TFLOPS,
            "unit": "TFLOP/s", "frac": round(trsm_tflops / FP64_PEAK_TFLOPS, 4),
            "traffic": traffic_full,
            "algorithmic_unit": "n^2 FLOP per SNP (LAPACK dtrsm count) x SNPs per launch",
            "peak_source": FP64_PEAK_SOURCE,
            "trsm_share_of_step": round(trsm_ms / (elapsed_ms / args.steps), 4),
        }

    if isinstance(clk, dict) and clk.get("sm_mhz") and clk.get("sm_max_mhz"):
        # the peak is quoted at the maximum SM clock; under the board's power cap the clock in the
        # timed region is lower -- the same peak scaled to the median measured clock
        scale = clk["sm_mhz"] / clk["sm_max_mhz"]
        roofline["peak_at_measured_clock"] = round(roofline["peak"] * scale, 1)
        roofline["frac_at_measured_clock"] = round(roofline["achieved"] / (roofline["peak"] * scale), 4)

    # ---- e2e through the public stream API with host buffers --------------------------------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, ctx, X if X is not None else Gres, n, m, world, rank, dev, np, torch,
                      dist if use_dist else None, pipeline)

    # ---- CPU baseline + sampled parity on rank 0 at N = 1 -----------------------------------
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, parity = run_cpu_baseline(M, XL, y, X if X is not None else Gres, n, beta, status,
                                       np)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(elapsed_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "dtype_detail": ("TRSM: exact int8 x int8 -> int32 tcgen05 products of a 7-slice split "
                             "of the FP64 inverse (+ integer diagonal head), one FP64 rounding per "
                             "element; reductions and p x p solves in FP64") if use_i8 else
                            "FP64 DMMA TRSM, FP64 reductions and solves",
            "config": {
                "workload": f"BASELINE config {args.config}: GLS sweep n={n}, p={p}, m={m} SNPs "
                            f"per GPU, FP64, blocks of {m_blk}; step = TRSM + fused epilogue "
                            f"over all m SNPs",
                "n": n, "p": p, "m_per_gpu": m, "m_total": m * world, "m_blk": m_blk,
                "blocks_per_step": len(plan), "parallelism": f"snp-shard x{world}",
                "resident": resident,
                "l2": "inputs larger than L2 (genotypes resident in HBM: "
                      f"{m * (np_ * 8 if resident == 'f64' else n) / 1e9:.1f} GB per GPU, "
                      f"{'FP64' if resident == 'f64' else 'int8, widened per block in the step'})",
                "t_prepare_s": round(t_prepare, 4),
                "prepare_device_ms": round(prepare_ms_device, 2),
                "t_generate_M_s": round(t_gen_m, 2),
                "step_fp64_tflops": round(step_tflops, 3),
                "all_snps_ok": ok_all,
            },
            "roofline": roofline,
            "gpu_launches": launches_per_block * len(plan) * args.steps,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "parity": parity,
        }
        if ncu is not None:
            line["roofline"]["traffic_source"] = ncu.get("source")
        print(json.dumps(line))
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, ctx, X, n, m, world, rank, dev, np, torch, dist, pipeline):
    """Same metric through the public stream API, pipeline.solve_array, with the genotypes in
    pinned host memory: every step H2D-copies all m markers (copy stream, double-buffered) and
    reads every block's results back.  Primary: int8 dosages on the host (the GWAI / config-2
    storage format, n bytes per SNP); also reported: FP64 host genotypes (8 n bytes per SNP,
    PCIe-bound) when host memory allows."""
    src = X[:, :n] if X.dtype == torch.float64 else X[:, :n]
    out = {}
    for dtype in ("i8", "f64"):
        if dtype == "f64":
            try:   # FP64 host genotypes need m*n*8 pinned bytes per rank
                import psutil

                if world * m * n * 8 > 0.5 * psutil.virtual_memory().available:
                    continue
            except ImportError:
                pass
        engine = pipeline.StreamEngine(ctx, args.block_snps, int8=dtype == "i8")
        tdt = torch.int8 if dtype == "i8" else torch.float64
        host_t = torch.empty((m, n), dtype=tdt).pin_memory()
        host_t.copy_(src.to(tdt))
        Xh = host_t.numpy().T                 # n x m, Fortran-ordered view of pinned memory
        res = pipeline.solve_array(ctx, Xh, engine=engine)      # warm-up
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        h0, d0 = engine.h2d_bytes, engine.d2h_bytes
        t0 = time.perf_counter()
        for _ in range(args.steps):
            res = pipeline.solve_array(ctx, Xh, engine=engine)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        out[dtype] = {
            "value": round(m * world * args.steps / dt, 1), "unit": UNIT,
            "h2d_bytes_per_step": int((engine.h2d_bytes - h0) // args.steps),
            "d2h_bytes_per_step": int((engine.d2h_bytes - d0) // args.steps),
            "api": "paper_1304_2272_b200.pipeline.solve_array (pinned host "
                   f"{'int8' if dtype == 'i8' else 'FP64'} genotypes, double-buffered H2D)",
            "all_snps_ok": bool(np.all(res.ok))}
        del host_t, engine, Xh
    e2e = dict(out["i8"])
    if "f64" in out:
        e2e["fp64_host"] = out["f64"]
    return e2e


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max((i.get("num_threads", 1) for i in threadpool_info()
                    if i.get("user_api") == "blas"), default=os.cpu_count())
    except Exception:   # pragma: no cover
        return os.cpu_count()


def run_cpu_baseline(M, XL, y, X, n, beta, status, np):
    """The CPU oracle (numpy/scipy restatement of the reference, oracle/gls_ref.py) on this
    host's cores: gls_prepare once, then one block of CPU_SAMPLE_SNPS markers; doubles as the
    sampled parity check of the GPU results."""
    from oracle import gls_ref as O

    S = CPU_SAMPLE_SNPS
    Xs = X[:S, :n].double().cpu().numpy().T.copy(order="F")
    t0 = time.perf_counter()
    octx = O.gls_prepare(M, XL, y)
    t_prep = time.perf_counter() - t0
    t0 = time.perf_counter()
    ob, ok = O.gls_solve_block(octx, Xs)
    t = time.perf_counter() - t0
    gb = beta[:S].cpu().numpy()
    gs = status[:S].cpu().numpy()
    gb = np.where((gs < 0)[:, None], gb, np.nan)
    rel, mism = O.compare(gb, ob)
    cpu = {"value": round(S / t, 2), "unit": UNIT, "cores": _blas_threads(), "kind": "port",
           "sample": f"oracle gls_solve_block on the first {S} SNPs of the workload at n={n} "
                     f"(prepare {t_prep:.2f} s excluded, like the GPU value)",
           "t_prepare_s": round(t_prep, 3)}
    parity = {"snps": S, "max_rel": rel, "status_mismatches": mism, "tol": 1e-9,
              "within": bool(mism == 0 and rel <= 1e-9)}
    return cpu, parity


# ---------------------------------------------------------------------------------------------
# reference arm: the reference's CPU implementation of the path (the oracle port) on host cores
# ---------------------------------------------------------------------------------------------

def run_reference(args):
    import numpy as np

    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import gls_ref as O
    from paper_1304_2272_b200 import datagen

    spec = datagen.CONFIGS[args.config]
    n, p = spec.n, spec.p
    S = REF_SAMPLE_SNPS
    t0 = time.perf_counter()
    M = datagen.kinship_covariance_host(spec)
    XL, y = datagen.covariates_host(spec)
    G = datagen.genotypes_host(spec.seed, n, spec.m, 0, S).astype(np.float64, order="F")
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    octx = O.gls_prepare(M, XL, y)
    t_prep = time.perf_counter() - t0
    for _ in range(args.warmup):
        O.gls_solve_block(octx, G)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.gls_solve_block(octx, G)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = S * args.steps / tot
    cores = _blas_threads()
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": f"BASELINE config {args.config}: GLS sweep n={n}, p={p}; each step "
                               f"= one {S}-SNP block through the reference CPU path",
                   "n": n, "p": p, "sample_snps_per_step": S, "t_prepare_s": round(t_prep, 3),
                   "t_generate_s": round(t_gen, 2)},
        "cpu_baseline": {"value": round(value, 2), "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{S}-SNP block of the config-{args.config} workload per step "
                                   "(oracle/gls_ref.py: scipy dtrsm + numpy reductions + batched "
                                   "p x p Cholesky, as kernel.py:315-342)"},
        "e2e": {"value": round(value, 2), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
