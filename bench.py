#!/usr/bin/env python
"""Benchmark of the GLS hot path on B200: BASELINE.json's metric on its headline configuration.

Headline workload (default, ``--config 3``): BASELINE configs[3] -- n = 40,000 individuals,
p = 8 (intercept + 6 N(0,1) covariates + SNP), m = 2,000,000 SNPs PER GPU, M = 0.5 K + 0.5 I,
blocks of 8,192 SNPs (244 full + one 1,152 tail), seeded synthetic BASELINE data (
no public dataset exists for this path).  It is the largest single-GPU configuration and the one
the "1/2/4/8 GPU" metric is quoted on.  One STEP is one full sweep of the rank's 2,000,000 SNPs:
per block one int8 tensor-core TRSM launch (Xbar = Linv * G with the per-SNP partial dots fused
into its TMEM epilogue) and one reduce + batched p x p solve launch.  The int8 dosages (80 GB per
GPU) are resident in HBM when the timed region starts -- far larger than L2, so no flush is
needed.  gls_prepare (Cholesky + inverse + slicing) runs once, outside the step, timed apart.

Also in the line:
  * e2e      -- the same metric through the reference-signature drop-in call
                kernel.gls_solve_block(ctx, SnpBlock(first, host_block)) (kernel.py:315-342) with
                the int8 dosages in pinned HOST memory: every step copies all m SNPs host->device
                and reads every block's results back (lazy ResultBlocks, resolved each step).
  * cpu_baseline + parity -- the CPU oracle (oracle/gls_ref.py, the reference's threads= path)
                on this host's cores: gls_prepare once (timed apart), then a sample of 2,048 SNPs
                -- 512 from each of the first block, two interior blocks and the last (partial)
                block -- which is also the parity set for the GPU results.
  * secondary -- BASELINE config 1 (n = 1e4, p = 4, m = 2e5, FP64-resident) measured the same
                way (value + roofline), for continuity with round 1.

Multi-GPU (``--gpus N``; the driver launches torchrun, a bare ``python bench.py --gpus N``
re-executes itself under torch.distributed.run): SNP-sharded weak scaling -- rank r owns markers
[r*m, (r+1)*m) of an N*m-marker panel; L is factored redundantly on every rank; no collective in
the timed region except the barriers that bracket it; time = max over ranks of the CUDA-event
time.

Other workloads: ``--config 2`` (n = 1e4, 1e7 SNPs, 100 GB of int8 dosages) at full size;
``--config 4`` (n = 1.5e5: M exceeds one GPU) runs the distributed engine's prepare -- every rank
generates its own blocks of M, the 2D block-cyclic Cholesky fused with the inverse, the int8
slices replicated -- and then the same sharded sweep with config 4's 1e6 markers spread 125,000
per GPU; ``--individuals N`` runs that form at a reduced n (one-GPU checks).  Both arms print the
same static ``config`` object (workload_config); measured prepare figures are under ``prepare``.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import socket
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
# int8 tensor-core peaks (the int8 TRSM's roofline), measured on this pool's B200 with the TRSM's
# own instruction shape (tools/i8_peak_pair.cu: tcgen05.mma.cta_group::2.kind::i8 M256 N224 K32
# back to back on 74 CTA pairs, operands resident in shared memory).  MEASURED_PEAKS.json has no
# int8 entry.  Burst = one 8-ms launch at full clock; sustained = back to back for 20 s (the board
# sits at its power cap) -- the denominator for a kernel timed inside a multi-second step.
I8_PEAK_BURST_TOPS = 4353.0
I8_PEAK_SUSTAINED_TOPS = float(os.environ.get("GG_I8_PEAK_SUSTAINED", "0")) or None
I8_PEAK_SOURCE = ("measured: tcgen05.mma.cta_group::2.kind::i8 M256 N224 K32 back to back on 148 "
                  "SMs (tools/i8_peak_pair.cu; burst: profiles/r01_i8_peak_pair.log; sustained "
                  "on the TRSM's operand statistics -- A {0,1,2}, B digits [0,127] -- under the "
                  "power cap: profiles/r02_peak_swap.log, profiles/i8_peak.json); "
                  "MEASURED_PEAKS.json has no int8 entry")
PEAK_FILE = os.path.join(REPO, "profiles", "i8_peak.json")
CPU_SAMPLE_PER_BLOCK = 512
REF_SAMPLE_SNPS = {0: 2048, 1: 2048, 2: 2048, 3: 512, 4: 128}


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--snps", type=int, default=None,
                    help="SNPs per GPU (default: config's m; config 4: its m over 8 GPUs)")
    # (names chosen not to abbreviate any torch.distributed.run option: its parser rejects "--n")
    ap.add_argument("--individuals", dest="n", type=int, default=None,
                    help="config 4 only: run its distributed form at a smaller n (one-GPU checks)")
    ap.add_argument("--grid-nb", dest="nb", type=int, default=512,
                    help="config 4: block-cyclic block size")
    ap.add_argument("--block-snps", type=int, default=8192)
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="timed e2e steps (default: min(steps, 5))")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the config-1 secondary measurement")
    ap.add_argument("--trsm", choices=["i8", "dmma"], default="i8",
                    help="TRSM engine: int8 tensor cores with the sliced inverse (default) or "
                         "the FP64 DMMA kernel")
    ap.add_argument("--resident", choices=["f64", "i8"], default=None,
                    help="genotype storage in HBM (default: FP64 if it fits, else int8)")
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_argv(args_list, gpus, port):
    """The torch.distributed.run command that runs this script on ``gpus`` ranks (one per GPU)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
            os.path.abspath(__file__)] + list(args_list)


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


def load_traffic(engine, n, snps):
    """Per-launch DRAM bytes of the TRSM kernel from the committed ncu --set full summaries
    (profiles/ncu_trsm_<engine>_summary*.json), for the capture whose workload matches."""
    import glob

    for path in sorted(glob.glob(os.path.join(REPO, "profiles", f"ncu_trsm_{engine}_summary*.json"))):
        try:
            with open(path) as f:
                d = json.load(f)
        except (OSError, ValueError):
            continue
        if d.get("n") == n and d.get("snps_per_launch") == snps:
            return d.get("dram_bytes_per_launch"), d
    return None, None


def measured_peaks():
    """The driver-written MEASURED_PEAKS.json (HBM GB/s, bf16 TF/s) when present."""
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def i8_peaks():
    """(burst, sustained) int8 TOPS of the TRSM's instruction shape (profiles/i8_peak.json when
    present: written from tools/i8_peak_pair runs on this pool's B200)."""
    burst, sust = I8_PEAK_BURST_TOPS, I8_PEAK_SUSTAINED_TOPS
    try:
        with open(PEAK_FILE) as f:
            d = json.load(f)
        burst = float(d.get("burst_tops", burst))
        sust = sust or d.get("sustained_tops")
    except (OSError, ValueError):
        pass
    return burst, (float(sust) if sust else None)


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------

class Sweep:
    """One rank's resident sweep of a BASELINE config: data on the device, gls_prepare done, and
    ``step()`` = one pass of the hot path over all the rank's markers."""

    def __init__(self, cfg, m, world, rank, dev, m_blk, trsm, resident, keep_host_M,
                 n=None, dist_prepare=None):
        import torch

        from paper_1304_2272_b200 import _capi, datagen, kernel, pipeline
        from paper_1304_2272_b200._capi import check, ptr

        self.torch, self.ptr, self.lib = torch, ptr, _capi.lib()
        base = datagen.CONFIGS[cfg]
        self.cfg = cfg
        self.m = m
        self.spec = spec = dataclasses.replace(base, m=m * world,      # the N*m-marker panel
                                               n=n or base.n)
        self.n, self.p = spec.n, spec.p
        n, q = spec.n, spec.p - 1
        self.q = q
        np_ = _capi.pad(n)
        self.np_ = np_
        self.m_blk = m_blk
        self.first_marker = rank * m
        self.XL, self.y = datagen.covariates_host(spec)
        if dist_prepare is not None:
            # config 4: M and L 2D block-cyclic over the ranks (never dense anywhere)
            self.ctx, self.t_gen_m, self.t_prepare, self.prepare_ms_device, self.dist_info = \
                dist_prepare(spec, self.XL, self.y)
            self.M = None
            if keep_host_M:     # reduced-n checks only: the dense bytes for the CPU oracle
                self.M = datagen.kinship_covariance_device(spec).cpu().numpy()
        else:
            t0 = time.perf_counter()
            Md = datagen.kinship_covariance_device(spec)          # (n, n) on the device
            torch.cuda.synchronize()
            self.t_gen_m = time.perf_counter() - t0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            self.ctx = kernel.gls_prepare(Md, self.XL, self.y)   # device-resident M, no host trip
            e1.record()
            torch.cuda.synchronize()
            self.t_prepare = time.perf_counter() - t0
            self.prepare_ms_device = e0.elapsed_time(e1)
            self.M = Md.cpu().numpy() if keep_host_M else None    # the CPU oracle's input bytes
            del Md
        d = self.d = self.ctx._dev
        free_b, _ = torch.cuda.mem_get_info(dev)
        self.resident = resident or default_resident(m, np_, free_b)
        self.use_i8 = trsm == "i8" and d.slices is not None
        n16 = self.n16 = -(-n // 16) * 16
        self.X = self.Gres = None
        if self.resident == "f64":
            self.X = torch.empty((m, np_), dtype=torch.float64, device=dev)
            self.X[:, n:].zero_()
            G = torch.empty((m_blk, n), dtype=torch.int8, device=dev)
            for j0 in range(0, m, m_blk):
                cnt = min(m_blk, m - j0)
                datagen.genotypes_device(spec, self.first_marker + j0, cnt, out=G)
                check(self.lib.gg_widen_i8_f64(n, cnt, ptr(G), n, ptr(self.X[j0:]), np_,
                                               _capi.stream_handle()), "widen")
            del G
        else:
            self.Gres = datagen.genotypes_device(spec, self.first_marker, m, ld=n16)
        # FP64-resident dosages are narrowed to int8 on a side stream, one block ahead, into a
        # double buffer: the HBM-bound narrow of block i+1 runs beside the TRSM of block i
        self.g8s = [torch.empty((m_blk, n16), dtype=torch.int8, device=dev) for _ in range(2)] \
            if (self.use_i8 and self.X is not None) else None
        self.side = torch.cuda.Stream(device=dev) if self.g8s is not None else None
        self.narrow_done = [torch.cuda.Event() for _ in range(2)]
        self.trsm_done = [torch.cuda.Event() for _ in range(2)]
        self.trsm_started = [False, False]
        from paper_1304_2272_b200._device import alloc_cols

        self.xin = alloc_cols(m_blk, np_) if (not self.use_i8 and self.X is None) else None
        self.xbar = alloc_cols(m_blk, np_, zero=False) if not self.use_i8 else None
        self.P = torch.empty(int(self.lib.gg_partials_bytes(n, m_blk, q)) // 8,
                             dtype=torch.float64, device=dev)
        self.bad = torch.zeros((1,), dtype=torch.int32, device=dev)
        self.W8 = _capi.i8_work(dev)
        self.beta = torch.empty((m, self.p), dtype=torch.float64, device=dev)
        self.status = torch.empty((m,), dtype=torch.int32, device=dev)
        self.plan = pipeline.block_plan(m, m_blk).blocks
        self.stream = torch.cuda.current_stream()
        self.sh = _capi.C.c_void_p(self.stream.cuda_stream)
        self.ev_pairs = [(torch.cuda.Event(enable_timing=True),
                          torch.cuda.Event(enable_timing=True)) for _ in self.plan]
        self.ev_rs = [(torch.cuda.Event(enable_timing=True),
                       torch.cuda.Event(enable_timing=True)) for _ in self.plan]
        self.rs_recorded = False
        self.launches_per_step = 0
        self._capi = _capi

    def step(self, record):
        self.torch.cuda.nvtx.range_push("step")
        try:
            self._step(record)
        finally:
            self.torch.cuda.nvtx.range_pop()

    def _step(self, record):
        lib, ptr, d, torch = self.lib, self.ptr, self.d, self.torch
        n, q, np_, n16 = self.n, self.q, self.np_, self.n16
        stream, sh = self.stream, self.sh
        nl = 0
        for i, (f, c) in enumerate(self.plan):
            rc = 0
            if self.use_i8:
                if self.X is not None:        # FP64 dosages -> int8 (exactness flag checked after)
                    slot = i % 2
                    with torch.cuda.stream(self.side):
                        if self.trsm_started[slot]:     # buffer free once its last TRSM is done
                            self.side.wait_event(self.trsm_done[slot])
                        rc |= lib.gg_narrow_f64_i8(n, c, ptr(self.X[f]), np_, ptr(self.g8s[slot]),
                                                   n16, ptr(self.bad),
                                                   self._capi.C.c_void_p(self.side.cuda_stream))
                        self.narrow_done[slot].record(self.side)
                    stream.wait_event(self.narrow_done[slot])
                    G, ldg = self.g8s[slot], n16
                    nl += 1
                else:
                    G, ldg = self.Gres[f:], n16
                if record:
                    self.ev_pairs[i][0].record(stream)
                rc |= lib.gg_trsm_lower_i8_partials(n, c, ptr(d.slices), ptr(d.expo), ptr(G), ldg,
                                                    q, ptr(d.XLy), ptr(d.ybar), ptr(self.P), None,
                                                    0, None, 0, ptr(self.W8), sh)
                if record:
                    self.ev_pairs[i][1].record(stream)
                if self.X is not None:
                    self.trsm_done[i % 2].record(stream)
                    self.trsm_started[i % 2] = True
                if record:
                    self.ev_rs[i][0].record(stream)
                rc |= lib.gg_gls_reduce_solve_f64(n, c, q, ptr(self.P), ptr(d.S_TL), ptr(d.b_T),
                                                  ptr(self.beta[f]), ptr(self.status[f]), None, sh)
                if record:
                    self.ev_rs[i][1].record(stream)
                    self.rs_recorded = True
                nl += 2
            else:
                if self.X is not None:
                    src = self.X[f]
                else:
                    rc |= lib.gg_widen_i8_f64(n, c, ptr(self.Gres[f]), n16, ptr(self.xin), np_, sh)
                    src = self.xin
                    nl += 1
                if record:
                    self.ev_pairs[i][0].record(stream)
                rc |= lib.gg_trsm_lower_packed_f64(n, c, ptr(d.LinvP), ptr(src), np_,
                                                   ptr(self.xbar), np_, sh)
                if record:
                    self.ev_pairs[i][1].record(stream)
                rc |= lib.gg_gls_epilogue_f64(n, c, q, ptr(self.xbar), np_, ptr(d.XLy), np_,
                                              ptr(d.ybar), ptr(d.S_TL), ptr(d.b_T),
                                              ptr(self.beta[f]), ptr(self.status[f]), None,
                                              ptr(self.P), sh)
                nl += 3          # TRSM + partials + reduce/solve
            if rc:
                raise RuntimeError(self._capi.last_error())
        self.launches_per_step = nl

    def trsm_ms(self):
        return sum(a.elapsed_time(b) for a, b in self.ev_pairs)   # the last recorded step

    def reduce_solve_hbm(self):
        """Achieved HBM GB/s of reduce_solve_kernel over the full blocks of the last recorded
        step: it reads the block's partials, 8 (q + 2) ceil(n / 32) bytes per SNP, once."""
        if not self.rs_recorded:
            return None
        full = [(i, c) for i, (f, c) in enumerate(self.plan) if c == self.m_blk] or \
               [(i, c) for i, (f, c) in enumerate(self.plan)]
        ms = statistics.median(self.ev_rs[i][0].elapsed_time(self.ev_rs[i][1]) for i, _ in full)
        c = full[0][1]
        nbytes = 8.0 * (self.q + 2) * c * (-(-self.n // 32))
        mp = measured_peaks() or {}
        peak = mp.get("hbm_gbs")
        gbs = nbytes / (ms / 1e3) / 1e9
        return {"kernel": "reduce_solve_kernel (partial sums in canonical order + p x p solves)",
                "ms_per_launch": round(ms, 4), "bytes_per_launch": int(nbytes),
                "achieved_gbs": round(gbs, 1), "peak_gbs": peak,
                "frac": round(gbs / peak, 4) if peak else None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peak else None}


def timed_sweep(sw, steps, warmup, use_dist, dist, local, dev):
    """W warm-up steps, then K timed steps bracketed by barrier + synchronize; returns
    (elapsed_ms max over ranks, clocks, trsm_ms of the last step)."""
    import torch

    def barrier():
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(warmup):
        sw.step(False)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record(sw.stream)
    for k in range(steps):
        sw.step(k == steps - 1)
    t_end.record(sw.stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    elapsed_ms = t_start.elapsed_time(t_end)
    barrier()
    if use_dist:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    return elapsed_ms, clk, sw.trsm_ms()


def roofline_obj(sw, steps, elapsed_ms, trsm_ms, clk, lib):
    n, m = sw.n, sw.m
    flops_per_step = float(n) * n * m
    trsm_tflops = flops_per_step / (trsm_ms / 1e3) / 1e12          # FP64-equivalent rate
    traffic, ncu = load_traffic("i8" if sw.use_i8 else "dmma", n, sw.m_blk)
    step_ms = elapsed_ms / steps
    if sw.use_i8:
        slices = int(lib.gg_i8_slices())
        tops = slices * flops_per_step / (trsm_ms / 1e3) / 1e12     # int8 ops: S slices x n^2
        burst, sustained = i8_peaks()
        long_step = step_ms > 1000.0
        peak = sustained if (long_step and sustained) else burst
        r = {
            "bound": "tensor",
            "kernel": "trsm_i8_dual_kernel (persistent CTA-pair TMA + tcgen05.mma.kind::i8 TRSM, "
                      "two row blocks per tile, fused reductions; inverse split into int8 slices)",
            "achieved": round(tops, 1), "peak": peak, "unit": "TOPS",
            "frac": round(tops / peak, 4),
            "traffic": traffic,
            "algorithmic_unit": f"{slices} slices x n^2 int8 ops per SNP (exact int32 products of "
                                "the sliced inverse with the dosages) x SNPs per launch",
            "algorithmic_bytes_per_launch": int(lib.gg_inverse_slices_bytes(n)) + n * sw.m_blk,
            "peak_kind": "sustained (kernel timed inside a multi-second step)"
                         if peak is sustained else "burst",
            "peak_burst": burst, "peak_sustained": sustained,
            "frac_of_burst": round(tops / burst, 4),
            "peak_source": I8_PEAK_SOURCE,
            "fp64_equivalent_tflops": round(trsm_tflops, 2),
            "fp64_equivalent_vs_dmma_peak": round(trsm_tflops / FP64_PEAK_TFLOPS, 3),
            "trsm_share_of_step": round(trsm_ms / step_ms, 4),
        }
        mp = measured_peaks()
        if mp:
            # the driver-measured file has no int8 figure; int8 dense is nominally 2x bf16 dense,
            # so 2x its cuBLAS bf16 rates are the int8 rates a library GEMM would imply -- lower
            # than our own measured tcgen05 int8 peaks, which stay the (stricter) denominator
            r["measured_peaks_json"] = {
                "bf16_tflops": mp.get("bf16_tflops"),
                "bf16_tflops_sustained": mp.get("bf16_tflops_sustained"),
                "implied_int8_tops_2x_bf16": (round(2 * mp["bf16_tflops"], 1)
                                              if mp.get("bf16_tflops") else None),
                "note": "no int8 entry in MEASURED_PEAKS.json; peak above is the stricter, "
                        "directly measured tcgen05 kind::i8 rate"}
    else:
        r = {
            "bound": "tensor",
            "kernel": "trsm_tma_kernel (persistent TMA + DMMA TRSM, Xbar = Linv*X)",
            "achieved": round(trsm_tflops, 3), "peak": FP64_PEAK_TFLOPS,
            "unit": "TFLOP/s", "frac": round(trsm_tflops / FP64_PEAK_TFLOPS, 4),
            "traffic": traffic,
            "algorithmic_unit": "n^2 FLOP per SNP (LAPACK dtrsm count) x SNPs per launch",
            "peak_source": FP64_PEAK_SOURCE,
            "trsm_share_of_step": round(trsm_ms / step_ms, 4),
        }
    if ncu is not None:
        r["traffic_source"] = ncu.get("source")
    if isinstance(clk, dict) and clk.get("sm_mhz") and clk.get("sm_max_mhz"):
        # the burst peak is quoted at the maximum SM clock; the same peak scaled to the median
        # clock measured in the timed region
        scale = clk["sm_mhz"] / clk["sm_max_mhz"]
        base = r.get("peak_burst", r["peak"])
        r["peak_at_measured_clock"] = round(base * scale, 1)
        r["frac_at_measured_clock"] = round(r["achieved"] / (base * scale), 4)
    return r


def fp64_path_sample(sw, blocks=3):
    """The same TRSM on the FP64 tensor pipe (trsm_tma_kernel: TMA-staged packed inverse, DMMA
    tiles) on one block of the workload, timed with CUDA events after a warm-up launch: the
    metric's "TRSM FP64 TFLOP/s vs FP64 peak" on the FP64 pipe itself, beside the int8 path's
    FP64-equivalent rate.  None when the context carries no packed FP64 inverse (config 4)."""
    import torch

    d = sw.d
    if getattr(d, "LinvP", None) is None:
        return None
    from paper_1304_2272_b200._device import alloc_cols

    lib, ptr, n, np_ = sw.lib, sw.ptr, sw.n, sw.np_
    f, c = sw.plan[0]
    xin = alloc_cols(c, np_)
    xbar = alloc_cols(c, np_, zero=False)
    if sw.X is not None:
        xin.copy_(sw.X[f:f + c])
    else:
        sw._capi.check(lib.gg_widen_i8_f64(n, c, ptr(sw.Gres[f]), sw.n16, ptr(xin), np_, sw.sh),
                       "widen")
    evs = []
    for i in range(blocks + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sw.stream)
        sw._capi.check(lib.gg_trsm_lower_packed_f64(n, c, ptr(d.LinvP), ptr(xin), np_, ptr(xbar),
                                                    np_, sw.sh), "gg_trsm_lower_packed_f64")
        e1.record(sw.stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in evs[1:])
    tf = float(n) * n * c / (ms / 1e3) / 1e12
    del xin, xbar
    return {"kernel": "trsm_tma_kernel (FP64 DMMA TRSM, the path of non-integer columns)",
            "snps": c, "ms_per_launch": round(ms, 3), "tflops": round(tf, 2),
            "peak": FP64_PEAK_TFLOPS, "frac": round(tf / FP64_PEAK_TFLOPS, 4),
            "snps_per_s": round(c / (ms / 1e3), 1), "peak_source": FP64_PEAK_SOURCE}


def default_resident(m, np_, free_bytes=None):
    """Genotype storage in HBM: FP64 when the m x np_ panel fits in 0.6 of the free memory (of a
    nominal 180 GB B200 when no device is queried: the reference arm), else int8."""
    free_b = 0.97 * 180e9 if free_bytes is None else free_bytes
    return "f64" if 8 * m * np_ < 0.6 * free_b else "i8"


def workload_config(cfg, m, world, m_blk, resident, n=None, nb=None):
    """The static description of the benched workload -- the same object on both arms."""
    from paper_1304_2272_b200 import datagen

    spec0 = datagen.CONFIGS[cfg]
    n, p = n or spec0.n, spec0.p
    from paper_1304_2272_b200._capi import pad

    np_ = pad(n)
    n16 = -(-n // 16) * 16
    gbytes = m * (np_ * 8 if resident == 'f64' else n16) / 1e9
    full_m = m == (spec0.m if cfg != 4 else spec0.m // 8)
    out = {
        "workload": f"BASELINE config {cfg}: GLS sweep n={n}, p={p}, m={m} SNPs "
                    f"per GPU ({'full m' if full_m else 'reduced m'}"
                    f"{'' if n == spec0.n else ', REDUCED n (the form of the config, not its size)'}"
                    f"), blocks of {m_blk}; step = TRSM + fused epilogue + p x p solves over all "
                    "m SNPs",
        "n": n, "p": p, "m_per_gpu": m, "m_total": m * world, "m_blk": m_blk,
        "blocks_per_step": -(-m // m_blk),
        "parallelism": f"snp-shard x{world}" if cfg != 4 else
                       f"prepare: M and L 2D block-cyclic (nb={nb}) over {world} ranks, distributed "
                       f"Cholesky + inverse, int8 slices replicated; sweep: snp-shard x{world}",
        "resident": resident,
        "l2": ("inputs larger than L2" if gbytes > 0.126 else
               "inputs SMALLER than L2 (a parity configuration, not a bench workload)")
              + f" (genotypes resident in HBM: {gbytes:.1f} GB per GPU, "
              f"{'FP64' if resident == 'f64' else 'int8'}); no flush",
    }
    return out


def make_dist_prepare(dist, world, rank, nb):
    """Config 4's prepare: every rank generates its own blocks of M on its
    GPU, the 2D block-cyclic Cholesky fused with the inverse (NCCL row / column broadcasts,
    look-ahead), the int8 slices assembled on every rank, [X_L | y] whitened from the
    block-cyclic inverse; no n x n array and no replicated FP64 inverse anywhere."""
    import numpy as np
    import torch

    from paper_1304_2272_b200 import distgrid, kernel
    from paper_1304_2272_b200.comm import as_comm

    def prepare(spec, XL, y):
        comm = as_comm(dist) if dist is not None else None
        ops = distgrid.DeviceOps()
        grid = distgrid.grid_create(world)
        nb_eff = min(nb, max(distgrid.SMALL_NB, -(-spec.n // 128) * 128))
        lay = distgrid.BlockCyclic(spec.n, nb_eff, grid, rank)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A, B = distgrid.local_from_spec(spec, lay, ops)
        torch.cuda.synchronize()
        t_gen = time.perf_counter() - t0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        distgrid.dist_potrf_inv(A, B, lay, ops, comm)
        del A
        torch.cuda.synchronize()
        t_factor = time.perf_counter() - t0
        S, e = distgrid.assemble_slices(B, lay, ops, comm)
        XLy = distgrid.whiten_blockcyclic(B, lay, ops, np.column_stack([XL, np.ravel(y)]), comm)
        del B
        ctx = kernel.prepare_from_inverse(None, spec.n, XL, y, slices=S, expo=e, XLy=XLy)
        e1.record()
        torch.cuda.synchronize()
        t_prep = time.perf_counter() - t0
        info = {"grid": f"{grid.r}x{grid.c}", "nb": nb_eff, "local_blocks": f"{lay.m_loc}x{lay.n_loc}",
                "t_factor_inverse_s": round(t_factor, 3),
                "t_slices_whiten_s": round(t_prep - t_factor, 3),
                "backend": str(dist.get_backend()) if dist is not None else "single rank"}
        return ctx, t_gen, t_prep, e0.elapsed_time(e1), info

    return prepare


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1304_2272_b200 import _capi, datagen

    rank, world, local = dist_env()
    if args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # one GPU per rank; GG_BENCH_BACKEND=gloo (a self-test of the multi-rank code path with several
    # ranks sharing a GPU) maps rank -> device modulo the device count
    backend = os.environ.get("GG_BENCH_BACKEND", "nccl")
    local = local % torch.cuda.device_count() if backend != "nccl" else local
    torch.cuda.set_device(local)
    use_dist = world > 1 or os.environ.get("GG_BENCH_FORCE_DIST") == "1"
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if world == 1:       # GG_BENCH_FORCE_DIST=1 without a launcher: a one-rank group
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
            os.environ.setdefault("MASTER_PORT", str(_free_port()))
        from paper_1304_2272_b200.comm import init_process_group

        init_process_group(backend, device=torch.device("cuda", local))
        # the communicator really spans N ranks
        t = torch.ones(1, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t)
        assert int(t.item()) == world == dist.get_world_size()
    dev = torch.device("cuda", local)
    lib = _capi.lib()
    spec0 = datagen.CONFIGS[args.config]
    dist_prepare = None
    if args.config == 4:
        # M (180 GB at n = 1.5e5) exceeds one GPU: the distributed engine's prepare, then the
        # SNP-sharded sweep on the replicated int8 slices; config 4's 1e6 markers over 8 GPUs
        m = args.snps or spec0.m // 8
        n_run = args.n or spec0.n
        dist_prepare = make_dist_prepare(dist if use_dist else None, world, rank, args.nb)
        # the CPU oracle needs the dense M and an O(n^3) factorisation: reduced-n checks only
        # (at N > 1 rank 0 still checks parity; the cpu_baseline object stays an N = 1 figure)
        want_cpu = rank == 0 and not args.no_cpu_baseline and n_run <= 20_000
    else:
        m = args.snps or spec0.m
        n_run = None
        # rank 0 checks parity at every N (its markers are the first m of the panel); the
        # cpu_baseline object itself stays an N = 1 figure (other ranks' spin-waits share the cores)
        want_cpu = rank == 0 and not args.no_cpu_baseline
    sw = Sweep(args.config, m, world, rank, dev, args.block_snps, args.trsm, args.resident,
               keep_host_M=want_cpu, n=n_run, dist_prepare=dist_prepare)
    elapsed_ms, clk, trsm_ms = timed_sweep(sw, args.steps, args.warmup, use_dist, dist, local,
                                           dev)
    if int(sw.bad.item()) != 0:
        raise RuntimeError("non-integer dosages reached the int8 path")
    ok_all = bool((sw.status >= 0).sum().item() == 0)
    value = m * world * args.steps / (elapsed_ms / 1e3)
    roofline = roofline_obj(sw, args.steps, elapsed_ms, trsm_ms, clk, lib)
    if sw.use_i8 and rank == 0:
        roofline["epilogue_hbm"] = sw.reduce_solve_hbm()
        roofline["fp64_dmma_path"] = fp64_path_sample(sw)
    beta_host = sw.beta.cpu().numpy()
    status_host = sw.status.cpu().numpy()

    # ---- CPU baseline + sampled parity (rank 0 at N = 1), before e2e frees nothing ----------
    cpu = parity = None
    if want_cpu:
        cpu, parity = run_cpu_baseline(sw, beta_host, status_host)
        sw.M = None
        if world > 1:
            cpu = None

    # ---- e2e through the reference-signature drop-in call with host buffers ------------------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, sw, world, rank, dev, use_dist, dist, beta_host)

    n, p = sw.n, sw.p
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(elapsed_ms / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "dtype_detail": ("TRSM: exact int8 x int8 -> int32 tcgen05 products of a 7-slice split "
                         "of the FP64 inverse (+ integer diagonal head), one FP64 rounding per "
                         "element; reductions and p x p solves in FP64") if sw.use_i8 else
                        "FP64 DMMA TRSM, FP64 reductions and solves",
        # static description of the workload: the reference arm prints the same object
        "config": workload_config(args.config, m, world, sw.m_blk, sw.resident, n=n_run,
                                  nb=args.nb),
        "prepare": {
            "t_prepare_s": round(sw.t_prepare, 4),
            "prepare_device_ms": round(sw.prepare_ms_device, 2),
            # SNPs/s end to end including the one-time prepare (one sweep + prepare)
            "snps_per_s_including_prepare": round(
                m * world / (elapsed_ms / 1e3 / args.steps + sw.t_prepare), 1),
            "t_generate_M_s": round(sw.t_gen_m, 2),
            **({"distributed": sw.dist_info} if dist_prepare is not None else {}),
        },
        "step_fp64_tflops": round(float(n) * n * m * args.steps / (elapsed_ms / 1e3) / 1e12, 3),
        "all_snps_ok": ok_all,
        "roofline": roofline,
        "gpu_launches": sw.launches_per_step * args.steps,
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity": parity,
    }
    del sw
    torch.cuda.empty_cache()
    if not args.no_secondary and args.config not in (1, 4):
        line["secondary"] = run_secondary(args, world, rank, local, dev, use_dist, dist)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()


def run_secondary(args, world, rank, local, dev, use_dist, dist):
    """BASELINE config 1 (n = 1e4, p = 4, m = 2e5 per GPU, FP64-resident), value + roofline."""
    import torch

    from paper_1304_2272_b200 import _capi, datagen

    m = datagen.CONFIGS[1].m
    sw = Sweep(1, m, world, rank, dev, args.block_snps, args.trsm, None, keep_host_M=False)
    steps, warmup = max(args.steps, 20), max(args.warmup, 5)
    elapsed_ms, clk, trsm_ms = timed_sweep(sw, steps, warmup, use_dist, dist, local, dev)
    out = {
        "workload": f"BASELINE config 1: GLS sweep n={sw.n}, p={sw.p}, m={m} SNPs per GPU, "
                    f"FP64-resident ({m * sw.np_ * 8 / 1e9:.1f} GB), blocks of {sw.m_blk}",
        "value": round(m * world * steps / (elapsed_ms / 1e3), 1), "unit": UNIT,
        "steps": steps, "warmup": warmup, "ms_per_step": round(elapsed_ms / steps, 3),
        "t_prepare_s": round(sw.t_prepare, 4),
        "all_snps_ok": bool((sw.status >= 0).sum().item() == 0),
        "roofline": roofline_obj(sw, steps, elapsed_ms, trsm_ms, clk, _capi.lib()),
        "gpu_launches": sw.launches_per_step * steps, "clocks": clk,
    }
    del sw
    torch.cuda.empty_cache()
    return out


def _host_register(arr):
    """Page-lock a numpy array in place (cudaHostRegister; no power-of-two rounding like the
    caching pinned allocator, which would turn 80 GB into 128 GB)."""
    import torch

    rt = torch._C._cudart
    err = rt.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
    if int(err) != 0:
        raise RuntimeError(f"cudaHostRegister failed ({err})")
    return lambda: rt.cudaHostUnregister(arr.ctypes.data)


def run_e2e(args, sw, world, rank, dev, use_dist, dist, beta_ref):
    """The metric end to end through the reference-signature call
    kernel.gls_solve_block(ctx, SnpBlock(first, data)) (kernel.py:315-342) with the int8
    dosages in pinned host memory: each step copies every block host->device (copy stream) and
    resolves every ResultBlock (device->host of beta and status)."""
    import numpy as np
    import torch

    from paper_1304_2272_b200 import _capi, kernel

    n, m, m_blk = sw.n, sw.m, sw.m_blk
    steps = args.e2e_steps if args.e2e_steps is not None else min(args.steps, 5)
    steps = max(1, steps)
    # host copy of the rank's dosages (n x m, F-order) when host memory allows; else a ring of
    # genuine blocks reused cyclically (same bytes per step, same H2D volume)
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except ImportError:   # pragma: no cover
        avail = 1 << 62
    if os.environ.get("GG_BENCH_E2E_HOST_GB"):     # self-test knob: pretend the host has this much
        avail = int(float(os.environ["GG_BENCH_E2E_HOST_GB"]) * 1e9)
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    fits = local_world * n * m < 0.6 * avail
    ring = None if fits else max(2, int(0.5 * avail / local_world / (n * m_blk)))
    cols = m if fits else min(m, ring * m_blk)
    while True:   # page-lock the host panel; on refusal (memlock limit, fragmentation) halve it
        host = np.empty((cols, n), dtype=np.int8)            # row j = marker j (n x cols F-order)
        try:
            unreg = _host_register(host)
            break
        except RuntimeError:
            if cols <= 2 * m_blk:
                raise
            fits = False
            cols = max(2 * m_blk, (cols // 2) // m_blk * m_blk)
            ring = cols // m_blk
            del host
    try:
        lib, sh = _capi.lib(), _capi.stream_handle()
        for j0 in range(0, cols, m_blk):
            c = min(m_blk, cols - j0)
            if sw.Gres is not None:
                blk, ld = sw.Gres[j0:j0 + c], sw.n16
            else:
                blk, ld = sw.X[j0:j0 + c, :n].to(torch.int8).contiguous(), n
            # pitched device -> pinned host copy (kind 2)
            _capi.check(lib.gg_memcpy2d_async(_capi.C.c_void_p(host.ctypes.data + j0 * n), n,
                                              _capi.C.c_void_p(blk.data_ptr()), ld, n, c, 2, sh),
                        "gg_memcpy2d_async")
            torch.cuda.synchronize()
        Xh = host.T                                           # n x cols, Fortran-ordered view
        plan = sw.plan

        def one_step(collect):
            blocks = []
            for f, c in plan:
                h0 = f % cols if not fits else f
                blocks.append(kernel.gls_solve_block(
                    sw.ctx, kernel.SnpBlock(sw.first_marker + f, Xh[:, h0:h0 + c])))
            arrays = [b.arrays for b in blocks]               # D2H of every block's results
            return arrays

        one_step(False)                                       # warm-up (engine creation)
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            arrays = one_step(True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if use_dist:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        beta = np.concatenate([a.beta for a in arrays])
        ok = np.concatenate([a.ok for a in arrays])
        # ring mode: only the first `cols` markers are the panel's own data (the later blocks
        # re-use ring blocks); those must still equal the resident sweep bit for bit
        ncmp = m if fits else cols
        same = bool(np.array_equal(beta[:ncmp], beta_ref[:ncmp], equal_nan=True))
    finally:
        unreg()
    p = sw.p
    return {
        "value": round(m * world * steps / dt, 1), "unit": UNIT,
        "h2d_bytes_per_step": int(n * m), "d2h_bytes_per_step": int(m * (8 * p + 4)),
        "host_link_gbs": round(n * m * steps / dt / 1e9, 2),
        "steps": steps,
        "api": "paper_1304_2272_b200.kernel.gls_solve_block(ctx, SnpBlock(first, host int8 "
               f"n x {m_blk} view)) per block -- the reference signature (kernel.py:315-342); "
               "pinned host dosages, copy stream overlapped with the previous block's compute, "
               "ResultBlocks resolved every step",
        "host_data": "full panel in pinned host memory" if fits else
                     f"ring of {ring} genuine blocks reused cyclically (host memory)",
        "all_snps_ok": bool(np.all(ok)),
        "bitwise_equal_to_device_resident_sweep": same,
        "bitwise_compared_snps": int(m if fits else cols),
    }


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max((i.get("num_threads", 1) for i in threadpool_info()
                    if i.get("user_api") == "blas"), default=os.cpu_count())
    except Exception:   # pragma: no cover
        return os.cpu_count()


_BLAS_LIMITS = []   # keeps the threadpoolctl limiter alive for the life of the process


def _host_cpu():
    """os.cpu_count() and the lscpu model name of the box."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.lower().startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_count": os.cpu_count(), "cpu_model": model}


def _host_threads():
    """BLAS threads the CPU arm may use: the library's own count, except under torchrun, which
    starts every rank with OMP_NUM_THREADS=1 -- there the host's cores are given back (the
    dpotrf of an n = 4e4 M on one thread takes minutes, and the reference arm is to run "with all
    the host threads it can use")."""
    cores = _blas_threads()
    if cores < (os.cpu_count() or 1) and os.environ.get("OMP_NUM_THREADS") == "1":
        try:
            from threadpoolctl import threadpool_limits

            _BLAS_LIMITS.append(threadpool_limits(limits=os.cpu_count(), user_api="blas"))
            cores = _blas_threads()
        except Exception:   # pragma: no cover
            pass
    return cores


def sample_columns(m, m_blk, per_block):
    """BASELINE.md §3 parity/baseline sample: the first block, two interior blocks and the last
    (partial) block -- per block its first and last per_block/2 markers (the block edges)."""
    import numpy as np

    nb = -(-m // m_blk)
    picks = sorted({0, nb // 3, (2 * nb) // 3, nb - 1})
    cols = []
    for b in picks:
        f = b * m_blk
        c = min(m_blk, m - f)
        h = min(per_block // 2, c // 2) if c >= 2 else c
        cols.extend(range(f, f + h))
        cols.extend(range(f + c - (per_block - h if c >= per_block else c - h), f + c))
    return np.unique(np.array(cols, dtype=np.int64)), picks


def run_cpu_baseline(sw, beta_gpu, status_gpu):
    """The CPU oracle (numpy/scipy restatement of the reference, oracle/gls_ref.py) on this
    host's cores: gls_prepare once (timed apart), then gls_solve_block(threads=cores) on the
    BASELINE.md §3 block sample; the same sample is the parity set of the GPU sweep."""
    import numpy as np

    from oracle import gls_ref as O

    cores = _host_threads()
    cols, picks = sample_columns(sw.m, sw.m_blk, CPU_SAMPLE_PER_BLOCK)
    if sw.Gres is not None:
        G = sw.Gres[cols][:, :sw.n]
    else:
        G = sw.X[cols][:, :sw.n]
    Xs = G.double().cpu().numpy().T.copy(order="F")
    t0 = time.perf_counter()
    octx = O.gls_prepare(sw.M, sw.XL, sw.y)
    t_prep = time.perf_counter() - t0
    t0 = time.perf_counter()
    ob, ok = O.gls_solve_block(octx, Xs, threads=cores)
    t = time.perf_counter() - t0
    gb = np.where((status_gpu[cols] < 0)[:, None], beta_gpu[cols], np.nan)
    rel, mism = O.compare(gb, ob)
    S = len(cols)
    cpu = {"value": round(S / t, 2), "unit": UNIT, "cores": cores, "kind": "port",
           "sample": f"oracle gls_solve_block(threads={cores}) on {S} SNPs of the workload "
                     f"(n={sw.n}): the first/last {CPU_SAMPLE_PER_BLOCK // 2} markers of blocks "
                     f"{picks} of {-(-sw.m // sw.m_blk)} (first, two interior, last partial); "
                     f"prepare {t_prep:.1f} s excluded, like the GPU value",
           "t_prepare_s": round(t_prep, 3), "t_sample_s": round(t, 3), **_host_cpu()}
    parity = {"snps": S, "blocks": picks, "max_rel": rel, "status_mismatches": mism, "tol": 1e-9,
              "within": bool(mism == 0 and rel <= 1e-9),
              "oracle": "oracle/gls_ref.py (scipy dpotrf/dtrsm + numpy reductions), same M bytes"}
    return cpu, parity


# ---------------------------------------------------------------------------------------------
# reference arm: the reference's CPU implementation of the path (the oracle port) on host cores
# ---------------------------------------------------------------------------------------------

def kinship_host_lean(spec):
    """M = a Z Z^T / m_k + (1 - a) I as datagen.kinship_covariance_host computes it (same
    operations, same bits), in place: at n = 4e4 the dense temporaries of the plain expression
    would need ~70 GB of host memory."""
    import numpy as np

    from paper_1304_2272_b200 import datagen

    Z = datagen.standardized_host(spec.seed, spec.n, spec.m_kin, spec.maf)
    K = Z @ Z.T
    del Z
    K /= spec.m_kin
    K *= spec.a
    K.flat[:: spec.n + 1] += (1.0 - spec.a)
    n, B = spec.n, 2048
    for i0 in range(0, n, B):                 # mirror the lower triangle (exact symmetry)
        i1 = min(n, i0 + B)
        K[i0:i1, i0:i1] = np.tril(K[i0:i1, i0:i1]) + np.tril(K[i0:i1, i0:i1], -1).T
        if i1 < n:
            K[i0:i1, i1:] = K[i1:, i0:i1].T
    return K


def run_reference(args):
    import numpy as np

    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import gls_ref as O
    from paper_1304_2272_b200 import datagen
    from paper_1304_2272_b200._capi import pad

    spec = datagen.CONFIGS[args.config]
    m_ws = args.snps or spec.m
    if args.config == 4:     # our arm's config-4 workload (and its reduced-n form, --n)
        spec = dataclasses.replace(spec, n=args.n or spec.n)
        m_ws = args.snps or spec.m // 8
    n, p = spec.n, spec.p
    if n > 60_000:
        # the CPU path needs the dense M (8 n^2 bytes of host memory) and an O(n^3) dpotrf:
        # 180 GB and ~1e15 flops at config 4's n = 1.5e5 -- not a bounded sample of minutes
        print(json.dumps({"impl": "reference", "unavailable":
                          f"config {args.config} at n={n}: the CPU reference needs a dense "
                          f"{8 * n * n / 1e9:.0f} GB M and an O(n^3) factorisation (hours on host "
                          "cores); run --individuals <= 60000 for the same form at a reduced n"}),
              flush=True)
        return
    S = REF_SAMPLE_SNPS.get(args.config, 512)
    cores = _host_threads()
    t0 = time.perf_counter()
    M = kinship_host_lean(spec)
    XL, y = datagen.covariates_host(spec)
    G = datagen.genotypes_host(spec.seed, n, spec.m, 0, S).astype(np.float64, order="F")
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    octx = O.gls_prepare(M, XL, y)
    t_prep = time.perf_counter() - t0
    del M
    for _ in range(args.warmup):
        O.gls_solve_block(octx, G, threads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.gls_solve_block(octx, G, threads=cores)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = S * args.steps / tot
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        # the workload of our arm (same static object); each step of this arm is a bounded
        # sample of it, described in "sample" / cpu_baseline.sample
        "config": workload_config(args.config, m_ws, world, args.block_snps,
                                  args.resident or default_resident(m_ws, pad(n)),
                                  n=args.n if args.config == 4 else None, nb=args.nb),
        "sample": {"snps_per_step": S, "t_prepare_s": round(t_prep, 3),
                   "t_generate_s": round(t_gen, 2),
                   "what": f"each step = one {S}-SNP block of the workload through the reference "
                           f"CPU path (gls_solve_block, threads={cores})"},
        "cpu_baseline": {"value": round(value, 2), "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{S}-SNP block of the config-{args.config} workload per step "
                                   f"(oracle/gls_ref.py: scipy dtrsm on {cores} BLAS threads + the "
                                   f"reference's threads={cores} column split of the per-SNP "
                                   "epilogue, kernel.py:315-342); gls_prepare timed apart",
                         **_host_cpu()},
        "e2e": {"value": round(value, 2), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main(argv=None):
    args = parse_args(argv)
    rank, world, _ = dist_env()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-run this script under torch.distributed.run
        cmd = relaunch_argv(sys.argv[1:] if argv is None else argv, args.gpus, _free_port())
        raise SystemExit(subprocess.call(cmd))
    if os.environ.get("GG_BENCH_LAUNCH_PROBE") == "1":
        launch_probe(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


def launch_probe(args):
    """Launcher self-test (CPU, gloo): every rank joins one process group and rank 0 prints how
    many ranks it saw -- proves ``--gpus N`` starts N ranks (tests/test_bench_contract.py)."""
    import torch
    import torch.distributed as dist

    rank, world, _ = dist_env()
    if args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    dist.init_process_group("gloo")
    t = torch.ones(1)
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"n_gpus": world, "ranks_seen": int(t.item())}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
