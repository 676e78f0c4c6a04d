#!/usr/bin/env python
"""Benchmark of the HSF path-evaluation hot path (BASELINE.json metric:
"HSF paths/s and output amplitudes/s at 1/2/4/8 B200; % of HBM/tensor roofline").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]

One step = one hsf_run over this rank's path range: path-tree simulation of
both halves + coefficient fold + path-sum (+ for N > 1 one NCCL collective).
Default workload: configs[1] = c2 (n=24 QFT, 4096 joint-cut paths, all 2^24
amplitudes, complex64).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "HSF paths/s"
# dram bytes read + written per launch of the dominant kernel, from one
# `ncu --set full` capture of the same workload (profiles/r01/*details.txt)
# L2-resident read bandwidth measured on the box (scripts/probe/l2bw.cu: 16 B
# __ldcg loads over a 64 MiB L2-resident buffer, 592 CTAs x 512 threads): the
# second denominator for kernels whose operands stay in L2 (frac > 1 vs HBM)
L2_READ_GBS = 19710.0
NCU_TRAFFIC = {("c2", "gemm"): 1.2576e9 + 0.1205e9}  # profiles/r01/h_c2_gemm_mn_details.txt (MN-major GEMM)


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--precision", default="auto")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--standard", action="store_true",
                    help="also time standard HSF (every crossing gate cut alone) on the same output: T/J")
    ap.add_argument("--collective", default="auto", choices=["auto", "reduce_scatter", "allreduce", "rows", "fused_rs"],
                    help="N>1 exchange (paper_2502_06959_b200/dist.py); auto = cheapest for the output mode; "
                         "fused_rs = GEMM epilogue reduce-adds into the owners' shards over peer memory")
    return ap.parse_args()


def _instance(name):
    from hsf_inputs import make_config
    return make_config(name)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _nvml_loop(self):
        """NVML polling every 2 ms (an nvidia-smi call takes ~50-100 ms, longer
        than c2's whole timed region); same fields as the nvidia-smi query."""
        import pynvml as N
        N.nvmlInit()
        try:
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            bits = [getattr(N, "nvmlClocksEventReasonHwSlowdown", 0x8), getattr(N, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                    getattr(N, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                    getattr(N, "nvmlClocksEventReasonSwPowerCap", 0x4)]
            while not self._stop.is_set():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(h) if hasattr(N, "nvmlDeviceGetCurrentClocksEventReasons") \
                    else N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.rows.append([str(sm), str(mx), hex(rs)] + ["Active" if rs & b else "Not Active" for b in bits])
                self._stop.wait(0.002)
        finally:
            N.nvmlShutdown()

    def _loop(self):
        try:
            self._nvml_loop()
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                r = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                    "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if r.returncode == 0 and r.stdout.strip():
                    self.rows.append([x.strip() for x in r.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "source": "NVML every 2 ms" if self.rows and self.rows[0][2].startswith("0x") else "nvidia-smi"}


# ------------------------------------------------------------ reference arm
_ORACLE_PLANS = {}


def cpu_oracle_rate(inst, budget_s: float = 15.0):
    """The oracle as it stands, on a bounded sample of the same workload:
    a prefix of the paths (both half-circuits from scratch per path) and the
    Kronecker path-sum of that prefix over the full output / bitstring set.
    Returns (paths/s, sample description, threads)."""
    from oracle import hsf_oracle as O
    n, g = O.parse_circuit(inst.text)
    t0 = time.perf_counter()
    if inst.name not in _ORACLE_PLANS:  # the plan is excluded from the rate: build it once
        blocks = O.find_cascades(g, inst.n_low)[0] if inst.blocks == "auto" else inst.blocks
        _ORACLE_PLANS[inst.name] = (O.plan(n, g, inst.n_low, blocks), time.perf_counter() - t0)
    P, t_plan = _ORACLE_PLANS[inst.name]
    k = 1
    done = 0
    t_sim = 0.0
    # full outputs beyond 2^24 amplitudes: the Kronecker sum over a row subset,
    # the rate scaled by the fraction of rows (c4: 2^34 outputs)
    rows_all = 1 << (n - inst.n_low)
    if inst.meta.get("prefix"):  # the workload itself is a row prefix (first 10^6 amplitudes)
        rows_all = -(-inst.meta["prefix"] // (1 << inst.n_low))
    rows = rows_all if inst.bitstrings is not None else max(1, min(rows_all, (1 << 24) >> inst.n_low))
    while True:
        t1 = time.perf_counter()
        A, B, c = O.half_states(P, done, min(P.n_paths, done + k))
        if inst.bitstrings is None:
            O.recombine_full(A[:rows], B, c)
        else:
            O.recombine_bits(A, B, c, inst.bitstrings, inst.n_low)
        t_sim += time.perf_counter() - t1
        done = min(P.n_paths, done + k)
        if t_sim > budget_s or done >= P.n_paths:
            break
        k = max(1, min(P.n_paths - done, int(k * 2)))
    threads = int(os.environ.get("OMP_NUM_THREADS", "0")) or len(os.sched_getaffinity(0))
    if inst.bitstrings is None:
        out = "full 2^%d output" % n if rows == rows_all else \
            "%d of %d output rows (rate scaled by the row fraction)" % (rows, rows_all)
    else:
        out = "%d bitstrings" % len(inst.bitstrings)
    # simulation of the half-states is per path and not scaled; the row
    # fraction only scales the recombination, so this rate is an upper bound
    rate = done / t_sim * (rows / rows_all)
    return rate, f"{done} of {P.n_paths} paths ({out}); plan {t_plan:.3f}s excluded", threads, t_sim / done


def reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    inst = _instance(a.config)
    budget = max(5.0, min(60.0, 120.0 / max(1, a.steps + a.warmup)))
    vals = []
    for _ in range(a.warmup):
        cpu_oracle_rate(inst, budget_s=budget / 4)
    for _ in range(a.steps):
        r, sample, thr, _ = cpu_oracle_rate(inst, budget_s=budget)
        vals.append(r)
    v = statistics.median(vals)
    npaths = _ORACLE_PLANS[inst.name][0].n_paths
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "paths/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * npaths / v, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": a.config, "n_qubits": inst.n, "n_low": inst.n_low, "n_paths": npaths},
            "cpu_baseline": {"value": v, "unit": "paths/s", "cores": thr, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "paths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------- standard HSF (T/J)
def standard_hsf(inst, precision, t_joint_ms, prefix_rows, out, bits_d, budget_s=20.0):
    """Standard HSF (every crossing gate cut alone) on the same output,
    run through the same library in path chunks accumulated in place
    (hsf_run accumulate=1).  Timed with CUDA events once after a warm-up
    chunk; beyond `budget_s` the remaining chunks are extrapolated and the
    time reported as a lower bound (the paper reports a timeout bound)."""
    import torch
    from paper_2502_06959_b200 import Plan
    Pi = Plan(inst.text, inst.n_low, None, dtype=inst.dtype, individual=True, log2_path_budget=62)
    m = max(Pi.n_a, Pi.n_b)
    chunk = max(1, min(Pi.n_paths, (1 << 33) >> (m + 3)))  # <= 8 GiB of leaves per half per chunk
    rr = (0, prefix_rows) if prefix_rows else None
    n_chunks = -(-Pi.n_paths // chunk)
    Pi.run(out, bitstrings=bits_d, path_range=(0, min(chunk, Pi.n_paths)), row_range=rr, precision=precision)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    done, t0 = 0, time.perf_counter()
    e0.record()
    for c in range(n_chunks):
        p0, p1 = c * chunk, min(Pi.n_paths, (c + 1) * chunk)
        Pi.run(out, bitstrings=bits_d, path_range=(p0, p1), row_range=rr, precision=precision, accumulate=c > 0)
        done = p1
        if time.perf_counter() - t0 > budget_s:
            break
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    full_ms = ms * Pi.n_paths / done
    return {"n_paths_individual": Pi.n_paths, "ms": full_ms, "measured_paths": done,
            "lower_bound": done < Pi.n_paths, "T_over_J": full_ms / t_joint_ms,
            "note": "same library, every crossing gate its own cut unit; chunks of %d paths accumulated on "
                    "the device" % chunk}


# ----------------------------------------------------------------- our arm
def main():
    a = _args()
    if a.impl == "reference":
        return reference_arm(a)
    import torch
    import torch.distributed as dist

    from paper_2502_06959_b200 import Plan, build
    from paper_2502_06959_b200 import dist as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus and rank == 0:
        print(f"note: --gpus {a.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    inst = _instance(a.config)
    t_plan0 = time.perf_counter()
    P = Plan(inst.text, inst.n_low, inst.blocks, dtype=inst.dtype)
    t_plan = time.perf_counter() - t_plan0
    if world > 1:
        h = torch.tensor([P.plan_hash & 0x7FFFFFFFFFFFFFFF], dtype=torch.int64, device="cuda")
        hs = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        if any(int(x.item()) != int(h.item()) for x in hs):
            raise RuntimeError("plan hash mismatch across ranks")
    full = inst.bitstrings is None
    prefix = inst.meta.get("prefix")
    prefix_rows = -(-prefix // (1 << P.n_b)) if prefix else None
    if prefix:  # small output (first `prefix` amplitudes): split paths, all-reduce
        mode = "allreduce"
    else:
        mode = a.collective if a.collective != "auto" else D.default_mode(full, P.n_paths, P.n_a, P.n_b, world)
    sh = D.make_shard(mode, P.n_paths, P.n_a, rank, world, full)
    pr = sh.path_range
    cdt = torch.complex64 if inst.dtype == "c64" else torch.complex128
    esz = 8 if inst.dtype == "c64" else 16
    stream = torch.cuda.current_stream()
    if full:
        N_out = prefix if prefix else 1 << inst.n
        rows = (sh.row_range[1] - sh.row_range[0]) if sh.row_range else (prefix_rows or (1 << P.n_a))
        out = torch.empty(rows << P.n_b, dtype=cdt, device="cuda")
        shard = torch.empty(N_out // world, dtype=cdt, device="cuda") if mode == "reduce_scatter" and world > 1 \
            else None
        if mode == "fused_rs":  # no partial output: each rank's shard, mapped into every rank (CUDA IPC)
            out = D.PeerShards(torch.zeros(N_out // world, dtype=cdt, device="cuda"))
        bits_d = None
    else:
        N_out = len(inst.bitstrings)
        out = torch.empty(N_out, dtype=cdt, device="cuda")
        bits_d = torch.from_numpy(inst.bitstrings.view(np.int64)).cuda()
        shard = None
    phases = []

    def step(timed=False):
        def partial(path_range, row_range, o):
            if prefix:
                row_range = (0, prefix_rows)
            if isinstance(o, D.PeerShards):
                ph = P.run(None, path_range=path_range, precision=a.precision, timings=timed, out_shards=o.ptrs)
            else:
                ph = P.run(o, bitstrings=bits_d, path_range=path_range, row_range=row_range, precision=a.precision,
                           timings=timed)
            if timed:
                phases.append(ph)
        D.sharded_step(sh, partial, out, shard)

    # L2 flush buffer (> 126 MB L2) written between timed steps, outside the events
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(max(3, a.warmup)):
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        # steps are enqueued back to back (the run returns once its work is
        # enqueued); the events on the launching stream bracket exactly one
        # run each, the L2 flush between them stays outside
        for i in range(a.steps):
            flush.fill_(i & 0xFF)
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = [s_.elapsed_time(e_) for s_, e_ in evs]
    # per-phase split (CUDA events inside the library, one synchronising run each)
    for i in range(min(5, a.steps)):
        flush.fill_(i & 0xFF)
        step(timed=True)
    phase = [statistics.mean(p_[i] for p_ in phases) for i in range(5)]
    t_step = statistics.mean(ms)
    if world > 1:
        t = torch.tensor([t_step], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step = float(t.item())
    value = P.n_paths / (t_step * 1e-3)
    amps = N_out / (t_step * 1e-3)

    # the full-output GEMM's other precision modes, timed the same way beside
    # the default (bf16x6 and tf32x3 reported beside bf16x3)
    prec_alt = None
    if full and world == 1 and a.precision in ("auto", "bf16x3") and inst.dtype == "c64" and \
            not isinstance(out, D.PeerShards):
        prec_alt = {}
        rr_alt = (0, prefix_rows) if prefix else None
        for alt in ("bf16x6", "tf32x3"):
            try:
                for _ in range(2):
                    P.run(out, path_range=None, row_range=rr_alt, precision=alt)
                ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
                for i in range(5):
                    flush.fill_(i & 0xFF)
                    ev2[i][0].record(stream)
                    P.run(out, path_range=None, row_range=rr_alt, precision=alt)
                    ev2[i][1].record(stream)
                torch.cuda.synchronize()
                t_alt = statistics.mean(s_.elapsed_time(e_) for s_, e_ in ev2)
                prec_alt[alt] = {"ms_per_step": t_alt, "value": P.n_paths / (t_alt * 1e-3)}
            except Exception as ex:  # noqa: BLE001 - reported, not fatal
                prec_alt[alt] = {"error": str(ex)[:200]}
        P.run(out, path_range=None, row_range=rr_alt, precision=a.precision)  # restore the default's workspace
        torch.cuda.synchronize()

    # end-to-end through the public API with host buffers: plan (host SVD etc.)
    # + table upload + run + copy of the result to pinned host memory
    e2e = None
    try:
        import psutil
        host_avail = psutil.virtual_memory().available
    except Exception:
        host_avail = 0
    if rank == 0 and N_out * esz > host_avail // 4:
        e2e = {"value": None, "unit": "paths/s", "skipped": "output of %d bytes exceeds a quarter of the host's "
               "available memory (%d bytes) for a pinned host buffer" % (N_out * esz, host_avail)}
    elif rank == 0:
        host_out = torch.empty(max(N_out, (rows << P.n_b) if full else 0), dtype=cdt, pin_memory=True)
        host_bits = None if full else torch.from_numpy(inst.bitstrings.view(np.int64)).pin_memory()
        # e2e: the public call with HOST buffers on a plan built beforehand (the
        # plan is excluded here as in the reference arm and the paper's
        # "simulation only" line; plan_s / e2e.with_plan_ms report it): per step
        # the H2D of the bitstrings, the run and the D2H of the amplitudes
        P2 = Plan(inst.text, inst.n_low, inst.blocks, dtype=inst.dtype)
        rr2 = (0, prefix_rows) if prefix else None
        hout = host_out[:rows << P.n_b] if full else host_out

        def e2e_step():
            P2.run(hout, bitstrings=host_bits, precision=a.precision, row_range=rr2)

        e2e_step()  # device setup (tables, workspace, JIT module lookup)
        tt = []
        for i in range(max(3, min(a.steps, 10))):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step()  # returns after the D2H of the result completed
            tt.append(time.perf_counter() - t0)
        te = statistics.median(tt)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P3 = Plan(inst.text, inst.n_low, inst.blocks, dtype=inst.dtype)
        P3.run(hout, bitstrings=host_bits, precision=a.precision, row_range=rr2)
        t_with_plan = time.perf_counter() - t0
        del P2, P3
        h2d = 0 if full else int(inst.bitstrings.nbytes)
        e2e = {"value": P.n_paths / te, "unit": "paths/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int((rows << P.n_b) * esz if full else N_out * esz), "ms_per_step": te * 1e3,
               "includes": "hsf_run through the C ABI with pinned host buffers: bitstring H2D + run + result "
                           "D2H (plan built beforehand)",
               "with_plan_ms": t_with_plan * 1e3}

    # roofline of the dominant kernel (the path-sum for full output)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs", 6650.0)
    bf16 = peaks.get("bf16_tflops", 1590.0)
    K = pr[1] - pr[0]
    core_ms = phase[3]
    prec = a.precision
    eff_prec = ("bf16x3" if inst.dtype == "c64" else "simt") if prec == "auto" else prec
    MA, MB = (rows if full else 1 << (inst.n - inst.n_low)), 1 << inst.n_low
    clk_mhz = peaks.get("clocks_under_load", {}).get("sm_mhz_median", 1305.0)
    # swapped path-sum (run.cu make_layout: <= 128 output rows, bf16 modes,
    # K > 64, n_low >= 8): GEMM M = 2^n_low (half B's leaves, MN-major), one
    # narrow N tile of the rows, then a transpose -- the M operand streams once
    Kp = (K + 31) // 32 * 32
    swap = (full and eff_prec in ("bf16x3", "bf16x1", "bf16x6") and MA <= 128 and inst.n_low >= 8
            and 2 * Kp > 128 and inst.dtype == "c64" and os.environ.get("HSF_TC_SWAP", "") != "0")
    if swap:
        nprod, planes = {"bf16x6": (6, 3), "bf16x3": (3, 2), "bf16x1": (1, 1)}[eff_prec]
        Rp = (MA + 1) // 2 * 2
        bn = (2 * Rp + 31) // 32 * 32
        tflop = nprod * 2.0 * MB * bn * (2 * K)  # executed (narrow tile incl. padding)
        obytes = planes * 2.0 * (2 * K) * (MB + bn) + MB * 2 * Rp * 4 + MA * MB * esz * 2
        t_tensor, t_hbm = tflop / (bf16 * 1e12), obytes / (hbm * 1e9)
        ach = obytes / (core_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "kernel": "tc_gemm2_kernel narrow-N swapped path-sum (tcgen05 bf16, split x%d) + transpose" % nprod,
                "traffic": None, "flops_per_launch": tflop, "bytes_per_launch": obytes,
                "tensor_time_fraction": t_tensor / (core_ms * 1e-3),
                "useful_complex_flops": 8.0 * MA * MB * K, "kernel_ms": core_ms,
                "note": "algorithmic bytes = M operand planes (half B's leaves, 2K x 2^n_low bf16 each) read "
                        "once + the fp32 [2^n_low][2 rows] GEMM output written + the transposed output"}
    elif full and eff_prec in ("bf16x3", "bf16x1", "bf16x6", "tf32x3"):
        # executed tensor-core flops: (6 | 3 | 1) real GEMMs of rows x 2MB x 2K;
        # algorithmic bytes: the fp32 output written once (+ bf16 operand planes)
        nprod, planes = {"bf16x6": (6, 3), "bf16x3": (3, 2), "bf16x1": (1, 1), "tf32x3": (3, 4)}[eff_prec]
        tflop = nprod * 2.0 * MA * (2 * MB) * (2 * K)
        obytes = MA * MB * esz + planes * 4.0 * K * (MA + 2 * MB)
        # tf32 runs at half the bf16 rate (nominal 1125 vs 2250 TFLOP/s dense)
        tpeak, tnom = (bf16 / 2, 1125.0) if eff_prec == "tf32x3" else (bf16, 2250.0)
        t_tensor, t_hbm = tflop / (tpeak * 1e12), obytes / (hbm * 1e9)
        if t_tensor >= t_hbm:
            ach = tflop / (core_ms * 1e-3) / 1e12
            roof = {"bound": "tensor", "achieved": ach, "peak": tpeak, "unit": "TFLOP/s", "frac": ach / tpeak,
                    "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst: torch/cuBLAS bf16 8192^3, itself "
                                   "%.0f%% of the 2250 TFLOP/s nominal dense peak)%s; sustained %.1f" %
                                   (100.0 * bf16 / 2250.0, " x 1/2 for tf32" if tnom < 2000 else "",
                                    peaks.get("bf16_tflops_sustained", 0.0)),
                    "frac_of_nominal": ach / tnom}
        else:
            ach = obytes / (core_ms * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
        pair = MA > 128
        roof.update({"kernel": "%s (tcgen05 bf16, split x%d)" % ("tc_gemm2_kernel CTA pairs" if pair else
                                                                 "tc_gemm_kernel", nprod),
                     "traffic": NCU_TRAFFIC.get((a.config, "gemm")),
                     "traffic_source": "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum per launch "
                                       "(profiles/r01)" if (a.config, "gemm") in NCU_TRAFFIC else None,
                     "flops_per_launch": tflop, "bytes_per_launch": obytes,
                     "useful_complex_flops": 8.0 * MA * MB * K, "kernel_ms": core_ms})
    elif full:
        alu_peak = 148 * 128 * 2 * clk_mhz * 1e6 / 1e12
        useful = 8.0 * MA * MB * K
        ach = useful / (core_ms * 1e-3) / 1e12
        roof = {"bound": "alu", "kernel": "simt_gemm_kernel (complex FMA path-sum)", "achieved": ach,
                "peak": alu_peak, "unit": "TFLOP/s", "frac": ach / alu_peak, "traffic": None, "kernel_ms": core_ms,
                "peak_source": "148 SM x 128 FP32 lanes x 2 x median SM clock under load (MEASURED_PEAKS.json)"}
    else:
        nb = len(inst.bitstrings)
        # folded trailing diagonal units shrink the operand rows (tree paths)
        Kt = K // (int(np.prod(P.ranks[len(P.ranks) - P.fold_units:])) if P.fold_units else 1)
        byts = nb * 2 * Kt * esz
        ach = byts / (core_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": "gather_dot (bitstring path-sum)", "achieved": ach, "peak": hbm,
                "unit": "GB/s", "frac": ach / hbm, "traffic": None, "kernel_ms": core_ms,
                "note": "algorithmic bytes = 2 operand rows of %d tree paths per sample (upper bound; rows "
                        "shared by samples hit L2, so frac > 1 means L2-resident operands)" % Kt,
                "frac_of_l2_read": ach / L2_READ_GBS, "l2_read_peak_gbs": L2_READ_GBS}

    # the simulator tree (both halves concurrently): algorithmic bytes of its
    # tile passes over this rank's share of the paths / the sim phase
    used_fold = (not full) and P.fold_units > 0
    tb = list(P.fold_tree_bytes if used_fold else P.tree_bytes)
    # full-output tensor-core runs evaluate each half's head/tail-folded tree
    # when the planner made one (hsf.h fold_trailing_diag)
    tc_full = full and eff_prec != "simt"
    halves_var = [tc_full and P.tail_passes[h] > 0 for h in (0, 1)]
    for h in (0, 1):
        if halves_var[h]:
            tb[h] = P.tail_tree_bytes[h]
    sim_ms = max(phase[0], phase[1])
    sim_bytes = (tb[0] + tb[1]) * (K / P.n_paths)
    cone = full and MA < (1 << (inst.n - inst.n_low))
    if cone:
        # row-range run: half A computes only the rows' light cone (run.cu
        # run_half), its bytes are not modelled -- count half B's tree alone
        # over B's phase (a lower bound on the simulator's traffic)
        sim_ms = phase[1]
        sim_bytes = tb[1] * (K / P.n_paths)
    sim_ach = sim_bytes / (sim_ms * 1e-3) / 1e9
    roof_sim = {"bound": "hbm", "kernel": "simulator tile passes (hsf_jit_pass, %s)" %
                ("half B; half A's light cone uncounted" if cone else "both halves"), "achieved": sim_ach,
                "peak": hbm, "unit": "GB/s", "frac": sim_ach / hbm, "traffic": None, "kernel_ms": sim_ms,
                "bytes": sim_bytes, "frac_of_l2_read": sim_ach / L2_READ_GBS, "l2_read_peak_gbs": L2_READ_GBS,
                "note": "algorithmic bytes = every pass reads + writes each output node state once; small "
                        "states stay L2/SMEM-resident, so frac can exceed 1"}
    if sim_ms > core_ms:
        roof, roof_other = roof_sim, roof
    else:
        roof_other = roof_sim

    std = None
    if a.standard and rank == 0 and world == 1:
        std = standard_hsf(inst, a.precision, t_step, prefix_rows, out, bits_d)

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        r, sample, thr, _ = cpu_oracle_rate(inst, budget_s=15.0)
        cpu = {"value": r, "unit": "paths/s", "cores": thr, "kind": "oracle", "sample": sample}

    # our kernels per step: simulator passes of both halves, then the path-sum:
    # full output = split_a + split_b + GEMM (SIMT: 1 kernel); bitstrings =
    # 2 transposes + gather (folded tree when the trailing units fold)
    # (full tensor-core runs: half B's last pass writes the GEMM operand itself
    # when B has no folded tree and K > 64, see hsf.h / run.cu)
    if used_fold:
        sim_launches = sum(P.fold_passes)
    else:
        sim_launches = sum(P.tail_passes[h] if halves_var[h] else P.passes[h] for h in (0, 1))
    fused_b = tc_full and not halves_var[1] and K > 64
    n_launch = sim_launches + (1 if (full and eff_prec == "simt") else (2 if fused_b else 3))
    if swap:  # split of A's rows (N operand) + GEMM + transpose (+ split of B's leaves unless fused)
        n_launch = sim_launches + (3 if (not halves_var[1] and eff_prec != "bf16x6") else 4)
    if not full:  # grouped gather (run.cu make_layout): + count, scan, scatter kernels
        Kt = K // (int(np.prod(P.ranks[len(P.ranks) - P.fold_units:])) if P.fold_units else 1)
        if inst.dtype == "c64" and Kt % 64 == 0 and Kt <= 512 and N_out >= 4 * (1 << P.n_a):
            n_launch += 3
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "paths/s", "n_gpus": world, "steps": a.steps,
                "warmup": max(3, a.warmup), "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": inst.dtype, "data": "synthetic",
                "config": {"workload": a.config, "n_qubits": inst.n, "n_low": inst.n_low,
                           "n_paths_joint": P.n_paths, "log2_n_paths_individual": P.log2_n_paths_individual,
                           "outputs": N_out, "precision": prec, "parallelism": f"{mode}{world}",
                           "l2": "flushed (256 MiB write) between timed steps"},
                "amplitudes_per_s": amps, "terms_per_s": amps * P.n_paths,
                "phase_ms": {"sim_A": phase[0], "sim_B": phase[1], "prep": phase[2], "core": phase[3],
                             "run_total": phase[4]},
                "plan_s": t_plan, "roofline": roof, "roofline_other": roof_other, "cpu_baseline": cpu,
                "e2e": e2e, "joint_blocks": P.n_joint_blocks, "separate_cuts": P.n_units - P.n_joint_blocks,
                "folded_units": P.fold_units if not full else 0, "standard_hsf": std,
                "gpu_launches": n_launch, "clocks": clk.summary(),
                "precision_modes": prec_alt}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()  # rank 0 ran the e2e / CPU legs alone; leave together
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
