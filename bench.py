#!/usr/bin/env python
"""Benchmark of the HSF path-evaluation hot path (BASELINE.json metric:
"HSF paths/s and output amplitudes/s at 1/2/4/8 B200; % of HBM/tensor roofline").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl reference]

One step = one hsf_run over this rank's path range: path-tree simulation of
both halves, coefficient fold, path-sum (+ for N > 1 the mode's collective).
Default workload: c5 (n=40, cut 20|20, 256 joint-cut paths, 2^22 seeded
bitstrings, complex64) -- the largest BASELINE.json configuration that fits
one GPU (c4's 2^34-amplitude output is the 8-GPU row-sharded config).  The
other configs are parity-test cases and `--config` lines.  Prints ONE JSON
line on rank 0.
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
DEFAULT_CONFIG = "c5"
# random 1 KiB-row read rate on the box (scripts/probe/rowgather.cu, 2^22 rows
# of a 2 GiB buffer, one warp per row): the bitstring gather's access pattern;
# context beside the copy peak of MEASURED_PEAKS.json
ROW_READ_GBS = 7267.0
# L2-resident read rate (scripts/probe/l2bw.cu: 16 B __ldcg over 64 MiB)
L2_READ_GBS = 19710.0


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--precision", default="auto")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--standard", action="store_true",
                    help="also time standard HSF (every crossing gate cut alone) on the same output: T/J")
    ap.add_argument("--collective", default="auto",
                    choices=["auto", "reduce_scatter", "allreduce", "rows", "fused_rs", "fused_bits", "nvls_bits"],
                    help="N>1 exchange (paper_2502_06959_b200/dist.py); auto = cheapest for the output mode")
    return ap.parse_args()


def _instance(name):
    from hsf_inputs import make_config
    return make_config(name)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region (NVML every
    2 ms; nvidia-smi if NVML is unavailable)."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self.source = "nvml"

    def _nvml_loop(self):
        import pynvml as N
        N.nvmlInit()
        try:
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            bits = [getattr(N, "nvmlClocksEventReasonHwSlowdown", 0x8),
                    getattr(N, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                    getattr(N, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                    getattr(N, "nvmlClocksEventReasonSwPowerCap", 0x4)]
            get = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self._stop.is_set():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                rs = get(h)
                self.rows.append((float(sm), float(mx), [bool(rs & b) for b in bits]))
                self._stop.wait(0.002)
        finally:
            N.nvmlShutdown()

    def _smi_loop(self):
        self.source = "nvidia-smi"
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                r = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                    "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                v = [x.strip() for x in r.stdout.strip().split(",")]
                if r.returncode == 0 and len(v) == 6:
                    self.rows.append((float(v[0]), float(v[1]), [x == "Active" for x in v[2:]]))
            except Exception:
                pass
            self._stop.wait(0.2)

    def _loop(self):
        try:
            self._nvml_loop()
        except Exception:
            self._smi_loop()

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, f in self.rows for i in range(4) if f[i]})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "source": self.source}


# ------------------------------------------------ the oracle on host cores
_ORACLE_PLANS = {}


def cpu_oracle_step(inst, paths: int | None = None, procs: int | None = None):
    """One bounded sample of the workload through the CPU oracle as it stands
    (oracle/hsf_oracle.py, complex128 NumPy), its path evaluations spread over
    all host cores by oracle/parallel.py (forked workers, one path chunk each;
    SURVEY.md §8(d)): the first `paths` paths (default 1 per core), both
    half-circuits from scratch per path, and their Kronecker path-sum over the
    workload's whole output (bitstrings / all rows; beyond 2^24 amplitudes a
    row subset, the rate scaled by the row fraction).  The plan is built once
    and excluded, as in the paper's "simulation only" line.
    Returns (paths/s, seconds, description, processes)."""
    from oracle import hsf_oracle as O
    from oracle import parallel as OP
    procs = procs or OP.n_procs()
    if inst.name not in _ORACLE_PLANS:
        n, g = O.parse_circuit(inst.text)
        blocks = O.find_cascades(g, inst.n_low)[0] if inst.blocks == "auto" else inst.blocks
        t0 = time.perf_counter()
        _ORACLE_PLANS[inst.name] = (O.plan(n, g, inst.n_low, blocks), time.perf_counter() - t0)
    P, t_plan = _ORACLE_PLANS[inst.name]
    n = inst.n
    k = min(P.n_paths, paths or procs)
    t0 = time.perf_counter()
    if inst.bitstrings is not None:
        OP.bits_amplitudes(P, inst.bitstrings, inst.n_low, 0, k, procs=procs)
        out = "%d bitstrings" % len(inst.bitstrings)
        scale = 1.0
    else:
        rows_all = 1 << (n - inst.n_low)
        if inst.meta.get("prefix"):
            rows_all = -(-inst.meta["prefix"] // (1 << inst.n_low))
        rows = max(1, min(rows_all, (1 << 24) >> inst.n_low))
        A, B, c = OP.half_state_rows(P, np.arange(rows), np.arange(1 << inst.n_low), 0, k, procs=procs)
        O.recombine_full(A, B, c)
        scale = rows / rows_all
        out = ("all %d output rows" % rows_all) if rows == rows_all else \
            "%d of %d output rows (rate scaled by the row fraction)" % (rows, rows_all)
    dt = time.perf_counter() - t0
    desc = "first %d of %d paths over %s, %d worker processes; plan %.3f s excluded" % (k, P.n_paths, out, procs,
                                                                                         t_plan)
    return k / dt * scale, dt, desc, procs


def reference_arm(a):
    """--impl reference: the oracle timed as it stands on the host cores (rank
    0 only; other ranks exit).  Each step is one bounded sample of the same
    workload (cpu_oracle_step); ms_per_step is that sample's measured time."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    inst = _instance(a.config)
    for _ in range(a.warmup):
        cpu_oracle_step(inst, paths=max(1, os.cpu_count() or 1))
    vals, secs = [], []
    desc, procs = "", 1
    for _ in range(a.steps):
        v, dt, desc, procs = cpu_oracle_step(inst)
        vals.append(v)
        secs.append(dt)
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "paths/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * statistics.mean(secs),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic",
            "config": {"workload": a.config, "n_qubits": inst.n, "n_low": inst.n_low,
                       "n_paths_joint": _ORACLE_PLANS[inst.name][0].n_paths,
                       "step": "one bounded sample: " + desc},
            "cpu_baseline": {"value": v, "unit": "paths/s", "cores": procs, "kind": "oracle", "sample": desc},
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


# --------------------------------------------------------------- rooflines
def _peaks():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        mp = {}
    # fallback: /opt/skills/guides/B200_PROFILING.md copy bandwidth / cuBLAS bf16
    hbm = mp.get("hbm_gbs", 6550.0)
    bf16 = mp.get("bf16_tflops", 1618.6)
    mhz = mp.get("sm_max_mhz", 1965.0)
    # FP32 (FFMA) and FP64 ALU peaks from unit counts x clock: 148 SMs x 128
    # FP32 lanes x 2 flops; FP64 at 1/2 the FP32 lane rate (B200 vector FP64)
    fp32 = 148 * 128 * 2 * mhz * 1e6 / 1e12
    return {"hbm": hbm, "bf16": bf16, "bf16_sustained": mp.get("bf16_tflops_sustained"), "fp32": fp32,
            "fp64": fp32 / 2, "mhz": mhz, "source": "MEASURED_PEAKS.json" if mp else "B200_PROFILING.md fallback"}


def _traffic(config, kernel):
    """dram bytes read + written per launch of `kernel` from the committed ncu
    capture of this config (profiles/traffic.json, scripts/traffic_table.py)."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        e = t[config][kernel]
        return e["dram_bytes_per_launch"], e["source"]
    except Exception:
        return None, None


def rooflines(cfg, desc, phase, pk, dtype, cone):
    """The path-sum kernel's and the simulator window's rooflines from the
    run's algorithmic work (hsf_run_describe) over CUDA-event times."""
    core_ms = phase[3]
    core = desc["core"]
    if core in ("tc_pair", "tc_single", "tc_swapped"):
        tpeak = pk["bf16"] / 2 if desc["tc_products"] == 3 and cfg.get("precision") == "tf32x3" else pk["bf16"]
        ex, useful, byts = desc["core_flops_executed"], desc["core_flops_useful"], desc["core_bytes"]
        t_tensor, t_hbm = ex / (tpeak * 1e12), byts / (pk["hbm"] * 1e9)
        kname = "tc_gemm2_kernel" if core == "tc_pair" else "tc_gemm_kernel"
        if t_tensor >= t_hbm:
            ach = ex / (core_ms * 1e-3) / 1e12
            r = {"bound": "tensor", "achieved": ach, "peak": tpeak, "unit": "TFLOP/s", "frac": ach / tpeak,
                 "frac_useful": useful / (core_ms * 1e-3) / 1e12 / tpeak,
                 "peak_source": pk["source"] + " bf16_tflops (burst, cuBLAS bf16 8192^3)"}
        else:
            ach = byts / (core_ms * 1e-3) / 1e9
            r = {"bound": "hbm", "achieved": ach, "peak": pk["hbm"], "unit": "GB/s", "frac": ach / pk["hbm"],
                 "frac_useful_tensor": useful / (core_ms * 1e-3) / 1e12 / tpeak,
                 "peak_source": pk["source"] + " hbm_gbs (copy)"}
        r.update({"kernel": kname + (" (swapped narrow-N) + transpose" if core == "tc_swapped" else ""),
                  "flops_executed_per_launch": ex, "flops_useful_per_launch": useful, "bytes_per_launch": byts,
                  "kernel_ms": core_ms,
                  "note": "executed = split-bf16 products actually issued (x%d); useful = 8 K flops per output "
                          "amplitude (the method's complex multiply-adds)" % desc["tc_products"]})
    elif core == "simt":
        alu = pk["fp32"] if dtype == "c64" else pk["fp64"]
        ach = desc["core_flops_useful"] / (core_ms * 1e-3) / 1e12
        r = {"bound": "alu", "kernel": "simt_gemm_kernel", "achieved": ach, "peak": alu, "unit": "TFLOP/s",
             "frac": ach / alu, "kernel_ms": core_ms, "flops_per_launch": desc["core_flops_useful"],
             "peak_source": "148 SM x 128 FP32 lanes x 2 x %.0f MHz%s" % (pk["mhz"], " / 2 (FP64)" if
                                                                              dtype != "c64" else "")}
        kname = "simt_gemm_kernel"
    else:
        byts = desc["core_bytes"]
        ach = byts / (core_ms * 1e-3) / 1e9
        kname = "gather_block_c64_kernel" if core == "block_gather" else "gather_dot_c64_vec_kernel"
        r = {"bound": "hbm", "kernel": kname, "achieved": ach, "peak": pk["hbm"], "unit": "GB/s",
             "frac": ach / pk["hbm"], "kernel_ms": core_ms, "bytes_per_launch": byts,
             "frac_of_row_read_probe": ach / ROW_READ_GBS, "row_read_probe_gbs": ROW_READ_GBS,
             "frac_of_l2_read": ach / L2_READ_GBS,
             "peak_source": pk["source"] + " hbm_gbs (copy)",
             "note": ("block gather: the direct half's leaves read once + one padded row of the other half, "
                      "sample index, bitstring and result per sample" if core == "block_gather" else
                      "per-sample gather: two K-rows, bitstring and result per sample")}
    tr, src = _traffic(cfg["workload"], kname)
    r["traffic"] = tr
    r["traffic_source"] = src
    if r["bound"] == "hbm" and tr is not None and tr < 0.5 * r["bytes_per_launch"]:
        # the committed capture shows the operands L2-resident (DRAM traffic
        # under half the algorithmic bytes, e.g. c3's 2 x 64 MiB leaves): the
        # bound is the L2 read rate, not HBM
        r.update({"bound": "l2", "peak": L2_READ_GBS, "frac": r["achieved"] / L2_READ_GBS, "frac_of_hbm_copy":
                  r["achieved"] / pk["hbm"], "peak_source": "scripts/probe/l2bw.cu (16 B __ldcg over 64 MiB, L2-resident "
                  "read rate); operands L2-resident per profiles/traffic.json"})
    # simulator window: both trees (concurrent streams) + the operand prep after them
    if cone:  # prefix outputs: half A computes only the rows' light cone (uncounted); half B alone
        t_w = phase[1]
        sb, sf = desc["sim_bytes"][1], desc["sim_flops"][1]
        what = "half B's tree (half A's light cone uncounted)"
    else:
        t_w = max(phase[0], phase[1]) + phase[2]
        sb = desc["sim_bytes"][0] + desc["sim_bytes"][1] + desc["prep_bytes"]
        sf = desc["sim_flops"][0] + desc["sim_flops"][1]
        what = "both trees + operand prep (transposes / split planes)"
    alu = pk["fp32"] if dtype == "c64" else pk["fp64"]
    t_hbm, t_alu = sb / (pk["hbm"] * 1e9), sf / (alu * 1e12)
    s = {"kernel": "simulator passes (hsf_jit_pass) + prep: " + what, "window_ms": t_w, "bytes": sb, "flops": sf,
         "hbm_gbs": sb / (t_w * 1e-3) / 1e9, "alu_tflops": sf / (t_w * 1e-3) / 1e12,
         "bound": "hbm" if t_hbm >= t_alu else "alu",
         "frac": max(t_hbm, t_alu) / (t_w * 1e-3), "frac_hbm": t_hbm / (t_w * 1e-3), "frac_alu": t_alu / (t_w * 1e-3),
         "peak_hbm_gbs": pk["hbm"], "peak_alu_tflops": alu,
         "note": "bytes: every pass reads and writes each node state once; flops: dense k-qubit op 8*2^k, "
                 "1-qubit gate 16, diagonal 6 per amplitude (FMA = 2); frac = max(bytes/HBM, flops/ALU) / window"}
    s["achieved"], s["peak"], s["unit"] = ((s["hbm_gbs"], pk["hbm"], "GB/s") if s["bound"] == "hbm" else
                                           (s["alu_tflops"], alu, "TFLOP/s"))
    s["traffic"] = None
    # `roofline` is the path-sum kernel (one launch, CUDA events around it);
    # the simulator window (many pass kernels + prep, concurrent streams) is
    # reported beside it
    return r, s


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
        D.check_plan_hash(P.plan_hash)
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
    bits_d = None
    if full:
        N_out = prefix if prefix else 1 << inst.n
        rows = (sh.row_range[1] - sh.row_range[0]) if sh.row_range else (prefix_rows or (1 << P.n_a))
        out = torch.empty(rows << P.n_b, dtype=cdt, device="cuda")
        shard = torch.empty(N_out // world, dtype=cdt, device="cuda") if mode == "reduce_scatter" and world > 1 \
            else None
        if mode == "fused_rs":  # no partial output: each rank's shard, mapped into every rank (CUDA IPC)
            out = D.PeerShards(torch.zeros(N_out // world, dtype=cdt, device="cuda"))
    else:
        N_out = len(inst.bitstrings)
        rows = 0
        out = torch.empty(N_out, dtype=cdt, device="cuda")
        bits_d = torch.from_numpy(inst.bitstrings.view(np.int64)).cuda()
        shard = None
        if mode == "fused_bits":
            out = D.PeerShards(torch.zeros(D.bits_shard_len(N_out, world), dtype=cdt, device="cuda"))
        if mode == "nvls_bits":  # every rank's copy of the multicast buffer receives the sum
            out = D.MulticastBuffer(N_out)
    rr_run = (0, prefix_rows) if prefix else sh.row_range
    phases = []
    # N > 1: the exchange step runs inside the library (its own NCCL
    # communicator, hsf_run_args.coll), captured in the run's graph
    lcomm = D.library_comm() if world > 1 else None

    def step(timed=False):
        D.run_sharded(P, out, sh, shard_out=shard, bitstrings=bits_d, precision=a.precision, row_range=rr_run,
                      comm=lcomm, phases=phases if timed else None)

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
        # steps enqueued back to back (a device-output run returns once its work
        # is enqueued); each step's events bracket exactly that step, the L2
        # flush between them stays outside
        for i in range(a.steps):
            flush.fill_(i & 0xFF)
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = [s_.elapsed_time(e_) for s_, e_ in evs]
    desc = P.describe(0 if full else N_out, path_range=pr, row_range=rr_run, precision=a.precision)
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
        for alt in ("bf16x6", "tf32x3"):
            try:
                for _ in range(2):
                    P.run(out, row_range=rr_run, precision=alt)
                ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
                for i in range(5):
                    flush.fill_(i & 0xFF)
                    ev2[i][0].record(stream)
                    P.run(out, row_range=rr_run, precision=alt)
                    ev2[i][1].record(stream)
                torch.cuda.synchronize()
                t_alt = statistics.mean(s_.elapsed_time(e_) for s_, e_ in ev2)
                prec_alt[alt] = {"ms_per_step": t_alt, "value": P.n_paths / (t_alt * 1e-3)}
            except Exception as ex:  # noqa: BLE001 - reported, not fatal
                prec_alt[alt] = {"error": str(ex)[:200]}
        P.run(out, row_range=rr_run, precision=a.precision)  # restore the default's graph
        torch.cuda.synchronize()

    e2e = end_to_end(a, inst, P, D, sh, mode, world, rank, full, prefix_rows, rows, N_out, cdt, esz)

    pk = _peaks()
    cfg = {"workload": a.config, "precision": a.precision}
    cone = full and prefix_rows is not None
    roof, roof_sim = rooflines(cfg, desc, phase, pk, inst.dtype, cone)

    std = None
    if a.standard and rank == 0 and world == 1:
        std = standard_hsf(inst, a.precision, t_step, prefix_rows, out, bits_d)

    cpu = None
    if rank == 0 and not a.no_cpu_baseline:
        r, dt, sample, procs = cpu_oracle_step(inst)
        cpu = {"value": r, "unit": "paths/s", "cores": procs, "kind": "oracle", "sample": sample,
               "seconds": dt}
    if world > 1:
        dist.barrier()  # rank 0's CPU leg runs alone

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "paths/s", "n_gpus": world, "steps": a.steps,
                "warmup": max(3, a.warmup), "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": inst.dtype, "data": "synthetic",
                "config": {"workload": a.config, "n_qubits": inst.n, "n_low": inst.n_low,
                           "n_paths_joint": P.n_paths, "log2_n_paths_individual": P.log2_n_paths_individual,
                           "outputs": N_out, "precision": a.precision, "parallelism": f"{mode}{world}",
                           "path_sum": desc["core"], "l2": "flushed (256 MiB write) between timed steps"},
                "amplitudes_per_s": amps, "terms_per_s": amps * P.n_paths,
                "phase_ms": {"sim_A": phase[0], "sim_B": phase[1], "prep": phase[2], "core": phase[3],
                             "run_total": phase[4]},
                "plan_s": t_plan, "roofline": roof, "roofline_sim": roof_sim, "cpu_baseline": cpu,
                "e2e": e2e, "joint_blocks": P.n_joint_blocks, "separate_cuts": P.n_units - P.n_joint_blocks,
                "folded_units": P.fold_units if not full else 0, "standard_hsf": std,
                "gpu_launches": desc["kernel_launches"] if desc["kernel_launches"] >= 0 else None,
                "gpu_launches_source": "kernel nodes of the run's captured CUDA graph (hsf_run_describe)",
                "clocks": clk.summary(), "precision_modes": prec_alt,
                "paper_context": {"note": "the paper's CPU joint-HSF rate on its own QAOA instances, 1x Threadripper "
                                          "PRO 5955WX (16 cores), P:218, Table I P:254-276: 1.9e3-3.3e3 paths/s; "
                                          "S/J up to ~237, T/J up to ~4247 (BASELINE.md); other workload and "
                                          "machine, context only"}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def end_to_end(a, inst, P, D, sh, mode, world, rank, full, prefix_rows, rows, N_out, cdt, esz):
    """The same metric through the public API with HOST buffers: per step the
    host->device copy of the step's inputs (bitstrings) from pinned memory,
    every rank's own path range, the collective, and the device->host copy of
    the result (each rank its shard / rank 0 the reduced vector).  Wall time,
    max over ranks.  At N = 1 this is one hsf_run call with host pointers (the
    library stages the copies itself)."""
    import torch
    import torch.distributed as dist
    try:
        import psutil
        host_avail = psutil.virtual_memory().available
    except Exception:
        host_avail = 1 << 40
    out_rows = (sh.out_rows[1] - sh.out_rows[0]) if (full and sh.out_rows) else (prefix_rows or (1 << P.n_a))
    res_elems = (out_rows << P.n_b) if full else N_out
    skip = res_elems * esz > host_avail // 4
    if world > 1:
        s = torch.tensor([int(skip)], device="cuda")
        dist.all_reduce(s, op=dist.ReduceOp.MAX)
        skip = bool(s.item())
    if skip:
        return {"value": None, "unit": "paths/s", "skipped": "result of %d bytes exceeds a quarter of the host's "
                "available memory for a pinned host buffer" % (res_elems * esz)}
    P2 = type(P)(inst.text, inst.n_low, inst.blocks, dtype=inst.dtype)
    rr2 = (0, prefix_rows) if prefix_rows else None
    host_bits = None if full else torch.from_numpy(inst.bitstrings.view(np.int64)).pin_memory()
    h2d = 0 if full else int(inst.bitstrings.nbytes)
    if world == 1:
        hout = torch.empty(res_elems, dtype=cdt, pin_memory=True)

        def e2e_step():
            P2.run(hout, bitstrings=host_bits, precision=a.precision, row_range=rr2)
        d2h = res_elems * esz
        how = "hsf_run through the C ABI with pinned host buffers: bitstring H2D + run + result D2H"
    else:
        bits_dev = None if full else torch.empty(N_out, dtype=torch.int64, device="cuda")
        dev_out = torch.empty((rows << P.n_b) if full else N_out, dtype=cdt, device="cuda")
        shard = torch.empty(N_out // world, dtype=cdt, device="cuda") if mode == "reduce_scatter" else None
        res_dev = shard if shard is not None else dev_out
        hout = torch.empty(res_dev.numel(), dtype=cdt, pin_memory=True)
        d2h = res_dev.numel() * esz
        if mode in ("fused_rs", "fused_bits", "nvls_bits"):
            return {"value": None, "unit": "paths/s", "skipped": "fused modes are measured by the device-timed "
                    "value only"}

        lcomm = D.library_comm()

        def e2e_step():
            if bits_dev is not None:
                bits_dev.copy_(host_bits, non_blocking=True)
            D.run_sharded(P2, dev_out, sh, shard_out=shard, bitstrings=bits_dev, precision=a.precision,
                          row_range=rr2, comm=lcomm)
            hout.copy_(res_dev, non_blocking=True)
            torch.cuda.synchronize()
        how = ("per rank: pinned H2D of the bitstrings, this rank's hsf_run (C ABI), the %s collective, D2H of "
               "the rank's result; wall time, max over ranks" % mode)
    e2e_step()  # device setup (tables, workspace, JIT module lookup, graph)
    tt = []
    for _ in range(max(3, min(a.steps, 10))):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_step()
        tt.append(time.perf_counter() - t0)
    te = statistics.median(tt)
    if world > 1:
        t = torch.tensor([te], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        te = float(t.item())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P3 = type(P)(inst.text, inst.n_low, inst.blocks, dtype=inst.dtype)
    t_plan = time.perf_counter() - t0
    del P2, P3
    return {"value": P.n_paths / te, "unit": "paths/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(d2h),
            "ms_per_step": te * 1e3, "includes": how + " (plan built beforehand; plan_ms beside it)",
            "plan_ms": t_plan * 1e3}


if __name__ == "__main__":
    sys.exit(main())
