#!/usr/bin/env python
"""SpAMM hot-path benchmark.  BASELINE.json metric: "SpAMM time & effective TFLOP/s vs tau at
1/2/4/8 B200; speedup vs cuBLAS GEMM", quoted on configs[4]:

  N = 65536 exponential-decay matrices a_ij = 0.999^|i-j|, A = B (C = A*A, the
  paper's a_ij = b_ij workloads), tile 32, headline tau = 1e-6, BF16 tcgen05 path (FP32 C),
  work-balanced row-block sharding at N GPUs (Sec. 3.4).

One STEP = one whole SpAMM through the C ABI: tile norms of A and B -> skip map -> masked
multiply into C (spamm_run; spamm_multiply_mgpu on N > 1 GPUs, C rows sharded by work).
Inputs are resident in HBM (8.6 GB, larger than the 126 MB L2, so no flush is needed between
steps; smaller sweep sizes flush L2 before every timed step).

  python bench.py [--gpus N --steps K --warmup W]       # our CUDA path (spawns N ranks itself
                                                         # when not started by torchrun)
  python bench.py --impl reference [...]                 # the float64 CPU oracle arm

The JSON line also carries: per-stage times, kept (non-skipped) TFLOP/s, the roofline of the
dominant kernel, a tau sweep at N = 65536 / 16384 (north_star's single-GPU target) / 8192 with
cuBLAS on the same box, an end-to-end number through the public API with host buffers, the
CPU-oracle baseline, clocks during the timed region and the count of our kernel launches.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

N_DEFAULT = 65536
LAM_DEFAULT = 0.999
TAU_HEADLINE = 1e-6
TAU5 = [1e-10, 1e-8, 1e-6, 1e-4, 1e-2]
TAU9 = [1e-10, 1e-9, 1e-8, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2]
TILE = 32
L2_BYTES = 126 * 1024 * 1024
METRIC = "SpAMM effective TFLOP/s (dense-equivalent 2N^3/t), configs[4]"
DT = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32, "fp32x3": torch.float32}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    out = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0,
           "source": "fallback (B200_PROFILING.md)"}
    if os.path.exists(p):
        d = json.load(open(p))
        out = {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
               "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
               "sm_max_mhz": d.get("sm_max_mhz", 1965.0), "source": "measured (MEASURED_PEAKS.json)"}
    # FP32 CUDA-core FFMA peak: measured by scripts/probe_ffma.cu on this pool's B200s
    f = os.path.join(ROOT, "profiles", "ffma_peak.json")
    if os.path.exists(f):
        d = json.load(open(f))
        out["fp32_tflops"] = d["tflops"]
        out["fp32_source"] = f"measured FFMA peak ({d.get('how', 'scripts/probe_ffma.cu')})"
    else:
        out["fp32_tflops"] = 148 * 128 * 2 * out["sm_max_mhz"] * 1e6 / 1e12
        out["fp32_source"] = "theoretical 148 SM x 128 FFMA x 2 x sm_max clock"
    return out


# ------------------------------------------------------------------ clocks ---
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.15)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "samples": len(sm),
                "reasons": sorted(reasons)}


# ------------------------------------------------------------- CPU oracle ---
def _cpu_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        threads = int(max(n)) if n else os.cpu_count()
    except Exception:
        threads = os.cpu_count()
    return threads, model


def _table(N, lam, prec):
    t = synth.decay_table("exp", N, lam).astype(np.float32)
    if prec == "bf16":
        t = synth.round_to_bf16(t)
    elif prec == "fp16":
        t = synth.round_to_fp16(t)
    return t


def _table_alg(N, prec):
    """The paper's algebraic-decay dataset a_ij = 0.1/(|i-j|^0.1 + 1) (configs[2])."""
    t = synth.decay_table("alg", N, 0.1, c=0.1).astype(np.float32)
    if prec == "bf16":
        t = synth.round_to_bf16(t)
    elif prec == "fp16":
        t = synth.round_to_fp16(t)
    return t


def _table1_taus(N):
    """(target valid ratio, tau) printed in Table 1 for this N, from the golden file."""
    path = os.path.join(ROOT, "tests", "golden", "table1_tau.csv")
    out = []
    with open(path) as f:
        for line in f:
            if line.startswith("#") or line.startswith("N,"):
                continue
            n, target, tau = line.strip().split(",")
            if int(n) == N:
                out.append((float(target), float(tau)))
    return out


def oracle_sample(N, lam, prec, tau, rows=8, cols=96, seed=0):
    """The float64 oracle (as it stands) on a bounded sample of the workload: the C tiles of
    `rows` middle tile rows x `cols` random tile columns, i.e. oracle.spamm(A[rows, :], B[:, cols])
    -- norms of exactly those operand strips (all of K) and every kept product of those C tiles,
    the same arithmetic those tiles get in the full problem.  Returns (seconds, dense-equivalent
    flops of the sample, description)."""
    import oracle
    table = _table(N, lam, prec)
    BD = N // TILE
    r0 = (BD - rows) // 2
    js = np.sort(np.random.default_rng(seed).choice(BD, size=cols, replace=False))
    As = synth.toeplitz_block(table, r0 * TILE, (r0 + rows) * TILE, 0, N)
    Bs = np.concatenate([synth.toeplitz_block(table, 0, N, j * TILE, (j + 1) * TILE) for j in js], axis=1)
    t0 = time.perf_counter()
    C = oracle.spamm(As, Bs, tau, TILE)
    dt = time.perf_counter() - t0
    assert C.shape == (rows * TILE, cols * TILE)
    desc = (f"{rows} middle tile rows x {cols} random tile columns of C ({rows * TILE} x {cols * TILE} of {N} x {N}), "
            f"full K: float64 numpy oracle.spamm incl. the operand strips' norm maps")
    return dt, 2.0 * rows * TILE * cols * TILE * N, desc


def run_reference(args, rank, world):
    """--impl reference: the oracle arm on rank 0 (other ranks exit without work)."""
    if rank != 0:
        return
    for w in range(args.warmup):
        oracle_sample(args.n, args.lam, args.precision, args.tau, seed=100 + w)
    times, flops, desc = [], 0.0, ""
    for s in range(args.steps):
        dt, flops, desc = oracle_sample(args.n, args.lam, args.precision, args.tau, seed=s)
        times.append(dt)
    ms = 1e3 * statistics.mean(times)
    value = flops / (ms / 1e3) / 1e12
    threads, model = _cpu_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(args, world),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "cpu": model, "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config(args, world):
    N = args.n
    big = N * N * (2 if args.precision in ("bf16", "fp16") else 4) > L2_BYTES
    return {"workload": f"configs[4]: N={N} exponential decay a_ij={args.lam}^|i-j| (A=B), tile 32, "
                        f"tau={args.tau:g}, {args.precision.upper()} path", "N": N, "tile": TILE,
            "lambda": args.lam, "tau": args.tau, "precision": args.precision,
            "parallelism": f"C row blocks balanced by skip-map work x{world}" if world > 1 else "single GPU",
            "l2": ("inputs larger than L2 (no flush)" if big else
                   "flushed before every timed step (512 MB write, then 512 MB read of another buffer)")}


# --------------------------------------------------------------- GPU path ---
def _flusher(dev):
    buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    rd = torch.zeros(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    out = torch.empty((), dtype=torch.float32, device=dev)

    def flush():
        buf.zero_()
        torch.sum(rd, dim=0, out=out)
    return flush


def _timed(fn, steps, warmup, flush, stream):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        if flush is not None:
            flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    return ms


def _roofline(st, prec, ms_mul, ms_norms, N, peaks, es, traffic):
    """Roofline of the multiply: its floor is max(kept tensor FLOPs / tensor peak, compulsory
    bytes / HBM peak) with the compulsory bytes = C written once + A read once (A = B)."""
    kept_flops = 2.0 * TILE ** 3 * st["kept"]
    mma_flops = kept_flops * (6 if prec == "fp32x3" else 1)   # fp32x3: six BF16 products per kept pair
    c_bytes = 4.0 * N * N + es * N * N
    if prec == "fp32":
        fpeak, fname = peaks["fp32_tflops"], peaks["fp32_source"]
    else:
        fpeak, fname = peaks["bf16_tflops"], peaks["source"] + " bf16 dense, burst"
    t_flop = mma_flops / (fpeak * 1e12)
    t_byte = c_bytes / (peaks["hbm_gbs"] * 1e9)
    tensor_bound = t_flop >= t_byte
    s = ms_mul / 1e3
    kname = {"fp32": "spamm_mul_simt_kernel", "fp32x3": "spamm_mul_x3_kernel"}.get(prec, "spamm_mul_dual_kernel")
    roof = {"kernel": kname, "bound": ("tensor" if prec != "fp32" else "alu") if tensor_bound else "hbm",
            "achieved": (mma_flops / s / 1e12) if tensor_bound else (c_bytes / s / 1e9),
            "peak": fpeak if tensor_bound else peaks["hbm_gbs"],
            "unit": "TFLOP/s" if tensor_bound else "GB/s",
            "traffic": traffic,
            "work_per_launch": (f"{'6*' if prec == 'fp32x3' else ''}2*32^3*kept = {mma_flops:.4g} FLOP "
                                f"(kept={st['kept']}); compulsory bytes {c_bytes:.4g} (C write + A read)"),
            "floor_ms": max(t_flop, t_byte) * 1e3, "peak_source": fname if tensor_bound else peaks["source"]}
    roof["frac"] = roof["achieved"] / roof["peak"]
    if prec != "fp32" and tensor_bound:
        roof["frac_vs_sustained_peak"] = (mma_flops / s / 1e12) / peaks["bf16_tflops_sustained"]
    norm_bytes = 1.0 * N * N * es + 2.0 * (N // TILE) ** 2 * 8      # A = B: read once, both maps written
    norms = {"kernel": "tile_norms_kernel (A = B: one read, both maps)", "bound": "hbm",
             "achieved": norm_bytes / (ms_norms / 1e3) / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
    norms["frac"] = norms["achieved"] / peaks["hbm_gbs"]
    return roof, norms, kept_flops


def _traffic(workload):
    """dram read+write bytes per launch of the dominant kernel from an ncu --set full capture of
    this exact workload (profiles/ncu_traffic.json, keyed by the config's workload string); null
    when no capture of this workload exists."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p)).get(workload, {}).get("multiply")
    except (OSError, ValueError, AttributeError):
        return None


def run_ours(args, rank, world, local_rank):
    from paper_2103_13042_b200 import spamm as sp
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    N, prec, tau = args.n, args.precision, args.tau
    peaks = _peaks()
    stream = torch.cuda.current_stream()
    es = 4 if prec in ("fp32", "fp32x3") else 2
    big = N * N * es > L2_BYTES
    flush = None if big else _flusher(dev)

    comm = None
    if world > 1:
        from paper_2103_13042_b200 import dist as spd
        comm = spd.nccl_comm(rank, world)

    A = synth.toeplitz_device(_table(N, args.lam, prec), N, DT[prec], device=dev)
    C = torch.empty((N, N), dtype=torch.float32, device=dev)
    plan = sp.Plan(N, N, N, tau, prec, flags=sp.SPAMM_FLAG_TIMING)

    def step():
        if world > 1:
            sp.spamm_multiply_mgpu(plan.handle, comm, rank, world, A, A, C, 0)
        else:
            sp.spamm_run(plan.handle, A, A, C)

    # ---------------- headline: W warm-up steps, then K timed steps (CUDA events per step,
    # barrier + synchronize on both sides of the timed region, max over ranks)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    _barrier(world)
    clocks = ClockSampler(local_rank)
    clocks.start()
    launches0 = sp.spamm_launch_count()
    step_ms, stage = [], {"norms": [], "skipmap": [], "multiply": []}
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        if flush is not None:
            flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        st = plan.stats()
        for k in stage:
            stage[k].append(st["ms_" + k])
    torch.cuda.synchronize()
    _barrier(world)
    wall_s = time.perf_counter() - t_wall
    launches = sp.spamm_launch_count() - launches0
    clk = clocks.stop()
    st = plan.stats()
    ms = _max_over_ranks(statistics.mean(step_ms), world)
    value = 2.0 * N ** 3 / (ms / 1e3) / 1e12
    mean = {k: statistics.mean(v) for k, v in stage.items()}
    cfg = _config(args, world)
    roof, norms_roof, kept_flops = _roofline(st, prec, mean["multiply"], mean["norms"], N, peaks, es,
                                             _traffic(cfg["workload"]))
    shares = {k: v / max(sum(mean.values()), 1e-9) for k, v in mean.items()}
    kept_all = _sum_over_ranks(st["kept"], world)

    e2e = None if args.no_e2e else _e2e(sp, plan, A, C, prec, N, args, world, rank, comm)
    sweep = None
    if not args.no_sweep and world == 1:
        sweep = _sweeps(sp, A, N, prec, args, flush, stream, dev)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        dt, fl, desc = oracle_sample(N, args.lam, prec, tau)
        threads, model = _cpu_info()
        cpu = {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": threads, "cpu": model, "kind": "oracle",
               "sample": f"{desc}; {dt:.2f} s"}
        try:   # the same oracle on one host thread (BLAS pinned to 1 thread), a quarter of the sample
            from threadpoolctl import threadpool_limits
            with threadpool_limits(limits=1):
                dt1, fl1, _ = oracle_sample(N, args.lam, prec, tau, rows=4, cols=48)
            cpu["value_1_thread"] = fl1 / dt1 / 1e12
            cpu["sample_1_thread"] = f"4 middle tile rows x 48 random tile columns; {dt1:.2f} s"
        except Exception as exc:   # noqa: BLE001 (reporting only)
            cpu["value_1_thread"] = None
            cpu["sample_1_thread"] = f"unavailable: {exc}"
    plan.close()
    if comm is not None:
        sp.spamm_nccl_comm_destroy(comm)
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": prec, "data": "synthetic (device-generated Toeplitz input)",
        "config": cfg, "stages_ms": mean, "stage_share": shares, "valid_ratio": st["valid_ratio"],
        "kept_pairs": kept_all, "kept_tflops": 2.0 * TILE ** 3 * kept_all / (ms / 1e3) / 1e12,
        "roofline": roof, "roofline_norms": norms_roof, "e2e": e2e, "gpu_launches": launches,
        "clocks": clk, "wall_s_timed_region": wall_s, "cpu_baseline": cpu, "sweep": sweep,
    }
    if sweep and sweep.get("cublas", {}).get(f"N={N}"):
        line["speedup_vs_cublas"] = sweep["cublas"][f"N={N}"]["ms"] / ms
    print(json.dumps(line), flush=True)


def _e2e(sp, plan, A, C, prec, N, args, world, rank, comm):
    """End to end through the public API with host buffers: every step copies the step's input
    A (C = A*A) from pinned host memory to the device, runs the SpAMM (spamm_run, or
    spamm_multiply_mgpu on this rank's share) and copies this rank's rows of C back to pinned
    host memory.  Two device buffer sets: step i+1's upload and step i-1's download overlap
    step i's compute (upload / compute / download streams)."""
    dev = A.device
    host_a = torch.empty((N, N), dtype=A.dtype, pin_memory=True)
    host_a.copy_(A)
    Ad = [A, torch.empty_like(A)]
    Cd = [C, torch.empty_like(C)]
    row_part = None
    if world > 1:
        sp.spamm_multiply_mgpu(plan.handle, comm, rank, world, A, A, C, 0)
        cut = sp.spamm_get_partition(plan.handle, world)
        row_part = (min(cut[rank] * TILE, N), min(cut[rank + 1] * TILE, N))
    r0, r1 = row_part or (0, N)
    host_c = torch.empty((max(r1 - r0, 1), N), dtype=torch.float32, pin_memory=True)
    s_up, s_cmp, s_dn = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev = {k: [torch.cuda.Event(), torch.cuda.Event()] for k in ("up", "cmp", "dn")}
    started = [False, False]

    def step(i):
        b = i % 2
        with torch.cuda.stream(s_up):
            if started[b]:
                s_up.wait_event(ev["cmp"][b])
            Ad[b].copy_(host_a, non_blocking=True)
            ev["up"][b].record(s_up)
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(ev["up"][b])
            if started[b]:
                s_cmp.wait_event(ev["dn"][b])
            if world > 1:
                sp.spamm_multiply_mgpu(plan.handle, comm, rank, world, Ad[b], Ad[b], Cd[b], 0, stream=s_cmp)
            else:
                sp.spamm_run(plan.handle, Ad[b], Ad[b], Cd[b], stream=s_cmp)
            ev["cmp"][b].record(s_cmp)
        with torch.cuda.stream(s_dn):
            s_dn.wait_event(ev["cmp"][b])
            if r1 > r0:
                host_c.copy_(Cd[b][r0:r1], non_blocking=True)
            ev["dn"][b].record(s_dn)
        started[b] = True

    for i in range(2):
        step(i)
    torch.cuda.synchronize()
    _barrier(world)
    n = max(3, min(args.steps, 6))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_up)
    for i in range(n):
        step(i)
    s_up.wait_stream(s_dn)
    e1.record(s_up)
    e1.synchronize()
    ms = _max_over_ranks(e0.elapsed_time(e1) / n, world)
    del Ad[1], Cd[1]
    torch.cuda.empty_cache()
    h2d = int(host_a.numel() * host_a.element_size()) * world
    d2h = int(N * N * 4)
    return {"value": 2.0 * N ** 3 / (ms / 1e3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": n,
            "note": "pinned host A -> device, SpAMM through the C ABI, this rank's C rows -> pinned host, every "
                    "step; pipelined over upload / compute / download streams with two device buffer sets"}


def _sweep_one(sp, A, N, prec, taus, flush, stream, reps=3, workload=None):
    out = []
    C = torch.empty((N, N), dtype=torch.float32, device=A.device)
    with sp.Plan(N, N, N, taus[0], prec, flags=sp.SPAMM_FLAG_TIMING) as plan:
        for tau in taus:
            plan.set_tau(tau)
            stages = {"norms": [], "skipmap": [], "multiply": []}
            ms_list = []
            for i in range(1 + reps):
                if flush is not None:
                    flush()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                sp.spamm_run(plan.handle, A, A, C)
                e1.record(stream)
                e1.synchronize()
                if i >= 1:
                    ms_list.append(e0.elapsed_time(e1))
                    s = plan.stats()
                    for k in stages:
                        stages[k].append(s["ms_" + k])
            s = plan.stats()
            ms = statistics.median(ms_list)
            ms_mul = statistics.median(stages["multiply"])
            roof, _, _ = _roofline(s, prec, ms_mul, statistics.median(stages["norms"]), N, _peaks(),
                                   4 if prec in ("fp32", "fp32x3") else 2, None)
            out.append({"N": N, "workload": workload, "precision": prec, "tau": tau, "ms": ms, "valid_ratio": s["valid_ratio"],
                        "kept": s["kept"], "stages_ms": {k: statistics.median(v) for k, v in stages.items()},
                        "tflops_dense_equiv": 2.0 * N ** 3 / (ms / 1e3) / 1e12,
                        "tflops_kept": 2.0 * TILE ** 3 * s["kept"] / (ms / 1e3) / 1e12,
                        "multiply_tflops_kept": 2.0 * TILE ** 3 * s["kept"] / (ms_mul / 1e3) / 1e12,
                        # multiply floor = max(kept MMA FLOPs / peak, (C write + A read) / HBM peak)
                        "multiply_roofline": {"bound": roof["bound"], "floor_ms": roof["floor_ms"],
                                              "frac": roof["floor_ms"] / ms_mul}})
    del C
    return out


def _cublas(A, flush, stream, reps):
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
    ms = statistics.median(_timed(lambda: torch.matmul(A, A), reps, 1, flush, stream))
    N = A.shape[0]
    return {"ms": ms, "tflops": 2.0 * N ** 3 / (ms / 1e3) / 1e12,
            "call": "torch.matmul (cuBLAS), " + ("FP32 SGEMM, TF32 off" if A.dtype == torch.float32
                                                else f"{str(A.dtype)[6:]} in, FP32 accumulate")}


def _low_only_point(sp, A, N, tau, flush, stream):
    """SPAMM_MUL_LOW_ONLY: the same SpAMM with the result written only as BF16
    (half the output bytes; C-write-bound at N = 16384), through spamm_multiply_chain."""
    Cl = torch.empty((N, N), dtype=A.dtype, device=A.device)
    with sp.Plan(N, N, N, tau, "bf16") as plan:
        fl = sp.SPAMM_MUL_AUTO | sp.SPAMM_MUL_LOW_ONLY
        ms = statistics.median(_timed(lambda: sp.spamm_multiply_chain(plan.handle, A, A, None, Cl, flags=fl),
                                      5, 2, flush, stream))
        st = plan.stats()
    return {"N": N, "precision": "bf16", "output": "bf16 only (SPAMM_MUL_LOW_ONLY)", "tau": tau, "ms": ms,
            "valid_ratio": st["valid_ratio"], "kept": st["kept"],
            "tflops_dense_equiv": 2.0 * N ** 3 / (ms / 1e3) / 1e12,
            "tflops_kept": 2.0 * TILE ** 3 * st["kept"] / (ms / 1e3) / 1e12}


def _sweeps(sp, A, N, prec, args, flush, stream, dev):
    """tau sweeps on configs[4] (the headline size), the north_star's N = 16384 exponential-decay
    target and configs[1] N = 8192, with cuBLAS dense GEMM on the same box and inputs."""
    res, cublas = [], {}
    res += _sweep_one(sp, A, N, prec, TAU5, flush, stream, workload=f"configs[4] lambda={args.lam}")
    cublas[f"N={N}"] = _cublas(A, flush, stream, 3)
    small_flush = _flusher(dev)
    for n2, lam2, precs, taus in ((16384, 0.99, ("bf16", "fp32x3", "fp32"), TAU5), (8192, 0.99, ("bf16", "fp32x3"), TAU9)):
        for p2 in precs:
            A2 = synth.toeplitz_device(_table(n2, lam2, p2), n2, DT[p2], device=dev)
            wl = "north_star target, lambda=0.99" if n2 == 16384 else "configs[1], lambda=0.99"
            res += _sweep_one(sp, A2, n2, p2, taus, small_flush, stream, workload=wl)
            if p2 != "fp32x3":
                cublas[f"N={n2} {p2}"] = _cublas(A2, small_flush, stream, 3)
            if p2 == "bf16" and n2 == 16384:
                res.append(_low_only_point(sp, A2, n2, 1e-6, small_flush, stream))
            del A2
    # configs[2]: the paper's own Table 2 workload -- N = 16384 algebraic decay at the six Table 1
    # tau (valid ratio 30 ... 5 %), next to cuBLAS on the same inputs
    alg = []
    t1 = _table1_taus(16384)
    for p2 in ("bf16", "fp32x3", "fp32"):
        A2 = synth.toeplitz_device(_table_alg(16384, p2), 16384, DT[p2], device=dev)
        pts = _sweep_one(sp, A2, 16384, p2, [tau for _, tau in t1], small_flush, stream, reps=2,
                         workload="configs[2] algebraic decay 0.1/(d^0.1+1), Table 1 tau")
        for r, (target, _) in zip(pts, t1):
            r["table1_target_valid_ratio"] = target
        if p2 != "fp32x3":
            cublas[f"N=16384 alg {p2}"] = _cublas(A2, small_flush, stream, 2)
        alg += pts
        del A2
    for r in alg:
        r["speedup_vs_cublas"] = cublas[f"N=16384 alg {'fp32' if r['precision'] == 'fp32x3' else r['precision']}"]["ms"] / r["ms"]
    for r in res:
        if "output" in r:
            r["speedup_vs_cublas"] = cublas[f"N={r['N']} bf16"]["ms"] / r["ms"]
            continue
        key = f"N={r['N']}" if r["N"] == N else f"N={r['N']} {'fp32' if r['precision'] == 'fp32x3' else r['precision']}"
        if key in cublas and (r["N"] != N or r["precision"] == prec):
            r["speedup_vs_cublas"] = cublas[key]["ms"] / r["ms"]
    res += alg
    torch.cuda.empty_cache()
    return {"points": res, "cublas": cublas,
            "workloads": {f"N={N}": f"configs[4] lambda={args.lam}", "N=16384": "north_star target, lambda=0.99",
                          "N=8192": "configs[1], lambda=0.99",
                          "N=16384 alg": "configs[2], the paper's algebraic decay (PAPER.md:257) at the Table 1 tau"}}


def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _max_over_ranks(x, world):
    if world <= 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(x, world):
    if world <= 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.int64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(args_list, n):
    """--gpus N started without a launcher: run N ranks under torch.distributed.run ourselves."""
    if torch.cuda.device_count() < n:
        sys.exit(f"bench.py: --gpus {n} requested but only {torch.cuda.device_count()} CUDA device(s) visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *args_list]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", choices=["bf16", "fp16", "fp32", "fp32x3"], default="bf16")
    ap.add_argument("--tau", type=float, default=TAU_HEADLINE)
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--lam", type=float, default=LAM_DEFAULT)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "ours":
        args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        _spawn(sys.argv[1:], args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if rank == 0:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using {world}", file=sys.stderr)
        args.gpus = world
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
