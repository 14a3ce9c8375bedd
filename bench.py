#!/usr/bin/env python
"""SpAMM hot-path benchmark (BASELINE.json metric: SpAMM time & effective TFLOP/s vs tau,
speedup vs cuBLAS GEMM) on BASELINE.json configs[1]: N=8192 exponential-decay matrices
a_ij = 0.99^|i-j|, tile 32, tau sweep 1e-10..1e-2, FP32 and BF16 paths.

One STEP = one whole SpAMM call through the C ABI (spamm_run): tile norms of A and B ->
skip map -> masked multiply into C, at the headline point (BF16 tcgen05 path,
tau = 1e-6).  Inputs are resident in HBM; L2 (126 MB) is flushed by writing a 512 MB
buffer and then reading another 512 MB buffer before every timed step, outside the
step's CUDA events.

  python bench.py [--gpus N --steps K --warmup W]            # our CUDA path
  python bench.py --impl reference [...]                      # the CPU float64 oracle arm

Multi-GPU (torchrun, one rank per GPU): the same problem is row-partitioned across
ranks with spamm_multiply_mgpu (Sec. 3.4 of the paper), strong scaling, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
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

N_DEFAULT = 8192
LAM = 0.99
TAU_HEADLINE = 1e-6
TAU_SWEEP = [1e-10, 1e-9, 1e-8, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2]
TILE = 32
ORACLE_SAMPLE_TILE_ROWS = 64     # bounded CPU sample: 64 middle tile rows (2048 rows) of C


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "sm_max_mhz": d.get("sm_max_mhz", 1965.0), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0,
            "source": "fallback (B200_PROFILING.md)"}


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
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.15)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
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
def _cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return int(max(n)) if n else os.cpu_count()
    except Exception:
        return os.cpu_count()


def oracle_sample(N: int, prec: str, tau: float, rows: int = ORACLE_SAMPLE_TILE_ROWS):
    """Time the float64 oracle (as it stands) on a bounded sample: C rows of `rows` middle
    tile rows of the same workload (their A rows times the full B; includes the norm
    maps of the sample's A rows and of all of B).  Returns (seconds, dense-equivalent flops)."""
    import oracle
    A = synth.decay_matrix(N, "exp", LAM)
    if prec == "bf16":
        A = synth.round_to_bf16(A)
    BM = N // TILE
    r0 = (BM - rows) // 2
    As = A[r0 * TILE:(r0 + rows) * TILE]
    t0 = time.perf_counter()
    C = oracle.spamm(As, A, tau, TILE)
    dt = time.perf_counter() - t0
    assert C.shape == (rows * TILE, N)
    return dt, 2.0 * rows * TILE * N * N


def run_reference(args, rank, world):
    """--impl reference: the oracle arm (rank 0 only; other ranks exit without work)."""
    if rank != 0:
        return
    prec = args.precision
    for _ in range(args.warmup):
        oracle_sample(args.n, prec, args.tau, rows=args.ref_rows)
    times, flops = [], 0.0
    for _ in range(args.steps):
        dt, flops = oracle_sample(args.n, prec, args.tau, rows=args.ref_rows)
        times.append(dt)
    ms = 1e3 * statistics.mean(times)
    value = flops / (ms / 1e3) / 1e12
    sample = (f"{args.ref_rows} middle tile rows ({args.ref_rows * TILE} of {args.n} rows of C) x full B, "
              f"float64 numpy oracle incl. norm maps")
    cores = _cpu_threads()
    line = {
        "impl": "reference", "metric": "SpAMM effective TFLOP/s (dense-equivalent 2MNK/t)", "value": value,
        "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config(args, prec),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config(args, prec):
    return {"workload": f"configs[1]: N={args.n} exponential decay a_ij=0.99^|i-j| (A=B), tile 32, "
                        f"tau={args.tau:g}, {prec.upper()} path", "N": args.n, "tile": TILE, "lambda": LAM,
            "tau": args.tau, "precision": prec,
            "parallelism": f"row-partition x{args.gpus}" if args.gpus > 1 else "single GPU",
            "l2": "flushed before every timed step (512 MB write, then 512 MB read of another buffer)"}


# --------------------------------------------------------------- GPU path ---
def _device_inputs(N, prec, dev):
    A32 = synth.decay_matrix(N, "exp", LAM)
    dt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32, "fp32x3": torch.float32}[prec]
    A = torch.from_numpy(A32).to(device=dev).to(dt)
    return A32, A


def _timed(fn, steps, warmup, flush, stream):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    return ms


def run_ours(args, rank, world, local_rank):
    from paper_2103_13042_b200 import spamm as sp
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    N, prec, tau = args.n, args.precision, args.tau
    peaks = _peaks()
    stream = torch.cuda.current_stream()
    # L2 flush between timed steps: write a 512 MB buffer (evicts everything), then read a
    # second 512 MB buffer so the flush's own dirty lines are written back before the timed
    # region instead of inside the first kernel of the step (L2 ends clean, holding none of
    # A, B, C or the plan's maps).
    flush_buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush_rd = torch.zeros(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush_out = torch.empty((), dtype=torch.float32, device=dev)

    def flush():
        flush_buf.zero_()
        torch.sum(flush_rd, dim=0, out=flush_out)

    comm = None
    if world > 1:
        import torch.distributed as dist
        uid = [sp.spamm_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = sp.spamm_nccl_comm_init(world, rank, uid[0])

    A32, A = _device_inputs(N, prec, dev)
    C = torch.empty((N, N), dtype=torch.float32, device=dev)
    plan = sp.Plan(N, N, N, tau, prec, flags=sp.SPAMM_FLAG_TIMING)

    def step():
        if world > 1:
            sp.spamm_multiply_mgpu(plan.handle, comm, rank, world, A, A, C, 0)
        else:
            sp.spamm_run(plan.handle, A, A, C)

    # ---------------- headline: K timed steps (each step bracketed by CUDA events)
    for _ in range(args.warmup):
        step()
    _barrier(world)
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    launches0 = sp.spamm_launch_count()
    step_ms, stage = [], {"norms": [], "skipmap": [], "multiply": []}
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        st = plan.stats()
        stage["norms"].append(st["ms_norms"])
        stage["skipmap"].append(st["ms_skipmap"])
        stage["multiply"].append(st["ms_multiply"])
    torch.cuda.synchronize()
    _barrier(world)
    wall_s = time.perf_counter() - t_wall
    launches = sp.spamm_launch_count() - launches0
    clk = clocks.stop()
    st = plan.stats()
    ms_local = statistics.mean(step_ms)
    ms = _max_over_ranks(ms_local, world)
    dense_flops = 2.0 * N * N * N
    value = dense_flops / (ms / 1e3) / 1e12

    # ---------------- roofline of the dominant kernel (device time inside the timed region)
    kept_flops = 2.0 * TILE ** 3 * st["kept"]
    es = 4 if prec in ("fp32", "fp32x3") else 2
    mean = {k: statistics.mean(v) for k, v in stage.items()}
    dominant = max(mean, key=mean.get)
    traffic = _ncu_traffic(prec)
    if dominant == "multiply":
        peak = peaks["bf16_tflops"] if prec != "fp32" else _fp32_peak(peaks)
        # fp32x3 executes six BF16 products per kept pair on the tensor cores
        mma_flops = kept_flops * (6 if prec == "fp32x3" else 1)
        achieved = mma_flops / (mean["multiply"] / 1e3) / 1e12
        # BF16/FP16: 256 x 256 macro-tiles (macro_i = 8) run multiply_dual.cu, 128 x 256 multiply_umma.cu
        tc_kernel = "spamm_mul_dual_kernel" if st.get("macro_i") == 8 else "spamm_mul_umma_kernel"
        kname = {"fp32": "spamm_mul_simt_kernel", "fp32x3": "spamm_mul_x3_kernel"}.get(prec, tc_kernel)
        work = (f"6*2*32^3*kept = {mma_flops:.4g} BF16 MMA FLOP (kept={st['kept']})" if prec == "fp32x3"
                else f"2*32^3*kept = {kept_flops:.4g} FLOP (kept={st['kept']})")
        roof = {"kernel": kname,
                "bound": "tensor" if prec != "fp32" else "alu", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic.get("multiply"),
                "work_per_launch": work,
                "peak_source": peaks["source"] + (" bf16 burst" if prec != "fp32" else
                                                  " FP32 CUDA-core 148 SM x 128 FMA x 2 x sm_max clock")}
    else:
        bytes_alg = 1.0 * N * N * es + 2.0 * (N // TILE) ** 2 * 8     # A = B: read once (norms.cu)
        achieved = bytes_alg / (mean["norms"] / 1e3) / 1e9
        roof = {"kernel": "tile_norms_kernel", "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic.get("norms"),
                "work_per_launch": f"read A and B once ({bytes_alg:.4g} B)", "peak_source": peaks["source"]}
    # secondary: the HBM-bound norm stage
    # A = B (C = A*A): the norm kernel reads the matrix once and writes both maps
    norm_bytes = 1.0 * N * N * es + 2.0 * (N // TILE) ** 2 * 8
    norms_roof = {"kernel": "tile_norms_kernel (A = B: one read, both maps)", "bound": "hbm",
                  "achieved": norm_bytes / (mean["norms"] / 1e3) / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
    norms_roof["frac"] = norms_roof["achieved"] / peaks["hbm_gbs"]

    # ---------------- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = _e2e(sp, A32, prec, N, tau, args, stream, flush, world, rank, comm)

    # ---------------- tau sweep, both paths, and cuBLAS on the same box
    sweep, cublas = None, None
    if not args.no_sweep and world == 1:
        sweep, cublas = _sweep(sp, N, stream, flush)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dt, fl = oracle_sample(N, prec, tau)
        cpu = {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": _cpu_threads(), "kind": "oracle",
               "sample": f"{ORACLE_SAMPLE_TILE_ROWS} middle tile rows ({ORACLE_SAMPLE_TILE_ROWS * TILE} of {N} rows "
                         f"of C) x full B, float64 numpy oracle incl. norm maps; {dt:.2f} s"}

    if comm is not None:
        sp.spamm_nccl_comm_destroy(comm)
    if rank != 0:
        return
    line = {
        "metric": "SpAMM effective TFLOP/s (dense-equivalent 2MNK/t)", "value": value, "unit": "TFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": prec, "data": "synthetic", "config": _config(args, prec),
        "stages_ms": mean, "valid_ratio": st["valid_ratio"], "kept_pairs": st["kept"],
        "macro_steps": st["macro_entries"],
        "kept_tflops": kept_flops / (ms / 1e3) / 1e12,
        "roofline": roof, "roofline_norms": norms_roof,
        "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        "wall_s_timed_region_incl_flush": wall_s,
        "cpu_baseline": cpu, "sweep": sweep, "cublas": cublas,
    }
    if cublas and prec in cublas:
        line["speedup_vs_cublas"] = cublas[prec]["ms"] / ms
    print(json.dumps(line), flush=True)


def _fp32_peak(peaks):
    return 148 * 128 * 2 * peaks["sm_max_mhz"] * 1e6 / 1e12


def _ncu_traffic(prec):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)).get(prec, {})
        except Exception:
            return {}
    return {}


def _e2e(sp, A32, prec, N, tau, args, stream, flush, world, rank, comm):
    """End to end through the public API: every step copies that step's A (the workload is
    C = A*A, so A is the only input) from pinned host memory, runs spamm_run, and copies C back
    to pinned host memory.  Steps are pipelined over three streams with double buffers (step
    i+1's upload and step i-1's download overlap step i's compute, as a streaming user would
    run it); the timed region spans the first upload to the last download.  Inputs are larger
    than L2 and arrive fresh from the host every step."""
    dt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32, "fp32x3": torch.float32}[prec]
    host = torch.from_numpy(A32).to(dt)
    dev = torch.device("cuda", torch.cuda.current_device())
    Ah = [host.pin_memory(), host.clone().pin_memory()]
    Ch = [torch.empty((N, N), dtype=torch.float32).pin_memory() for _ in range(2)]
    Ad = [torch.empty_like(host, device=dev) for _ in range(2)]
    Cd = [torch.empty((N, N), dtype=torch.float32, device=dev) for _ in range(2)]
    plan = sp.Plan(N, N, N, tau, prec)
    s_up, s_cmp, s_dn = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev = {k: [torch.cuda.Event(), torch.cuda.Event()] for k in ("up", "cmp", "dn")}
    started = [[False, False]]

    def step(i):
        b = i % 2
        with torch.cuda.stream(s_up):
            if started[0][b]:
                s_up.wait_event(ev["cmp"][b])          # Ad[b] free: its previous product is done
            Ad[b].copy_(Ah[b], non_blocking=True)
            ev["up"][b].record(s_up)
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(ev["up"][b])
            if started[0][b]:
                s_cmp.wait_event(ev["dn"][b])          # Cd[b] free: its previous download is done
            if world > 1:
                sp.spamm_multiply_mgpu(plan.handle, comm, rank, world, Ad[b], Ad[b], Cd[b], sp.SPAMM_MGPU_GATHER_C,
                                       stream=s_cmp)
            else:
                sp.spamm_run(plan.handle, Ad[b], Ad[b], Cd[b], stream=s_cmp)
            ev["cmp"][b].record(s_cmp)
        with torch.cuda.stream(s_dn):
            s_dn.wait_event(ev["cmp"][b])
            Ch[b].copy_(Cd[b], non_blocking=True)
            ev["dn"][b].record(s_dn)
        started[0][b] = True

    for i in range(2):
        step(i)
    torch.cuda.synchronize()
    _barrier(world)
    n = max(4, args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_up)
    for i in range(n):
        step(i)
    s_up.wait_stream(s_dn)
    e1.record(s_up)
    e1.synchronize()
    ms = _max_over_ranks(e0.elapsed_time(e1) / n, world)
    plan.close()
    return {"value": 2.0 * N ** 3 / (ms / 1e3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "h2d_bytes_per_step": int(host.numel() * host.element_size()),
            "d2h_bytes_per_step": int(N * N * 4), "steps": n,
            "note": "pinned host A -> device, spamm_run (C = A*A), C -> pinned host, every step; "
                    "pipelined over upload/compute/download streams with double buffers"}


def _sweep(sp, N, stream, flush):
    out = []
    A32 = synth.decay_matrix(N, "exp", LAM)
    dev = torch.device("cuda", torch.cuda.current_device())
    cublas = {}
    for prec in ("fp32", "fp32x3", "bf16"):
        dt = {"bf16": torch.bfloat16, "fp32": torch.float32, "fp32x3": torch.float32}[prec]
        A = torch.from_numpy(A32).to(device=dev).to(dt)
        C = torch.empty((N, N), dtype=torch.float32, device=dev)
        plan = sp.Plan(N, N, N, TAU_SWEEP[0], prec, flags=sp.SPAMM_FLAG_TIMING)
        for tau in TAU_SWEEP:
            plan.set_tau(tau)
            stages = {"norms": [], "skipmap": [], "multiply": []}

            def step():
                sp.spamm_run(plan.handle, A, A, C)

            ms_list = []
            for i in range(2 + 5):
                flush()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step()
                e1.record(stream)
                e1.synchronize()
                if i >= 2:
                    ms_list.append(e0.elapsed_time(e1))
                    s = plan.stats()
                    for k in stages:
                        stages[k].append(s["ms_" + k])
            s = plan.stats()
            ms = statistics.median(ms_list)
            out.append({"precision": prec, "tau": tau, "ms": ms, "valid_ratio": s["valid_ratio"],
                        "kept": s["kept"], "stages_ms": {k: statistics.median(v) for k, v in stages.items()},
                        "tflops_dense_equiv": 2.0 * N ** 3 / (ms / 1e3) / 1e12,
                        "tflops_kept": 2.0 * TILE ** 3 * s["kept"] / (ms / 1e3) / 1e12})
        plan.close()
        # cuBLAS dense GEMM on the same matrices (torch.matmul -> cublas), same flush protocol
        torch.backends.cuda.matmul.allow_tf32 = False
        torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
        gemm = lambda: torch.matmul(A, A)  # noqa: E731
        if prec == "fp32x3":   # same FP32 inputs and accuracy class: compared with the SGEMM
            ms_c = cublas["fp32"]["ms"]
        else:
            ms_c = statistics.median(_timed(gemm, 3 if prec == "fp32" else 5, 2, flush, stream))
            cublas[prec] = {"ms": ms_c, "tflops": 2.0 * N ** 3 / (ms_c / 1e3) / 1e12,
                            "call": "torch.matmul (cuBLAS), " + ("FP32 SGEMM, TF32 off" if prec == "fp32"
                                                                else "BF16 in, FP32 accumulate")}
        for r in out:
            if r["precision"] == prec:
                r["speedup_vs_cublas"] = ms_c / r["ms"]
        del A, C
    return out, cublas


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", choices=["bf16", "fp16", "fp32", "fp32x3"], default="bf16")
    ap.add_argument("--tau", type=float, default=TAU_HEADLINE)
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--ref-rows", type=int, default=16, help="oracle sample (tile rows) per reference step")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
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
