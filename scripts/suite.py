#!/usr/bin/env python
"""Measurement suite over every BASELINE.json config on one GPU.

For each workload and tau: per-stage device times (CUDA events recorded by the library,
median over reps, L2 flushed by a 512 MB write + 512 MB read before every rep), total time,
dense-equivalent TFLOP/s (2MNK/t), kept TFLOP/s (2*32^3*P/t), the multiply's fraction of
its roofline (BF16 burst peak from MEASURED_PEAKS.json; FP32 = 148 SMs x 128 FMA x 2 x max
clock), the norm stage's HBM fraction, and cuBLAS dense GEMM (torch.matmul) on the same
shape and precision.  Writes one JSON document (default gpurun_out/suite.json).

  python scripts/suite.py [--configs 1,2,3,4a,4b,5] [--reps 5] [--out gpurun_out/suite.json]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2103_13042_b200 import spamm as sp  # noqa: E402

T = 32
DT = {"fp32": torch.float32, "fp32x3": torch.float32, "bf16": torch.bfloat16}
TAUS = [1e-10, 1e-8, 1e-6, 1e-4, 1e-2]


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    return {"hbm": d.get("hbm_gbs", 6650.0), "bf16": d.get("bf16_tflops", 1590.0),
            "fp32": 148 * 128 * 2 * d.get("sm_max_mhz", 1965.0) * 1e6 / 1e12}


PK = None
FLUSH = FLUSH_RD = FLUSH_OUT = None


def flush():
    FLUSH.zero_()                        # evict (write 512 MB) ...
    torch.sum(FLUSH_RD, dim=0, out=FLUSH_OUT)   # ... then write the dirty lines back outside the timing


def dev(x, prec):
    m, n = x.shape
    buf = torch.zeros((m, -(-n // 8) * 8), dtype=DT[prec], device="cuda")
    buf[:, :n] = torch.from_numpy(np.ascontiguousarray(x)).to(DT[prec])
    return buf[:, :n]


_CUBLAS = {}


def cublas_ms(A, B, reps):
    key = (tuple(A.shape), tuple(B.shape), A.dtype, A.data_ptr() == B.data_ptr())
    if key in _CUBLAS:   # fp32x3 is compared with the same SGEMM as fp32
        return _CUBLAS[key]
    _CUBLAS[key] = _cublas_ms(A, B, reps)
    return _CUBLAS[key]


def _cublas_ms(A, B, reps):
    out = torch.empty((A.shape[0], B.shape[1]), dtype=A.dtype, device="cuda")
    torch.backends.cuda.matmul.allow_tf32 = False
    for _ in range(2):
        torch.matmul(A, B, out=out)
    ms = []
    for _ in range(reps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(A, B, out=out)
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    del out
    return statistics.median(ms)


def measure(name, A, B, prec, taus, reps, dense_ms=None):
    M, K = A.shape
    N = B.shape[1]
    C = torch.empty((M, -(-N // 4) * 4), dtype=torch.float32, device="cuda")[:, :N]
    es = 4 if prec in ("fp32", "fp32x3") else 2
    rows = []
    with sp.Plan(M, N, K, taus[0], prec, flags=sp.SPAMM_FLAG_TIMING) as plan:
        for tau in taus:
            plan.set_tau(tau)
            for _ in range(2):
                plan.run(A, B, C)
            torch.cuda.synchronize()
            tot, st_ms = [], {"norms": [], "skipmap": [], "multiply": []}
            for _ in range(reps):
                flush()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan.run(A, B, C)
                e1.record()
                e1.synchronize()
                tot.append(e0.elapsed_time(e1))
                st = plan.stats()
                for k in st_ms:
                    st_ms[k].append(st["ms_" + k])
            st = plan.stats()
            ms = statistics.median(tot)
            stages = {k: statistics.median(v) for k, v in st_ms.items()}
            kept_fl = 2.0 * T ** 3 * st["kept"]
            mul_peak = PK["fp32"] if prec == "fp32" else PK["bf16"]
            mma_fl = kept_fl * (6 if prec == "fp32x3" else 1)   # fp32x3: six BF16 products per kept pair
            same = A.data_ptr() == B.data_ptr() and A.stride() == B.stride() and M == K == N
            norm_bytes = (M * K + (0 if same else K * N)) * es   # A = B is read once (norms.cu)
            row = {"config": name, "precision": prec, "M": M, "N": N, "K": K, "tau": tau,
                   "kept": st["kept"], "valid_ratio": st["valid_ratio"], "ms": ms, "stages_ms": stages,
                   "tflops_dense_equiv": 2.0 * M * N * K / (ms / 1e3) / 1e12,
                   "tflops_kept": kept_fl / (ms / 1e3) / 1e12,
                   "multiply_roofline_frac": (mma_fl / (stages["multiply"] / 1e3) / 1e12) / mul_peak
                   if stages["multiply"] > 0 else None,
                   "norms_hbm_frac": (norm_bytes / (stages["norms"] / 1e3) / 1e9) / PK["hbm"]}
            if dense_ms is not None:
                row["cublas_ms"] = dense_ms
                row["speedup_vs_cublas"] = dense_ms / ms
            rows.append(row)
            print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in row.items()
                              if k != "stages_ms"}), flush=True)
    del C
    return rows


def cfg_toeplitz(name, kind, lam, c, N, taus, reps, precs, device_gen=False):
    out = []
    table = synth.decay_table(kind, N, lam, c).astype(np.float32)
    for prec in precs:
        if device_gen:
            tb = synth.round_to_bf16(table) if prec == "bf16" else table
            A = synth.toeplitz_device(tb, N, DT[prec])
        else:
            A = dev(synth.toeplitz(table, N, N), prec)
        dense = cublas_ms(A, A, max(1, min(reps, 3)))
        out += measure(name, A, A, prec, taus, reps, dense)
        del A
        torch.cuda.empty_cache()
    return out


def main():
    global PK, FLUSH, FLUSH_RD, FLUSH_OUT
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4a,4b,5")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "suite.json"))
    ap.add_argument("--precs", default="fp32,fp32x3,bf16")
    args = ap.parse_args()
    PK = peaks()
    FLUSH = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    FLUSH_RD = torch.zeros(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    FLUSH_OUT = torch.empty((), dtype=torch.float32, device="cuda")
    precs = args.precs.split(",")
    cfgs = args.configs.split(",")
    res = {"peaks": PK, "device": torch.cuda.get_device_name(0), "rows": []}
    t0 = time.time()
    if "1" in cfgs:
        for lam in (0.9, 0.99):
            res["rows"] += cfg_toeplitz(f"configs[0] N=1024 exp lam={lam}", "exp", lam, 1.0, 1024, [1e-4],
                                        args.reps, precs)
    if "2" in cfgs:
        res["rows"] += cfg_toeplitz("configs[1] N=8192 exp lam=0.99", "exp", 0.99, 1.0, 8192,
                                    [1e-10, 1e-9, 1e-8, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2], args.reps, precs)
    if "3" in cfgs:
        res["rows"] += cfg_toeplitz("configs[2] N=16384 algebraic 0.1/(d^0.1+1)", "alg", 0.1, 0.1, 16384,
                                    [0.0, 0.997847, 1.012852, 1.03536, 1.06537, 1.110386, 1.170407],
                                    args.reps, precs)
        res["rows"] += cfg_toeplitz("configs[2] N=16384 exp lam=0.99", "exp", 0.99, 1.0, 16384, TAUS,
                                    args.reps, precs)
    if "4a" in cfgs:
        W = synth.water_cluster_matrix()
        for prec in precs:
            A = dev(synth.round_to_bf16(W) if prec == "bf16" else W, prec)
            res["rows"] += measure("configs[3] water cluster N=13656", A, A, prec, TAUS, args.reps,
                                   cublas_ms(A, A, 3))
            del A
    if "4b" in cfgs:
        for layer in ("conv21", "conv31"):
            W32, X32 = synth.im2col_gemm(layer)
            # tau at the target valid ratios from the library's own norm maps (input recipe)
            with sp.Plan(W32.shape[0], X32.shape[1], W32.shape[1], 0.0, "fp32") as p0:
                p0.norms(dev(W32, "fp32"), dev(X32, "fp32"))
                nA, nBt = sp.spamm_get_norms(p0.handle)
            nA, nB = nA.cpu().numpy(), nBt.cpu().numpy().T
            prods = np.unique(nA[:, :, None] * nB[None, :, :])
            taus = [float(0.5 * (prods[q] + prods[q + 1]))
                    for q in (int((1 - vr) * (len(prods) - 1)) for vr in (0.97, 0.85, 0.63, 0.43))]
            for prec in precs:
                A, B = dev(W32, prec), dev(X32, prec)
                res["rows"] += measure(f"configs[3] im2col {layer}", A, B, prec, taus, args.reps,
                                       cublas_ms(A, B, 5))
    if "5" in cfgs:
        res["rows"] += cfg_toeplitz("configs[4] N=65536 exp lam=0.999", "exp", 0.999, 1.0, 65536, TAUS,
                                    max(2, args.reps // 2), precs, device_gen=True)
    res["wall_s"] = time.time() - t0
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
