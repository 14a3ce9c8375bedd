"""Fixed-cost view of the SpAMM pipeline on the small BASELINE.json shapes (configs[0] N = 1024
exponential decay; configs[3] im2col layers) and configs[1] N = 8192: spamm_run eager (CUDA events
around the call) and replayed from a captured CUDA graph, next to cuBLAS on the same inputs.
Prints one JSON line; L2 flushed before every timed repetition."""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2103_13042_b200 import spamm as sp  # noqa: E402

DT = {"bf16": torch.bfloat16, "fp32": torch.float32, "fp32x3": torch.float32}
flush_buf = torch.empty(512 * 1024 * 1024 // 4, device="cuda")


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        flush_buf.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


def case(name, A32, B32, tau, prec):
    M, K = A32.shape
    N = B32.shape[1]
    A = torch.from_numpy(A32).to(DT[prec]).cuda()
    B = torch.from_numpy(B32).to(DT[prec]).cuda()
    C = torch.empty((M, N), device="cuda")
    plan = sp.Plan(M, N, K, tau, prec, flags=sp.SPAMM_FLAG_TIMING)
    plan.run(A, B, C)
    torch.cuda.synchronize()
    st = plan.stats()
    eager = timed(lambda: sp.spamm_run(plan.handle, A, B, C))
    st = plan.stats()
    def graph_time(flags):
        g = torch.cuda.CUDAGraph()
        plan2 = sp.Plan(M, N, K, tau, prec, flags=flags)
        plan2.run(A, B, C)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            sp.spamm_run(plan2.handle, A, B, C)
        return timed(g.replay)
    graph = graph_time(0)
    graph_staged = graph_time(sp.SPAMM_FLAG_STAGED)   # norm -> skip-map -> multiply kernels
    torch.backends.cuda.matmul.allow_tf32 = False
    cub = timed(lambda: torch.matmul(A, B))
    return {"case": name, "precision": prec, "M": M, "N": N, "K": K, "tau": tau, "valid_ratio": st["valid_ratio"],
            "eager_ms": eager, "graph_ms": graph, "graph_staged_ms": graph_staged, "cublas_ms": cub, "speedup_graph_vs_cublas": cub / graph,
            "stages_ms": {k: st["ms_" + k] for k in ("norms", "skipmap", "multiply")}}


def main():
    out = []
    for lam in (0.9, 0.99):
        A = synth.decay_matrix(1024, "exp", lam)
        for prec in ("bf16", "fp32", "fp32x3"):
            out.append(case(f"configs[0] N=1024 lambda={lam}", A, A, 1e-4, prec))
    for layer in ("conv21", "conv31"):
        W, B = synth.im2col_gemm(layer)
        nA, nB = oracle.tile_norms(W, 32), oracle.tile_norms(B, 32)
        prods = np.unique(nA[:, :, None] * nB[None, :, :])
        for vr in (0.97, 0.43):
            q = int((1.0 - vr) * (len(prods) - 1))
            tau = float(0.5 * (prods[q] + prods[q + 1]))
            for prec in ("bf16", "fp32x3"):
                out.append(case(f"im2col {layer} vr~{vr}", W, B, tau, prec))
    A = synth.decay_matrix(8192, "exp", 0.99)
    for prec in ("bf16", "fp32x3"):
        out.append(case("configs[1] N=8192 lambda=0.99", A, A, 1e-6, prec))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
