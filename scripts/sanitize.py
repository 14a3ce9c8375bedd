"""Small SpAMM runs for compute-sanitizer (memcheck / racecheck / synccheck): every product kernel
(norms, pyramid, skip map + order pass, BF16 dual multiply, FP32 SIMT, FP32X3, multi-rank emulation,
im2col) on ragged shapes.  Exit code 0 when every result matches the float64 oracle."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2103_13042_b200 import spamm as sp  # noqa: E402

DT = {"fp32": torch.float32, "fp32x3": torch.float32, "bf16": torch.bfloat16}


def dev(x, prec):
    m, n = x.shape
    buf = torch.zeros((m, -(-n // 8) * 8), dtype=DT[prec], device="cuda")
    buf[:, :n] = torch.from_numpy(x).to(DT[prec])
    return buf[:, :n]


def main():
    M, N, K = 300, 520, 257
    bad = 0
    for prec in ("bf16", "fp32", "fp32x3"):
        A = synth.perturbed_decay_matrix(K, 0.95, seed=1, m=M)
        B = synth.perturbed_decay_matrix(N, 0.95, seed=2, m=K)
        if prec == "bf16":
            A, B = synth.round_to_bf16(A), synth.round_to_bf16(B)
        nA, nB = oracle.tile_norms(A, 32), oracle.tile_norms(B, 32)
        tau = float(np.median(nA[:, :, None] * nB[None, :, :]))
        C = torch.zeros((M, -(-N // 4) * 4), device="cuda")[:, :N]
        with sp.Plan(M, N, K, tau, prec) as plan:
            plan.run(dev(A, prec), dev(B, prec), C)
            torch.cuda.synchronize()
            sp.spamm_get_skipmap(plan.handle)
        ref = oracle.spamm(A, B, tau, 32, nA, nB)
        err = np.linalg.norm(C.cpu().numpy() - ref) / np.linalg.norm(ref)
        print(f"{prec}: rel err {err:.2e}")
        bad += err > 1e-5
        # two virtual ranks
        plans = [sp.Plan(M, N, K, tau, prec) for _ in range(2)]
        Cs = [torch.zeros((M, -(-N // 4) * 4), device="cuda")[:, :N] for _ in range(2)]
        sp.spamm_multiply_mgpu_local([p.handle for p in plans], dev(A, prec), dev(B, prec), Cs, sp.SPAMM_MGPU_GATHER_C)
        torch.cuda.synchronize()
        err2 = np.linalg.norm(Cs[1].cpu().numpy() - ref) / np.linalg.norm(ref)
        print(f"{prec} 2 ranks: rel err {err2:.2e}")
        bad += err2 > 1e-5
        for p in plans:
            p.close()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
