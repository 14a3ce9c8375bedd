"""One small SpAMM (configs[0] N = 1024 lambda = 0.9 BF16 tau = 1e-4, or an im2col layer) run a few
times -- for ncu launch lists of the small-problem fixed costs."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2103_13042_b200 import spamm as sp  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "n1024"
if which.startswith("n"):   # n1024 (lambda = 0.9), n<N>:<lambda>
    n = int(which.split(":")[0][1:])
    A32 = B32 = synth.decay_matrix(n, "exp", float(which.split(":")[1]) if ":" in which else 0.9)
    tau = 1e-4
else:
    A32, B32 = synth.im2col_gemm(which)
    nA, nB = oracle.tile_norms(A32, 32), oracle.tile_norms(B32, 32)
    prods = np.unique(nA[:, :, None] * nB[None, :, :])
    q = int(0.03 * (len(prods) - 1))
    tau = float(0.5 * (prods[q] + prods[q + 1]))
A = torch.from_numpy(A32).to(torch.bfloat16).cuda()
B = torch.from_numpy(B32).to(torch.bfloat16).cuda()
M, K = A.shape
N = B.shape[1]
C = torch.empty((M, N), device="cuda")
plan = sp.Plan(M, N, K, tau, "bf16")
for _ in range(4):
    sp.spamm_run(plan.handle, A, B, C)
torch.cuda.synchronize()
print(which, plan.stats()["valid_ratio"])
