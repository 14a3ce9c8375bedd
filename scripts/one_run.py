"""spamm_run on an exponential-decay Toeplitz matrix (A = B), a few times -- the target of ncu
captures of one kernel:  python scripts/one_run.py N lambda tau precision [runs]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2103_13042_b200 import spamm as sp  # noqa: E402

N, lam, tau, prec = int(sys.argv[1]), float(sys.argv[2]), float(sys.argv[3]), sys.argv[4]
runs = int(sys.argv[5]) if len(sys.argv) > 5 else 3
dt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32, "fp32x3": torch.float32}[prec]
tb = synth.decay_table("exp", N, lam, 1.0).astype(np.float32)
if prec == "bf16":
    tb = synth.round_to_bf16(tb)
A = synth.toeplitz_device(tb, N, dt)
C = torch.empty((N, N), dtype=torch.float32, device="cuda")
with sp.Plan(N, N, N, tau, prec, flags=sp.SPAMM_FLAG_TIMING) as plan:
    for _ in range(runs):
        plan.run(A, A, C)
    torch.cuda.synchronize()
    st = plan.stats()
    print({k: st[k] for k in ("kept", "valid_ratio", "ms_norms", "ms_skipmap", "ms_multiply")})
