"""One N = 65536 (configs[4], exp. decay 0.999, BF16) multiply with the dual kernel's profiling
counters on (library built with SPAMM_NVCC_FLAGS=-DSPAMM_PROFILE python -m paper_2103_13042_b200.build --force):
   python scripts/prof_n65536.py [tau]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2103_13042_b200 import spamm as sp  # noqa: E402

N = 65536
tau = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-6
tb = synth.round_to_bf16(synth.decay_table("exp", N, 0.999, 1.0).astype(np.float32))
A = synth.toeplitz_device(tb, N, torch.bfloat16)
C = torch.empty((N, N), dtype=torch.float32, device="cuda")
with sp.Plan(N, N, N, tau, "bf16", flags=sp.SPAMM_FLAG_TIMING) as plan:
    for _ in range(2):
        plan.run(A, A, C)
    torch.cuda.synchronize()
    st = plan.stats()
    print({k: st[k] for k in ("kept", "valid_ratio", "ms_norms", "ms_skipmap", "ms_multiply")})
