"""Per-32x32-tile relative error of the tensor path vs the oracle (debug helper)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth, oracle  # noqa: E402
from paper_2103_13042_b200 import spamm as sp  # noqa: E402


def _run(sp, A32, B32, tau, prec):
    M, K = A32.shape
    N = B32.shape[1]
    plan = sp.Plan(M, N, K, tau, prec)
    dt = torch.bfloat16
    A = torch.from_numpy(np.ascontiguousarray(A32)).to(dt).cuda()
    B = torch.from_numpy(np.ascontiguousarray(B32)).to(dt).cuda()
    C = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    plan.norms(A, B)
    plan.build_skipmap()
    plan.multiply(A, B, C)
    torch.cuda.synchronize()
    return plan, C.cpu().numpy()


_rounded = lambda x, p: synth.round_to_bf16(x)  # noqa: E731

for (M, N, K) in [tuple(map(int, a.split("x"))) for a in (sys.argv[1:] or ["256x256x256", "512x512x512", "300x512x256"])]:
    A = _rounded(synth.perturbed_decay_matrix(K, 0.95, seed=11, m=M), "bf16")
    B = _rounded(synth.perturbed_decay_matrix(N, 0.95, seed=12, m=K), "bf16")
    plan, C = _run(sp, A, B, 0.0, "bf16")
    ref = A.astype(np.float64) @ B.astype(np.float64)
    bm, bn = -(-M // 32), -(-N // 32)
    bad = np.zeros((bm, bn))
    for i in range(bm):
        for j in range(bn):
            r = ref[32 * i:32 * i + 32, 32 * j:32 * j + 32]
            c = C[32 * i:32 * i + 32, 32 * j:32 * j + 32]
            bad[i, j] = np.linalg.norm(c - r) / max(np.linalg.norm(r), 1e-30)
    print((M, N, K), "max tile err", bad.max())
    print((bad > 1e-2).astype(int))
    if bad.max() > 1e-2:
        i, j = np.unravel_index(np.argmax(bad), bad.shape)
        r = ref[32 * i:32 * i + 32, 32 * j:32 * j + 32]; c = C[32 * i:32 * i + 32, 32 * j:32 * j + 32]
        print("ratio c/r sample", (c / r)[:4, :4])
