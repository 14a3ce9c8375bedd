"""GPU: the fused small-problem path (spamm_run on plans of at most one 128 x 128 macro-tile per
SM -- BF16/FP16 small problems, FP32X3 and FP32: the multiply's producer warps decide their own
tiles' skip lists, no skip-map launch) against
the staged path (SPAMM_FLAG_STAGED: norm -> skip-map -> multiply kernels) on the same inputs.

Both take every decision with the same float64 predicate keep <=> !(nA*nB < tau) (PAPER.md:47,
Alg. 2 l.5) and multiply the kept k of a tile in ascending order with the same MMA
runs, so the skip maps must be IDENTICAL (lists, counts, row work, totals) and C bitwise equal;
the oracle parity of the fused path itself is covered by every small-shape test of
test_gpu_parity.py / test_gpu_dual.py (which run it by default)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import BAR, T, cbuf, dev, rounded

pytestmark = pytest.mark.gpu

STAGED = 4   # SPAMM_FLAG_STAGED

SHAPES = [(1024, 1024, 1024), (300, 257, 129), (40, 32, 32), (129, 1000, 384), (64, 256, 4096), (1, 1, 1),
          (256, 6400, 1152)]


@pytest.fixture(scope="module")
def sp():
    from paper_2103_13042_b200 import spamm
    return spamm


def _tau_at(nA, nB, q):
    if q == 0.0:
        return 0.0
    prods = np.unique(nA[:, :, None] * nB[None, :, :])
    if q >= 1.0:
        return float(prods[-1] * 2.0 + 1.0)
    i = min(int(q * (len(prods) - 1)), len(prods) - 2)
    return float(0.5 * (prods[i] + prods[i + 1]))


def _inputs(shape, prec, seed):
    M, N, K = shape
    A = rounded(synth.perturbed_decay_matrix(K, 0.97, seed=seed, m=M), prec)
    B = rounded(synth.perturbed_decay_matrix(N, 0.97, seed=seed + 1, m=K), prec)
    return A, B


def _lists(sp, plan):
    start, count, ent, order, GM, GN = sp.spamm_get_macro(plan.handle)
    start, count, ent, order = start.cpu().numpy(), count.cpu().numpy(), ent.cpu().numpy(), order.cpu().numpy()
    lists = [ent[s:s + c].tolist() for s, c in zip(start, count)]
    assert sorted(order.tolist()) == list(range(GM * GN)), "claim order is not a permutation"
    return lists


def _compare(sp, fused, staged, A_d, B_d, M, N):
    Cf, Cs = cbuf(M, N), cbuf(M, N)
    staged.run(A_d, B_d, Cs)
    fused.run(A_d, B_d, Cf)
    torch.cuda.synchronize()
    sf, ss = fused.stats(), staged.stats()
    assert sf["macro_i"] == ss["macro_i"] == 4
    assert sf["kept"] == ss["kept"] and sf["macro_entries"] == ss["macro_entries"]
    assert _lists(sp, fused) == _lists(sp, staged)
    Vf, rwf = sp.spamm_get_counts(fused.handle)
    Vs, rws = sp.spamm_get_counts(staged.handle)
    assert torch.equal(Vf, Vs) and torch.equal(rwf, rws)
    assert torch.equal(Cf, Cs), "fused and staged C differ"
    return Cf, sf


@pytest.mark.parametrize("prec", ["bf16", "fp16", "fp32x3", "fp32"])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("q", [0.0, 0.5, 0.9, 1.0])
def test_fused_equals_staged(sp, prec, shape, q):
    M, N, K = shape
    if prec in ("fp32x3", "fp32") and shape == (256, 6400, 1152) and q in (0.5, 0.9):
        pytest.skip("covered by q = 0 / 1 (oracle on the large shape is slow)")
    A, B = _inputs(shape, prec, 31)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    tau = _tau_at(nA, nB, q)
    fused = sp.Plan(M, N, K, tau, prec)
    staged = sp.Plan(M, N, K, tau, prec, flags=STAGED)
    A_d, B_d = dev(A, prec), dev(B, prec)
    C, st = _compare(sp, fused, staged, A_d, B_d, M, N)
    assert st["kept"] == oracle.count_kept(nA, nB, tau)
    if max(M, N, K) <= 1024:
        ref = oracle.spamm(A, B, tau, T, nA, nB)
        d = np.linalg.norm(C.cpu().numpy().astype(np.float64) - ref)
        s = np.linalg.norm(ref)
        assert (d == 0.0) if s == 0.0 else d / s <= BAR[prec]
    # a second run on the same plans (counters and totals are re-zeroed by the norm kernel)
    _compare(sp, fused, staged, A_d, B_d, M, N)


@pytest.mark.parametrize("lam", [0.9, 0.99])
@pytest.mark.parametrize("prec", ["bf16", "fp32x3", "fp32"])
def test_fused_configs0(sp, lam, prec):
    """configs[0]: N = 1024 exponential decay, tau = 1e-4 (Table 1's N)."""
    N = 1024
    A = rounded(synth.decay_matrix(N, "exp", lam), prec)
    fused = sp.Plan(N, N, N, 1e-4, prec)
    staged = sp.Plan(N, N, N, 1e-4, prec, flags=STAGED)
    A_d = dev(A, prec)
    _compare(sp, fused, staged, A_d, A_d, N, N)
    nA = oracle.tile_norms(A, T)
    assert fused.stats()["kept"] == oracle.count_kept(nA, nA, 1e-4)


def test_fused_chain_outputs(sp):
    """Chained outputs (alpha, C_low, nC) through the fused path equal the staged path's."""
    M, N, K = 300, 384, 257
    prec = "bf16"
    A, B = _inputs((M, N, K), prec, 41)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    tau = _tau_at(nA, nB, 0.4)
    out = []
    for flags in (0, STAGED):
        plan = sp.Plan(M, N, K, tau, prec, flags=flags)
        plan.set_scalars(0.5, 0.0)
        C = cbuf(M, N)
        Cl = torch.zeros((M, N), dtype=torch.bfloat16, device="cuda")
        sp.spamm_multiply_chain(plan.handle, dev(A, prec), dev(B, prec), C, Cl,
                                flags=sp.SPAMM_MUL_AUTO | sp.SPAMM_MUL_OUTPUT_NORMS)
        torch.cuda.synchronize()
        out.append((C.clone(), Cl.clone(), sp.spamm_get_output_norms(plan.handle).clone()))
        plan.close()
    for a, b in zip(out[0], out[1]):
        assert torch.equal(a, b)


def test_fused_graph_capture(sp):
    """The fused spamm_run (norm kernel -> fused multiply, PDL) replays from a CUDA graph."""
    N = 1024
    prec = "bf16"
    A = rounded(synth.decay_matrix(N, "exp", 0.9), prec)
    A_d = dev(A, prec)
    plan = sp.Plan(N, N, N, 1e-4, prec)
    ref = cbuf(N, N)
    plan.run(A_d, A_d, ref)
    torch.cuda.synchronize()
    C = cbuf(N, N)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        plan.run(A_d, A_d, C)   # warm-up on the capture stream
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        plan.run(A_d, A_d, C)
    for _ in range(3):
        C.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(C, ref)
    nA = oracle.tile_norms(A, T)
    assert plan.stats()["kept"] == oracle.count_kept(nA, nA, 1e-4)
