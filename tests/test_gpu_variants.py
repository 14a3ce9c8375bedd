"""GPU parity of every tensor-path kernel variant (SPAMM_UMMA_VARIANT, read at plan creation)
against the float64 oracle: 0 = 128x256 tiles, 2 CTAs/SM (default); 1 = same, 64-deep merged
k-steps; 2/4 = 1 CTA/SM split issuers; 5 (default) = 256x256 tiles, one CTA per SM, two MMA
issuers (multiply_dual.cu), with 1 or 2 k-steps per ring stage (SPAMM_DUAL_PACK).  Same bars as test_gpu_parity.py: skip map bit-exact outside
the 1e-6 tie band, C within 2e-2 (north_star) and 1e-5 (FP32 accumulation of exactly rounded
inputs) relative Frobenius error.  The variants only change the schedule, never the kept set."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_parity import T, _check_skipmap, _dev, _rel_fro, _rounded, sp  # noqa: F401

pytestmark = pytest.mark.gpu

# "5:1" = variant 5 with one k-step per ring stage (SPAMM_DUAL_PACK=1; default 2)
VARIANTS = os.environ.get("SPAMM_TEST_VARIANTS", "0,1,2,4,5,5:1").split(",")
SHAPES = [(256, 256, 256), (300, 512, 129), (1000, 768, 600), (64, 256, 4096), (513, 1024, 300), (40, 32, 32),
          (300, 257, 129), (129, 1000, 384)]   # the last two: N % 32 != 0 (2-D B boxes, clipped stores)


def _tau_at(nA, nB, q):
    prods = np.unique(nA[:, :, None] * nB[None, :, :])
    i = min(int(q * (len(prods) - 1)), len(prods) - 2)
    return float(0.5 * (prods[i] + prods[i + 1]))


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("q", [0.0, 0.5, 0.9])
def test_variant_parity(sp, monkeypatch, variant, shape, q):
    v, _, pack = variant.partition(":")
    monkeypatch.setenv("SPAMM_UMMA_VARIANT", v)
    monkeypatch.setenv("SPAMM_DUAL_PACK", pack or "2")
    M, N, K = shape
    prec = "bf16"
    A = _rounded(synth.perturbed_decay_matrix(K, 0.97, seed=11, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.97, seed=12, m=K), prec)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    tau = 0.0 if q == 0.0 else _tau_at(nA, nB, q)
    plan = sp.Plan(M, N, K, tau, prec)
    Ad, Bd = _dev(A, prec), _dev(B, prec)
    Cbuf = torch.full((M, -(-N // 4) * 4), float("nan"), dtype=torch.float32, device="cuda")
    C = Cbuf[:, :N]
    plan.run(Ad, Bd, C)
    torch.cuda.synchronize()
    assert plan.stats()["kept"] == oracle.count_kept(nA, nB, tau)
    _check_skipmap(sp, plan, nA, nB, tau)
    err = _rel_fro(C.cpu().numpy(), oracle.spamm(A, B, tau, T, nA, nB))
    assert err <= 2e-2 and err <= 1e-5, err
    # repeat on the same plan (self-resetting counters / tickets)
    C.fill_(float("nan"))
    plan.run(Ad, Bd, C)
    torch.cuda.synchronize()
    assert _rel_fro(C.cpu().numpy(), oracle.spamm(A, B, tau, T, nA, nB)) <= 1e-5


@pytest.mark.parametrize("prec", ["bf16", "fp16"])
def test_dual_decay_band(sp, monkeypatch, prec):
    """Variant 5 on a banded exponential-decay product (the bench workload's structure, N = 2048):
    most macro-tiles are empty (zero-filled by the epilogue warps), the band's are dense."""
    monkeypatch.setenv("SPAMM_UMMA_VARIANT", "5")
    N = 2048
    A = _rounded(synth.decay_matrix(N, "exp", 0.99), prec)
    nA = oracle.tile_norms(A, T)
    tau = 1e-6
    plan = sp.Plan(N, N, N, tau, prec)
    Ad = _dev(A, prec)
    C = torch.full((N, N), float("nan"), dtype=torch.float32, device="cuda")
    plan.run(Ad, Ad, C)
    torch.cuda.synchronize()
    assert plan.stats()["kept"] == oracle.count_kept(nA, nA, tau)
    err = _rel_fro(C.cpu().numpy(), oracle.spamm(A, A, tau, T, nA, nA))
    assert err <= 1e-5, err


@pytest.mark.parametrize("alpha,beta", [(-0.5, 0.0), (2.0, 1.5), (0.0, 0.5)])
def test_dual_alpha_beta(sp, monkeypatch, alpha, beta):
    monkeypatch.setenv("SPAMM_UMMA_VARIANT", "5")
    M, N, K = 300, 512, 129
    prec = "bf16"
    A = _rounded(synth.perturbed_decay_matrix(K, 0.95, seed=91, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.95, seed=92, m=K), prec)
    C0 = synth.random_matrix(M, N, seed=93)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    tau = _tau_at(nA, nB, 0.7)
    plan = sp.Plan(M, N, K, tau, prec)
    plan.set_scalars(alpha, beta)
    Cbuf = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    if beta != 0.0:
        Cbuf[:] = torch.from_numpy(C0).cuda()
    plan.run(_dev(A, prec), _dev(B, prec), Cbuf)
    torch.cuda.synchronize()
    ref = oracle.spamm_axpby(A, B, tau, T, alpha, beta, C0, nA, nB)
    assert _rel_fro(Cbuf.cpu().numpy(), ref) <= 5e-6


def test_dual_chain(sp, monkeypatch):
    """Chained outputs from the variant-5 epilogue: C, C_low = RNE(C), nC = Eq. 2 of C_low."""
    monkeypatch.setenv("SPAMM_UMMA_VARIANT", "5")
    M, N, K = 300, 512, 129
    prec = "bf16"
    A = _rounded(synth.perturbed_decay_matrix(K, 0.95, seed=101, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.95, seed=102, m=K), prec)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    tau = _tau_at(nA, nB, 0.4)
    plan = sp.Plan(M, N, K, tau, prec)
    C = torch.empty((M, N), dtype=torch.float32, device="cuda")
    Cl = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    plan.multiply_chain(_dev(A, prec), _dev(B, prec), C, Cl, flags=sp.SPAMM_MUL_AUTO | sp.SPAMM_MUL_OUTPUT_NORMS)
    torch.cuda.synchronize()
    Cn = C.cpu().numpy()
    assert _rel_fro(Cn, oracle.spamm(A, B, tau, T, nA, nB)) <= 1e-5
    np.testing.assert_array_equal(Cl.cpu().float().numpy(), synth.round_to_bf16(Cn))
    np.testing.assert_allclose(plan.output_norms().cpu().numpy(), oracle.tile_norms(Cl.cpu().float().numpy(), T),
                               rtol=1e-12, atol=0)


@pytest.mark.parametrize("n_split", [1, 10, 1000])
def test_dual_k_split(sp, monkeypatch, n_split):
    """Variant 5 with the LPT tail's last tiles split into k-halves (C = P1 + P2, the second half's
    epilogue adds onto the first's stores after a per-tile handshake); forced on a small grid."""
    monkeypatch.setenv("SPAMM_UMMA_VARIANT", "5")
    monkeypatch.setenv("SPAMM_DUAL_SPLIT", str(n_split))
    M, N, K = 1000, 1024, 1536
    prec = "bf16"
    A = _rounded(synth.perturbed_decay_matrix(K, 0.995, seed=21, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.995, seed=22, m=K), prec)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    tau = _tau_at(nA, nB, 0.3)
    plan = sp.Plan(M, N, K, tau, prec)
    Ad, Bd = _dev(A, prec), _dev(B, prec)
    ref = oracle.spamm(A, B, tau, T, nA, nB)
    for _ in range(3):   # repeated launches: the handshake counters reset themselves
        C = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
        plan.run(Ad, Bd, C)
        torch.cuda.synchronize()
        assert _rel_fro(C.cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("alpha,beta", [(1.0, 0.0), (2.0, 1.5)])
def test_dual_blocked_order(sp, monkeypatch, alpha, beta):
    """Variant 5 with the blocked (12 x 12 super-block) claim order forced (SPAMM_DUAL_ORDER=2;
    automatic when every CTA gets >= 16 tiles): empty tiles are zero-filled (beta = 0) or go
    through the pipeline (beta != 0)."""
    monkeypatch.setenv("SPAMM_UMMA_VARIANT", "5")
    monkeypatch.setenv("SPAMM_DUAL_ORDER", "2")
    M, N, K = 1000, 1024, 1536
    prec = "bf16"
    A = _rounded(synth.perturbed_decay_matrix(K, 0.99, seed=41, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.99, seed=42, m=K), prec)
    C0 = synth.random_matrix(M, N, seed=43)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    tau = _tau_at(nA, nB, 0.8)
    plan = sp.Plan(M, N, K, tau, prec)
    plan.set_scalars(alpha, beta)
    C = torch.from_numpy(C0).cuda() if beta != 0.0 else torch.full((M, N), float("nan"), device="cuda")
    plan.run(_dev(A, prec), _dev(B, prec), C)
    torch.cuda.synchronize()
    ref = oracle.spamm_axpby(A, B, tau, T, alpha, beta, C0, nA, nB)
    assert _rel_fro(C.cpu().numpy(), ref) <= 5e-6


def test_fp32x3_blocked_order(sp, monkeypatch):
    """FP32X3 multiply with the blocked claim order forced (SPAMM_X3_ORDER=2; automatic with >= 16
    tiles with k-steps per CTA): every tile, with or without k-steps, is claimed exactly once."""
    monkeypatch.setenv("SPAMM_X3_ORDER", "2")
    M, N, K = 1000, 1000, 1536
    A = synth.perturbed_decay_matrix(K, 0.99, seed=51, m=M)
    B = synth.perturbed_decay_matrix(N, 0.99, seed=52, m=K)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    tau = _tau_at(nA, nB, 0.8)
    plan = sp.Plan(M, N, K, tau, "fp32x3")
    C = torch.full((M, N), float("nan"), device="cuda")
    plan.run(_dev(A, "fp32x3"), _dev(B, "fp32x3"), C)
    torch.cuda.synchronize()
    assert _rel_fro(C.cpu().numpy(), oracle.spamm(A, B, tau, T, nA, nB)) <= 1e-5
