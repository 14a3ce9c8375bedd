"""GPU parity of the BF16/FP16 tensor-core multiplies -- multiply_dual.cu (256 x 256 macro-tiles,
two MMA issuers; forced with SPAMM_FLAG_LARGE_TILES on small shapes) and the 128 x 128 path of
small problems (multiply_x3.cu with one plane: "auto" on these shapes) -- on shapes that exercise
their schedules -- ragged edges, N % 32 != 0 (2-D B boxes, clipped stores), K much larger than M,
one-tile grids, banded products with mostly empty macro-tiles -- and their general epilogues
(alpha / beta, chained outputs, BF16/FP16-only output).  Bars: skip map bit-exact outside the 1e-6 tie band,
C within 2e-2 (north_star) and 1e-5 (FP32 accumulation of the same rounded inputs).
PAPER.md:127 (the product), 187 (FP32 accumulation), 47 (alpha, beta)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_parity import T, _check_skipmap, _dev, _rel_fro, _rounded, sp  # noqa: F401

pytestmark = pytest.mark.gpu

SHAPES = [(256, 256, 256), (300, 512, 129), (1000, 768, 600), (64, 256, 4096), (513, 1024, 300), (40, 32, 32),
          (300, 257, 129), (129, 1000, 384)]   # the last two: N % 32 != 0


TILES = {"large": 2, "auto": 0, "staged": 4}   # plan flags: SPAMM_FLAG_LARGE_TILES / automatic / SPAMM_FLAG_STAGED


def _tau_at(nA, nB, q):
    prods = np.unique(nA[:, :, None] * nB[None, :, :])
    i = min(int(q * (len(prods) - 1)), len(prods) - 2)
    return float(0.5 * (prods[i] + prods[i + 1]))


@pytest.mark.parametrize("tiles", ["large", "auto", "staged"])
@pytest.mark.parametrize("prec", ["bf16", "fp16"])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("q", [0.0, 0.5, 0.9])
def test_dual_parity(sp, prec, shape, q, tiles):
    M, N, K = shape
    A = _rounded(synth.perturbed_decay_matrix(K, 0.97, seed=11, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.97, seed=12, m=K), prec)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    tau = 0.0 if q == 0.0 else _tau_at(nA, nB, q)
    plan = sp.Plan(M, N, K, tau, prec, flags=TILES[tiles])
    assert plan.stats()["macro_i"] == (8 if tiles == "large" else 4)
    Ad, Bd = _dev(A, prec), _dev(B, prec)
    Cbuf = torch.full((M, -(-N // 4) * 4), float("nan"), dtype=torch.float32, device="cuda")
    C = Cbuf[:, :N]
    plan.run(Ad, Bd, C)
    torch.cuda.synchronize()
    assert plan.stats()["kept"] == oracle.count_kept(nA, nB, tau)
    _check_skipmap(sp, plan, nA, nB, tau)
    ref = oracle.spamm(A, B, tau, T, nA, nB)
    err = _rel_fro(C.cpu().numpy(), ref)
    assert err <= 2e-2 and err <= 1e-5, err
    # repeat on the same plan (self-resetting counters / tickets)
    C.fill_(float("nan"))
    plan.run(Ad, Bd, C)
    torch.cuda.synchronize()
    assert _rel_fro(C.cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("tiles", ["large", "auto"])
@pytest.mark.parametrize("prec", ["bf16", "fp16"])
def test_dual_decay_band(sp, prec, tiles):
    """A banded exponential-decay product (the bench workload's structure, N = 2048): most
    macro-tiles are empty (zero-filled by the epilogue warps), the band's are dense."""
    N = 2048
    A = _rounded(synth.decay_matrix(N, "exp", 0.99), prec)
    nA = oracle.tile_norms(A, T)
    tau = 1e-6
    plan = sp.Plan(N, N, N, tau, prec, flags=TILES[tiles])
    Ad = _dev(A, prec)
    C = torch.full((N, N), float("nan"), dtype=torch.float32, device="cuda")
    plan.run(Ad, Ad, C)
    torch.cuda.synchronize()
    assert plan.stats()["kept"] == oracle.count_kept(nA, nA, tau)
    err = _rel_fro(C.cpu().numpy(), oracle.spamm(A, A, tau, T, nA, nA))
    assert err <= 1e-5, err


@pytest.mark.parametrize("tiles", ["large", "auto"])
@pytest.mark.parametrize("alpha,beta", [(-0.5, 0.0), (2.0, 1.5), (0.0, 0.5)])
def test_dual_alpha_beta(sp, alpha, beta, tiles):
    M, N, K = 300, 512, 129
    prec = "bf16"
    A = _rounded(synth.perturbed_decay_matrix(K, 0.95, seed=91, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.95, seed=92, m=K), prec)
    C0 = synth.random_matrix(M, N, seed=93)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    tau = _tau_at(nA, nB, 0.7)
    plan = sp.Plan(M, N, K, tau, prec, flags=TILES[tiles])
    plan.set_scalars(alpha, beta)
    Cbuf = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    if beta != 0.0:
        Cbuf[:] = torch.from_numpy(C0).cuda()
    plan.run(_dev(A, prec), _dev(B, prec), Cbuf)
    torch.cuda.synchronize()
    ref = oracle.spamm_axpby(A, B, tau, T, alpha, beta, C0, nA, nB)
    assert _rel_fro(Cbuf.cpu().numpy(), ref) <= 5e-6


@pytest.mark.parametrize("tiles", ["large", "auto"])
def test_dual_chain(sp, tiles):
    """Chained outputs: C, C_low = RNE(C), nC = Eq. 2 of C_low."""
    M, N, K = 300, 512, 129
    prec = "bf16"
    A = _rounded(synth.perturbed_decay_matrix(K, 0.95, seed=101, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.95, seed=102, m=K), prec)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    tau = _tau_at(nA, nB, 0.4)
    plan = sp.Plan(M, N, K, tau, prec, flags=TILES[tiles])
    C = torch.empty((M, N), dtype=torch.float32, device="cuda")
    Cl = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    plan.multiply_chain(_dev(A, prec), _dev(B, prec), C, Cl, flags=sp.SPAMM_MUL_AUTO | sp.SPAMM_MUL_OUTPUT_NORMS)
    torch.cuda.synchronize()
    Cn = C.cpu().numpy()
    assert _rel_fro(Cn, oracle.spamm(A, B, tau, T, nA, nB)) <= 1e-5
    np.testing.assert_array_equal(Cl.cpu().float().numpy(), synth.round_to_bf16(Cn))
    np.testing.assert_allclose(plan.output_norms().cpu().numpy(), oracle.tile_norms(Cl.cpu().float().numpy(), T),
                               rtol=1e-12, atol=0)


@pytest.mark.parametrize("tiles", ["large", "auto"])
@pytest.mark.parametrize("prec", ["bf16", "fp16"])
@pytest.mark.parametrize("alpha", [1.0, -2.0])
def test_dual_low_precision_output_only(sp, prec, alpha, tiles):
    """SPAMM_MUL_LOW_ONLY: the result is written only as BF16/FP16 (RNE of the
    FP32 accumulator times alpha); no FP32 C is passed or written.  Equals rounding the oracle's
    product up to the FP32 accumulation (compared after rounding both: the bits may differ only
    where the FP32 value sits on a rounding boundary, so compare within one ulp of the type)."""
    M, N, K = 513, 1000, 300
    A = _rounded(synth.perturbed_decay_matrix(K, 0.95, seed=111, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.95, seed=112, m=K), prec)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    tau = _tau_at(nA, nB, 0.5)
    dt = torch.bfloat16 if prec == "bf16" else torch.float16
    plan = sp.Plan(M, N, K, tau, prec, flags=TILES[tiles])
    plan.set_scalars(alpha, 0.0)
    Cl = torch.full((M, -(-N // 8) * 8), float("nan"), dtype=dt, device="cuda")[:, :N]
    sp.spamm_multiply_chain(plan.handle, _dev(A, prec), _dev(B, prec), None, Cl,
                            flags=sp.SPAMM_MUL_AUTO | sp.SPAMM_MUL_OUTPUT_NORMS | sp.SPAMM_MUL_LOW_ONLY)
    torch.cuda.synchronize()
    got = Cl.cpu().float().numpy().astype(np.float64)
    ref = alpha * oracle.spamm(A, B, tau, T, nA, nB)
    ulp = 2.0 ** -7 if prec == "bf16" else 2.0 ** -10
    assert np.all(np.isfinite(got))
    assert np.all(np.abs(got - ref) <= ulp * np.abs(ref) + 1e-30 + 1e-6 * np.abs(ref).max())
    np.testing.assert_allclose(plan.output_norms().cpu().numpy(), oracle.tile_norms(got, T), rtol=1e-12, atol=0)


def test_dense_many_tiles_blocked_claims(sp):
    """tau = 0 on a 13000 x 13000 output (ragged, 51 x 51 = 2601 macro-tiles >= 16 per CTA: the
    blocked super-block claim order): every tile is claimed once and C = A B."""
    M = N = 13000
    K = 256
    A = synth.random_matrix(M, K, seed=121)
    B = synth.random_matrix(K, N, seed=122)
    Ab, Bb = synth.round_to_bf16(A), synth.round_to_bf16(B)
    plan = sp.Plan(M, N, K, 0.0, "bf16")
    C = torch.full((M, -(-N // 4) * 4), float("nan"), dtype=torch.float32, device="cuda")[:, :N]
    plan.run(_dev(Ab, "bf16"), _dev(Bb, "bf16"), C)
    torch.cuda.synchronize()
    ref = Ab.astype(np.float64) @ Bb.astype(np.float64)
    assert _rel_fro(C.cpu().numpy(), ref) <= 1e-6


@pytest.mark.parametrize("prec", ["bf16", "fp32", "fp32x3"])
def test_spamm_run_graph_capture(sp, prec):
    """spamm_run is stream-ordered with no host synchronisation, so a whole SpAMM (norms -> pyramid
    -> skip map -> multiply, PDL-chained) can be captured in a CUDA graph and replayed; replays
    pick up new operand values in the same buffers."""
    M, N, K = 1000, 768, 600
    A1 = _rounded(synth.perturbed_decay_matrix(K, 0.97, seed=171, m=M), prec)
    A2 = _rounded(synth.perturbed_decay_matrix(K, 0.97, seed=172, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.97, seed=173, m=K), prec)
    nA1, nA2, nB = oracle.tile_norms(A1, T), oracle.tile_norms(A2, T), oracle.tile_norms(B, T)
    tau = _tau_at(nA1, nB, 0.5)
    plan = sp.Plan(M, N, K, tau, prec)
    Ad, Bd = _dev(A1, prec), _dev(B, prec)
    C = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    plan.run(Ad, Bd, C)                       # warm-up outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        sp.spamm_run(plan.handle, Ad, Bd, C)
    bar = 1e-5
    for A, nA in ((A2, nA2), (A1, nA1), (A2, nA2)):
        Ad.copy_(torch.from_numpy(A).to(Ad.dtype))
        C.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert _rel_fro(C.cpu().numpy(), oracle.spamm(A, B, tau, T, nA, nB)) <= bar
        assert plan.stats()["kept"] == oracle.count_kept(nA, nB, tau)
