"""GPU parity: the CUDA path through the C ABI vs the float64 oracle, same seeded inputs.

Bars (BASELINE.json north_star): skip map bit-exact except triples whose norm product
lies within 1e-6 relative of tau (counted, reported); C within 1e-5 relative
Frobenius error for the FP32 path and 2e-2 for BF16/FP16.  Norm maps are float64 on
both sides and agree to ~1e-15 relative (different summation order); we require 1e-12.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import tile_max_rel

pytestmark = pytest.mark.gpu

T = 32
BAND = 1e-6


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2103_13042_b200 import build
    build.build()
    from paper_2103_13042_b200 import spamm
    return spamm


def _dev(x: np.ndarray, prec: str, ld_mult: int = 8):
    """Device copy of float32 host array x in the path's dtype, with a padded ld."""
    m, n = x.shape
    ld = -(-n // ld_mult) * ld_mult
    dt = {"fp32": torch.float32, "fp32x3": torch.float32, "bf16": torch.bfloat16, "fp16": torch.float16}[prec]
    buf = torch.zeros((m, ld), dtype=dt, device="cuda")
    buf[:, :n] = torch.from_numpy(np.ascontiguousarray(x)).to(dt)
    return buf[:, :n]


def _rounded(x: np.ndarray, prec: str) -> np.ndarray:
    if prec == "bf16":
        return synth.round_to_bf16(x)
    if prec == "fp16":
        return synth.round_to_fp16(x)
    return x


def _rel_fro(C, ref):
    ref = np.asarray(ref, dtype=np.float64)
    d = np.asarray(C, dtype=np.float64) - ref
    nr = math.sqrt(float(np.sum(ref * ref)))
    return math.sqrt(float(np.sum(d * d))) / (nr if nr > 0 else 1.0)


def _run(sp, A32, B32, tau, prec, flags=0):
    M, K = A32.shape
    N = B32.shape[1]
    plan = sp.Plan(M, N, K, tau, prec, flags=flags)
    A, B = _dev(A32, prec), _dev(B32, prec)
    Cbuf = torch.full((M, -(-N // 4) * 4), float("nan"), dtype=torch.float32, device="cuda")
    C = Cbuf[:, :N]
    plan.norms(A, B)
    plan.build_skipmap()
    plan.multiply(A, B, C)
    torch.cuda.synchronize()
    return plan, C.cpu().numpy()


def _gpu_keep(sp, plan, BM, BK, BN):
    start, kidx = sp.spamm_get_skipmap(plan.handle)
    V = sp.spamm_get_counts(plan.handle)[0].cpu().numpy().reshape(-1)
    start, kidx = start.cpu().numpy(), kidx.cpu().numpy()
    keep = np.zeros((BM, BK, BN), dtype=bool)
    for t in range(BM * BN):
        ks = kidx[start[t]:start[t] + V[t]]
        assert np.all(np.diff(ks) > 0), "k lists must be strictly ascending"
        keep[t // BN, ks, t % BN] = True
    return keep


def _check_skipmap(sp, plan, nA, nB, tau):
    BM, BK = nA.shape
    BN = nB.shape[1]
    keep_o = oracle.keep_mask(nA, nB, tau)
    keep_g = _gpu_keep(sp, plan, BM, BK, BN)
    p = nA[:, :, None] * nB[None, :, :]
    band = np.abs(p - tau) <= BAND * tau
    diff = keep_o != keep_g
    assert not np.any(diff & ~band), f"{int(np.sum(diff & ~band))} skip decisions differ outside the tie band"
    V, rw = sp.spamm_get_counts(plan.handle)
    V, rw = V.cpu().numpy(), rw.cpu().numpy()
    np.testing.assert_array_equal(V, keep_g.sum(axis=1))
    np.testing.assert_array_equal(rw, keep_g.sum(axis=(1, 2)))
    return int(np.sum(diff)), int(np.sum(band))


SHAPES = [(256, 256, 256), (100, 70, 45), (300, 257, 129), (129, 520, 384), (1, 1, 1), (33, 1000, 64)]


@pytest.mark.parametrize("prec", ["fp32", "bf16", "fp16"])
@pytest.mark.parametrize("shape", SHAPES)
def test_norms_match_oracle(sp, prec, shape):
    M, N, K = shape
    A = _rounded(synth.perturbed_decay_matrix(K, 0.97, seed=1, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.97, seed=2, m=K), prec)
    plan = sp.Plan(M, N, K, 0.0, prec)
    plan.norms(_dev(A, prec), _dev(B, prec))
    nA_g, nBt_g = sp.spamm_get_norms(plan.handle)
    np.testing.assert_allclose(nA_g.cpu().numpy(), oracle.tile_norms(A, T), rtol=1e-12, atol=0)
    np.testing.assert_allclose(nBt_g.cpu().numpy().T, oracle.tile_norms(B, T), rtol=1e-12, atol=0)


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_norms_toeplitz_bit_identical(sp, prec):
    """Equal tiles (same block diagonal of a Toeplitz matrix) get bit-identical norms."""
    N = 1024
    A = _rounded(synth.decay_matrix(N, "exp", 0.99), prec)
    plan = sp.Plan(N, N, N, 0.0, prec)
    Ad = _dev(A, prec)
    plan.norms(Ad, Ad)
    nA = sp.spamm_get_norms(plan.handle)[0].cpu().numpy()
    BD = N // T
    for d in range(-BD + 1, BD):
        diag = np.diagonal(nA, offset=d)
        assert np.all(diag == diag[0]), d


@pytest.mark.parametrize("prec", ["fp32", "bf16", "fp16", "fp32x3"])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("q", [0.0, 0.3, 0.7, 1.01])
def test_spamm_parity_ragged(sp, prec, shape, q):
    """Skip map bit-exact + C vs float64 oracle, ragged shapes, tau at product quantiles."""
    M, N, K = shape
    A = _rounded(synth.perturbed_decay_matrix(K, 0.95, seed=11, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.95, seed=12, m=K), prec)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    prods = np.sort((nA[:, :, None] * nB[None, :, :]).ravel())
    tau = 0.0 if q == 0.0 else (float(prods[-1]) * 2 if q > 1 else float(prods[int(q * (len(prods) - 1))]) * (1 + 1e-9))
    plan, C = _run(sp, A, B, tau, prec)
    _check_skipmap(sp, plan, nA, nB, tau)
    ref = oracle.spamm(A, B, tau, T, nA, nB)
    assert C.shape == ref.shape
    if q > 1:
        assert np.all(C == 0.0)
        return
    err = _rel_fro(C, ref)
    bar = 1e-5 if prec in ("fp32", "fp32x3") else 2e-2
    assert err <= bar, err
    # tighter regression guards: FP32 accumulation of exactly-representable products (fp32,
    # bf16/fp16 with the same rounded inputs on both sides), FP32-level split products (fp32x3)
    assert err <= {"fp32": 2e-6, "fp32x3": 5e-6}.get(prec, 1e-5), err
    # per C tile, relative to the same tile of SpAMM(|A|, |B|) (same keep set): a single wrong
    # tile cannot hide inside the global norm
    absref = oracle.spamm(np.abs(A), np.abs(B), tau, T, nA, nB)
    assert tile_max_rel(C, ref, absref) <= {"fp32": 2e-6, "fp32x3": 5e-6}.get(prec, 1e-5)


def test_macro_lists_match_oracle(sp):
    M = N = K = 520
    for prec in ("fp32", "bf16"):
        A = _rounded(synth.perturbed_decay_matrix(K, 0.95, seed=21, m=M), prec)
        B = _rounded(synth.perturbed_decay_matrix(N, 0.95, seed=22, m=K), prec)
        nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
        prods = np.unique(nA[:, :, None] * nB[None, :, :])
        mid = len(prods) // 2
        tau = float(0.5 * (prods[mid] + prods[mid + 1]))   # in a gap: no product in the tie band
        plan, _ = _run(sp, A, B, tau, prec)
        st = plan.stats()
        MI, MJ = st["macro_i"], st["macro_j"]
        start, count, ent, order, GM, GN = sp.spamm_get_macro(plan.handle)
        start, count = start.cpu().numpy(), count.cpu().numpy()
        ent = ent.cpu().numpy().astype(np.uint64)
        ref = oracle.macro_lists(nA, nB, tau, MI, MJ)
        np.testing.assert_array_equal(count, np.diff(ref["ptr"]))
        for t in range(GM * GN):
            np.testing.assert_array_equal(ent[start[t]:start[t] + count[t]],
                                          ref["entries"][ref["ptr"][t]:ref["ptr"][t + 1]])
        o = order.cpu().numpy()
        assert sorted(o.tolist()) == list(range(GM * GN))
        lens = count[o]
        assert np.all(np.diff(lens) <= 0), "LPT order must be descending in work"


@pytest.mark.parametrize("prec", ["fp32", "bf16", "fp32x3"])
def test_tau_zero_is_dense(sp, prec):
    N = 384
    A = _rounded(synth.random_matrix(N, N, seed=5), prec)
    B = _rounded(synth.random_matrix(N, N, seed=6), prec)
    plan, C = _run(sp, A, B, 0.0, prec)
    st = plan.stats()
    assert st["kept"] == (N // T) ** 3 and st["valid_ratio"] == 1.0
    err = _rel_fro(C, oracle.dense_product(A, B))
    assert err <= {"fp32": 1e-6, "fp32x3": 2e-6}.get(prec, 1e-5), err


def test_nan_propagates_like_gemm(sp):
    N = 128
    A = synth.random_matrix(N, N, seed=7)
    A[5, 40] = np.nan
    B = synth.random_matrix(N, N, seed=8)
    plan, C = _run(sp, A, B, 1e30, "fp32")
    # only pairs (i=0, k=1, j) have a NaN norm product -> kept; all others skipped
    assert np.all(np.isnan(C[5, :]))
    assert np.all(C[32:, :] == 0.0)
    st = plan.stats()
    assert st["kept"] == N // T


def test_table1_counts_n2048(sp):
    """The paper's dataset at Table 1's tau, N=2048:
    GPU kept counts = oracle counts (no triple lies in the 1e-6 band there)."""
    N = 2048
    A = synth.decay_matrix(N, "alg", 0.1, c=0.1)
    nA = oracle.tile_norms(A, T)
    taus = [1.310666, 1.330525, 1.360312, 1.40003, 1.449676, 1.548969]
    plan = sp.Plan(N, N, N, taus[0], "fp32")
    Ad = _dev(A, "fp32")
    plan.norms(Ad, Ad)
    for tau in taus:
        plan.set_tau(tau)
        plan.build_skipmap()
        diff, band = _check_skipmap(sp, plan, nA, nA, tau)
        assert diff == 0 and band == 0
        assert plan.stats()["kept"] == oracle.count_kept(nA, nA, tau)


def test_table3_error_n1024_gpu(sp):
    """End to end on the GPU (FP32): ||E||_F at the Table 3 valid ratios."""
    N = 1024
    A = synth.decay_matrix(N, "alg", 0.1, c=0.1)
    AB = oracle.dense_product(A, A)
    for tau, printed in ((1.4500655430308595, 996), (1.6619009145139256, 1302), (1.820188128117199, 1387)):
        _, C = _run(sp, A, A, tau, "fp32")
        err = math.sqrt(float(np.sum((AB - C.astype(np.float64)) ** 2)))
        assert abs(err - printed) < 1.0, (tau, err)


def test_errors_and_state(sp):
    plan = sp.Plan(64, 64, 64, 1.0, "fp32")
    A = torch.zeros((64, 64), device="cuda")
    C = torch.zeros((64, 64), device="cuda")
    with pytest.raises(sp.SpammError) as e:
        plan.multiply(A, A, C)
    assert e.value.status == sp.SPAMM_E_STATE
    with pytest.raises(sp.SpammError) as e:
        sp.spamm_norms(plan.handle, torch.zeros((64, 64)), A)     # host pointer through the raw ABI
    assert e.value.status == sp.SPAMM_E_INVALID
    with pytest.raises(ValueError):                               # the Plan wrapper checks dtype / shape
        plan.norms(torch.zeros((64, 64), device="cuda", dtype=torch.bfloat16), A)
    with pytest.raises(ValueError):
        plan.norms(torch.zeros((64, 32), device="cuda"), A)
    with pytest.raises(sp.SpammError) as e:
        sp.Plan(64, 64, 64, 1.0, "fp32", tile=64)
    assert e.value.status == sp.SPAMM_E_UNSUPPORTED


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_mgpu_single_rank_equals_single_gpu(sp, prec):
    N = 640
    A = _rounded(synth.perturbed_decay_matrix(N, 0.95, seed=31), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.95, seed=32), prec)
    tau = 0.05
    _, C1 = _run(sp, A, B, tau, prec)
    plan = sp.Plan(N, N, N, tau, prec)
    Ad, Bd = _dev(A, prec), _dev(B, prec)
    C = torch.zeros((N, N), device="cuda")
    sp.spamm_multiply_mgpu(plan.handle, None, 0, 1, Ad, Bd, C, 0)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(C.cpu().numpy(), C1)
    assert sp.spamm_get_partition(plan.handle, 1) == [0, N // T]


@pytest.mark.parametrize("prec", ["fp32", "bf16", "fp32x3"])
def test_full_size_bench_config_sampled(sp, prec):
    """configs[1] at full size (N=8192, exp. decay lam=0.99, tau=1e-6) in the bench launch
    configuration: exact kept count vs oracle, sampled C tiles vs oracle tiles."""
    N, lam, tau = 8192, 0.99, 1e-6
    A32 = _rounded(synth.decay_matrix(N, "exp", lam), prec)
    nA = oracle.tile_norms(A32, T)
    plan = sp.Plan(N, N, N, tau, prec)
    Ad = _dev(A32, prec)
    C = torch.empty((N, N), device="cuda")
    plan.run(Ad, Ad, C)
    torch.cuda.synchronize()
    st = plan.stats()
    band = oracle.band_count(nA, nA, tau)
    assert abs(st["kept"] - oracle.count_kept(nA, nA, tau)) <= band
    rng = np.random.default_rng(0)
    BD = N // T
    tiles = [(int(i), int(j)) for i, j in rng.integers(0, BD, size=(24, 2))]
    tiles += [(d, d) for d in range(0, BD, 37)] + [(0, 1), (BD - 1, BD - 2), (BD - 1, BD - 1)]
    Cn = C.cpu().numpy()
    for i, j in tiles:
        ref = oracle.spamm_tile(A32, A32, tau, T, i, j, nA, nA)
        got = Cn[i * T:(i + 1) * T, j * T:(j + 1) * T]
        nr = np.linalg.norm(ref)
        if nr == 0:
            assert np.all(got == 0)
        else:
            assert np.linalg.norm(got - ref) / nr <= (1e-5 if prec in ("fp32", "fp32x3") else 2e-2), (i, j)


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("N", [256, 1000])
def test_aliased_a_equals_b_norms(sp, prec, N):
    """A and B the same buffer (C = A*A): the norm kernel reads it once and writes both maps;
    they must be bit-identical to normalising a separate copy as B."""
    A = _rounded(synth.perturbed_decay_matrix(N, 0.95, seed=51), prec)
    Ad = _dev(A, prec)
    Bd = Ad.clone()
    p1 = sp.Plan(N, N, N, 0.0, prec)
    p1.norms(Ad, Ad)
    p2 = sp.Plan(N, N, N, 0.0, prec)
    p2.norms(Ad, Bd)
    a1, bt1 = sp.spamm_get_norms(p1.handle)
    a2, bt2 = sp.spamm_get_norms(p2.handle)
    assert torch.equal(a1, a2) and torch.equal(bt1, bt2)
    assert torch.equal(bt1, a1.T)
    np.testing.assert_allclose(a1.cpu().numpy(), oracle.tile_norms(A, T), rtol=1e-12, atol=0)


def test_bf16_norms_special_values(sp):
    """BF16 norms with subnormal, zero, Inf and NaN entries (the integer bf16->f64 fast path
    must hand these to the exact conversion) vs the oracle."""
    N = 256
    A = synth.round_to_bf16(synth.random_matrix(N, N, seed=71))
    A[3, 5] = np.float32(1e-40)      # bf16 subnormal (rounds to a subnormal bf16)
    A[40, 70] = np.float32(-3e-39)
    A[100, 200] = np.inf
    A[200, 10] = np.nan
    A[0:32, 32:64] = 0.0
    A = synth.round_to_bf16(A)
    plan = sp.Plan(N, N, N, 0.0, "bf16")
    Bd = _dev(np.ones((N, N), np.float32), "bf16")
    plan.norms(_dev(A, "bf16"), Bd)
    got = sp.spamm_get_norms(plan.handle)[0].cpu().numpy()
    np.testing.assert_allclose(got, oracle.tile_norms(A, T), rtol=1e-12, atol=0, equal_nan=True)


@pytest.mark.parametrize("prec", ["fp32", "bf16", "fp32x3"])
@pytest.mark.parametrize("alpha,beta", [(1.0, 0.0), (-0.5, 0.0), (2.0, 1.5), (1.0, -1.0), (0.0, 0.5)])
def test_alpha_beta_update(sp, prec, alpha, beta):
    """C = alpha*SpAMM(A, B) + beta*C vs oracle.spamm_axpby; beta = 0 must not
    read C (a NaN-filled C stays out of the result)."""
    M, N, K = 300, 257, 129
    A = _rounded(synth.perturbed_decay_matrix(K, 0.95, seed=91, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.95, seed=92, m=K), prec)
    C0 = synth.random_matrix(M, N, seed=93)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    prods = np.unique(nA[:, :, None] * nB[None, :, :])
    tau = float(0.5 * (prods[len(prods) // 2] + prods[len(prods) // 2 + 1]))
    plan = sp.Plan(M, N, K, tau, prec)
    plan.set_scalars(alpha, beta)
    Cbuf = torch.full((M, -(-N // 4) * 4), float("nan"), dtype=torch.float32, device="cuda")
    if beta != 0.0:
        Cbuf[:, :N] = torch.from_numpy(C0).cuda()
    plan.run(_dev(A, prec), _dev(B, prec), Cbuf[:, :N])
    torch.cuda.synchronize()
    got = Cbuf[:, :N].cpu().numpy()
    ref = oracle.spamm_axpby(A, B, tau, T, alpha, beta, C0, nA, nB)
    err = _rel_fro(got, ref)
    assert err <= (1e-5 if prec != "bf16" else 2e-2), err
    assert err <= 5e-6, err
    with pytest.raises(sp.SpammError):
        plan.set_scalars(float("nan"), 0.0)


# ------------------------------------------------------------ chained SpAMM (f3) ---
@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_chain_output_norms_and_low_copy(sp, prec):
    """spamm_multiply_chain: C as spamm_multiply; C_low = RNE(C) to bf16; nC = tile norms (Eq. 2)
    of the stored values (C_low's for BF16 plans, reading R4)."""
    M, N, K = 300, 257, 129
    A = _rounded(synth.perturbed_decay_matrix(K, 0.95, seed=101, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.95, seed=102, m=K), prec)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    prods = np.unique(nA[:, :, None] * nB[None, :, :])
    tau = float(0.5 * (prods[len(prods) // 3] + prods[len(prods) // 3 + 1]))
    plan = sp.Plan(M, N, K, tau, prec)
    Ad, Bd = _dev(A, prec), _dev(B, prec)
    C = torch.empty((M, -(-N // 4) * 4), dtype=torch.float32, device="cuda")[:, :N]
    Cl = torch.empty((M, -(-N // 8) * 8), dtype=torch.bfloat16, device="cuda")[:, :N] if prec == "bf16" else None
    plan.multiply_chain(Ad, Bd, C, Cl, flags=sp.SPAMM_MUL_AUTO | sp.SPAMM_MUL_OUTPUT_NORMS)
    torch.cuda.synchronize()
    Cn = C.cpu().numpy()
    assert _rel_fro(Cn, oracle.spamm(A, B, tau, T, nA, nB)) <= (2e-6 if prec == "fp32" else 1e-5)
    stored = Cn
    if prec == "bf16":
        np.testing.assert_array_equal(Cl.cpu().float().numpy(), synth.round_to_bf16(Cn))
        stored = Cl.cpu().float().numpy()
    np.testing.assert_allclose(plan.output_norms().cpu().numpy(), oracle.tile_norms(stored, T), rtol=1e-12, atol=0)


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_chain_matrix_square_twice(sp, prec):
    """X -> X^2 -> X^4 by repeated SpAMM squaring, the second step's norm maps taken from the
    first step's epilogue (spamm_set_norms), never from re-reading X^2.  Each step vs the
    oracle on that step's actual input: skip map outside the tie band, C within the bar."""
    N = 520
    X = _rounded(synth.perturbed_decay_matrix(N, 0.9, seed=103), prec)
    n1 = oracle.tile_norms(X, T)
    tau = float(np.quantile(n1[:, :, None] * n1[None, :, :], 0.6))
    dt = torch.float32 if prec == "fp32" else torch.bfloat16
    p1 = sp.Plan(N, N, N, tau, prec)
    Xd = _dev(X, prec)
    X2 = torch.empty((N, N), dtype=torch.float32, device="cuda")
    X2l = torch.empty((N, N), dtype=dt, device="cuda") if prec == "bf16" else None
    p1.multiply_chain(Xd, Xd, X2, X2l, flags=sp.SPAMM_MUL_AUTO | sp.SPAMM_MUL_OUTPUT_NORMS)
    nC = p1.output_norms()
    X2in = X2 if prec == "fp32" else X2l
    p2 = sp.Plan(N, N, N, tau * 1e-2, prec)
    p2.set_norms(nC, nC)
    p2.build_skipmap()
    X4 = torch.empty((N, N), dtype=torch.float32, device="cuda")
    p2.multiply(X2in, X2in, X4)
    torch.cuda.synchronize()
    X2h = X2in.cpu().float().numpy()
    n2 = oracle.tile_norms(X2h, T)
    np.testing.assert_allclose(nC.cpu().numpy(), n2, rtol=1e-12, atol=0)
    diff, _ = _check_skipmap(sp, p2, n2, n2, tau * 1e-2)
    err = _rel_fro(X4.cpu().numpy(), oracle.spamm(X2h, X2h, tau * 1e-2, T, n2, n2))
    assert err <= (2e-6 if prec == "fp32" else 1e-5), err
    with pytest.raises(sp.SpammError) as e:
        sp.Plan(N, N, N, tau, "fp32x3").set_norms(nC, nC)
    assert e.value.status == sp.SPAMM_E_UNSUPPORTED
