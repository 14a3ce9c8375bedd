"""GPU parity on every BASELINE.json config and tau sweep the north_star names (round 2).

  configs[0]  N = 1024 exponential decay lam = 0.9 / 0.99 (and a signed A != B variant),
              tau = 1e-4, full oracle (skip map, C, per-tile error), FP32 / FP32X3 / BF16 / FP16;
  configs[1]  N = 8192, lam = 0.99, all nine tau 1e-10 .. 1e-2, every precision: kept count,
              skip lists of sampled tile rows, sampled C tiles;
  configs[2]  N = 16384 exponential decay lam = 0.99 (the north_star's single-GPU target), tau
              1e-10 .. 1e-2, every precision;
  configs[4]  N = 65536 with lam = 0.99 (the overhead-dominated variant), BF16 and FP32X3.
Bars: tests/gpu_helpers.py.  PAPER.md:45 (decay classes, Sec. 2.1), 127 (the product), 257.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import (BAR, GUARD, T, ToeplitzTiles, cbuf, check_norms, check_rows, check_tiles, dev,
                         rounded, sample_tiles, tile_max_rel, toeplitz_oracle_norms)

pytestmark = pytest.mark.gpu

PRECS = ["fp32", "fp32x3", "bf16", "fp16"]
TAU9 = [1e-10, 1e-9, 1e-8, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2]
TAU5 = [1e-10, 1e-8, 1e-6, 1e-4, 1e-2]


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2103_13042_b200 import build
    build.build()
    from paper_2103_13042_b200 import spamm
    return spamm


# ------------------------------------------------------------------ configs[0] ---
@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("case", ["exp0.9", "exp0.99", "signed"])
def test_config1_n1024_full_oracle(sp, prec, case):
    """N = 1024, tile 32, tau = 1e-4 (configs[0]): the whole skip map bit-exact outside the tie
    band, C vs the float64 oracle globally and per tile."""
    N, tau = 1024, 1e-4
    if case == "signed":   # A != B, signed, ties of the Toeplitz inputs broken
        A32 = synth.perturbed_decay_matrix(N, 0.95, seed=2103 + 1)
        B32 = synth.perturbed_decay_matrix(N, 0.95, seed=2103 + 11)
    else:
        A32 = B32 = synth.decay_matrix(N, "exp", float(case[3:]))
    A, B = rounded(A32, prec), rounded(B32, prec)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    Ad, Bd = dev(A, prec), (dev(B, prec) if case == "signed" else None)
    Bd = Ad if Bd is None else Bd
    C = cbuf(N, N)
    with sp.Plan(N, N, N, tau, prec) as plan:
        plan.norms(Ad, Bd)
        plan.build_skipmap()
        plan.multiply(Ad, Bd, C)
        torch.cuda.synchronize()
        check_norms(sp, plan, nA, nB)
        BD = N // T
        check_rows(sp, plan, nA, nB, tau, range(BD))       # every tile row: the full skip map
        st = plan.stats()
        band = oracle.band_count(nA, nB, tau)
        assert abs(st["kept"] - oracle.count_kept(nA, nB, tau)) <= band
        if prec in ("fp32", "fp32x3") and case != "signed":   # SURVEY.md 8(d) configs 1 (no band)
            assert st["kept"] == {"exp0.9": 1758, "exp0.99": 32362}[case]
    ref = oracle.spamm(A, B, tau, T, nA, nB)
    got = C.cpu().numpy()
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= BAR[prec] and err <= GUARD[prec], err
    absref = oracle.spamm(np.abs(A), np.abs(B), tau, T, nA, nB)
    assert tile_max_rel(got, ref, absref) <= GUARD[prec]


# ------------------------------------------------------------------ configs[1] ---
@pytest.fixture(scope="module")
def cfg2():
    return synth.decay_matrix(8192, "exp", 0.99)


@pytest.mark.parametrize("prec", PRECS)
def test_config2_n8192_all_tau(sp, cfg2, prec):
    """configs[1] at full size, every tau of the sweep (bench.py's second workload)."""
    N = 8192
    A = rounded(cfg2, prec)
    nA = oracle.tile_norms(A, T)
    BD = N // T
    Ad = dev(A, prec)
    C = cbuf(N, N)
    with sp.Plan(N, N, N, TAU9[0], prec) as plan:
        plan.norms(Ad, Ad)
        check_norms(sp, plan, nA, nA)
        for n, tau in enumerate(TAU9):
            plan.set_tau(tau)
            plan.build_skipmap()
            plan.multiply(Ad, Ad, C)
            torch.cuda.synchronize()
            band = oracle.band_count(nA, nA, tau)
            assert abs(plan.stats()["kept"] - oracle.count_kept(nA, nA, tau)) <= band, tau
            check_rows(sp, plan, nA, nA, tau, [0, 1, BD // 3, BD - 1])
            check_tiles(C, A, A, tau, nA, nA, sample_tiles(BD, BD, 70 + n, 10), GUARD[prec])


# ------------------------------------------------------------------ configs[2] ---
@pytest.fixture(scope="module")
def cfg3exp():
    return synth.decay_matrix(16384, "exp", 0.99)


@pytest.mark.parametrize("prec", PRECS)
def test_config3_n16384_exp_sweep(sp, cfg3exp, prec):
    """The north_star's single-GPU target: N = 16384 exponential decay (lam = 0.99), tau sweep."""
    N = 16384
    A = rounded(cfg3exp, prec)
    nA = oracle.tile_norms(A, T)
    BD = N // T
    Ad = dev(A, prec)
    C = cbuf(N, N)
    with sp.Plan(N, N, N, TAU5[0], prec) as plan:
        plan.norms(Ad, Ad)
        check_norms(sp, plan, nA, nA)
        for n, tau in enumerate(TAU5):
            plan.set_tau(tau)
            plan.build_skipmap()
            plan.multiply(Ad, Ad, C)
            torch.cuda.synchronize()
            band = oracle.band_count(nA, nA, tau)
            assert abs(plan.stats()["kept"] - oracle.count_kept(nA, nA, tau)) <= band, tau
            check_rows(sp, plan, nA, nA, tau, [0, BD // 2, BD - 1])
            check_tiles(C, A, A, tau, nA, nA, sample_tiles(BD, BD, 90 + n, 10), GUARD[prec])


# ------------------------------------------------------------------ configs[4] ---
@pytest.mark.parametrize("prec,tau", [("bf16", 1e-6), ("bf16", 1e-2), ("fp16", 1e-6), ("fp32x3", 1e-6)])
def test_config5_n65536_lam099(sp, prec, tau):
    """N = 65536 exponential decay lam = 0.99 (configs[4]'s overhead-dominated variant), A = B:
    full norm map and kept count, skip lists of sampled tile rows, sampled C tiles."""
    N, lam = 65536, 0.99
    table = rounded(synth.decay_table("exp", N, lam).astype(np.float32)[None, :], prec)[0]
    nA = toeplitz_oracle_norms(table, N)
    BD = N // T
    Ad = synth.toeplitz_device(table, N, {"bf16": torch.bfloat16, "fp16": torch.float16,
                                          "fp32x3": torch.float32}[prec])
    C = torch.empty((N, N), dtype=torch.float32, device="cuda")
    with sp.Plan(N, N, N, tau, prec) as plan:
        plan.run(Ad, Ad, C)
        torch.cuda.synchronize()
        check_norms(sp, plan, nA, nA)
        band = oracle.band_count(nA, nA, tau)
        assert abs(plan.stats()["kept"] - oracle.count_kept(nA, nA, tau)) <= band
        check_rows(sp, plan, nA, nA, tau, [0, BD // 2, BD - 1])
    del Ad
    At = ToeplitzTiles(table, N)
    check_tiles(C, At, At, tau, nA, nA, sample_tiles(BD, BD, 7, 12), GUARD[prec])
    del C
    torch.cuda.empty_cache()
