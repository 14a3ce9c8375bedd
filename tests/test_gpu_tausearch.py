"""GPU parity of the tau search (Sec. 3.5.2) and of
the count-only kept-triple kernel it evaluates, through the C ABI, against the oracle.

Pins: Table 1 (tests/golden/table1_tau.csv) -- the search on the device
norm maps reproduces every printed tau to one unit of its last printed digit, and agrees
with oracle.tau_search (same iteration count, same valid ratio, tau to 1e-12 relative).
"""
import csv
import os

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
T = 32
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2103_13042_b200 import build
    build.build()
    from paper_2103_13042_b200 import spamm
    return spamm


def _table1():
    with open(os.path.join(GOLD, "table1_tau.csv")) as f:
        return list(csv.DictReader(r for r in f if not r.startswith("#")))


def _dev(x, prec="fp32"):
    dt = {"fp32": torch.float32, "bf16": torch.bfloat16}[prec]
    m, n = x.shape
    buf = torch.zeros((m, -(-n // 8) * 8), dtype=dt, device="cuda")
    buf[:, :n] = torch.from_numpy(np.ascontiguousarray(x)).to(dt)
    return buf[:, :n]


@pytest.mark.parametrize("N", [1024, 2048, 4096, 8192])
def test_tau_search_reproduces_table1(sp, N):
    A = synth.decay_matrix(N, "alg", 0.1, c=0.1)
    nA = oracle.tile_norms(A, T)
    Ad = _dev(A)
    plan = sp.Plan(N, N, N, 0.0, "fp32")
    plan.norms(Ad, Ad)
    for r in _table1():
        if int(r["N"]) != N:
            continue
        target, printed = float(r["target"]), r["tau"]
        decimals = len(printed.split(".")[1])
        tau, vr, it = plan.tau_search(target, 0.01, 20)
        tau_o, vr_o, it_o = oracle.tau_search(nA, nA, target, iters=20, tol=0.01)
        assert it == it_o and vr == vr_o, (N, target, it, it_o, vr, vr_o)
        assert abs(tau - tau_o) <= 1e-12 * tau_o
        assert abs(tau - float(printed)) <= 1.01 * 10.0 ** (-decimals), (N, printed, tau)
        # the plan's tau is now the searched one: the skip map built from it keeps vr
        plan.build_skipmap()
        assert plan.stats()["kept"] == round(vr * (N // T) ** 3)


@pytest.mark.parametrize("shape", [(300, 257, 129), (1, 1, 1), (33, 1000, 64), (2100, 700, 1500)])
def test_count_kept_matches_oracle(sp, shape):
    M, N, K = shape
    A = synth.perturbed_decay_matrix(K, 0.95, seed=61, m=M)
    B = synth.perturbed_decay_matrix(N, 0.95, seed=62, m=K)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    plan = sp.Plan(M, N, K, 0.0, "fp32")
    plan.norms(_dev(A), _dev(B))
    nA_g, nBt_g = sp.spamm_get_norms(plan.handle)
    nA_g, nB_g = nA_g.cpu().numpy(), nBt_g.cpu().numpy().T
    # the count kernel is the keep predicate over the device maps: bit-exact against the
    # oracle predicate on those same maps, at exact product values too (">=")
    prods = np.unique(nA_g[:, :, None] * nB_g[None, :, :])
    taus = [0.0, float(prods[0]), float(prods[len(prods) // 2]), float(prods[-1]), float(prods[-1]) * 2]
    for tau in taus:
        assert plan.count_kept(tau) == oracle.count_kept(nA_g, nB_g, tau), tau
        # and against the oracle's own maps, up to the 1e-6 tie band
        assert abs(plan.count_kept(tau) - oracle.count_kept(nA, nB, tau)) <= oracle.band_count(nA, nB, tau)


def test_count_kept_nan_and_state(sp):
    N = 128
    A = synth.random_matrix(N, N, seed=63)
    A[5, 40] = np.nan
    B = synth.random_matrix(N, N, seed=64)
    plan = sp.Plan(N, N, N, 0.0, "fp32")
    with pytest.raises(sp.SpammError) as e:
        plan.count_kept(1.0)
    assert e.value.status == sp.SPAMM_E_STATE
    plan.norms(_dev(A), _dev(B))
    assert plan.count_kept(1e30) == N // T           # NaN products are kept (reading R2)
    with pytest.raises(sp.SpammError) as e:
        plan.tau_search(1.5)
    assert e.value.status == sp.SPAMM_E_INVALID


@pytest.mark.parametrize("bad", ["zero", "nan", "inf"])
def test_tau_search_degenerate_maps_fail_cleanly(sp, bad):
    """All-zero maps (a chain converged to 0) or non-finite norms: the Sec. 3.5.2 bracket
    [0, k*ave] is undefined; the search must return SPAMM_E_INVALID instead of looping."""
    N = 128
    A = np.zeros((N, N), np.float32) if bad == "zero" else synth.random_matrix(N, N, seed=65)
    if bad == "nan":
        A[3, 3] = np.nan
    if bad == "inf":
        A[3, 3] = np.inf
    plan = sp.Plan(N, N, N, 0.0, "fp32")
    plan.norms(_dev(A), _dev(A))
    with pytest.raises(sp.SpammError) as e:
        plan.tau_search(0.3)
    assert e.value.status == sp.SPAMM_E_INVALID
    assert plan.count_kept(0.0) == (N // T) ** 3        # the plan stays usable


def test_tau_search_heavy_tail_terminates(sp):
    """One huge tile among tiny ones: ave is far below the largest products, so the paper's
    k += 1 bracket widening would need ~1e6 count evaluations; the widening turns geometric
    after 64 steps and the search ends within max_iter bisection steps."""
    N = 256
    A = synth.random_matrix(N, N, seed=66, scale=1e-6)
    A[:32, :32] = 1e6
    plan = sp.Plan(N, N, N, 0.0, "fp32")
    Ad = _dev(A)
    plan.norms(Ad, Ad)
    # target 0: vr(k*ave) > 0 until k*ave passes the largest product (~512 ave)
    tau, vr, it = plan.tau_search(0.0, tol=1e-4, max_iter=40)
    assert np.isfinite(tau) and vr <= 1.0 / 512 and it <= 40
