"""The multi-GPU path (Sec. 3.4, Alg. 4; load balance Sec. 3.5.1,
PAPER.md:230-234) emulated on one GPU through spamm_multiply_mgpu_local: the same three phases
and kernels as spamm_multiply_mgpu, with the NCCL collectives replaced by device copies between
the ranks' plans.  The survey's P4 invariant:
  * each rank's C rows are BITWISE the single-GPU C rows (every C tile is computed by the same
    per-tile instruction sequence, whichever rank or CTA runs it), rows outside the rank's range
    are untouched;
  * the union of the ranks' skip maps is the single-GPU skip map;
  * the device cut equals spamm_partition_rows on the single-GPU row work summed per macro row;
  * with GATHER_C every rank ends with the whole single-GPU C.
"""
import numpy as np
import pytest
import torch

import synth
from test_gpu_parity import T, _dev, _rounded, sp  # noqa: F401

pytestmark = pytest.mark.gpu


def _single(sp, A, B, tau, prec, M, N, K):
    plan = sp.Plan(M, N, K, tau, prec)
    C = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    plan.run(A, B, C)
    torch.cuda.synchronize()
    return plan, C.cpu().numpy()


def _leaf_lists(sp, plan, rows, BN):
    start, kidx = sp.spamm_get_skipmap(plan.handle)
    V = sp.spamm_get_counts(plan.handle)[0].cpu().numpy()
    start, kidx = start.cpu().numpy(), kidx.cpu().numpy()
    return {(i, j): tuple(kidx[start[i * BN + j]:start[i * BN + j] + V[i, j]]) for i in rows for j in range(BN)}


@pytest.mark.parametrize("prec", ["fp32", "bf16", "fp32x3", "bf16-small"])
@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_p4_ranks_equal_single_gpu(sp, prec, nranks):
    # several macro rows per rank, ragged edge; "bf16-small": the 128 x 128 BF16 path (tiles fit one wave)
    M = N = K = {"bf16": 4100, "bf16-small": 1000}.get(prec, 2080)
    prec = "bf16" if prec == "bf16-small" else prec
    lam = 0.995
    A = _rounded(synth.perturbed_decay_matrix(K, lam, seed=131, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, lam, seed=132, m=K), prec)
    Ad, Bd = _dev(A, prec), _dev(B, prec)
    tau = 1e-3
    single, C1 = _single(sp, Ad, Bd, tau, prec, M, N, K)
    st1 = single.stats()
    plans = [sp.Plan(M, N, K, tau, prec) for _ in range(nranks)]
    Cs = [torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda") for _ in range(nranks)]
    sp.spamm_multiply_mgpu_local([p.handle for p in plans], Ad, Bd, Cs, 0)
    torch.cuda.synchronize()
    cut = sp.spamm_get_partition(plans[0].handle, nranks)          # tile rows
    for p in plans[1:]:
        assert sp.spamm_get_partition(p.handle, nranks) == cut
    # the device cut = the host rule on the single-GPU row work grouped by macro rows
    MI = st1["macro_i"]
    rw = sp.spamm_get_counts(single.handle)[1].cpu().numpy()
    mw = [int(rw[g * MI:(g + 1) * MI].sum()) for g in range(-(-len(rw) // MI))]
    host = sp.spamm_partition_rows(mw, nranks)
    assert [min(c * MI, st1["BM"]) for c in host] == cut
    BN = st1["BN"]
    kept = 0
    for q in range(nranks):
        r0, r1 = min(cut[q] * T, M), min(cut[q + 1] * T, M)
        Cq = Cs[q].cpu().numpy()
        np.testing.assert_array_equal(Cq[r0:r1], C1[r0:r1])       # bitwise
        assert np.all(np.isnan(Cq[:r0])) and np.all(np.isnan(Cq[r1:]))
        st = plans[q].stats()
        assert (st["row_begin"], st["row_end"]) == (cut[q], cut[q + 1])
        kept += st["kept"]
        rows = range(cut[q], cut[q + 1])
        assert _leaf_lists(sp, plans[q], rows, BN) == _leaf_lists(sp, single, rows, BN)
    assert kept == st1["kept"]


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
def test_p4_gather_c(sp, prec):
    M, N, K = 3000, 2100, 1900
    nranks = 4
    A = _rounded(synth.perturbed_decay_matrix(K, 0.99, seed=141, m=M), prec)
    B = _rounded(synth.perturbed_decay_matrix(N, 0.99, seed=142, m=K), prec)
    Ad, Bd = _dev(A, prec), _dev(B, prec)
    ldc = -(-N // 4) * 4
    _, C1 = _single(sp, Ad, Bd, 1e-2, prec, M, N, K)
    plans = [sp.Plan(M, N, K, 1e-2, prec) for _ in range(nranks)]
    Cb = [torch.full((M, ldc), float("nan"), dtype=torch.float32, device="cuda") for _ in range(nranks)]
    sp.spamm_multiply_mgpu_local([p.handle for p in plans], Ad, Bd, [c[:, :N] for c in Cb], sp.SPAMM_MGPU_GATHER_C)
    torch.cuda.synchronize()
    for c in Cb:
        np.testing.assert_array_equal(c[:, :N].cpu().numpy(), C1)


def test_p4_repeated_steps_and_single_rank(sp):
    """Steady state (the bench loop): repeated multi-rank steps on the same plans stay bitwise
    equal; one rank through spamm_multiply_mgpu (no communicator) equals spamm_run."""
    M = N = K = 2048
    prec = "bf16"
    A = _rounded(synth.perturbed_decay_matrix(K, 0.995, seed=151, m=M), prec)
    Ad = _dev(A, prec)
    _, C1 = _single(sp, Ad, Ad, 1e-4, prec, M, N, K)
    plans = [sp.Plan(M, N, K, 1e-4, prec) for _ in range(2)]
    Cs = [torch.zeros((M, N), dtype=torch.float32, device="cuda") for _ in range(2)]
    for _ in range(3):
        sp.spamm_multiply_mgpu_local([p.handle for p in plans], Ad, Ad, Cs, sp.SPAMM_MGPU_GATHER_C)
        torch.cuda.synchronize()
        for c in Cs:
            np.testing.assert_array_equal(c.cpu().numpy(), C1)
    plan = sp.Plan(M, N, K, 1e-4, prec)
    C = torch.zeros((M, N), device="cuda")
    sp.spamm_multiply_mgpu(plan.handle, None, 0, 1, Ad, Ad, C, 0)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(C.cpu().numpy(), C1)
    assert sp.spamm_get_partition(plan.handle, 1) == [0, M // T]


def test_nccl_communicator_single_rank(sp):
    """The NCCL plumbing of spamm_multiply_mgpu on real hardware as far as one GPU allows: a
    communicator from spamm_nccl_unique_id / spamm_nccl_comm_init (NCCL's own bootstrap, one rank),
    handed to spamm_multiply_mgpu (Alg. 4) with GATHER_C, equals spamm_run; the
    collectives themselves need nranks > 1, i.e. more than the one GPU of this box (their phases are
    verified above through spamm_multiply_mgpu_local)."""
    M = N = K = 1024
    prec = "bf16"
    A = _rounded(synth.perturbed_decay_matrix(K, 0.99, seed=161, m=M), prec)
    Ad = _dev(A, prec)
    _, C1 = _single(sp, Ad, Ad, 1e-4, prec, M, N, K)
    comm = sp.spamm_nccl_comm_init(1, 0, sp.spamm_nccl_unique_id())
    try:
        plan = sp.Plan(M, N, K, 1e-4, prec)
        C = torch.zeros((M, N), device="cuda")
        for _ in range(2):
            sp.spamm_multiply_mgpu(plan.handle, comm, 0, 1, Ad, Ad, C, sp.SPAMM_MGPU_GATHER_C)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(C.cpu().numpy(), C1)
    finally:
        sp.spamm_nccl_comm_destroy(comm)
