"""World-size-2 gloo tests (CPU) of the multi-rank host logic of the row-partitioned
SpAMM (Sec. 3.4; load balance Sec. 3.5.1).

Each rank computes the kept-pair row work of its provisional tile rows (with the
float64 oracle -- test infrastructure), the work vectors are all-reduced, and the
C ABI's host partitioner cuts the rows.  Checked: every rank gets the same cuts, the
cuts are balanced, the shards' skip sets reassemble the single-process skip set, and
the shards' C rows reassemble single-process C (invariant P4)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2103_13042_b200 import dist as sd
        T, N = 32, 640
        A = synth.perturbed_decay_matrix(N, 0.95, seed=41)
        B = synth.perturbed_decay_matrix(N, 0.95, seed=42)
        nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
        tau = 0.05
        BM = nA.shape[0]
        r0, r1 = sd.provisional_rows(BM, rank, world)
        local = np.zeros(BM, dtype=np.int64)
        sm = oracle.skipmap(nA[r0:r1], nB, tau)
        local[r0:r1] = sm["row_work"]
        cuts = sd.balanced_cuts(local, world)
        c0, c1 = cuts[rank], cuts[rank + 1]
        mine = oracle.spamm(A[c0 * T:c1 * T], B, tau, T, nA[c0:c1], nB) if c1 > c0 else np.zeros((0, N))
        uid = sd.agree_unique_id(rank, world)
        gathered = [None] * world
        dist.all_gather_object(gathered, (cuts, mine, uid, rank))
        tmax = sd.max_over_ranks(float(rank + 1))
        if rank == 0:
            out.put((gathered, tmax))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def built():
    from paper_2103_13042_b200 import build
    build.build()


def test_row_partition_two_ranks_gloo(built):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cuts = [g[0] for g in gathered]
    assert cuts[0] == cuts[1], "every rank must compute the identical partition"
    assert gathered[0][2] == gathered[1][2] and len(gathered[0][2]) == 128, "NCCL unique id must agree"
    assert tmax == 2.0
    # reference: single process
    T, N = 32, 640
    A = synth.perturbed_decay_matrix(N, 0.95, seed=41)
    B = synth.perturbed_decay_matrix(N, 0.95, seed=42)
    nA, nB = oracle.tile_norms(A, T), oracle.tile_norms(B, T)
    sm = oracle.skipmap(nA, nB, 0.05)
    w = sm["row_work"]
    c = cuts[0]
    loads = [int(w[c[r]:c[r + 1]].sum()) for r in range(world)]
    assert max(loads) <= w.sum() / world + w.max()
    C = np.concatenate([g[1] for g in sorted(gathered, key=lambda g: g[3])], axis=0)
    np.testing.assert_array_equal(C, oracle.spamm(A, B, 0.05, T, nA, nB))
