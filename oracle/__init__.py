"""CPU float64 oracle for the SpAMM hot path (cuSpAMM, arXiv 2103.13042).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import or call
anything under ``oracle/``.  The product path (``paper_2103_13042_b200``) never
imports it and shares no code with it; the only shared module is ``synth``
(seeded inputs, no method arithmetic).

Every function is the plain definition from the paper, in float64, with no
blocking, fusion or reordering beyond what the definition states.  Citations are
lines of /root/reference/PAPER.md.

Definitions followed (flat leaf-level semantics, Alg. 2 lines 3-8):
  * pad to a multiple of the tile LoNum with zeros;
  * ``nA[i,k] = ||A[i,k]||_F`` (Eq. 2; normmap PAPER.md:103);
  * keep (i,k,j)  iff  ``nA[i,k] * nB[k,j] >= tau`` ("no smaller than",
    Alg. 1 line 7/10 PAPER.md:63, Alg. 2 line 5 PAPER.md:155).  NaN products are
    kept (reading R2: keep iff ``not (p < tau)``);
  * ``C[i,j] = sum_{kept k, ascending} A[i,k] @ B[k,j]``, alpha=1, beta=0
    (PAPER.md:47);
  * valid ratio ``sum V / (BM*BK*BN)`` (reading R10);
  * error ``||AB - SpAMM(A,B,tau)||_F`` (Eq. 5).
Also: the recursive Alg. 1 as an independent cross-check, and
the Sec. 3.5.2 tau search.

Parity pins: every function here is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_pins.py`` (paper tables, closed forms, brute force); none is
"parity unpinned".  ``spamm_tile`` (reference of every sampled full-size tile check):
hand-enumerated N=4 tiles, tau=0 = the plain product's block on ragged edges, a tile with
one kept k = that block product, and agreement with ``spamm``; ``band_count``: products
placed by hand inside/outside the 1e-6 band; ``tile_error_bound``: hand values and
equality with the true error for aligned rank-one tiles (where the bound is tight);
``macro_lists``: a hand-enumerated 8 x 8 (64-bit mask) case with a ragged second group.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "pad_to_tiles", "tile_norms", "keep_mask", "skipmap", "spamm", "spamm_tile",
    "spamm_recursive", "valid_ratio", "count_kept", "error_fnorm", "tile_error_bound",
    "tau_search", "band_count", "dense_product", "macro_lists", "spamm_axpby",
]


def _nblk(n: int, T: int) -> int:
    return (n + T - 1) // T


def pad_to_tiles(X: np.ndarray, T: int) -> np.ndarray:
    """Zero-pad X (float64 copy) to multiples of the tile size T."""
    X = np.asarray(X)
    m, n = X.shape
    P = np.zeros((_nblk(m, T) * T, _nblk(n, T) * T), dtype=np.float64)
    P[:m, :n] = X
    return P


def tile_norms(X: np.ndarray, T: int) -> np.ndarray:
    """normmap[i][k] = ||X[i,k]||_F = sqrt(sum of squares of the T x T tile), Eq. 2.

    PAPER.md:51 (Eq. 2), PAPER.md:103 (normmap), PAPER.md:99 (zero padding).
    Returns a float64 array of shape (ceil(m/T), ceil(n/T)).  Computed one tile
    row at a time only to bound memory; each tile's sum is the plain float64 sum.
    """
    X = np.asarray(X)
    m, n = X.shape
    BM, BK = _nblk(m, T), _nblk(n, T)
    out = np.empty((BM, BK), dtype=np.float64)
    for i in range(BM):
        strip = np.zeros((T, BK * T), dtype=np.float64)
        rows = X[i * T:min(m, (i + 1) * T)]
        strip[:rows.shape[0], :n] = rows
        sq = strip * strip
        out[i] = np.sqrt(sq.reshape(T, BK, T).sum(axis=(0, 2)))
    return out


def keep_mask(nA: np.ndarray, nB: np.ndarray, tau: float) -> np.ndarray:
    """Boolean keep[i,k,j] = (nA[i,k]*nB[k,j] >= tau), NaN kept (Alg. 2 lines 3-8).

    PAPER.md:152-158 (Alg. 2 lines 3-8; ``bitmap[i]`` read as ``bitmap[k]``,
    DESIGN.md reading R7), PAPER.md:47/63 (">= tau").  Small problems only: the
    result has BM*BK*BN entries.
    """
    p = nA[:, :, None] * nB[None, :, :]
    return ~(p < tau)


def count_kept(nA: np.ndarray, nB: np.ndarray, tau: float) -> int:
    """Number of kept (i,k,j) triples, sum of V[i][j]."""
    total = 0
    for i in range(nA.shape[0]):
        p = nA[i][:, None] * nB
        total += int(np.count_nonzero(~(p < tau)))
    return total


def valid_ratio(nA: np.ndarray, nB: np.ndarray, tau: float) -> float:
    """valid ratio = sum V / BDIM^3; BM*BK*BN for rectangular shapes."""
    BM, BK = nA.shape
    BN = nB.shape[1]
    return count_kept(nA, nB, tau) / float(BM * BK * BN)


def skipmap(nA: np.ndarray, nB: np.ndarray, tau: float) -> dict:
    """Per-C-tile ascending k-lists (CSR), V and row work.

    ``map_offset`` of Alg. 2 (Fig. 3) is the ascending list of
    valid k for one C tile; here it is stored for every tile (i,j), row-major,
    as ``k_idx[tile_ptr[i*BN+j] : tile_ptr[i*BN+j+1]]``.
    V[i][j] = list length; row_work[i] = sum_j V[i][j].
    """
    BM, BK = nA.shape
    BN = nB.shape[1]
    V = np.zeros((BM, BN), dtype=np.int64)
    lists = []
    for i in range(BM):
        keep = ~((nA[i][:, None] * nB) < tau)          # (BK, BN)
        V[i] = keep.sum(axis=0)
        for j in range(BN):
            lists.append(np.nonzero(keep[:, j])[0].astype(np.int64))
    tile_ptr = np.zeros(BM * BN + 1, dtype=np.int64)
    tile_ptr[1:] = np.cumsum(V.reshape(-1))
    k_idx = np.concatenate(lists) if lists else np.zeros(0, dtype=np.int64)
    return {"tile_ptr": tile_ptr, "k_idx": k_idx, "V": V,
            "row_work": V.sum(axis=1), "kept": int(tile_ptr[-1])}


def macro_lists(nA: np.ndarray, nB: np.ndarray, tau: float, MI: int, MJ: int) -> dict:
    """Union k-lists of MI x MJ groups of C tiles with per-tile keep bits.

    Not a paper construct: the grouping the GPU scheduler uses, written out from
    the keep definition (bit ``li*MJ + lj`` of entry k of group (I,J) is
    keep(I*MI+li, k, J*MJ+lj)).  Returns dict with ``ptr`` (GM*GN+1) and
    ``entries`` (n, 2) uint64 rows (k, mask).
    """
    BM, BK = nA.shape
    BN = nB.shape[1]
    GM, GN = _nblk(BM, MI), _nblk(BN, MJ)
    ptr = [0]
    ents = []
    for I in range(GM):
        for J in range(GN):
            for k in range(BK):
                mask = 0
                for li in range(MI):
                    i = I * MI + li
                    if i >= BM:
                        continue
                    for lj in range(MJ):
                        j = J * MJ + lj
                        if j >= BN:
                            continue
                        if not (nA[i, k] * nB[k, j] < tau):
                            mask |= 1 << (li * MJ + lj)
                if mask:
                    ents.append((k, mask))
            ptr.append(len(ents))
    # uint64: 8 x 8 groups use all 64 mask bits
    return {"ptr": np.asarray(ptr, dtype=np.int64),
            "entries": np.asarray(ents, dtype=np.uint64).reshape(-1, 2)}


def spamm(A: np.ndarray, B: np.ndarray, tau: float, T: int,
          nA: np.ndarray | None = None, nB: np.ndarray | None = None) -> np.ndarray:
    """Flat SpAMM in float64: C[i,j] = sum over kept k (ascending) of A[i,k] @ B[k,j].

    PAPER.md:127 (``C[i,j] = sum A[i,k] x B[k,j] x bitmap[k]``), PAPER.md:103 (the
    flat re-design is equivalent to Alg. 1), alpha=1, beta=0.
    Returns C of shape (m, n) (padding removed).
    """
    m, K = A.shape
    K2, n = B.shape
    assert K == K2
    Ap, Bp = pad_to_tiles(A, T), pad_to_tiles(B, T)
    if nA is None:
        nA = tile_norms(A, T)
    if nB is None:
        nB = tile_norms(B, T)
    BM, BK = nA.shape
    BN = nB.shape[1]
    C = np.zeros((BM * T, BN * T), dtype=np.float64)
    for i in range(BM):
        keep = ~((nA[i][:, None] * nB) < tau)            # (BK, BN)
        for j in range(BN):
            ks = np.nonzero(keep[:, j])[0]
            if ks.size == 0:
                continue
            a = Ap[i * T:(i + 1) * T].reshape(T, BK, T)[:, ks, :].reshape(T, -1)
            b = Bp[:, j * T:(j + 1) * T].reshape(BK, T, T)[ks].reshape(-1, T)
            C[i * T:(i + 1) * T, j * T:(j + 1) * T] = a @ b
    return C[:m, :n]


def spamm_axpby(A: np.ndarray, B: np.ndarray, tau: float, T: int, alpha: float, beta: float,
                C0: np.ndarray | None, nA: np.ndarray | None = None, nB: np.ndarray | None = None) -> np.ndarray:
    """The problem statement in full, ``C = alpha*A*B + beta*C`` with A*B the SpAMM product
    (the paper then fixes alpha = 1, beta = 0).  float64.  beta == 0 ignores C0
    entirely (BLAS convention: NaN in C0 does not propagate)."""
    P = spamm(A, B, tau, T, nA, nB)
    if beta == 0.0:
        return alpha * P
    return alpha * P + beta * np.asarray(C0, dtype=np.float64)


def spamm_tile(A: np.ndarray, B: np.ndarray, tau: float, T: int, i: int, j: int,
               nA: np.ndarray, nB: np.ndarray) -> np.ndarray:
    """One C tile (i,j) of flat SpAMM in float64 (for sampled checks at full size)."""
    m, K = A.shape
    n = B.shape[1]
    BK = nA.shape[1]
    out = np.zeros((T, T), dtype=np.float64)
    r0, r1 = i * T, min(m, (i + 1) * T)
    c0, c1 = j * T, min(n, (j + 1) * T)
    for k in range(BK):
        if nA[i, k] * nB[k, j] < tau:
            continue
        k0, k1 = k * T, min(K, (k + 1) * T)
        a = np.asarray(A[r0:r1, k0:k1], dtype=np.float64)
        b = np.asarray(B[k0:k1, c0:c1], dtype=np.float64)
        out[:r1 - r0, :c1 - c0] += a @ b
    return out[:r1 - r0, :c1 - c0]


def _fnorm(X: np.ndarray) -> float:
    return math.sqrt(float(np.sum(np.asarray(X, dtype=np.float64) ** 2)))


def spamm_recursive(A: np.ndarray, B: np.ndarray, tau: float, T: int) -> np.ndarray:
    """Alg. 1 literally: quadtree recursion (Eq. 1).

    Requires square power-of-two multiples of T.  At the lowest level (size T)
    returns A@B; otherwise for each quadrant C_ij, T0 = SpAMM(A_i0, B_0j) if
    ||A_i0||_F ||B_0j||_F >= tau else 0, T1 likewise with (A_i1, B_1j), and
    C_ij = T0 + T1.  Norms per Eq. 2.
    """
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    n = A.shape[0]
    assert A.shape == (n, n) and B.shape == (n, n)
    assert n >= T and n % T == 0 and ((n // T) & (n // T - 1)) == 0

    def rec(a, b):
        s = a.shape[0]
        if s == T:                                   # line 3-4: lowest level
            return a @ b
        h = s // 2
        c = np.zeros((s, s), dtype=np.float64)
        for i in range(2):                            # lines 5-15
            for j in range(2):
                a0, b0 = a[i * h:(i + 1) * h, :h], b[:h, j * h:(j + 1) * h]
                a1, b1 = a[i * h:(i + 1) * h, h:], b[h:, j * h:(j + 1) * h]
                t0 = rec(a0, b0) if not (_fnorm(a0) * _fnorm(b0) < tau) else 0.0
                t1 = rec(a1, b1) if not (_fnorm(a1) * _fnorm(b1) < tau) else 0.0
                c[i * h:(i + 1) * h, j * h:(j + 1) * h] = t0 + t1
        return c

    return rec(A, B)


def dense_product(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Exact-in-float64 reference product AB (the tau = 0 limit; Eq. 5's AB)."""
    return np.asarray(A, dtype=np.float64) @ np.asarray(B, dtype=np.float64)


def error_fnorm(A: np.ndarray, B: np.ndarray, C: np.ndarray) -> float:
    """||E||_F with E = AB - SpAMM(A,B,tau) (Eq. 5), float64."""
    return _fnorm(dense_product(A, B) - np.asarray(C, dtype=np.float64))


def tile_error_bound(nA: np.ndarray, nB: np.ndarray, tau: float) -> float:
    """sqrt(sum_{i,j} (sum_{skipped k} nA[i,k] nB[k,j])^2): an upper bound on ||E||_F.

    By the triangle inequality and ||XY||_F <= ||X||_F ||Y||_F applied to each
    skipped product ("error bound").  Not a paper formula; the paper's
    asymptotic law has no pinned constant.
    """
    BM = nA.shape[0]
    BN = nB.shape[1]
    s = np.zeros((BM, BN), dtype=np.float64)
    for i in range(BM):
        p = nA[i][:, None] * nB
        s[i] = np.where(p < tau, p, 0.0).sum(axis=0)
    return math.sqrt(float(np.sum(s * s)))


def band_count(nA: np.ndarray, nB: np.ndarray, tau: float, rel: float = 1e-6) -> int:
    """Number of triples whose norm product lies within rel*tau of tau (tie band)."""
    total = 0
    for i in range(nA.shape[0]):
        p = nA[i][:, None] * nB
        total += int(np.count_nonzero(np.abs(p - tau) <= rel * tau))
    return total


def tau_search(nA: np.ndarray, nB: np.ndarray, target: float, iters: int = 20,
               tol: float = 0.01) -> tuple[float, float, int]:
    """Sec. 3.5.2 tau search for a target valid ratio.

    ``ave`` = average of the norm products of all sub-matrix pairs (reading R17:
    mean over all BM*BK*BN triples).  Binary search on [0, k*ave], initial value
    ave, k starts at 1 and grows by one whenever the upper bound still keeps too
    many pairs.  Stops when |vr - target| < tol (absolute, reading R16) or after
    ``iters`` evaluations.  Returns (tau, vr(tau), iterations used).
    """
    BM, BK = nA.shape
    BN = nB.shape[1]
    ave = float(np.sum(nA.sum(axis=0) * nB.sum(axis=1))) / float(BM * BK * BN)
    tau, lo, hi, k = ave, 0.0, ave, 1
    vr = valid_ratio(nA, nB, tau)
    it = 1
    while it < iters and abs(vr - target) >= tol:
        if vr > target:
            lo = tau
            while valid_ratio(nA, nB, hi) > target:
                k += 1
                hi = k * ave
        else:
            hi = tau
        tau = 0.5 * (lo + hi)
        vr = valid_ratio(nA, nB, tau)
        it += 1
    return tau, vr, it
