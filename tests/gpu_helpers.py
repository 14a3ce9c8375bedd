"""Shared helpers of the GPU parity tests (import only; no tests here).

Bars (BASELINE.json north_star): skip decisions bit-exact outside the 1e-6 relative tie band
around tau; C within 1e-5 relative Frobenius error (FP32 paths) / 2e-2 (BF16/FP16 tensor path).
Per-tile check: every C tile's error is also bounded relative to the same tile of the SpAMM of
|A| and |B| with the same keep set (the magnitude its FP32 accumulation works on), so a single
wrong tile cannot hide inside a global Frobenius norm, and cancellation inside a tile does not
make the bound meaningless.
"""
import numpy as np
import torch

import oracle
import synth

T = 32
BAND = 1e-6
BAR = {"fp32": 1e-5, "fp32x3": 1e-5, "bf16": 2e-2, "fp16": 2e-2}
# regression guards below the north_star bars: FP32 accumulation of exactly representable
# products (fp32; bf16/fp16 with the same rounded inputs on both sides), split products (fp32x3)
GUARD = {"fp32": 2e-6, "fp32x3": 5e-6, "bf16": 1e-5, "fp16": 5e-5}
DT = {"fp32": torch.float32, "fp32x3": torch.float32, "bf16": torch.bfloat16, "fp16": torch.float16}


def rounded(x: np.ndarray, prec: str) -> np.ndarray:
    if prec == "bf16":
        return synth.round_to_bf16(x)
    if prec == "fp16":
        return synth.round_to_fp16(x)
    return x


def dev(x: np.ndarray, prec: str, ld_mult: int = 8):
    """Device copy in the path's dtype with the leading dimension padded to ld_mult."""
    m, n = x.shape
    ld = -(-n // ld_mult) * ld_mult
    buf = torch.zeros((m, ld), dtype=DT[prec], device="cuda")
    buf[:, :n] = torch.from_numpy(np.ascontiguousarray(x)).to(DT[prec])
    return buf[:, :n]


def cbuf(M, N):
    """NaN-filled C (unwritten tiles show up as NaN)."""
    return torch.full((M, -(-N // 4) * 4), float("nan"), dtype=torch.float32, device="cuda")[:, :N]


def tile_max_rel(C, ref, absref):
    """max over C tiles of ||C_t - ref_t||_F / ||absref_t||_F (absref = SpAMM(|A|,|B|), same
    keep set); tiles with absref_t = 0 must be exactly zero (returned as inf otherwise)."""
    C = np.asarray(C, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    absref = np.asarray(absref, dtype=np.float64)
    m, n = ref.shape
    worst = 0.0
    for r0 in range(0, m, T):
        for c0 in range(0, n, T):
            d = C[r0:r0 + T, c0:c0 + T] - ref[r0:r0 + T, c0:c0 + T]
            na = np.linalg.norm(absref[r0:r0 + T, c0:c0 + T])
            if na == 0.0:
                if np.any(C[r0:r0 + T, c0:c0 + T] != 0.0):
                    return float("inf")
                continue
            worst = max(worst, float(np.linalg.norm(d)) / na)
    return worst


def check_norms(sp, plan, nA, nB):
    nA_g, nBt_g = sp.spamm_get_norms(plan.handle)
    np.testing.assert_allclose(nA_g.cpu().numpy(), nA, rtol=1e-12, atol=0)
    np.testing.assert_allclose(nBt_g.cpu().numpy().T, nB, rtol=1e-12, atol=0)


def check_rows(sp, plan, nA, nB, tau, rows):
    """Skip lists of every C tile in the given tile rows vs the oracle predicate (outside the
    tie band); lists strictly ascending."""
    BN = nB.shape[1]
    start, kidx = sp.spamm_get_skipmap(plan.handle)
    V = sp.spamm_get_counts(plan.handle)[0]
    for i in rows:
        keep_o = ~((nA[i][:, None] * nB) < tau)
        p = nA[i][:, None] * nB
        band = np.abs(p - tau) <= BAND * tau
        s = start[i * BN:(i + 1) * BN].cpu().numpy()
        v = V[i].cpu().numpy()
        lo, hi = int(s.min()), int((s + v).max())
        ks = kidx[lo:hi].cpu().numpy()
        keep_g = np.zeros_like(keep_o)
        for j in range(BN):
            lst = ks[s[j] - lo:s[j] - lo + v[j]]
            assert np.all(np.diff(lst) > 0), (i, j)
            keep_g[lst, j] = True
        bad = (keep_g != keep_o) & ~band
        assert not np.any(bad), f"row {i}: {int(bad.sum())} decisions differ outside the tie band"


def check_tiles(C, A, B, tau, nA, nB, tiles, bar, absA=None, absB=None):
    """Sampled C tiles vs oracle.spamm_tile, one by one (A, B host arrays or tile views)."""
    Cn = C if isinstance(C, np.ndarray) else None
    for i, j in tiles:
        ref = oracle.spamm_tile(A, B, tau, T, i, j, nA, nB)
        got = Cn[i * T:i * T + ref.shape[0], j * T:j * T + ref.shape[1]] if Cn is not None else \
            C[i * T:i * T + ref.shape[0], j * T:j * T + ref.shape[1]].cpu().numpy()
        scale = np.linalg.norm(ref)
        if absA is not None:
            scale = np.linalg.norm(oracle.spamm_tile(absA, absB, tau, T, i, j, nA, nB))
        if scale == 0:
            assert np.all(got == 0), (i, j)
        else:
            assert np.linalg.norm(got.astype(np.float64) - ref) / scale <= bar, (i, j)


def sample_tiles(BM, BN, seed, n=24):
    rng = np.random.default_rng(seed)
    t = [(int(i), int(j)) for i, j in zip(rng.integers(0, BM, n), rng.integers(0, BN, n))]
    t += [(d, d) for d in range(0, min(BM, BN), max(1, min(BM, BN) // 12))]
    t += [(0, 0), (0, BN - 1), (BM - 1, 0), (BM - 1, BN - 1), (BM - 1, max(0, BN - 2))]
    return t


def toeplitz_oracle_norms(table, N):
    """Oracle norm map of the Toeplitz matrix a_ij = table[|i-j|] from two strips: tile (i, k)
    depends only on D = k - i, so the oracle's norms of the first tile row (D >= 0) and first tile
    column (D <= 0) give every tile's norm."""
    r = oracle.tile_norms(synth.toeplitz_block(table, 0, T, 0, N), T)[0]
    c = oracle.tile_norms(synth.toeplitz_block(table, 0, N, 0, T), T)[:, 0]
    BD = N // T
    d = np.arange(BD)[None, :] - np.arange(BD)[:, None]
    return np.where(d >= 0, r[np.clip(d, 0, None)], c[np.clip(-d, 0, None)])


class ToeplitzTiles:
    """Host view of tiles of a Toeplitz matrix for oracle.spamm_tile (never materialised)."""

    def __init__(self, table, n):
        self.t, self.shape = table, (n, n)

    def __getitem__(self, idx):
        rs, cs = idx
        return synth.toeplitz_block(self.t, rs.start, rs.stop, cs.start, cs.stop)
