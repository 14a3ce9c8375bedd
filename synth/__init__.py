"""Seeded synthetic inputs for the SpAMM hot path.

This module is shared by the CPU oracle (``oracle/``) and the CUDA product path
(``paper_2103_13042_b200``).  It holds NONE of the method's arithmetic (no tile
norms, no thresholding, no products): only the matrices the paper's workloads
are made of, generated deterministically so that both sides see bit-identical
inputs.

Workload shapes (cited to /root/reference/PAPER.md):
  * decay matrices, PAPER.md:45 (Sec. 2.1): exponential ``|a_ij| < c*lam**|i-j|``
    and algebraic ``|a_ij| < c/(|i-j|**lam + 1)``.
  * the paper's synthetic dataset, PAPER.md:257 (Sec. 4.1):
    ``a_ij = b_ij = 0.1/(|i-j|**0.1 + 1)``.
  * a signed, perturbed exponential variant (A != B) that breaks the Toeplitz
    ties of the plain generators.

Recipe ("Inputs"): a 1-D decay table ``f(d), d = 0..n-1`` is evaluated
in float64 on the host and rounded ONCE to float32; ``a_ij = f(|i-j|)``.  The
perturbed variant multiplies in float64 by ``(0.5 + u_ij) * s_ij`` where ``u_ij``
and the sign ``s_ij`` come from a counter-based splitmix64 hash of
``(seed, i*ncols + j)``, then rounds once to float32.  Low-precision copies
(BF16 / FP16) are round-to-nearest-even of those float32 values.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "splitmix64", "uniform01", "decay_table", "toeplitz", "decay_matrix",
    "perturbed_decay_matrix", "fp32_to_bf16_bits", "bf16_bits_to_fp32",
    "round_to_bf16", "round_to_fp16", "random_matrix", "CONFIG_SEED",
]

# seed = 2103 + config number.
CONFIG_SEED = {1: 2104, 2: 2105, 3: 2106, 4: 2107, 5: 2108}

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Counter-based splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, counter: np.ndarray) -> np.ndarray:
    """Uniform [0,1) float64 from the top 53 bits of splitmix64(seed<<40 ^ counter)."""
    base = np.uint64((int(seed) << 40) & 0xFFFFFFFFFFFFFFFF)
    h = splitmix64(np.asarray(counter, dtype=np.uint64) ^ base)
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def decay_table(kind: str, n: int, lam: float, c: float = 1.0) -> np.ndarray:
    """float64 table f(d), d = 0..n-1.

    kind="exp": f(d) = c * lam**d.   kind="alg": f(d) = c / (d**lam + 1).
    """
    d = np.arange(n, dtype=np.float64)
    if kind == "exp":
        return c * np.power(float(lam), d)
    if kind == "alg":
        return c / (np.power(d, float(lam)) + 1.0)
    raise ValueError(f"unknown decay kind {kind!r}")


def toeplitz(table32: np.ndarray, m: int, n: int) -> np.ndarray:
    """a_ij = table32[|i-j|] as a C-contiguous (m, n) array of table32's dtype."""
    out = np.empty((m, n), dtype=table32.dtype)
    cols = np.arange(n, dtype=np.int64)
    step = max(1, (1 << 24) // max(n, 1))
    for r0 in range(0, m, step):
        rows = np.arange(r0, min(m, r0 + step), dtype=np.int64)
        out[r0:r0 + len(rows)] = table32[np.abs(rows[:, None] - cols[None, :])]
    return out


def decay_matrix(n: int, kind: str = "exp", lam: float = 0.99, c: float = 1.0,
                 m: int | None = None) -> np.ndarray:
    """float32 decay matrix a_ij = fp32(f(|i-j|)); square unless ``m`` is given.

    The paper's dataset is ``decay_matrix(N, "alg", 0.1, c=0.1)``.
    """
    m = n if m is None else m
    t = decay_table(kind, max(m, n), lam, c).astype(np.float32)
    return toeplitz(t, m, n)


def perturbed_decay_matrix(n: int, lam: float, seed: int, kind: str = "exp",
                           c: float = 1.0, m: int | None = None) -> np.ndarray:
    """float32 a_ij = fp32(f(|i-j|) * (0.5 + u_ij) * s_ij), u, s from splitmix64."""
    m = n if m is None else m
    t = decay_table(kind, max(m, n), lam, c)
    out = np.empty((m, n), dtype=np.float32)
    cols = np.arange(n, dtype=np.int64)
    step = max(1, (1 << 22) // max(n, 1))
    for r0 in range(0, m, step):
        rows = np.arange(r0, min(m, r0 + step), dtype=np.int64)
        ctr = (rows[:, None] * n + cols[None, :]).astype(np.uint64)
        u = uniform01(seed, ctr)
        sgn = np.where(uniform01(seed + 0x5151, ctr) < 0.5, -1.0, 1.0)
        out[r0:r0 + len(rows)] = (t[np.abs(rows[:, None] - cols[None, :])] * (0.5 + u) * sgn).astype(np.float32)
    return out


def random_matrix(m: int, n: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """float32 matrix with entries scale*(2u-1), u ~ splitmix64 uniform (edge-case tests)."""
    ctr = np.arange(m * n, dtype=np.uint64).reshape(m, n)
    return (scale * (2.0 * uniform01(seed, ctr) - 1.0)).astype(np.float32)


def fp32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 bit patterns (uint16). NaN stays NaN."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    lsb = (u >> np.uint32(16)) & np.uint32(1)
    with np.errstate(over="ignore"):
        r = (u + np.uint32(0x7FFF) + lsb) >> np.uint32(16)
    nan = (u & np.uint32(0x7FFFFFFF)) > np.uint32(0x7F800000)
    r = np.where(nan, (u >> np.uint32(16)) | np.uint32(0x40), r)
    return r.astype(np.uint16)


def bf16_bits_to_fp32(b: np.ndarray) -> np.ndarray:
    """Exact widening of bfloat16 bit patterns to float32."""
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """float32 array holding the RNE-bfloat16 values of x (what the BF16 path multiplies)."""
    return bf16_bits_to_fp32(fp32_to_bf16_bits(x))


def round_to_fp16(x: np.ndarray) -> np.ndarray:
    """float32 array holding the RNE-float16 values of x."""
    return np.asarray(x, dtype=np.float32).astype(np.float16).astype(np.float32)
