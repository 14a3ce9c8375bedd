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


# --------------------------------------------------------------------------------------------
# configs[3]: electronic-structure-like banded decay and ReLU-sparsified im2col GEMM shapes
# --------------------------------------------------------------------------------------------

def normal01(seed: int, counter: np.ndarray) -> np.ndarray:
    """Standard normal float64 via Box-Muller from two splitmix64 uniforms per counter."""
    c = np.asarray(counter, dtype=np.uint64)
    u1 = uniform01(seed, c * np.uint64(2))
    u2 = uniform01(seed, c * np.uint64(2) + np.uint64(1))
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


def water_cluster_centres(n_mol: int = 569, spacing: float = 3.1, jitter: float = 0.3,
                          seed: int = 2107) -> np.ndarray:
    """(n_mol, 3) molecule centres in Angstrom, Morton (Z-curve) ordered.

    The n_mol points of a cubic lattice (spacing 3.1 A, about the O-O distance in water)
    nearest the origin (ties broken lexicographically), each jittered by N(0, jitter^2)
    per axis.  The shape stands in for the ergo water-cluster density matrices the
    paper multiplies (PAPER.md:320, 569 molecules at the size used there); no chemistry.
    """
    R = int(np.ceil((3.0 * n_mol / (4.0 * np.pi)) ** (1.0 / 3.0))) + 2
    g = np.arange(-R, R + 1)
    pts = np.stack(np.meshgrid(g, g, g, indexing="ij"), axis=-1).reshape(-1, 3)
    d2 = (pts * pts).sum(axis=1)
    order = np.lexsort((pts[:, 2], pts[:, 1], pts[:, 0], d2))[:n_mol]
    pos = spacing * pts[order].astype(np.float64)
    ctr = np.arange(3 * n_mol, dtype=np.uint64).reshape(n_mol, 3)
    pos = pos + jitter * normal01(seed, ctr)
    # Morton order of 10-bit quantised coordinates
    q = pos - pos.min(axis=0)
    q = np.minimum((q / max(float(q.max()), 1e-12) * 1023.0).astype(np.int64), 1023)
    code = np.zeros(n_mol, dtype=np.int64)
    for b in range(10):
        for a in range(3):
            code |= ((q[:, a] >> b) & 1) << (3 * b + a)
    return pos[np.argsort(code, kind="stable")]


def water_cluster_matrix(n_mol: int = 569, nbf: int = 24, alpha: float = 1.0,
                         seed: int = 2107) -> np.ndarray:
    """float32 (n, n), n = n_mol*nbf: a_ij = exp(-alpha * r(m(i), m(j))) * g_ij.

    m(i) = i // nbf is the molecule of basis function i, r the centre distance in A,
    g symmetric uniform in [-1, 1) from splitmix64 of (seed, min(i,j)*n + max(i,j)).
    A = B ("power" of a density-like matrix).  n = 13656 for the default
    569 molecules x 24 functions, which is not a multiple of 32 (exercises padding).
    """
    pos = water_cluster_centres(n_mol, seed=seed)
    n = n_mol * nbf
    mol = np.arange(n) // nbf
    out = np.empty((n, n), dtype=np.float32)
    cols = np.arange(n, dtype=np.int64)
    step = max(1, (1 << 22) // n)
    for r0 in range(0, n, step):
        rows = np.arange(r0, min(n, r0 + step), dtype=np.int64)
        dr = pos[mol[rows]][:, None, :] - pos[mol[cols]][None, :, :]
        r = np.sqrt((dr * dr).sum(axis=-1))
        lo = np.minimum(rows[:, None], cols[None, :]).astype(np.uint64)
        hi = np.maximum(rows[:, None], cols[None, :]).astype(np.uint64)
        g = 2.0 * uniform01(seed + 0x77, lo * np.uint64(n) + hi) - 1.0
        out[r0:r0 + len(rows)] = (np.exp(-alpha * r) * g).astype(np.float32)
    return out


# VGG13 layers whose im2col GEMMs the paper sparsifies (reading R15):
# name -> (C_out, C_in, H = W, batch)
IM2COL_LAYERS = {"conv21": (128, 64, 16, 100), "conv31": (256, 128, 8, 100)}


def conv_weight(c_out: int, c_in: int, seed: int, prune: float = 0.5) -> np.ndarray:
    """float32 (c_out, c_in*9) 3x3 conv weights ~ N(0, 2/fan_in), the smallest |w| fraction
    ``prune`` set to zero (magnitude pruning)."""
    fan = c_in * 9
    w = normal01(seed, np.arange(c_out * fan, dtype=np.uint64)).reshape(c_out, fan) * np.sqrt(2.0 / fan)
    if prune > 0:
        thr = np.quantile(np.abs(w), prune)
        w = np.where(np.abs(w) <= thr, 0.0, w)
    return w.astype(np.float32)


def relu_activations(batch: int, c: int, h: int, seed: int) -> np.ndarray:
    """float32 (batch, c, h, h): ReLU(N(b_c, 1)) * s_{n,c}, b_c ~ N(-0.5, 0.5^2),
    s ~ LogNormal(0, 0.5^2); >= 50 % zeros like post-ReLU feature maps."""
    b = -0.5 + 0.5 * normal01(seed, np.arange(c, dtype=np.uint64))
    s = np.exp(0.5 * normal01(seed + 1, np.arange(batch * c, dtype=np.uint64))).reshape(batch, c)
    z = normal01(seed + 2, np.arange(batch * c * h * h, dtype=np.uint64)).reshape(batch, c, h, h)
    x = np.maximum(z + b[None, :, None, None], 0.0) * s[:, :, None, None]
    return x.astype(np.float32)


def im2col(x: np.ndarray) -> np.ndarray:
    """(batch, c, h, w) -> (c*9, batch*h*w) columns of a 3x3, stride-1, pad-1 convolution;
    row index c*9 + ky*3 + kx, column index (n*h + y)*w + x."""
    nb, c, h, w = x.shape
    xp = np.zeros((nb, c, h + 2, w + 2), dtype=x.dtype)
    xp[:, :, 1:-1, 1:-1] = x
    cols = np.empty((c, 3, 3, nb, h, w), dtype=x.dtype)
    for ky in range(3):
        for kx in range(3):
            cols[:, ky, kx] = xp[:, :, ky:ky + h, kx:kx + w].transpose(1, 0, 2, 3)
    return np.ascontiguousarray(cols.reshape(c * 9, nb * h * w))


def im2col_gemm(layer: str, seed: int = 2107) -> tuple[np.ndarray, np.ndarray]:
    """(A, B) = (pruned weights W [C_out x C_in*9], im2col(X) [C_in*9 x batch*H*W]) for a
    VGG13 layer of IM2COL_LAYERS: conv21 128x576x25600, conv31 256x1152x6400."""
    c_out, c_in, h, nb = IM2COL_LAYERS[layer]
    W = conv_weight(c_out, c_in, seed)
    X = relu_activations(nb, c_in, h, seed + 10)
    return W, im2col(X)


def toeplitz_block(table32: np.ndarray, r0: int, r1: int, c0: int, c1: int) -> np.ndarray:
    """Rows r0:r1, columns c0:c1 of the Toeplitz matrix a_ij = table32[|i-j|]."""
    rows = np.arange(r0, r1, dtype=np.int64)
    cols = np.arange(c0, c1, dtype=np.int64)
    return table32[np.abs(rows[:, None] - cols[None, :])]


def toeplitz_device(table32: np.ndarray, n: int, dtype, device="cuda"):
    """Device-resident (n, n) torch tensor a_ij = table32[|i-j|] in ``dtype`` (configs[4]:
    N = 65536 does not fit comfortably in host memory).  Pure indexing: the same values
    ``toeplitz(table32, n, n)`` holds, converted to ``dtype`` by torch's RNE cast."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(table32)).to(device)
    out = torch.empty((n, n), dtype=dtype, device=device)
    cols = torch.arange(n, device=device)
    step = max(1, (1 << 26) // n)
    for r0 in range(0, n, step):
        rows = torch.arange(r0, min(n, r0 + step), device=device)
        out[r0:r0 + len(rows)] = t[(rows[:, None] - cols[None, :]).abs()].to(dtype)
    return out
