"""Thin Python binding of libspamm.so (include/spamm.h) -- argument marshalling only.

Every function has the name of the C entry point it calls.  Matrices are torch CUDA
tensors (row-major, unit column stride); the binding passes ``data_ptr()`` and
``stride(0)`` and the caller's current CUDA stream.  There is no fallback: if the
extension is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
import re

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libspamm.so")
HEADER = os.path.join(os.path.dirname(_PKG), "include", "spamm.h")

SPAMM_OK, SPAMM_E_INVALID, SPAMM_E_UNSUPPORTED, SPAMM_E_CUDA, SPAMM_E_NOMEM, SPAMM_E_NCCL, SPAMM_E_STATE = range(7)
SPAMM_FP32, SPAMM_BF16, SPAMM_FP16, SPAMM_FP32X3 = 0, 1, 2, 3
SPAMM_FLAG_NONE, SPAMM_FLAG_TIMING, SPAMM_FLAG_LARGE_TILES, SPAMM_FLAG_STAGED = 0, 1, 2, 4
SPAMM_MUL_AUTO, SPAMM_MUL_OUTPUT_NORMS, SPAMM_MUL_LOW_ONLY = 1, 2, 4
SPAMM_MGPU_INPUTS_REPLICATED, SPAMM_MGPU_INPUTS_ON_ROOT, SPAMM_MGPU_GATHER_C = 0, 1, 2

DTYPE_OF = {SPAMM_FP32: torch.float32, SPAMM_BF16: torch.bfloat16, SPAMM_FP16: torch.float16,
            SPAMM_FP32X3: torch.float32}
PREC_OF = {"fp32": SPAMM_FP32, "bf16": SPAMM_BF16, "fp16": SPAMM_FP16, "fp32x3": SPAMM_FP32X3}


class SpammError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_status_name(status)}: {msg}")
        self.status = status


class spamm_stats(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int64), ("N", ctypes.c_int64), ("K", ctypes.c_int64),
                ("BM", ctypes.c_int64), ("BK", ctypes.c_int64), ("BN", ctypes.c_int64),
                ("tile", ctypes.c_int32), ("macro_i", ctypes.c_int32), ("macro_j", ctypes.c_int32),
                ("kept", ctypes.c_int64), ("macro_entries", ctypes.c_int64),
                ("valid_ratio", ctypes.c_double), ("tau", ctypes.c_double),
                ("ms_norms", ctypes.c_float), ("ms_skipmap", ctypes.c_float), ("ms_multiply", ctypes.c_float),
                ("precision", ctypes.c_int32), ("row_begin", ctypes.c_int32), ("row_end", ctypes.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libspamm.so not built ({LIB_PATH}); run `python -m paper_2103_13042_b200.build`")
    lib = ctypes.CDLL(LIB_PATH)
    P, I64, I32, D, U32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_uint32
    PP = ctypes.POINTER(ctypes.c_void_p)
    PI64 = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "spamm_plan": [PP, I64, I32, D, ctypes.c_int],
        "spamm_plan_ex": [PP, I64, I64, I64, I32, D, ctypes.c_int, U32],
        "spamm_plan_destroy": [P],
        "spamm_set_tau": [P, D],
        "spamm_norms": [P, P, I64, P, I64, P],
        "spamm_build_skipmap": [P, P],
        "spamm_multiply": [P, P, I64, P, I64, P, I64, U32, P],
        "spamm_run": [P, P, I64, P, I64, P, I64, P],
        "spamm_nccl_unique_id": [ctypes.c_char_p],
        "spamm_nccl_comm_init": [PP, ctypes.c_int, ctypes.c_int, ctypes.c_char_p],
        "spamm_nccl_comm_destroy": [P],
        "spamm_partition_rows": [PI64, I64, ctypes.c_int, PI64],
        "spamm_multiply_mgpu": [P, P, ctypes.c_int, ctypes.c_int, P, I64, P, I64, P, I64, U32, P],
        "spamm_multiply_mgpu_local": [PP, ctypes.c_int, P, I64, P, I64, PP, I64, U32, P],
        "spamm_conv2d_im2col": [P, P, I64, P, I64, I64, I64, I64, I32, I32, I32, I32, P, I64, P],
        "spamm_get_norms": [P, PP, PP, PI64, PI64, PI64],
        "spamm_get_skipmap": [P, PP, PP, PI64],
        "spamm_get_counts": [P, PP, PP],
        "spamm_get_macro": [P, PP, PP, PP, PP, PI64, PI64],
        "spamm_get_partition": [P, PI64, ctypes.c_int],
        "spamm_get_stats": [P, ctypes.POINTER(spamm_stats)],
        "spamm_count_kept": [P, D, PI64, P],
        "spamm_set_scalars": [P, D, D],
        "spamm_multiply_chain": [P, P, I64, P, I64, P, I64, P, I64, U32, P],
        "spamm_get_output_norms": [P, PP],
        "spamm_set_norms": [P, P, P, P],
        "spamm_tau_search": [P, D, D, I32, ctypes.POINTER(D), ctypes.POINTER(D), ctypes.POINTER(I32), P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.spamm_status_string.argtypes = [ctypes.c_int]
    lib.spamm_status_string.restype = ctypes.c_char_p
    lib.spamm_last_error.argtypes = []
    lib.spamm_last_error.restype = ctypes.c_char_p
    lib.spamm_launch_count.argtypes = []
    lib.spamm_launch_count.restype = ctypes.c_int64
    return lib


_lib = _load()


def _status_name(s: int) -> str:
    return _lib.spamm_status_string(int(s)).decode()


def _check(status: int):
    if status != SPAMM_OK:
        raise SpammError(status, _lib.spamm_last_error().decode())


def declared_functions() -> list[str]:
    """Entry points declared in include/spamm.h (for the export test)."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(spamm_[a-z0-9_]+)\s*\(", txt)) - {"spamm_plan_t"})


def library():
    return _lib


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _mat(t):
    """(pointer, leading dimension) of a row-major 2-D tensor with unit column stride."""
    if t is None:
        return ctypes.c_void_p(0), 0
    if t.dim() != 2 or (t.stride(1) != 1 and t.shape[1] > 1):
        raise ValueError("matrices must be 2-D, row-major with unit column stride")
    return ctypes.c_void_p(t.data_ptr()), int(t.stride(0)) if t.shape[0] > 1 else int(max(t.stride(0), t.shape[1]))


# ------------------------------------------------------------------ plans ---
def spamm_plan(N: int, tile: int, tau: float, prec: int) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _check(_lib.spamm_plan(ctypes.byref(h), int(N), int(tile), float(tau), int(prec)))
    return h


def spamm_plan_ex(M: int, N: int, K: int, tile: int, tau: float, prec: int, flags: int = 0) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _check(_lib.spamm_plan_ex(ctypes.byref(h), int(M), int(N), int(K), int(tile), float(tau), int(prec),
                              int(flags)))
    return h


def spamm_plan_destroy(plan) -> None:
    _check(_lib.spamm_plan_destroy(plan))


def spamm_set_tau(plan, tau: float) -> None:
    _check(_lib.spamm_set_tau(plan, float(tau)))


def spamm_set_scalars(plan, alpha: float, beta: float) -> None:
    """C = alpha * SpAMM(A, B) + beta * C for later multiplies."""
    _check(_lib.spamm_set_scalars(plan, float(alpha), float(beta)))


# ----------------------------------------------------------------- stages ---
def spamm_norms(plan, A, B, stream=None) -> None:
    a, lda = _mat(A)
    b, ldb = _mat(B)
    _check(_lib.spamm_norms(plan, a, lda, b, ldb, _stream(stream)))


def spamm_build_skipmap(plan, stream=None) -> None:
    _check(_lib.spamm_build_skipmap(plan, _stream(stream)))


def spamm_multiply(plan, A, B, C, flags: int = 0, stream=None) -> None:
    a, lda = _mat(A)
    b, ldb = _mat(B)
    c, ldc = _mat(C)
    _check(_lib.spamm_multiply(plan, a, lda, b, ldb, c, ldc, int(flags), _stream(stream)))


def spamm_run(plan, A, B, C, stream=None) -> None:
    a, lda = _mat(A)
    b, ldb = _mat(B)
    c, ldc = _mat(C)
    _check(_lib.spamm_run(plan, a, lda, b, ldb, c, ldc, _stream(stream)))


# ---------------------------------------------------------- chained SpAMM ---
def spamm_multiply_chain(plan, A, B, C, C_low=None, flags: int = SPAMM_MUL_OUTPUT_NORMS, stream=None) -> None:
    a, lda = _mat(A)
    b, ldb = _mat(B)
    c, ldc = _mat(C)
    cl, ldcl = _mat(C_low)
    _check(_lib.spamm_multiply_chain(plan, a, lda, b, ldb, c, ldc, cl, ldcl, int(flags), _stream(stream)))


def spamm_get_output_norms(plan):
    """nC [BM, BN] float64 copy of the last chained multiply's output tile norms."""
    st = spamm_get_stats(plan)
    d = ctypes.c_void_p()
    _check(_lib.spamm_get_output_norms(plan, ctypes.byref(d)))
    torch.cuda.synchronize()
    return _view(d.value, (st["BM"], st["BN"]), "<f8", torch.float64)


def spamm_set_norms(plan, nA, nB, stream=None) -> None:
    """Stage 1 from device float64 maps nA [BM, BK] and nB [BK, BN] (contiguous)."""
    nA, nB = nA.contiguous(), nB.contiguous()
    _check(_lib.spamm_set_norms(plan, ctypes.c_void_p(nA.data_ptr()), ctypes.c_void_p(nB.data_ptr()),
                                _stream(stream)))


# ------------------------------------------------------- convolution drop-in ---
def spamm_conv2d_im2col(plan, W, X, Y, kh: int = 3, kw: int = 3, stride: int = 1, pad: int = 1,
                        stream=None) -> None:
    """Y = SpAMM(W, im2col(X)) (Sec. 4.3.2).  X: contiguous (batch, C_in, H, W) CUDA tensor."""
    if X.dim() != 4 or not X.is_contiguous():
        raise ValueError("X must be a contiguous NCHW tensor")
    w, ldw = _mat(W)
    y, ldy = _mat(Y)
    nb, ci, h, wd = X.shape
    _check(_lib.spamm_conv2d_im2col(plan, w, ldw, ctypes.c_void_p(X.data_ptr()), nb, ci, h, wd, kh, kw, stride, pad,
                                    y, ldy, _stream(stream)))


# -------------------------------------------------------------- tau search ---
def spamm_count_kept(plan, tau: float, stream=None) -> int:
    out = ctypes.c_int64()
    _check(_lib.spamm_count_kept(plan, float(tau), ctypes.byref(out), _stream(stream)))
    return out.value


def spamm_tau_search(plan, target: float, tol: float = 0.01, max_iter: int = 20,
                     stream=None) -> tuple[float, float, int]:
    """Sec. 3.5.2 search; returns (tau, valid_ratio, iterations)."""
    t, vr, it = ctypes.c_double(), ctypes.c_double(), ctypes.c_int32()
    _check(_lib.spamm_tau_search(plan, float(target), float(tol), int(max_iter), ctypes.byref(t),
                                 ctypes.byref(vr), ctypes.byref(it), _stream(stream)))
    return t.value, vr.value, it.value


# -------------------------------------------------------------- multi-GPU ---
def spamm_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.spamm_nccl_unique_id(buf))
    return buf.raw


def spamm_nccl_comm_init(nranks: int, rank: int, uid: bytes) -> ctypes.c_void_p:
    comm = ctypes.c_void_p()
    _check(_lib.spamm_nccl_comm_init(ctypes.byref(comm), int(nranks), int(rank), uid))
    return comm


def spamm_nccl_comm_destroy(comm) -> None:
    _check(_lib.spamm_nccl_comm_destroy(comm))


def spamm_partition_rows(row_work, nranks: int) -> list[int]:
    w = (ctypes.c_int64 * len(row_work))(*[int(x) for x in row_work])
    out = (ctypes.c_int64 * (nranks + 1))()
    _check(_lib.spamm_partition_rows(w, len(row_work), int(nranks), out))
    return list(out)


def spamm_multiply_mgpu(plan, comm, rank: int, nranks: int, A, B, C, flags: int = 0, stream=None) -> None:
    a, lda = _mat(A)
    b, ldb = _mat(B)
    c, ldc = _mat(C)
    _check(_lib.spamm_multiply_mgpu(plan, comm, int(rank), int(nranks), a, lda, b, ldb, c, ldc, int(flags),
                                    _stream(stream)))


def spamm_multiply_mgpu_local(plans, A, B, Cs, flags: int = 0, stream=None) -> None:
    """nranks = len(plans) ranks of spamm_multiply_mgpu emulated on one GPU (verification)."""
    n = len(plans)
    a, lda = _mat(A)
    b, ldb = _mat(B)
    ptrs = [_mat(c) for c in Cs]
    if len({ld for _, ld in ptrs}) != 1:
        raise ValueError("all C buffers must share one leading dimension")
    hp = (ctypes.c_void_p * n)(*[p.value if isinstance(p, ctypes.c_void_p) else p for p in plans])
    cp = (ctypes.c_void_p * n)(*[c.value for c, _ in ptrs])
    _check(_lib.spamm_multiply_mgpu_local(hp, n, a, lda, b, ldb, cp, ptrs[0][1], int(flags), _stream(stream)))


# ---------------------------------------------------------- introspection ---
class _DevArray:
    """__cuda_array_interface__ view of plan-owned device memory (for torch.as_tensor)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(int(s) for s in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2, "strides": None}


def _view(ptr, shape, typestr, dtype):
    n = 1
    for s in shape:
        n *= int(s)
    if n == 0:
        return torch.zeros(shape, dtype=dtype, device="cuda")
    return torch.as_tensor(_DevArray(ptr, shape, typestr), device="cuda").clone()


def spamm_get_norms(plan):
    """(nA [BM,BK], nB^T [BN,BK]) float64 copies."""
    a, bt = ctypes.c_void_p(), ctypes.c_void_p()
    BM, BK, BN = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.spamm_get_norms(plan, ctypes.byref(a), ctypes.byref(bt), ctypes.byref(BM), ctypes.byref(BK),
                                ctypes.byref(BN)))
    torch.cuda.synchronize()
    return (_view(a.value, (BM.value, BK.value), "<f8", torch.float64),
            _view(bt.value, (BN.value, BK.value), "<f8", torch.float64))


def spamm_get_skipmap(plan):
    """(tile_start int64 [BM*BN], k_idx int32 [n]) copies: the k list of C tile t is
    k_idx[tile_start[t] : tile_start[t] + V[t]] (V from spamm_get_counts).  k_idx covers
    the storage in use (lists may sit in fixed per-tile regions)."""
    st = spamm_get_stats(plan)
    tp, ki = ctypes.c_void_p(), ctypes.c_void_p()
    kept = ctypes.c_int64()
    _check(_lib.spamm_get_skipmap(plan, ctypes.byref(tp), ctypes.byref(ki), ctypes.byref(kept)))
    start = _view(tp.value, (st["BM"] * st["BN"],), "<i8", torch.int64)
    V = spamm_get_counts(plan)[0].reshape(-1)
    n = int((start + V).max().item()) if V.numel() else 0
    k = _view(ki.value, (n,), "<u2", torch.uint16) if n else torch.zeros(0, dtype=torch.uint16, device="cuda")
    return start, k.to(torch.int32)


def spamm_get_counts(plan):
    """(V int64 [BM,BN], row_work int64 [BM]) copies."""
    st = spamm_get_stats(plan)
    v, rw = ctypes.c_void_p(), ctypes.c_void_p()
    _check(_lib.spamm_get_counts(plan, ctypes.byref(v), ctypes.byref(rw)))
    return (_view(v.value, (st["BM"], st["BN"]), "<i8", torch.int64),
            _view(rw.value, (st["BM"],), "<i8", torch.int64))


def spamm_get_macro(plan):
    """(start int64 [GM*GN], count int64 [GM*GN], entries [n, 2] int64 (k, mask) over all
    entry storage in use, order int32 [GM*GN], GM, GN); macro-tile t's list is
    entries[start[t] : start[t] + count[t]].  Masks of 8 x 8 groups (the BF16/FP16 path) use
    all 64 bits: view them as uint64."""
    st = spamm_get_stats(plan)
    ps, pc, e, o = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    GM, GN = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.spamm_get_macro(plan, ctypes.byref(ps), ctypes.byref(pc), ctypes.byref(e), ctypes.byref(o),
                                ctypes.byref(GM), ctypes.byref(GN)))
    nmac = GM.value * GN.value
    start = _view(ps.value, (nmac,), "<i8", torch.int64)
    count = _view(pc.value, (nmac,), "<i8", torch.int64)
    n = int((start + count).max().item()) if nmac else 0
    wide = st["macro_i"] * st["macro_j"] > 32   # 8 x 8 tiles: (k, mask_lo, mask_hi, 0) words
    if not n:
        ent = torch.zeros((0, 2), dtype=torch.int64, device="cuda")
    elif wide:
        w = _view(e.value, (n, 4), "<u4", torch.uint32).to(torch.int64)
        ent = torch.stack([w[:, 0], w[:, 1] | (w[:, 2] << 32)], dim=1)   # mask bit 63 wraps to negative int64
    else:
        ent = _view(e.value, (n, 2), "<u4", torch.uint32).to(torch.int64)
    order = _view(o.value, (nmac,), "<i4", torch.int32)
    return start, count, ent, order, GM.value, GN.value


def spamm_get_partition(plan, nranks: int) -> list[int]:
    out = (ctypes.c_int64 * (nranks + 1))()
    _check(_lib.spamm_get_partition(plan, out, int(nranks)))
    return list(out)


def spamm_get_stats(plan) -> dict:
    s = spamm_stats()
    _check(_lib.spamm_get_stats(plan, ctypes.byref(s)))
    return s.as_dict()


def spamm_launch_count() -> int:
    return int(_lib.spamm_launch_count())


# ------------------------------------------------------------- convenience ---
class Plan:
    """RAII wrapper: ``with Plan(M, N, K, tau, "bf16") as p: p.run(A, B, C)``."""

    def __init__(self, M: int, N: int, K: int, tau: float, precision="fp32", tile: int = 32, flags: int = 0):
        self.prec = PREC_OF[precision] if isinstance(precision, str) else int(precision)
        self.handle = spamm_plan_ex(M, N, K, tile, tau, self.prec, flags)
        self.shape = (M, N, K)

    @property
    def dtype(self):
        return DTYPE_OF[self.prec]

    def close(self):
        if self.handle is not None:
            spamm_plan_destroy(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_tau(self, tau):
        spamm_set_tau(self.handle, tau)

    def set_scalars(self, alpha, beta):
        spamm_set_scalars(self.handle, alpha, beta)

    def _check_ops(self, A, B, C=None):
        """Operands against the plan (the C ABI sees only pointers and leading dimensions): a
        float32 tensor given to a bf16 plan would be read as bf16, a short one past its end."""
        M, N, K = self.shape
        for name, t, shape, dt in (("A", A, (M, K), self.dtype), ("B", B, (K, N), self.dtype),
                                   ("C", C, (M, N), torch.float32)):
            if t is None:
                continue
            if not t.is_cuda:
                raise ValueError(f"{name} must be a CUDA tensor")
            if tuple(t.shape) != shape:
                raise ValueError(f"{name} has shape {tuple(t.shape)}, the plan expects {shape}")
            if t.dtype != dt:
                raise ValueError(f"{name} has dtype {t.dtype}, the plan expects {dt}")

    def norms(self, A, B, stream=None):
        self._check_ops(A, B)
        spamm_norms(self.handle, A, B, stream)

    def build_skipmap(self, stream=None):
        spamm_build_skipmap(self.handle, stream)

    def multiply(self, A, B, C, flags=0, stream=None):
        self._check_ops(A, B, C)
        spamm_multiply(self.handle, A, B, C, flags, stream)

    def run(self, A, B, C=None, stream=None):
        if C is None:
            C = torch.empty((self.shape[0], self.shape[1]), dtype=torch.float32, device=A.device)
        self._check_ops(A, B, C)
        spamm_run(self.handle, A, B, C, stream)
        return C

    def stats(self):
        return spamm_get_stats(self.handle)

    def multiply_chain(self, A, B, C, C_low=None, flags=SPAMM_MUL_OUTPUT_NORMS, stream=None):
        self._check_ops(A, B, C)
        spamm_multiply_chain(self.handle, A, B, C, C_low, flags, stream)

    def output_norms(self):
        return spamm_get_output_norms(self.handle)

    def set_norms(self, nA, nB, stream=None):
        spamm_set_norms(self.handle, nA, nB, stream)

    def count_kept(self, tau, stream=None):
        return spamm_count_kept(self.handle, tau, stream)

    def tau_search(self, target, tol=0.01, max_iter=20, stream=None):
        return spamm_tau_search(self.handle, target, tol, max_iter, stream)
