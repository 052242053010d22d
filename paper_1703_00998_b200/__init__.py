"""B200-native randUTV (arXiv 1703.00998): thin Python binding of the C ABI.

Argument marshalling only: every step of the factorization runs in the sm_100a
kernels of ``_randutv.so`` (built from ``csrc/`` by ``build.py``).  There is no
CPU fallback -- importing a function that needs the library raises if the
library is missing or cannot be loaded.

Matrices are column-major.  A torch tensor ``X`` of shape (r, c) is accepted
as-is when its strides are (1, ld >= r) -- e.g. ``X = Xt.t()`` for a
contiguous ``Xt`` of shape (c, r); other layouts are copied to column-major.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import flops  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("RANDUTV_LIB") or os.path.join(_HERE, "_randutv.so")
_lib = None

c_i64, c_i32, c_u64, c_u32, c_dbl, c_vp = (ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint32,
                                           ctypes.c_double, ctypes.c_void_p)


class RandUTVError(RuntimeError):
    def __init__(self, code: int, where: str):
        msg = lib().randutv_strerror(code).decode() if _lib is not None else str(code)
        super().__init__(f"{where}: randutv error {code}: {msg}")
        self.code = code


class _Opts(ctypes.Structure):
    _fields_ = [("stream", c_vp), ("tol", c_dbl), ("no_reortho", c_i32), ("qr_mode", c_i32),
                ("workspace", c_vp), ("workspace_bytes", ctypes.c_size_t), ("oversample", c_i32),
                ("reserved1", c_i32)]


class _Info(ctypes.Structure):
    _fields_ = [("k_done", c_i64), ("steps", c_i32), ("final_block", c_i32), ("max_sweeps", c_i32),
                ("qr_fallbacks", c_i32), ("trailing_fro", c_dbl), ("a_fro", c_dbl)]


@dataclass
class Info:
    k_done: int
    steps: int
    final_block: bool
    max_sweeps: int
    trailing_fro: float
    a_fro: float
    qr_fallbacks: int = 0


def lib():
    """Load (building first if stale and nvcc exists) the CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH) or os.environ.get("RANDUTV_REBUILD"):
        from .build import build
        build()
    L = ctypes.CDLL(_LIB_PATH)
    L.randutv_factor_ex.argtypes = [ctypes.POINTER(_Opts), c_i64, c_i64, c_vp, c_i64, c_i64, c_i32, c_u64, c_i64,
                                    c_vp, c_vp, c_vp, ctypes.POINTER(_Info)]
    L.randutv_factor_ex.restype = ctypes.c_int
    L.randutv_factor.argtypes = [c_i64, c_i64, c_vp, c_i64, c_i64, c_i32, c_u64, c_i64, c_vp, c_vp, c_vp]
    L.randutv_factor.restype = ctypes.c_int
    L.randutv_workspace_size.argtypes = [c_i64, c_i64, c_i64, c_i32, c_i32]
    L.randutv_workspace_size.restype = ctypes.c_size_t
    L.randutv_workspace_size_ex.argtypes = [c_i64, c_i64, c_i64, c_i32, c_i32, c_i32]
    L.randutv_workspace_size_ex.restype = ctypes.c_size_t
    L.randutv_strerror.argtypes = [ctypes.c_int]
    L.randutv_strerror.restype = ctypes.c_char_p
    L.randutv_version.restype = ctypes.c_char_p
    L.randutv_gaussian.argtypes = [c_vp, c_i64, c_i64, c_i64, c_u64, c_u32, c_u32, c_vp]
    L.randutv_rsvd.argtypes = [ctypes.POINTER(_Opts), c_i64, c_i64, c_vp, c_i64, c_i64, c_i32, c_u64, c_vp, c_i64,
                               c_vp, c_vp, c_i64]
    L.randutv_rsvd.restype = ctypes.c_int
    L.randutv_dgemm.argtypes = [c_i32, c_i32, c_i64, c_i64, c_i64, c_dbl, c_vp, c_i64, c_vp, c_i64, c_dbl, c_vp,
                                c_i64, c_vp]
    L.randutv_panel_qr.argtypes = [c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp]
    L.randutv_panel_qr_ex.argtypes = [c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_i64, c_i32,
                                      ctypes.POINTER(c_i32), c_vp]
    L.randutv_small_svd_batched.argtypes = [c_i32, c_i32, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]
    L.randutv_launch_count.restype = ctypes.c_longlong
    L.randutv_profile_begin.restype = ctypes.c_int
    L.randutv_profile_end.argtypes = [c_vp, c_vp, c_vp]
    L.randutv_profile_end.restype = ctypes.c_int
    L.randutv_profile_timeline.argtypes = [c_vp, ctypes.c_longlong]
    L.randutv_profile_timeline.restype = ctypes.c_longlong
    L.randutv_profile_class_name.argtypes = [ctypes.c_int]
    L.randutv_profile_class_name.restype = ctypes.c_char_p
    for f in ("randutv_gaussian", "randutv_dgemm", "randutv_panel_qr", "randutv_panel_qr_ex",
              "randutv_small_svd_batched"):
        getattr(L, f).restype = ctypes.c_int
    _lib = L
    return L


EXPORTED = ["randutv_factor", "randutv_factor_ex", "randutv_workspace_size", "randutv_workspace_size_ex",
            "randutv_strerror",
            "randutv_version", "randutv_gaussian", "randutv_dgemm", "randutv_panel_qr", "randutv_panel_qr_ex",
            "randutv_small_svd_batched", "randutv_launch_count", "randutv_profile_begin",
            "randutv_profile_end", "randutv_profile_class_name", "randutv_profile_timeline", "randutv_nccl_unique_id",
            "randutv_comm_init_nccl", "randutv_comm_init_loopback", "randutv_comm_destroy",
            "randutv_comm_local_ranks", "randutv_dist_local_cols", "randutv_dist_global_col",
            "randutv_factor_dist", "randutv_rsvd", "randutv_comm_stats"]


def launch_count() -> int:
    """Kernel launches issued by the library since load."""
    return int(lib().randutv_launch_count())


def profile_begin():
    _check(lib().randutv_profile_begin(), "randutv_profile_begin")


def profile_end() -> dict:
    """Per-class event time (ms), algorithmic flops and launches since profile_begin()."""
    L = lib()
    ms = (ctypes.c_double * 16)()
    fl = (ctypes.c_double * 16)()
    ln = (ctypes.c_longlong * 16)()
    _check(L.randutv_profile_end(ms, fl, ln), "randutv_profile_end")
    out = {}
    for i in range(16):
        name = L.randutv_profile_class_name(i)
        if name is None:
            break
        out[name.decode()] = {"ms": ms[i], "flops": fl[i], "launches": ln[i]}
    return out


def profile_timeline():
    """Per-launch (class name, stream slot, start ms, end ms) of the last profile window."""
    L = lib()
    n = L.randutv_profile_timeline(None, 0)
    buf = (ctypes.c_double * (4 * max(n, 1)))()
    L.randutv_profile_timeline(buf, n)
    names = {}
    out = []
    for i in range(n):
        c = int(buf[4 * i])
        if c not in names:
            nm = L.randutv_profile_class_name(c)
            names[c] = nm.decode() if nm else str(c)
        out.append((names[c], int(buf[4 * i + 1]), buf[4 * i + 2], buf[4 * i + 3]))
    return out


# --------------------------------------------------------------------------- layout helpers
def _torch():
    import torch
    return torch


def empty_cm(rows: int, cols: int, device="cuda"):
    """Uninitialised column-major fp64 (rows x cols) tensor."""
    torch = _torch()
    return torch.empty(cols, rows, dtype=torch.float64, device=device).t()


def as_colmajor(X):
    """Column-major fp64 view (or copy) of a torch tensor."""
    torch = _torch()
    if X.dtype != torch.float64:
        X = X.to(torch.float64)
    r, c = X.shape
    if X.stride(0) == 1 and (c <= 1 or X.stride(1) >= max(r, 1)):
        return X
    return X.t().contiguous().t()


def _ld(X) -> int:
    r, c = X.shape
    return max(int(X.stride(1)) if c > 1 else r, r, 1)


def _stream(stream, device=None):
    """cudaStream_t of ``stream`` (a torch.cuda.Stream or a raw handle); None:
    torch's current stream."""
    if stream is not None:
        return ctypes.c_void_p(int(getattr(stream, "cuda_stream", stream)))
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _check(rc: int, where: str):
    if rc != 0:
        raise RandUTVError(rc, where)


# --------------------------------------------------------------------------- the factorization
def randutv(A, b: int, q: int, seed: int, k_stop: int = 0, tol: float = 0.0, reortho: bool = True,
            with_uv: bool = True, stream=None, out=None, qr_mode: int = 0, oversample: int = 0):
    """A = U T V^T (Fig. fig:randUTV) on the GPU.

    ``A``: torch CUDA tensor (m x n, m >= n) or a numpy array (host buffers,
    staged through device memory inside the C call).  Returns (U, T, V, info);
    U = V = None when ``with_uv`` is False (the paper's "no orthonormal
    matrices" mode).  ``out`` = (U, T, V) preallocated column-major tensors.
    """
    L = lib()
    if isinstance(A, np.ndarray):
        return _randutv_host(A, b, q, seed, k_stop, tol, reortho, with_uv, qr_mode, oversample)
    torch = _torch()
    A = as_colmajor(A)
    m, n = A.shape
    if out is not None:
        U, T, V = out
    else:
        T = empty_cm(m, n, A.device)
        U = empty_cm(m, m, A.device) if with_uv else None
        V = empty_cm(n, n, A.device) if with_uv else None
    opts = _Opts(stream=_stream(stream, A.device).value, tol=float(tol), no_reortho=0 if reortho else 1,
                 qr_mode=int(qr_mode), oversample=int(oversample))
    info = _Info()
    rc = L.randutv_factor_ex(ctypes.byref(opts), m, n, A.data_ptr(), _ld(A), int(b), int(q), int(seed) & (2**64 - 1),
                             int(k_stop), U.data_ptr() if U is not None else None, T.data_ptr(),
                             V.data_ptr() if V is not None else None, ctypes.byref(info))
    _check(rc, "randutv_factor_ex")
    del torch
    return U, T, V, Info(info.k_done, info.steps, bool(info.final_block), info.max_sweeps, info.trailing_fro,
                         info.a_fro, info.qr_fallbacks)


def _randutv_host(A: np.ndarray, b, q, seed, k_stop, tol, reortho, with_uv, qr_mode=0, oversample=0):
    L = lib()
    A = np.asfortranarray(A, dtype=np.float64)
    m, n = A.shape
    T = np.empty((m, n), order="F")
    U = np.empty((m, m), order="F") if with_uv else None
    V = np.empty((n, n), order="F") if with_uv else None
    opts = _Opts(stream=None, tol=float(tol), no_reortho=0 if reortho else 1, qr_mode=int(qr_mode),
                 oversample=int(oversample))
    info = _Info()
    p = lambda X: X.ctypes.data if X is not None else None  # noqa: E731
    rc = L.randutv_factor_ex(ctypes.byref(opts), m, n, p(A), m, int(b), int(q), int(seed) & (2**64 - 1),
                             int(k_stop), p(U), p(T), p(V), ctypes.byref(info))
    _check(rc, "randutv_factor_ex(host)")
    return U, T, V, Info(info.k_done, info.steps, bool(info.final_block), info.max_sweeps, info.trailing_fro,
                         info.a_fro, info.qr_fallbacks)


def factor_raw(m, n, A_ptr, lda, b, q, seed, k_stop, U_ptr, T_ptr, V_ptr) -> int:
    """Direct randutv_factor call on raw pointers (host or device)."""
    return lib().randutv_factor(m, n, A_ptr, lda, b, q, seed, k_stop, U_ptr, T_ptr, V_ptr)


def rsvd(A, b: int, q: int, seed: int, oversample: int = 0, reortho: bool = True, qr_mode: int = 0, stream=None):
    """Randomized SVD (Remark remark:RSVD): A ~ U diag(D) V^T, rank b.  Returns (U, D, V)."""
    torch = _torch()
    A = as_colmajor(A)
    m, n = A.shape
    U = empty_cm(m, b, A.device)
    V = empty_cm(n, b, A.device)
    D = torch.empty(b, dtype=torch.float64, device=A.device)
    opts = _Opts(stream=_stream(stream, A.device).value, no_reortho=0 if reortho else 1, qr_mode=int(qr_mode),
                 oversample=int(oversample))
    _check(lib().randutv_rsvd(ctypes.byref(opts), m, n, A.data_ptr(), _ld(A), int(b), int(q),
                              int(seed) & (2**64 - 1), U.data_ptr(), _ld(U), D.data_ptr(), V.data_ptr(), _ld(V)),
           "randutv_rsvd")
    return U, D, V


def workspace_size(m, n, b, q, with_uv=True) -> int:
    return int(lib().randutv_workspace_size(m, n, b, q, 1 if with_uv else 0))


# --------------------------------------------------------------------------- components
def gaussian(rows: int, cols: int, seed: int, step: int, purpose: int = 0, device="cuda", stream=None):
    """G (rows x cols) of step ``step`` (0-based), PAPER.md:941 (R2)."""
    G = empty_cm(rows, cols, device)
    _check(lib().randutv_gaussian(G.data_ptr(), _ld(G), rows, cols, int(seed) & (2**64 - 1), step, purpose,
                                  _stream(stream)), "randutv_gaussian")
    return G


def dgemm(transa: bool, transb: bool, alpha: float, A, B, beta: float, C, stream=None):
    """C = alpha op(A) op(B) + beta C in place (DMMA kernels); returns C."""
    A, B = as_colmajor(A), as_colmajor(B)
    assert C.stride(0) == 1, "C must be column-major"
    M, N = C.shape
    K = A.shape[0] if transa else A.shape[1]
    _check(lib().randutv_dgemm(1 if transa else 0, 1 if transb else 0, M, N, K, float(alpha), A.data_ptr(), _ld(A),
                               B.data_ptr(), _ld(B), float(beta), C.data_ptr(), _ld(C), _stream(stream)),
           "randutv_dgemm")
    return C


def panel_qr(P, stream=None, mode: int = 0, return_fallback: bool = False):
    """Householder QR of an m x b panel (copied).  Returns (V, R, tau, Tw) with
    H_1...H_b = I - V Tw V^T and P = (I - V Tw V^T)[:, :b] R.  mode 0:
    CholeskyQR2 + Householder reconstruction (Householder fallback); mode 1:
    column-by-column Householder.  return_fallback adds whether the fallback ran."""
    torch = _torch()
    m, b = P.shape
    V = empty_cm(m, b, P.device)
    V.copy_(P)
    R = empty_cm(b, b, P.device)
    Tw = empty_cm(b, b, P.device)
    tau = torch.empty(b, dtype=torch.float64, device=P.device)
    fb = c_i32(0)
    _check(lib().randutv_panel_qr_ex(m, b, V.data_ptr(), _ld(V), R.data_ptr(), _ld(R), tau.data_ptr(),
                                     Tw.data_ptr(), _ld(Tw), int(mode), ctypes.byref(fb), _stream(stream)),
           "randutv_panel_qr_ex")
    if return_fallback:
        return V, R, tau, Tw, bool(fb.value)
    return V, R, tau, Tw


def small_svd_batched(R, stream=None):
    """R: (batch, k, k) torch tensor of matrices (each taken as given, i.e.
    R[i] is the k x k matrix).  Returns (D, Us, Vs, sweeps) with
    R[i] = Us[i] diag(D[i]) Vs[i]^T."""
    torch = _torch()
    batch, k, _ = R.shape
    Rc = R.transpose(1, 2).contiguous()  # column-major blocks: Rc[i] stored = R[i]^T row-major
    D = torch.empty(batch, k, dtype=torch.float64, device=R.device)
    Us = torch.empty(batch, k, k, dtype=torch.float64, device=R.device)
    Vs = torch.empty(batch, k, k, dtype=torch.float64, device=R.device)
    sw = torch.zeros(batch, dtype=torch.int32, device=R.device)
    _check(lib().randutv_small_svd_batched(batch, k, Rc.data_ptr(), k, k * k, D.data_ptr(), Us.data_ptr(),
                                           Vs.data_ptr(), sw.data_ptr(), _stream(stream)),
           "randutv_small_svd_batched")
    # blocks were written column-major: transpose back to (row, col) indexing
    return D, Us.transpose(1, 2), Vs.transpose(1, 2), sw
