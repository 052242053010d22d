"""Multi-GPU randUTV: thin binding of randutv_factor_dist (include/randutv.h).

Layout: 1-D block-cyclic column blocks of
width b -- global column block j lives on rank j mod P, and a rank stores its
blocks in increasing j as one m x n_loc column-major matrix.  torch.distributed
is plumbing only (exchanging the NCCL unique id, barriers, timing); every
arithmetic step and every data-path collective runs inside the library
(NCCL called from C++ on the factorization's stream).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import (RandUTVError, _check, _Info, _ld, _Opts, _stream, as_colmajor, empty_cm, Info, lib)

c_i64, c_i32, c_vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
NCCL_ID_BYTES = 128


def _lib():
    L = lib()
    if not getattr(L, "_dist_ready", False):
        L.randutv_nccl_unique_id.argtypes = [c_vp]
        L.randutv_comm_init_nccl.argtypes = [c_i32, c_i32, c_vp, ctypes.POINTER(c_vp)]
        L.randutv_comm_init_loopback.argtypes = [c_i32, ctypes.POINTER(c_vp)]
        L.randutv_comm_destroy.argtypes = [c_vp]
        L.randutv_comm_local_ranks.argtypes = [c_vp, ctypes.POINTER(c_i32), ctypes.POINTER(c_i32), c_i32]
        L.randutv_comm_stats.argtypes = [c_vp, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_longlong)]
        L.randutv_dist_local_cols.argtypes = [c_i64, c_i64, c_i32, c_i32]
        L.randutv_dist_local_cols.restype = c_i64
        L.randutv_dist_global_col.argtypes = [c_i64, c_i64, c_i32, c_i32]
        L.randutv_dist_global_col.restype = c_i64
        L.randutv_factor_dist.argtypes = [ctypes.POINTER(_Opts), c_vp, c_i64, c_i64, ctypes.POINTER(c_vp),
                                          ctypes.POINTER(c_i64), c_i64, c_i32, ctypes.c_uint64, c_i64,
                                          ctypes.POINTER(c_vp), ctypes.POINTER(c_i64),
                                          ctypes.POINTER(c_vp), ctypes.POINTER(c_i64),
                                          ctypes.POINTER(c_vp), ctypes.POINTER(c_i64), ctypes.POINTER(_Info)]
        for f in ("randutv_nccl_unique_id", "randutv_comm_init_nccl", "randutv_comm_init_loopback",
                  "randutv_comm_destroy", "randutv_comm_local_ranks", "randutv_factor_dist", "randutv_comm_stats"):
            getattr(L, f).restype = ctypes.c_int
        L._dist_ready = True
    return L


# --------------------------------------------------------------------------- layout (host only)
def local_cols(n: int, b: int, rank: int, nranks: int) -> int:
    """Number of columns of an n-column matrix held by ``rank`` (block-cyclic, width b)."""
    v = _lib().randutv_dist_local_cols(n, b, rank, nranks)
    if v < 0:
        raise ValueError("invalid layout arguments")
    return int(v)


def global_cols(n: int, b: int, rank: int, nranks: int) -> np.ndarray:
    """Global column indices of ``rank``'s local columns, in local order."""
    blocks = np.arange(rank, -(-n // b), nranks)
    if blocks.size == 0:
        return np.zeros(0, dtype=np.int64)
    cols = (blocks[:, None] * b + np.arange(b)[None, :]).reshape(-1)
    return cols[cols < n].astype(np.int64)


def shard(A, b: int, rank: int, nranks: int):
    """Rank ``rank``'s column shard of A (numpy or torch), column-major torch
    tensor on A's device (a copy)."""
    import torch
    cols = global_cols(A.shape[1], b, rank, nranks)
    if isinstance(A, np.ndarray):
        A = torch.from_numpy(np.ascontiguousarray(A))
    idx = torch.as_tensor(cols, device=A.device)
    S = A.index_select(1, idx)
    return S.t().contiguous().t()


def assemble(shards, n: int, b: int):
    """Full matrix from the P shards (list in rank order) -- test/harness helper."""
    import torch
    P = len(shards)
    m = shards[0].shape[0]
    out = torch.empty(n, m, dtype=shards[0].dtype, device=shards[0].device).t()
    for r, S in enumerate(shards):
        cols = global_cols(n, b, r, P)
        if cols.size:
            out[:, torch.as_tensor(cols, device=out.device)] = S
    return out


# --------------------------------------------------------------------------- communicators
class Comm:
    """A randutv_comm handle (NCCL or loopback)."""

    def __init__(self, handle: int):
        self.h = c_vp(handle)
        L = _lib()
        world = c_i32(0)
        ranks = (c_i32 * 4096)()
        nl = L.randutv_comm_local_ranks(self.h, ctypes.byref(world), ranks, 4096)
        if nl < 0:
            raise RandUTVError(nl, "randutv_comm_local_ranks")
        self.world = int(world.value)
        self.ranks = [int(ranks[i]) for i in range(nl)]

    def stats(self) -> dict:
        """Collectives issued so far and their payload per rank (bytes):
        {"allreduce": (count, bytes), "bcast": ..., "allgather": ..., "aborted": bool}."""
        cnt = (ctypes.c_longlong * 3)()
        byt = (ctypes.c_longlong * 3)()
        rc = _lib().randutv_comm_stats(self.h, cnt, byt)
        if rc < 0:
            raise RandUTVError(rc, "randutv_comm_stats")
        out = {k: (int(cnt[i]), int(byt[i])) for i, k in enumerate(("allreduce", "bcast", "allgather"))}
        out["aborted"] = rc != 0
        return out

    def close(self):
        if self.h:
            _lib().randutv_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def loopback(nranks: int) -> Comm:
    """All ``nranks`` ranks driven by this process on the current device."""
    h = c_vp()
    _check(_lib().randutv_comm_init_loopback(nranks, ctypes.byref(h)), "randutv_comm_init_loopback")
    return Comm(h.value)


def nccl_from_torch(group=None) -> Comm:
    """NCCL communicator over the ranks of an initialised torch.distributed
    group (one process per GPU; call after torch.cuda.set_device).  Rank 0
    creates the unique id; torch.distributed broadcasts it (plumbing)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    buf = torch.zeros(NCCL_ID_BYTES, dtype=torch.uint8)
    if rank == 0:
        raw = (ctypes.c_ubyte * NCCL_ID_BYTES)()
        _check(_lib().randutv_nccl_unique_id(raw), "randutv_nccl_unique_id")
        buf = torch.tensor(list(raw), dtype=torch.uint8)
    dev = buf.cuda() if dist.get_backend(group) == "nccl" else buf
    dist.broadcast(dev, src=0, group=group)
    raw = (ctypes.c_ubyte * NCCL_ID_BYTES)(*dev.cpu().tolist())
    h = c_vp()
    _check(_lib().randutv_comm_init_nccl(world, rank, raw, ctypes.byref(h)), "randutv_comm_init_nccl")
    return Comm(h.value)


# --------------------------------------------------------------------------- the factorization
def factor(comm: Comm, shards, m: int, n: int, b: int, q: int, seed: int, k_stop: int = 0, tol: float = 0.0,
           reortho: bool = True, qr_mode: int = 0, out=None, stream=None, with_uv: bool = False,
           oversample: int = 0):
    """Distributed A = U T V^T.  ``shards``: one column-major CUDA tensor per
    rank driven by ``comm`` (comm.ranks order), rank r's shard being
    m x local_cols(n, b, r, P).  Returns (T shards, Info), or with ``with_uv``
    (U shards, T shards, V shards, Info) -- U's shard of rank r is
    m x local_cols(m, b, r, P), V's n x local_cols(n, b, r, P)."""
    L = _lib()
    nl = len(comm.ranks)
    assert len(shards) == nl, "one shard per local rank"
    shards = [as_colmajor(S) for S in shards]
    if out is None:
        out = [empty_cm(m, S.shape[1], S.device) for S in shards]
    Ap = (c_vp * nl)(*[S.data_ptr() for S in shards])
    lda = (c_i64 * nl)(*[_ld(S) for S in shards])
    Tp = (c_vp * nl)(*[T.data_ptr() for T in out])
    ldt = (c_i64 * nl)(*[_ld(T) for T in out])
    Up = Vp = ldu = ldv = None
    if with_uv:
        bb = min(int(b), n)
        Us = [empty_cm(m, max(local_cols(m, bb, r, comm.world), 1), S.device) for r, S in zip(comm.ranks, shards)]
        Vs = [empty_cm(n, max(local_cols(n, bb, r, comm.world), 1), S.device) for r, S in zip(comm.ranks, shards)]
        Up = (c_vp * nl)(*[U.data_ptr() for U in Us])
        Vp = (c_vp * nl)(*[V.data_ptr() for V in Vs])
        ldu = (c_i64 * nl)(*[_ld(U) for U in Us])
        ldv = (c_i64 * nl)(*[_ld(V) for V in Vs])
    opts = _Opts(stream=_stream(stream, shards[0].device).value, tol=float(tol), no_reortho=0 if reortho else 1,
                 qr_mode=int(qr_mode), oversample=int(oversample))
    info = _Info()
    rc = L.randutv_factor_dist(ctypes.byref(opts), comm.h, m, n, Ap, lda, int(b), int(q), int(seed) & (2**64 - 1),
                               int(k_stop), Up, ldu, Tp, ldt, Vp, ldv, ctypes.byref(info))
    _check(rc, "randutv_factor_dist")
    inf = Info(info.k_done, info.steps, bool(info.final_block), info.max_sweeps, info.trailing_fro, info.a_fro,
               info.qr_fallbacks)
    if with_uv:
        Us = [U[:, :local_cols(m, min(int(b), n), r, comm.world)] for r, U in zip(comm.ranks, Us)]
        Vs = [V[:, :local_cols(n, min(int(b), n), r, comm.world)] for r, V in zip(comm.ranks, Vs)]
        return Us, out, Vs, inf
    return out, inf
