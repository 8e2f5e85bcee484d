"""Thin ctypes binding of libknng.so (include/knng.h) -- argument marshalling
only.  Every step of the GNND path runs in the library's CUDA kernels; this
module turns torch tensors (device memory, PyTorch is plumbing here) and
numpy arrays (host buffers) into pointers and raises on a non-OK status.

There is no CPU fallback: if the shared library is missing or fails to load,
importing the binding raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libknng.so")

KNNG_OK, KNNG_E_USAGE, KNNG_E_DOMAIN, KNNG_E_NOMEM, KNNG_E_CUDA, KNNG_E_NCCL, KNNG_E_INTERNAL = range(7)
KNNG_L2SQ, KNNG_COSINE, KNNG_CHI2 = 0, 1, 2
KNNG_F32, KNNG_U8 = 0, 1
METRICS = {"l2": KNNG_L2SQ, "l2sq": KNNG_L2SQ, "cosine": KNNG_COSINE, "chi2": KNNG_CHI2}


class KnngError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


_STATUS = {0: "KNNG_OK", 1: "KNNG_E_USAGE", 2: "KNNG_E_DOMAIN", 3: "KNNG_E_NOMEM",
           4: "KNNG_E_CUDA", 5: "KNNG_E_NCCL", 6: "KNNG_E_INTERNAL"}


class IterStats(C.Structure):
    _fields_ = [("joins", C.c_int64), ("sum_m", C.c_int64), ("sum_q", C.c_int64),
                ("dist_evals", C.c_int64), ("candidates", C.c_int64), ("appended", C.c_int64),
                ("accepted", C.c_int64), ("rows", C.c_int64), ("recomputed", C.c_int64)]

    def as_dict(self) -> dict:
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


# (name, restype, argtypes) of every exported symbol; tests check this list
# against include/knng.h.
P, i32, i64, u32, u64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_size_t
SIGNATURES = [
    ("knng_build_workspace_bytes", sz, [i32, i64, i32, i32, i32, i32]),
    ("knng_build", i32, [P, i32, i64, i32, i32, i32, i32, i32, u64, P, P, P, sz, P]),
    ("knng_build_host", i32, [P, i32, i64, i32, i32, i32, i32, i32, u64, P, P, P]),
    ("knng_merge_workspace_bytes", sz, [i32, i64, i64, i32, i32, i32, i32]),
    ("knng_merge", i32, [P, i64, P, P, P, i64, P, P, i32, i32, i32, i32, i32, i32, i32, u64, P, P, P, sz, P]),
    ("knng_extend", i32, [P, i64, P, P, P, i64, i32, i32, i32, i32, i32, i32, i32, u64, P, P, P]),
    ("knng_get_unique_id", i32, [P]),
    ("knng_comm_init", i32, [i32, i32, P, P]),
    ("knng_comm_init_local", i32, [i32, P]),
    ("knng_comm_destroy", i32, [P]),
    ("knng_build_sharded", i32, [P, P, i64, i64, i64, i32, i32, i32, i32, i32, i32, P, i32, u64, P, P, P]),
    ("knng_bruteforce", i32, [P, i32, i64, i32, i32, P, i64, i32, P, P, P]),
    ("knng_build_ooc", i32, [P, i32, i64, i32, i32, i32, i32, i32, i32, u64, i32, P, P, P]),
    ("knng_debug_init", i32, [P, i32, i64, i32, i32, i32, u64, P, P, P]),
    ("knng_debug_iterate", i32, [P, i32, i64, i32, i32, i32, i32, u32, u64, i64, P, P, P, P, sz, P]),
    ("knng_debug_sample", i32, [i64, i32, i32, u32, u64, P, P, P, P, P, P, P, sz, P]),
    ("knng_debug_philox", i32, [P, i64, u64, P, P]),
    ("knng_set_option", i32, [C.c_char_p, i64]),
    ("knng_get_option", i32, [C.c_char_p, P]),
    ("knng_last_stats", i32, [P, i32]),
    ("knng_launch_count", i64, []),
    ("knng_set_timing", None, [i32]),
    ("knng_reset_timing", None, []),
    ("knng_kernel_time", i32, [C.c_char_p, P, P]),
    ("knng_last_error", C.c_char_p, []),
    ("knng_status_string", C.c_char_p, [i32]),
    ("knng_abi_version", i32, []),
]

_lib = None


def lib():
    """Load libknng.so (raises if it is missing: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `make` or __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int):
    if status != KNNG_OK:
        raise KnngError(status, lib().knng_last_error().decode())


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _dtype_code(t) -> int:
    name = str(t.dtype)
    if name.endswith("float32"):
        return KNNG_F32
    if name.endswith("uint8"):
        return KNNG_U8
    raise TypeError(f"vectors must be float32 or uint8, got {t.dtype}")


def _metric(metric) -> int:
    return METRICS[metric] if isinstance(metric, str) else int(metric)


def _workspace(nbytes: int, device):
    import torch
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)


# ------------------------------------------------------------------ build
def knng_build_workspace_bytes(dtype: int, n: int, d: int, k: int, sample_size: int, metric="l2") -> int:
    return int(lib().knng_build_workspace_bytes(dtype, n, d, k, sample_size, _metric(metric)))


def knng_build(vectors, k: int, iters: int, sample_size: int, seed: int = 0, metric="l2",
               out_ids=None, out_dists=None, workspace=None, stream=None):
    """GNND build (Alg. 1) on a CUDA tensor [n, d] (float32 or uint8).
    Returns (ids u32-as-int32 tensor [n, k], dists float32 [n, k])."""
    import torch
    assert vectors.is_cuda and vectors.is_contiguous() and vectors.dim() == 2
    n, d = vectors.shape
    dt = _dtype_code(vectors)
    if out_ids is None:
        out_ids = torch.empty((n, k), dtype=torch.int32, device=vectors.device)
    if out_dists is None:
        out_dists = torch.empty((n, k), dtype=torch.float32, device=vectors.device)
    ws_ptr, ws_bytes = None, 0
    if workspace is not None:
        ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    _check(lib().knng_build(_ptr(vectors), dt, n, d, k, _metric(metric), iters, sample_size, seed,
                            _ptr(out_ids), _ptr(out_dists), ws_ptr, ws_bytes, _stream(stream)))
    return out_ids, out_dists


def knng_build_host(vectors: np.ndarray, k: int, iters: int, sample_size: int, seed: int = 0,
                    metric="l2", out_ids=None, out_dists=None, stream=None):
    """End-to-end build from HOST buffers (copies in, builds, copies out)."""
    assert vectors.flags.c_contiguous and vectors.ndim == 2
    n, d = vectors.shape
    if out_ids is None:
        out_ids = np.empty((n, k), np.uint32)
    if out_dists is None:
        out_dists = np.empty((n, k), np.float32)
    _check(lib().knng_build_host(_ptr(vectors), _dtype_code(vectors), n, d, k, _metric(metric), iters,
                                 sample_size, seed, _ptr(out_ids), _ptr(out_dists), _stream(stream)))
    return out_ids, out_dists


def knng_build_ooc(vectors: np.ndarray, k: int, iters: int, merge_iters: int, sample_size: int, shards: int,
                   seed: int = 0, metric="l2", out_ids=None, out_dists=None, stream=None):
    """The paper's out-of-memory construction from HOST buffers:
    GNND per shard, GGM of every pair of sub-graphs, running top-k lists."""
    assert vectors.flags.c_contiguous and vectors.ndim == 2
    n, d = vectors.shape
    if out_ids is None:
        out_ids = np.empty((n, k), np.uint32)
    if out_dists is None:
        out_dists = np.empty((n, k), np.float32)
    _check(lib().knng_build_ooc(_ptr(vectors), _dtype_code(vectors), n, d, k, _metric(metric), iters, merge_iters,
                                sample_size, seed, shards, _ptr(out_ids), _ptr(out_dists), _stream(stream)))
    return out_ids, out_dists


def knng_merge(vecA, idsA, distsA, vecB, idsB, distsB, k: int, merge_iters: int, sample_size: int,
               seed: int = 0, level: int = 0, metric="l2", workspace=None, stream=None):
    """GGM (Alg. 3): returns (ids, dists) [nA + nB, k]; B ids re-based by nA."""
    import torch
    nA, d = vecA.shape
    nB = vecB.shape[0]
    dt = _dtype_code(vecA)
    # the C side trusts these shapes (it copies nB * d elements of vecB and
    # reads k entries per list): check them here
    if vecB.dim() != 2 or vecB.shape[1] != d or vecA.dtype != vecB.dtype:
        raise ValueError(f"vecB must be [nB, {d}] of dtype {vecA.dtype}, got {tuple(vecB.shape)} {vecB.dtype}")
    for name, t, rows, dtypes in (("idsA", idsA, nA, ("int32", "uint32")), ("distsA", distsA, nA, ("float32",)),
                                  ("idsB", idsB, nB, ("int32", "uint32")), ("distsB", distsB, nB, ("float32",))):
        if tuple(t.shape) != (rows, k) or not any(str(t.dtype).endswith(x) for x in dtypes):
            raise ValueError(f"{name} must be [{rows}, {k}] {dtypes[0]}, got {tuple(t.shape)} {t.dtype}")
    for t in (vecA, vecB, idsA, distsA, idsB, distsB):
        if not (t.is_cuda and t.is_contiguous()):
            raise ValueError("knng_merge needs contiguous CUDA tensors")
    out_ids = torch.empty((nA + nB, k), dtype=torch.int32, device=vecA.device)
    out_dists = torch.empty((nA + nB, k), dtype=torch.float32, device=vecA.device)
    ws_ptr, ws_bytes = None, 0
    if workspace is not None:
        ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    _check(lib().knng_merge(_ptr(vecA), nA, _ptr(idsA), _ptr(distsA), _ptr(vecB), nB, _ptr(idsB),
                            _ptr(distsB), dt, d, k, _metric(metric), merge_iters, sample_size, level, seed,
                            _ptr(out_ids), _ptr(out_dists), ws_ptr, ws_bytes, _stream(stream)))
    return out_ids, out_dists


def knng_extend(vec_old, ids_old, dists_old, vec_new, k: int, iters: int, merge_iters: int, sample_size: int,
                seed: int = 0, metric="l2", stream=None):
    """Incremental construction: GNND on the batch, GGM into the
    existing graph.  Returns (ids, dists) [n_old + n_new, k]."""
    import torch
    n_old, d = vec_old.shape
    n_new = vec_new.shape[0]
    if vec_new.dim() != 2 or vec_new.shape[1] != d or vec_new.dtype != vec_old.dtype:
        raise ValueError("vec_new must match vec_old's width and dtype")
    if tuple(ids_old.shape) != (n_old, k) or tuple(dists_old.shape) != (n_old, k):
        raise ValueError(f"ids_old/dists_old must be [{n_old}, {k}]")
    for t in (vec_old, ids_old, dists_old, vec_new):
        if not (t.is_cuda and t.is_contiguous()):
            raise ValueError("knng_extend needs contiguous CUDA tensors")
    out_ids = torch.empty((n_old + n_new, k), dtype=torch.int32, device=vec_old.device)
    out_dists = torch.empty((n_old + n_new, k), dtype=torch.float32, device=vec_old.device)
    _check(lib().knng_extend(_ptr(vec_old), n_old, _ptr(ids_old), _ptr(dists_old), _ptr(vec_new), n_new,
                             _dtype_code(vec_old), d, k, _metric(metric), iters, merge_iters, sample_size, seed,
                             _ptr(out_ids), _ptr(out_dists), _stream(stream)))
    return out_ids, out_dists


# ------------------------------------------------------------------ multi-GPU
def knng_get_unique_id() -> bytes:
    """NCCL unique id (128 bytes) for knng_comm_init; rank 0 creates it."""
    buf = C.create_string_buffer(128)
    _check(lib().knng_get_unique_id(buf))
    return buf.raw


def knng_comm_init(rank: int, world: int, uid: bytes) -> int:
    """NCCL communicator handle of this rank (the current CUDA device)."""
    assert len(uid) == 128
    h = C.c_void_p()
    _check(lib().knng_comm_init(rank, world, C.create_string_buffer(uid, 128), C.byref(h)))
    return h.value


def knng_comm_init_local(world: int) -> list[int]:
    """`world` in-process communicators (one per host thread)."""
    arr = (C.c_void_p * world)()
    _check(lib().knng_comm_init_local(world, arr))
    return [arr[i] for i in range(world)]


def knng_comm_destroy(comm: int):
    _check(lib().knng_comm_destroy(comm))


def knng_build_sharded(comm: int, rank: int, world: int, local_vectors, k: int, iters: int, merge_iters,
                       sample_size: int, seed: int = 0, metric="l2", out_ids=None, out_dists=None, stream=None):
    """Collective GNND + log-depth GGM tree (include/knng.h): this rank's rows
    [rank n_local, (rank+1) n_local) -> their lists with global ids.
    merge_iters: one count, or one per tree level."""
    import torch
    assert local_vectors.is_cuda and local_vectors.is_contiguous() and local_vectors.dim() == 2
    nl, d = local_vectors.shape
    if out_ids is None:
        out_ids = torch.empty((nl, k), dtype=torch.int32, device=local_vectors.device)
    if out_dists is None:
        out_dists = torch.empty((nl, k), dtype=torch.float32, device=local_vectors.device)
    levels = max(0, world.bit_length() - 1)
    if isinstance(merge_iters, int):
        lv, mi = None, merge_iters
    else:
        its = [int(x) for x in merge_iters]
        its = (its + its[-1:] * levels)[:max(levels, 1)]
        lv, mi = (C.c_int32 * len(its))(*its), its[0]
    _check(lib().knng_build_sharded(comm, _ptr(local_vectors), nl, rank * nl, world * nl, _dtype_code(local_vectors),
                                    d, k, _metric(metric), iters, mi, lv, sample_size, seed, _ptr(out_ids),
                                    _ptr(out_dists), _stream(stream)))
    return out_ids, out_dists


def knng_bruteforce(vectors, queries, kq: int, metric="l2", stream=None):
    """Exact top-kq (excluding self) of the query rows: (ids, dists) [nq, kq]."""
    import torch
    n, d = vectors.shape
    q = queries.to(device=vectors.device, dtype=torch.int64).contiguous()
    out_ids = torch.empty((q.numel(), kq), dtype=torch.int32, device=vectors.device)
    out_dists = torch.empty((q.numel(), kq), dtype=torch.float32, device=vectors.device)
    _check(lib().knng_bruteforce(_ptr(vectors), _dtype_code(vectors), n, d, _metric(metric), _ptr(q), q.numel(),
                                 kq, _ptr(out_ids), _ptr(out_dists), _stream(stream)))
    return out_ids, out_dists


# ------------------------------------------------------------------ debug ABI
def knng_debug_init(vectors, k: int, seed: int, metric="l2", stream=None):
    import torch
    n, d = vectors.shape
    keys = torch.empty((n, k), dtype=torch.int64, device=vectors.device)
    flags = torch.empty((n, k), dtype=torch.uint8, device=vectors.device)
    _check(lib().knng_debug_init(_ptr(vectors), _dtype_code(vectors), n, d, k, _metric(metric), seed,
                                 _ptr(keys), _ptr(flags), _stream(stream)))
    return keys, flags


def knng_debug_iterate(vectors, keys, flags, sample_size: int, tword: int, seed: int, boundary: int = -1,
                       metric="l2", stream=None) -> dict:
    """One iteration in place on device (keys int64-as-u64 [n, k], flags u8)."""
    n, d = vectors.shape
    k = keys.shape[1]
    st = IterStats()
    _check(lib().knng_debug_iterate(_ptr(vectors), _dtype_code(vectors), n, d, k, _metric(metric), sample_size,
                                    tword, seed, boundary, _ptr(keys), _ptr(flags), C.addressof(st), None, 0,
                                    _stream(stream)))
    return st.as_dict()


def knng_debug_sample(keys, flags, sample_size: int, tword: int, seed: int, stream=None):
    import torch
    n, k = keys.shape
    cap = 2 * sample_size
    dev = keys.device
    Gn = torch.empty((n, cap), dtype=torch.int32, device=dev)
    Go = torch.empty((n, cap), dtype=torch.int32, device=dev)
    cn = torch.empty((n,), dtype=torch.int32, device=dev)
    co = torch.empty((n,), dtype=torch.int32, device=dev)
    _check(lib().knng_debug_sample(n, k, sample_size, tword, seed, _ptr(keys), _ptr(flags), _ptr(Gn), _ptr(cn),
                                   _ptr(Go), _ptr(co), None, 0, _stream(stream)))
    return Gn, cn, Go, co


def knng_debug_philox(ctr, seed: int, stream=None):
    import torch
    out = torch.empty_like(ctr)
    _check(lib().knng_debug_philox(_ptr(ctr), ctr.shape[0], seed, _ptr(out), _stream(stream)))
    return out


# ------------------------------------------------------------------ introspection
def knng_last_stats(max_iters: int = 256) -> list[dict]:
    arr = (IterStats * max_iters)()
    m = lib().knng_last_stats(arr, max_iters)
    return [arr[i].as_dict() for i in range(m)]


def knng_launch_count() -> int:
    return int(lib().knng_launch_count())


def knng_set_timing(enable: bool):
    lib().knng_set_timing(1 if enable else 0)


def knng_reset_timing():
    lib().knng_reset_timing()


def knng_kernel_time(name: str) -> tuple[float, int]:
    ms = C.c_double()
    cnt = C.c_int64()
    lib().knng_kernel_time(name.encode(), C.addressof(ms), C.addressof(cnt))
    return ms.value, cnt.value


def knng_set_option(name: str, value: int):
    _check(lib().knng_set_option(name.encode(), int(value)))


def knng_get_option(name: str) -> int:
    v = C.c_int64()
    _check(lib().knng_get_option(name.encode(), C.addressof(v)))
    return v.value


def knng_last_error() -> str:
    return lib().knng_last_error().decode()


def knng_abi_version() -> int:
    return int(lib().knng_abi_version())
