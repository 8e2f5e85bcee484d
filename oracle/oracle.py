"""ctypes front end of the C oracle (knng_oracle.c) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module.  It shares no code with the
CUDA product (paper_2103_15386_b200/) and never imports it.

Graph state format (see knng_oracle.h): keys u64 [n, k] ascending, where
key = float_bits(dist) << 32 | id; flags u8 [n, k], 1 = NEW.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
SENTINEL = np.uint64(0xFFFFFFFFFFFFFFFF)
L2SQ, COSINE, CHI2 = 0, 1, 2
UPDATE_SELECTIVE, UPDATE_FULL = 0, 1
F32, U8 = 0, 1


def compile_lib(force: bool = False) -> str:
    """Compile the oracle shared library (plain C, gcc, no fast math)."""
    src = os.path.join(_HERE, "knng_oracle.c")
    hdr = os.path.join(_HERE, "knng_oracle.h")
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return _LIB_PATH
    cmd = ["gcc", "-std=gnu99", "-O2", "-ffp-contract=off", "-fno-fast-math",
           "-fPIC", "-shared", "-Wall", "-Wextra", "-Wno-unused-parameter",
           "-o", _LIB_PATH, src, "-lm"]
    subprocess.check_call(cmd)
    return _LIB_PATH


class _Stats(C.Structure):
    _fields_ = [("dist_evals", C.c_int64), ("candidates", C.c_int64),
                ("accepted", C.c_int64), ("joins", C.c_int64),
                ("sum_m", C.c_int64), ("sum_q", C.c_int64)]

    def as_dict(self) -> dict:
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


_lib = None


def lib():
    global _lib
    if _lib is None:
        compile_lib()
        L = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        i64, i32, u32, u64, dbl = C.c_int64, C.c_int, C.c_uint32, C.c_uint64, C.c_double
        L.orc_philox4x32_10.argtypes = [P, P, P]
        L.orc_uniform.argtypes = [P, u64]
        L.orc_uniform.restype = u64
        L.orc_distance.argtypes = [P, i32, i64, i32, i32, i64, i64]
        L.orc_distance.restype = C.c_float
        L.orc_init.argtypes = [P, i32, i64, i32, i32, i32, u64, P, P]
        L.orc_sample.argtypes = [i64, i32, i32, u32, u64, P, P, P, P, P, P, P, P, P, P]
        L.orc_iterate.argtypes = [P, i32, i64, i32, i32, i32, i32, u32, u64, i64, P, P, P, P]
        L.orc_build.argtypes = [P, i32, i64, i32, i32, i32, i32, i32, u64, P, P, P]
        L.orc_ggm_seed.argtypes = [P, i32, i64, i32, i32, i32, i64, i32, u64, P, P, P, P]
        L.orc_ggm_finalize.argtypes = [i64, i32, P, P]
        L.orc_merge.argtypes = [P, i32, i64, i32, i32, i32, i32, i64, i32, i32, u64, P, P, P]
        L.orc_bruteforce.argtypes = [P, i32, i64, i32, i32, P, i64, i32, P]
        L.orc_recall.argtypes = [i64, i32, P, i32, P, i32]
        L.orc_recall.restype = dbl
        L.orc_phi.argtypes = [i64, i32, P]
        L.orc_phi.restype = dbl
        L.orc_pair_index.argtypes = [i64, P, P]
        L.orc_list_insert.argtypes = [P, P, i32, u64]
        L.orc_list_insert_seg.argtypes = [P, P, i32, i32, u64]
        L.orc_set_option.argtypes = [C.c_char_p, i32]
        L.orc_segments.argtypes = [i32]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(rc: int, what: str):
    if rc != 0:
        raise RuntimeError(f"oracle {what} failed with status {rc}")


def _dtype_code(X: np.ndarray) -> int:
    if X.dtype == np.float32:
        return F32
    if X.dtype == np.uint8:
        return U8
    raise TypeError(f"unsupported dtype {X.dtype}")


def _c(X):
    return np.ascontiguousarray(X)


# ---------------------------------------------------------------- primitives
def philox(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def uniform(words, N: int) -> int:
    w = np.asarray(words, dtype=np.uint32)
    return int(lib().orc_uniform(_p(w), N))


def distance(X: np.ndarray, a: int, b: int, metric: int = L2SQ) -> float:
    X = _c(X)
    n, d = X.shape
    return float(lib().orc_distance(_p(X), _dtype_code(X), n, d, metric, a, b))


def key(dist, ids) -> np.ndarray:
    dist = np.asarray(dist, dtype=np.float32)
    return (dist.view(np.uint32).astype(np.uint64) << np.uint64(32)) | np.asarray(ids, dtype=np.uint64)


def key_ids(keys: np.ndarray) -> np.ndarray:
    return (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def key_dists(keys: np.ndarray) -> np.ndarray:
    return (keys >> np.uint64(32)).astype(np.uint32).view(np.float32)


def pair_index(t: int):
    u = C.c_int64(); v = C.c_int64()
    lib().orc_pair_index(t, C.byref(u), C.byref(v))
    return u.value, v.value


def list_insert(keys: np.ndarray, flags: np.ndarray, key_: int) -> bool:
    """In-place InsertIntoNNList on one list (u64 keys[k], u8 flags[k])."""
    assert keys.dtype == np.uint64 and flags.dtype == np.uint8
    return bool(lib().orc_list_insert(_p(keys), _p(flags), len(keys), int(key_)))


def list_insert_seg(keys: np.ndarray, flags: np.ndarray, s: int, key_: int) -> bool:
    """Segmented InsertIntoNNList on one list kept as the
    sorted union of s segments (id v in segment v % s)."""
    assert keys.dtype == np.uint64 and flags.dtype == np.uint8
    r = lib().orc_list_insert_seg(_p(keys), _p(flags), len(keys), s, int(key_))
    if r < 0:
        raise ValueError("bad segment count")
    return bool(r)


def set_option(name: str, value: int):
    """'update': UPDATE_SELECTIVE (GNND) / UPDATE_FULL (GNND-r1);
    'segment_size': entries per list segment (default 32)."""
    _check(lib().orc_set_option(name.encode(), int(value)), f"set_option {name}")


def segments(k: int) -> int:
    return int(lib().orc_segments(k))


class options:
    """Context manager: temporarily set oracle options, e.g.
    with orc.options(update=orc.UPDATE_FULL): ..."""

    def __init__(self, **kw):
        self.kw = kw

    def __enter__(self):
        for n, v in self.kw.items():
            set_option(n, v)
        return self

    def __exit__(self, *a):
        set_option("update", UPDATE_SELECTIVE)
        set_option("segment_size", 32)
        return False


# ---------------------------------------------------------------- algorithm
def init(X, k, seed, metric=L2SQ):
    X = _c(X)
    n, d = X.shape
    keys = np.zeros((n, k), dtype=np.uint64)
    flags = np.zeros((n, k), dtype=np.uint8)
    _check(lib().orc_init(_p(X), _dtype_code(X), n, d, metric, k, seed, _p(keys), _p(flags)), "init")
    return keys, flags


def sample(keys, flags, p, tword, seed):
    n, k = keys.shape
    FN = np.zeros((n, p), np.uint32); fnc = np.zeros(n, np.int32)
    FO = np.zeros((n, p), np.uint32); foc = np.zeros(n, np.int32)
    Gn = np.zeros((n, 2 * p), np.uint32); cn = np.zeros(n, np.int32)
    Go = np.zeros((n, 2 * p), np.uint32); co = np.zeros(n, np.int32)
    _check(lib().orc_sample(n, k, p, tword, seed, _p(_c(keys)), _p(_c(flags)), _p(FN), _p(fnc),
                            _p(FO), _p(foc), _p(Gn), _p(cn), _p(Go), _p(co)), "sample")
    return dict(FN=FN, fnc=fnc, FO=FO, foc=foc, Gn=Gn, cn=cn, Go=Go, co=co)


def iterate(X, keys, flags, p, tword, seed, metric=L2SQ, boundary=-1, target_mask=None):
    """One GNND iteration in place on (keys, flags); returns stats dict."""
    X = _c(X)
    n, d = X.shape
    k = keys.shape[1]
    assert keys.flags.c_contiguous and flags.flags.c_contiguous
    st = _Stats()
    tm = None if target_mask is None else _c(target_mask.astype(np.uint8))
    _check(lib().orc_iterate(_p(X), _dtype_code(X), n, d, metric, k, p, tword, seed, boundary,
                             _p(keys), _p(flags), _p(tm), C.byref(st)), "iterate")
    return st.as_dict()


def build(X, k, p, iters, seed, metric=L2SQ, with_stats=False):
    X = _c(X)
    n, d = X.shape
    ids = np.zeros((n, k), np.uint32)
    dists = np.zeros((n, k), np.float32)
    stats = (_Stats * iters)()
    _check(lib().orc_build(_p(X), _dtype_code(X), n, d, metric, k, p, iters, seed,
                           _p(ids), _p(dists), stats), "build")
    if with_stats:
        return ids, dists, [s.as_dict() for s in stats]
    return ids, dists


def ggm_seed(X, keys_in, nA, k, seed, level=0, metric=L2SQ):
    X = _c(X)
    n, d = X.shape
    kr = k - (k + 1) // 2
    keys = np.zeros((n, k), np.uint64)
    flags = np.zeros((n, k), np.uint8)
    reserved = np.zeros((n, max(kr, 1)), np.uint64)
    _check(lib().orc_ggm_seed(_p(X), _dtype_code(X), n, d, metric, k, nA, level, seed,
                              _p(_c(keys_in)), _p(keys), _p(flags), _p(reserved)), "ggm_seed")
    return keys, flags, reserved[:, :kr]


def ggm_finalize(keys, reserved):
    n, k = keys.shape
    keys = keys.copy()
    _check(lib().orc_ggm_finalize(n, k, _p(_c(reserved)), _p(keys)), "ggm_finalize")
    return keys


def merge(X, keys_in, nA, k, p, merge_iters, seed, level=0, metric=L2SQ, with_stats=False):
    """GGM over the combined set X = [S1; S2]; keys_in: combined lists with
    S2 ids already re-based by nA."""
    X = _c(X)
    n, d = X.shape
    out = np.zeros((n, k), np.uint64)
    stats = (_Stats * max(1, merge_iters))()
    _check(lib().orc_merge(_p(X), _dtype_code(X), n, d, metric, k, p, nA, merge_iters, level,
                           seed, _p(_c(keys_in)), _p(out), stats), "merge")
    if with_stats:
        return out, [s.as_dict() for s in stats][:merge_iters]
    return out


def bruteforce(X, queries, kq, metric=L2SQ):
    X = _c(X)
    n, d = X.shape
    q = _c(np.asarray(queries, dtype=np.int64))
    out = np.zeros((len(q), kq), np.uint64)
    _check(lib().orc_bruteforce(_p(X), _dtype_code(X), n, d, metric, _p(q), len(q), kq, _p(out)),
           "bruteforce")
    return out


def recall(graph_keys, truth_keys, at_k=10) -> float:
    g = _c(np.asarray(graph_keys, dtype=np.uint64))
    t = _c(np.asarray(truth_keys, dtype=np.uint64))
    r = lib().orc_recall(g.shape[0], g.shape[1], _p(g), t.shape[1], _p(t), at_k)
    if r < 0:
        raise ValueError("bad recall arguments")
    return float(r)


def phi(keys) -> float:
    keys = _c(np.asarray(keys, dtype=np.uint64))
    return float(lib().orc_phi(keys.shape[0], keys.shape[1], _p(keys)))


def tree_build(X, shards, k, p, iters, merge_iters, seed, metric=L2SQ):
    """Log-depth divide and conquer (D26): GNND on `shards`
    contiguous equal shards (per-shard seed = seed + g), then at level l
    every group of 2^(l+1) shards is GGM(left half, right half)."""
    X = _c(X)
    n = X.shape[0]
    assert shards >= 1 and (shards & (shards - 1)) == 0 and n % shards == 0
    ns = n // shards
    keys = np.zeros((n, k), np.uint64)
    for g in range(shards):
        ids, dists = build(X[g * ns:(g + 1) * ns], k, p, iters, seed + g, metric)
        keys[g * ns:(g + 1) * ns] = key(dists, ids.astype(np.uint64) + np.uint64(g * ns))
    level = 0
    width = 1
    while width < shards:
        for g0 in range(0, shards, 2 * width):
            lo, mid, hi = g0 * ns, (g0 + width) * ns, (g0 + 2 * width) * ns
            local = keys[lo:hi].copy()
            ids = key_ids(local).astype(np.int64) - lo
            local = key(key_dists(local), ids.astype(np.uint64))
            merged = merge(X[lo:hi], local, mid - lo, k, p, merge_iters, seed, level, metric)
            keys[lo:hi] = key(key_dists(merged), key_ids(merged).astype(np.uint64) + np.uint64(lo))
        width *= 2
        level += 1
    return keys


def extend(X_old, keys_old, X_new, k, p, iters, merge_iters, seed, metric=L2SQ):
    """Incremental construction: GNND on the new batch (seed), then
    GGM of the existing graph (A, ids < n_old) with the batch graph (B, ids
    re-based by n_old), level 0, the same seed.  Returns keys [n_old + n_new, k]."""
    n_old = X_old.shape[0]
    ids, dists = build(X_new, k, p, iters, seed, metric)
    keys_in = np.concatenate([keys_old, key(dists, ids.astype(np.uint64) + np.uint64(n_old))])
    return merge(np.concatenate([X_old, X_new]), keys_in, n_old, k, p, merge_iters, seed, 0, metric)


def shard_bounds(n: int, shards: int) -> list:
    """Contiguous shard g = rows [g n / S, (g+1) n / S) ("partitioned
    into multiple shards")."""
    return [g * n // shards for g in range(shards + 1)]


def allpairs_level(i: int, h: int, shards: int) -> int:
    """Philox level word of the merge of shards i < h (D41): i * S + h."""
    return i * shards + h


def allpairs_build(X, shards, k, p, iters, merge_iters, seed, metric=L2SQ, order=None):
    """The paper's out-of-memory scheme (D41): GNND builds the
    sub-graph G_g of every shard g (seed + g, local ids); then GGM merges
    every pair of sub-graphs (i < h) once -- Alg. 3 on S_i U S_h with A = G_i,
    B = G_h, Philox level i * S + h -- and "each k-NN list in either
    sub-graph retains the top-k neighbors": the merged lists are folded into
    the running lists R of both shards (R(x) <- k smallest unique keys of
    R(x) U M(x), InsertIntoNNList per entry, D17).  R starts as the shards'
    own graphs with global ids.  `order`: the sequence of pairs (default
    (0,1), (0,2), ..., (S-2,S-1)); the result does not depend on it.
    Returns keys [n, k] with global ids."""
    X = _c(X)
    n = X.shape[0]
    b = shard_bounds(n, shards)
    G, R = [], np.zeros((n, k), np.uint64)
    for g in range(shards):
        ids, dists = build(X[b[g]:b[g + 1]], k, p, iters, seed + g, metric)
        G.append(key(dists, ids))
        R[b[g]:b[g + 1]] = key(dists, ids.astype(np.uint64) + np.uint64(b[g]))
    pairs = order if order is not None else [(i, h) for i in range(shards) for h in range(i + 1, shards)]
    flags = np.zeros(k, np.uint8)
    for i, h in pairs:
        nA = b[i + 1] - b[i]
        Xp = np.concatenate([X[b[i]:b[i + 1]], X[b[h]:b[h + 1]]])
        keys_in = np.concatenate([G[i], key(key_dists(G[h]), key_ids(G[h]).astype(np.uint64) + np.uint64(nA))])
        M = merge(Xp, keys_in, nA, k, p, merge_iters, seed, allpairs_level(i, h, shards), metric)
        mid = key_ids(M).astype(np.int64)
        gid = np.where(mid < nA, mid + b[i], mid - nA + b[h]).astype(np.uint64)
        Mg = key(key_dists(M), gid)
        rows = list(range(b[i], b[i + 1])) + list(range(b[h], b[h + 1]))
        for r, x in enumerate(rows):
            lst = R[x].copy()
            for kk in Mg[r]:
                list_insert(lst, flags, int(kk))
            R[x] = lst
    return R
