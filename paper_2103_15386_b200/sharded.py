"""Sharded GNND build: divide and conquer over GPUs with a log-depth GGM tree.

Two entry points:
  * knng_build_sharded_nccl -- the product multi-GPU path: the C ABI's
    knng_build_sharded (every tree level merged by all GPUs of its group,
    records exchanged over NCCL inside libknng.so, SURVEY.md 8(e) stage B).
    torch.distributed only broadcasts the NCCL unique id (nccl_comm).
  * knng_build_sharded -- stage A host plumbing below: per-level block
    transfers with torch.distributed send/recv and one knng_merge per group
    on its leader.  It runs over any backend (gloo on CPU in the tests, with
    the oracle injected as compute) and is kept as the staged fallback.

The paper's out-of-memory scheme (Sec. 4.2): the set is split into
shards, "sub-graphs are constructed by GNND ... on different GPUs",
then the sub-graphs are joined by the GPU graph merge GGM (Alg. 3).
This module is the host-side plumbing of that scheme; every step of the
method runs in libknng.so (knng_build, knng_merge through the ctypes binding).
PyTorch supplies only device memory and torch.distributed send/recv (NCCL
over NVLink on a GPU box; gloo stages through host memory).

Schedule (D26, stage A):
  * `shards` S contiguous, equal shards of the global id range; rank r of P
    owns shards [r S/P, (r+1) S/P) -- its rows are contiguous.
  * shard g is built with seed + g (the oracle's tree_build, oracle/oracle.py).
  * level l = 0, 1, ...: every group of 2^(l+1) shards is GGM(left half, right
    half) with the group's id range numbered from 0 and Philox level l.  When
    both halves live on one rank the merge is local; otherwise the owner of
    the right half sends its block (vectors, ids, dists) to the owner of the
    left half (the group leader), which runs knng_merge.
  * after the top level rank 0 holds the whole graph (global ids); with
    scatter=True every rank receives its own rows back (node-partitioned
    output, as knng_build_sharded in SURVEY.md section 8(b)).

Because the tree is fixed by S (not by P), the result is bit-identical for
every P that divides S -- tests check P = 1 and P = 2 against the oracle's
tree_build.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class MergeStep:
    level: int
    g0: int          # first shard of the group
    width: int       # shards per half
    leader: int      # rank owning the left half (runs the merge)
    partner: int     # rank owning the right half (== leader: local merge)


def plan(shards: int, world: int) -> list[list[MergeStep]]:
    """Log-depth merge schedule: one list of MergeSteps per tree level."""
    if shards < 1 or shards & (shards - 1):
        raise ValueError("shards must be a power of two")
    if world < 1 or shards % world:
        raise ValueError("world size must divide the shard count")
    per = shards // world
    levels = []
    width, level = 1, 0
    while width < shards:
        levels.append([MergeStep(level, g0, width, g0 // per, (g0 + width) // per)
                       for g0 in range(0, shards, 2 * width)])
        width *= 2
        level += 1
    return levels


class CudaOps:
    """The product compute: libknng.so through the ctypes binding."""

    def __init__(self, stream=None):
        from . import knng as K
        K.lib()  # raises if the library is missing: there is no fallback
        self.K = K
        self.stream = stream

    def build(self, X, k, iters, p, seed, metric):
        return self.K.knng_build(X, k, iters, p, seed, metric, stream=self.stream)

    def merge(self, XA, ia, da, XB, ib, db, k, merge_iters, p, seed, level, metric):
        return self.K.knng_merge(XA, ia, da, XB, ib, db, k, merge_iters, p, seed=seed, level=level, metric=metric,
                                 stream=self.stream)


class _Comm:
    """Point-to-point block exchange over torch.distributed (NCCL moves device
    tensors directly; gloo moves host tensors, so device data is staged)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.active = dist.is_available() and dist.is_initialized()
        self.gloo = self.active and dist.get_backend(group) == "gloo"

    def send(self, t, dst):
        if self.gloo and t.is_cuda:
            t = t.cpu()
        self.dist.send(t.contiguous(), dst, group=self.group)

    def recv_into(self, t, src):
        if self.gloo and t.is_cuda:
            h = t.new_empty(t.shape, device="cpu")
            self.dist.recv(h, src, group=self.group)
            t.copy_(h)
        else:
            self.dist.recv(t, src, group=self.group)


def knng_build_sharded(local_vectors, shards: int, k: int, iters: int, merge_iters, sample_size: int,
                       seed: int = 0, metric="l2", group=None, ops=None, scatter: bool = True, timeline=None):
    """GNND on every shard + log-depth GGM tree across ranks.

    local_vectors: this rank's rows [n_local, d], n_local = shard_rows * S/P
    (all ranks equal).  merge_iters: one count for every level, or a
    sequence with one count per tree level (D23: higher levels merge larger
    sets and need more refine iterations).  Returns (ids int32 [n_local, k] with GLOBAL ids,
    dists float32) when scatter, else the whole graph on rank 0 and None on
    the other ranks.  timeline: optional list receiving (phase, level) marks
    (host-side order of events, for tests)."""
    import torch

    # every copy, exchange and library call of the tree runs on one stream:
    # the ops' stream when it is a torch stream, else the current one
    ops = ops or CudaOps()
    st = getattr(ops, "stream", None)
    if st is not None and local_vectors.is_cuda and hasattr(st, "cuda_stream"):
        with torch.cuda.stream(st):
            return _build_sharded(local_vectors, shards, k, iters, merge_iters, sample_size, seed, metric, group,
                                  ops, scatter, timeline)
    return _build_sharded(local_vectors, shards, k, iters, merge_iters, sample_size, seed, metric, group, ops,
                          scatter, timeline)


def _build_sharded(local_vectors, shards, k, iters, merge_iters, sample_size, seed, metric, group, ops, scatter,
                   timeline):
    import torch

    comm = _Comm(group)
    world = comm.dist.get_world_size(group) if comm.active else 1
    rank = comm.dist.get_rank(group) if comm.active else 0
    n_local, d = local_vectors.shape
    per = shards // world
    if shards % world or n_local % per:
        raise ValueError("local rows must split into S/P equal shards")
    ns = n_local // per
    steps = plan(shards, world)
    dev = local_vectors.device
    if isinstance(merge_iters, int):
        level_iters = [merge_iters] * len(steps)
    else:
        level_iters = [int(m) for m in merge_iters]
        if len(level_iters) < len(steps):
            raise ValueError(f"merge_iters needs one count per level ({len(steps)})")

    # Vectors of the largest block this rank leads, local rows first: a
    # received right half lands right after the left half, so merged blocks
    # stay contiguous without re-copying.
    lead_rows = n_local
    for lvl in steps:
        for s in lvl:
            if s.leader == rank and s.partner != rank:
                lead_rows = max(lead_rows, 2 * s.width * ns)
    if lead_rows > n_local:
        X = torch.empty((lead_rows, d), dtype=local_vectors.dtype, device=dev)
        X[:n_local].copy_(local_vectors)
    else:
        X = local_vectors

    # 1. GNND per shard, ids local to the shard.
    blocks = {}  # first shard -> (ids, dists) with block-local ids
    first = rank * per
    for j in range(per):
        g = first + j
        ids, dists = ops.build(X[j * ns:(j + 1) * ns], k, iters, sample_size, seed + g, metric)
        blocks[g] = (ids, dists)
        if timeline is not None:
            timeline.append(("build", g))

    # 2. log-depth GGM tree (Alg. 3 per group).
    for lvl in steps:
        for s in lvl:
            gA, gB = s.g0, s.g0 + s.width
            rows = s.width * ns
            if rank == s.partner and s.partner != s.leader:
                ib, db = blocks.pop(gB)
                lo = (gB - first) * ns
                comm.send(X[lo:lo + rows], s.leader)
                comm.send(ib, s.leader)
                comm.send(db, s.leader)
                if timeline is not None:
                    timeline.append(("send", s.level))
            elif rank == s.leader:
                ia, da = blocks.pop(gA)
                loA = (gA - first) * ns
                if s.partner != rank:
                    loB = loA + rows
                    comm.recv_into(X[loB:loB + rows], s.partner)
                    ib = torch.empty((rows, k), dtype=torch.int32, device=dev)
                    db = torch.empty((rows, k), dtype=torch.float32, device=dev)
                    comm.recv_into(ib, s.partner)
                    comm.recv_into(db, s.partner)
                else:
                    ib, db = blocks.pop(gB)
                    loB = (gB - first) * ns
                blocks[gA] = ops.merge(X[loA:loA + rows], ia, da, X[loB:loB + rows], ib, db, k,
                                       level_iters[s.level], sample_size, seed, s.level, metric)
                if timeline is not None:
                    timeline.append(("merge", s.level))

    # 3. output: rank 0 holds block 0 = the whole graph with global ids.
    if not scatter:
        return blocks.get(0, (None, None)) if rank == 0 else (None, None)
    if world == 1:
        return blocks[0]
    if rank == 0:
        ids, dists = blocks[0]
        for r in range(1, world):
            comm.send(ids[r * n_local:(r + 1) * n_local], r)
            comm.send(dists[r * n_local:(r + 1) * n_local], r)
        return ids[:n_local], dists[:n_local]
    ids = torch.empty((n_local, k), dtype=torch.int32, device=dev)
    dists = torch.empty((n_local, k), dtype=torch.float32, device=dev)
    comm.recv_into(ids, 0)
    comm.recv_into(dists, 0)
    return ids, dists


# ---------------------------------------------------------------- stage B (C ABI)
_COMMS = {}


def nccl_comm(group=None):
    """The libknng NCCL communicator of this rank for `group` (cached): rank 0
    creates the unique id, torch.distributed broadcasts it (the only role of
    torch here), every rank calls knng_comm_init on its current device."""
    import torch.distributed as dist

    from . import knng as K
    key = id(group)
    if key in _COMMS:
        return _COMMS[key]
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [K.knng_get_unique_id() if rank == 0 else None]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(obj, src=src, group=group)
    comm = (K.knng_comm_init(rank, world, obj[0]), rank, world)
    _COMMS[key] = comm
    return comm


def knng_build_sharded_nccl(local_vectors, k: int, iters: int, merge_iters, sample_size: int, seed: int = 0,
                            metric="l2", group=None, stream=None):
    """Collective build over the ranks of `group` (one GPU each): this rank's
    rows [rank n_local, (rank+1) n_local) -> their lists, global ids."""
    from . import knng as K
    comm, rank, world = nccl_comm(group)
    return K.knng_build_sharded(comm, rank, world, local_vectors, k, iters, merge_iters, sample_size, seed, metric,
                                stream=stream)
