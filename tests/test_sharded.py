"""Sharded build (log-depth GGM tree over ranks, D26, SURVEY.md
section 8(e)): the host plumbing of paper_2103_15386_b200/sharded.py.

CPU tests (gloo, world size 1 and 2) drive the exchange and schedule with the
oracle standing in for the compute -- only the tests inject it; the product
default is the CUDA library -- and require the result to equal the oracle's
tree_build bit for bit.  GPU tests run the same with libknng.so.
"""
import os
import socket

import numpy as np
import pytest

import datagen
import oracle.oracle as orc
from paper_2103_15386_b200.sharded import knng_build_sharded, plan

torch = pytest.importorskip("torch")


class OracleOps:
    """Test-only compute backend: the oracle on host tensors."""

    def build(self, X, k, iters, p, seed, metric):
        ids, dists = orc.build(X.cpu().numpy(), k, p, iters, seed, _m(metric))
        return torch.from_numpy(ids.view(np.int32).copy()), torch.from_numpy(dists)

    def merge(self, XA, ia, da, XB, ib, db, k, merge_iters, p, seed, level, metric):
        nA = XA.shape[0]
        X = np.concatenate([XA.cpu().numpy(), XB.cpu().numpy()])
        keys = np.concatenate([orc.key(da.numpy(), ia.numpy().view(np.uint32)),
                               orc.key(db.numpy(), ib.numpy().view(np.uint32).astype(np.uint64) + np.uint64(nA))])
        out = orc.merge(X, keys, nA, k, p, merge_iters, seed, level, _m(metric))
        return (torch.from_numpy(orc.key_ids(out).astype(np.uint32).view(np.int32).copy()),
                torch.from_numpy(orc.key_dists(out).copy()))


def _m(metric):
    return orc.COSINE if metric == "cosine" else orc.L2SQ


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASE = dict(n=2400, shards=4, k=10, p=6, iters=6, merge_iters=5, seed=3)


def _expected():
    X = datagen.make("c1", CASE["n"], seed=11)
    keys = orc.tree_build(X, CASE["shards"], CASE["k"], CASE["p"], CASE["iters"], CASE["merge_iters"], CASE["seed"])
    return X, keys


def _worker(rank, world, port, use_cuda, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X = datagen.make("c1", CASE["n"], seed=11)
        nl = CASE["n"] // world
        Xl = torch.from_numpy(X[rank * nl:(rank + 1) * nl].copy())
        ops = OracleOps()
        if use_cuda:
            from paper_2103_15386_b200.sharded import CudaOps
            Xl = Xl.cuda()
            ops = CudaOps()
        ids, dists = knng_build_sharded(Xl, CASE["shards"], CASE["k"], CASE["iters"], CASE["merge_iters"],
                                        CASE["p"], CASE["seed"], ops=ops)
        np.save(os.path.join(out_dir, f"ids{rank}.npy"), ids.cpu().numpy())
        np.save(os.path.join(out_dir, f"dists{rank}.npy"), dists.cpu().numpy())
    finally:
        dist.destroy_process_group()


def _run_world(world, use_cuda, tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _free_port(), use_cuda, str(tmp_path)), nprocs=world, join=True)
    ids = np.concatenate([np.load(tmp_path / f"ids{r}.npy") for r in range(world)])
    dists = np.concatenate([np.load(tmp_path / f"dists{r}.npy") for r in range(world)])
    return orc.key(dists, ids.view(np.uint32))


# ------------------------------------------------------------------ schedule
def test_plan_levels_and_owners():
    lv = plan(8, 4)
    assert [len(x) for x in lv] == [4, 2, 1]
    assert all(s.leader == s.partner for s in lv[0])            # 2 shards per rank: level 0 local
    assert [(s.leader, s.partner) for s in lv[1]] == [(0, 1), (2, 3)]
    assert [(s.leader, s.partner) for s in lv[2]] == [(0, 2)]
    assert plan(1, 1) == []
    assert [(s.g0, s.width) for s in plan(4, 1)[1]] == [(0, 2)]
    for bad in [(3, 1), (4, 3), (2, 4)]:
        with pytest.raises(ValueError):
            plan(*bad)


def test_plan_every_shard_merged_once_per_level():
    for S in [1, 2, 4, 8, 16]:
        for P in [p for p in [1, 2, 4, 8] if S % p == 0]:
            for lvl in plan(S, P):
                covered = sorted(g for s in lvl for g in range(s.g0, s.g0 + 2 * s.width))
                assert covered == list(range(S))


# ------------------------------------------------------------------ CPU (gloo) exchange, oracle compute
def test_sharded_world1_equals_oracle_tree():
    X, expect = _expected()
    ids, dists = knng_build_sharded(torch.from_numpy(X), CASE["shards"], CASE["k"], CASE["iters"],
                                    CASE["merge_iters"], CASE["p"], CASE["seed"], ops=OracleOps())
    got = orc.key(dists.numpy(), ids.numpy().view(np.uint32))
    assert np.array_equal(got, expect)


def test_sharded_gloo_world2_equals_oracle_tree(tmp_path):
    _, expect = _expected()
    got = _run_world(2, False, tmp_path)
    assert np.array_equal(got, expect)


def test_sharded_timeline_order():
    X, _ = _expected()
    tl = []
    knng_build_sharded(torch.from_numpy(X), 4, CASE["k"], 2, 1, CASE["p"], CASE["seed"], ops=OracleOps(),
                       timeline=tl)
    assert tl == [("build", 0), ("build", 1), ("build", 2), ("build", 3), ("merge", 0), ("merge", 0),
                  ("merge", 1)]


# ------------------------------------------------------------------ GPU: libknng.so compute
@pytest.mark.gpu
def test_gpu_sharded_world1_equals_oracle_tree():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    X, expect = _expected()
    ids, dists = knng_build_sharded(torch.from_numpy(X).cuda(), CASE["shards"], CASE["k"], CASE["iters"],
                                    CASE["merge_iters"], CASE["p"], CASE["seed"])
    got = orc.key(dists.cpu().numpy(), ids.cpu().numpy().view(np.uint32))
    assert np.array_equal(got, expect)


@pytest.mark.gpu
def test_gpu_sharded_two_ranks_equals_oracle_tree(tmp_path):
    # two processes on one GPU (gloo moves the blocks): the multi-rank path
    # with the CUDA compute, bit-identical to the oracle tree
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    _, expect = _expected()
    got = _run_world(2, True, tmp_path)
    assert np.array_equal(got, expect)


@pytest.mark.gpu
def test_gpu_sharded_medium_eight_shards_equals_oracle_tree():
    # 8 shards x 4000 rows (3 tree levels, many join batches per level): the
    # libknng tree equals the oracle's tree_build bit for bit
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    X = datagen.make("c1", 32000, seed=21)
    k, p, iters, mi, seed = 10, 8, 6, 5, 9
    expect = orc.tree_build(X, 8, k, p, iters, mi, seed)
    ids, dists = knng_build_sharded(torch.from_numpy(X).cuda(), 8, k, iters, mi, p, seed)
    got = orc.key(dists.cpu().numpy(), ids.cpu().numpy().view(np.uint32))
    assert np.array_equal(got, expect)
    # per-level merge iterations (D23): same as the oracle with the same count per level
    ids2, dists2 = knng_build_sharded(torch.from_numpy(X).cuda(), 8, k, iters, [mi, mi, mi], p, seed)
    assert np.array_equal(ids2.cpu().numpy(), ids.cpu().numpy())


def test_sharded_per_level_merge_iters():
    X, _ = _expected()
    with pytest.raises(ValueError):
        knng_build_sharded(torch.from_numpy(X), 4, CASE["k"], 2, [1], CASE["p"], CASE["seed"], ops=OracleOps())
    # a list with one count per level equals the oracle tree with that count
    ids, dists = knng_build_sharded(torch.from_numpy(X), 4, CASE["k"], CASE["iters"],
                                    [CASE["merge_iters"]] * 2, CASE["p"], CASE["seed"], ops=OracleOps())
    _, expect = _expected()
    assert np.array_equal(orc.key(dists.numpy(), ids.numpy().view(np.uint32)), expect)


# ------------------------------------------------------------------ stage B plumbing (CPU, gloo)
def _uid_worker(rank, world, port, out_dir):
    import torch.distributed as dist

    import paper_2103_15386_b200.knng as K
    from paper_2103_15386_b200 import sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # the unique-id broadcast of nccl_comm, without the GPU-side init
        obj = [K.knng_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        with open(os.path.join(out_dir, f"uid{rank}.bin"), "wb") as f:
            f.write(obj[0])
        assert sharded._COMMS == {}
    finally:
        dist.destroy_process_group()


def test_stage_b_unique_id_broadcast_gloo_world2(tmp_path):
    """knng_build_sharded_nccl's rendezvous (torch provides
    only the ncclUniqueId broadcast): rank 0's 128-byte NCCL id from
    libknng.so reaches every rank of a world-size-2 gloo group intact."""
    import paper_2103_15386_b200.knng as K
    try:
        K.knng_get_unique_id()
    except K.KnngError as e:  # no NCCL on this host: nothing to broadcast
        pytest.skip(str(e))
    import torch.multiprocessing as mp
    mp.spawn(_uid_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    a = (tmp_path / "uid0.bin").read_bytes()
    b = (tmp_path / "uid1.bin").read_bytes()
    assert len(a) == 128 and a == b and any(a)


def test_build_sharded_abi_validation_without_gpu():
    """Host-side checks of knng_build_sharded run before any CUDA call."""
    import ctypes as C

    import paper_2103_15386_b200.knng as K
    L = K.lib()
    comms = K.knng_comm_init_local(2)
    try:
        ok = dict(n_local=100, goff=0, ntot=200, k=10, iters=3, mi=2, p=5)

        def call(comm, **kw):
            a = dict(ok, **kw)
            return L.knng_build_sharded(comm, None, a["n_local"], a["goff"], a["ntot"], K.KNNG_F32, 8, a["k"],
                                        K.KNNG_L2SQ, a["iters"], a["mi"], None, a["p"], 1, None, None, None)
        assert call(comms[0], ntot=300) == K.KNNG_E_USAGE          # unequal shards
        assert call(comms[1], goff=0) == K.KNNG_E_USAGE            # rank 1 must start at n_local
        assert call(comms[0], p=10) == K.KNNG_E_USAGE              # p < k
        assert call(comms[0], mi=-1) == K.KNNG_E_USAGE
        assert call(None) == K.KNNG_E_USAGE
        three = (C.c_void_p * 3)()
        assert L.knng_comm_init_local(3, three) == K.KNNG_OK
        assert L.knng_build_sharded(three[0], None, 100, 0, 300, 0, 8, 10, 0, 3, 2, None, 5, 1, None, None,
                                    None) == K.KNNG_E_USAGE  # world not a power of two
        for h in three:
            K.knng_comm_destroy(h)
    finally:
        for c in comms:
            K.knng_comm_destroy(c)
