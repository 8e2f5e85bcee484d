"""Distributed build through the C ABI (knng_build_sharded, SURVEY.md section
8(e) stage B): P ranks, every level of the log-depth GGM tree merged by all
ranks of its group with records exchanged between them.

The ranks here are host threads of one process on one GPU
(knng_comm_init_local: the exchange layer copies device buffers after CUDA
events); NCCL cannot place two ranks on one device, and the round's GPU
budget is one B200.  Everything except the ncclSend/ncclRecv calls is the
code path a multi-GPU run takes.  Expected values: the oracle's log-depth
tree of P shards (oracle.tree_build), element by element."""
import threading

import numpy as np
import pytest

import datagen
import oracle.oracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2103_15386_b200.knng as K
    K.lib()
    return K


def run_ranks(K, X, P, k, iters, merge_iters, p, seed, metric="l2"):
    """knng_build_sharded on P thread-ranks; returns the concatenated graph
    (ids, dists) and each rank's counters."""
    n = X.shape[0]
    nl = n // P
    comms = K.knng_comm_init_local(P)
    out = [None] * P
    stats = [None] * P
    errs = []

    def rank(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                Xl = torch.from_numpy(np.ascontiguousarray(X[r * nl:(r + 1) * nl])).cuda()
                ids, dists = K.knng_build_sharded(comms[r], r, P, Xl, k, iters, merge_iters, p, seed, metric,
                                                  stream=st)
                st.synchronize()
                out[r] = (ids.cpu().numpy().view(np.uint32), dists.cpu().numpy())
                stats[r] = K.knng_last_stats()
        except Exception as e:  # noqa: BLE001 -- reported below
            errs.append(e)

    th = [threading.Thread(target=rank, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for c in comms:
        K.knng_comm_destroy(c)
    assert not errs, errs
    ids = np.concatenate([o[0] for o in out])
    dists = np.concatenate([o[1] for o in out])
    return ids, dists, stats


CASES = [
    # (shape, n, d, k, p, iters, merge_iters, P, dtype, metric)
    ("c1", 2400, 16, 10, 6, 6, 5, 2, "f32", "l2"),
    ("c1", 2400, 16, 10, 6, 6, 4, 4, "f32", "l2"),
    ("sift", 4000, 128, 16, 8, 5, 4, 4, "f32", "l2"),      # integer-valued: the exact-u8 tensor-core join
    ("sift", 3200, 128, 32, 16, 4, 3, 2, "u8", "l2"),
    ("deep", 4000, 96, 16, 8, 5, 3, 8, "f32", "l2"),       # float join, 3 levels
    ("deep", 2400, 96, 16, 8, 5, 4, 2, "f32", "cosine"),
]


def _data(shape, n, d, dtype):
    if shape == "sift":
        return datagen.make("sift", n, seed=21, dtype=dtype)
    return datagen.make(shape, n, seed=21, d=d)


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[1]}-k{c[3]}-P{c[7]}-{c[8]}-{c[9]}")
def test_sharded_equals_oracle_tree(K, case):
    shape, n, d, k, p, iters, mi, P, dtype, metric = case
    X = _data(shape, n, d, dtype)
    m = orc.COSINE if metric == "cosine" else orc.L2SQ
    expect = orc.tree_build(X, P, k, p, iters, mi, 9, m)
    ids, dists, stats = run_ranks(K, X, P, k, iters, mi, p, 9, metric)
    assert np.array_equal(ids, orc.key_ids(expect))
    assert np.array_equal(dists, orc.key_dists(expect))
    levels = P.bit_length() - 1
    for r in range(P):
        assert len(stats[r]) == iters + levels * mi
        # the refine joins of every rank evaluate cross pairs only, some
        assert sum(s["dist_evals"] for s in stats[r][iters:]) > 0


def test_sharded_per_level_iterations(K):
    X = datagen.make("c1", 3200, seed=22, d=8)
    P, k, p, iters = 4, 12, 6, 5
    # the oracle tree with 3 then 5 refine iterations, composed by hand
    ns = 800
    keys = np.zeros((3200, k), np.uint64)
    for g in range(P):
        i_, d_ = orc.build(X[g * ns:(g + 1) * ns], k, p, iters, 9 + g)
        keys[g * ns:(g + 1) * ns] = orc.key(d_, i_.astype(np.uint64) + np.uint64(g * ns))
    for level, (width, mi) in enumerate([(1, 3), (2, 5)]):
        for g0 in range(0, P, 2 * width):
            lo, mid, hi = g0 * ns, (g0 + width) * ns, (g0 + 2 * width) * ns
            loc = orc.key(orc.key_dists(keys[lo:hi]), orc.key_ids(keys[lo:hi]).astype(np.uint64) - np.uint64(lo))
            mg = orc.merge(X[lo:hi], loc, mid - lo, k, p, mi, 9, level)
            keys[lo:hi] = orc.key(orc.key_dists(mg), orc.key_ids(mg).astype(np.uint64) + np.uint64(lo))
    ids, dists, _ = run_ranks(K, X, P, k, iters, [3, 5], p, 9)
    assert np.array_equal(ids, orc.key_ids(keys))
    assert np.array_equal(dists, orc.key_dists(keys))


def test_sharded_rejects_mismatched_parameters(K):
    # every rank sees the mismatch (collective check) and returns KNNG_E_USAGE
    X = datagen.make("c1", 800, seed=3, d=8)
    comms = K.knng_comm_init_local(2)
    errs = [None, None]

    def rank(r):
        torch.cuda.set_device(0)
        Xl = torch.from_numpy(np.ascontiguousarray(X[r * 400:(r + 1) * 400])).cuda()
        try:
            K.knng_build_sharded(comms[r], r, 2, Xl, 10, 4, 3, 5, seed=1 + r)  # seeds differ
        except K.KnngError as e:
            errs[r] = e.status

    th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join(timeout=120) for t in th]
    for c in comms:
        K.knng_comm_destroy(c)
    assert errs == [K.KNNG_E_USAGE, K.KNNG_E_USAGE]
