"""Pins of the oracle GGM (Alg. 3), brute force, recall (Eq. 4) and phi
(Eq. 3): SPEC worked examples, brute force on tiny inputs, invariants."""
import numpy as np
import pytest

import datagen
import oracle.oracle as orc


def _split_build(X, nA, k, p, iters, seed):
    """Sub-graphs of S1 = X[:nA] and S2 = X[nA:], combined with S2 re-based."""
    ia, da = orc.build(X[:nA], k, p, iters, seed)
    ib, db = orc.build(X[nA:], k, p, iters, seed + 1)
    keys = np.concatenate([orc.key(da, ia), orc.key(db, ib.astype(np.uint64) + np.uint64(nA))])
    return keys


def test_ggm_seed_spec_example_and_cross_draws():
    # k=4: keep first 2 (OLD), reserve last 2, draw 2 distinct
    # ids of the other subset, NEW; every NEW entry of an S1 list is >= nA.
    X = datagen.make("c1", 300, seed=2, d=6)
    nA, k = 120, 4
    keys_in = _split_build(X, nA, k, 2, 3, 2)
    keys, flags, reserved = orc.ggm_seed(X, keys_in, nA, k, 9)
    ids = orc.key_ids(keys).astype(np.int64)
    for i in range(len(X)):
        own_b = i >= nA
        kept = set(orc.key_ids(keys_in[i, :2]))
        assert set(orc.key_ids(reserved[i])) == set(orc.key_ids(keys_in[i, 2:]))
        new_ids = ids[i][flags[i] == 1]
        old_ids = ids[i][flags[i] == 0]
        assert set(old_ids) == kept and len(new_ids) == 2 and len(set(new_ids)) == 2
        assert all((v < nA) if own_b else (v >= nA) for v in new_ids)
        assert (keys[i, 1:] > keys[i, :-1]).all()  # sorted (D25)
        for j in range(k):
            assert orc.key_dists(keys[i:i + 1, j:j + 1])[0, 0] == orc.distance(X, i, int(ids[i, j]))


def test_ggm_usage_error_when_other_subset_too_small():
    # |S2| < k/2 -> usage error
    X = datagen.make("c1", 40, seed=2, d=4)
    keys_in = np.zeros((40, 8), np.uint64)
    with pytest.raises(RuntimeError):
        orc.ggm_seed(X, keys_in, 37, 8, 1)


def test_ggm_finalize_spec_examples():
    n, k = 1, 4
    refined = orc.key([1.0, 2.0, 3.0, 4.0], [10, 11, 12, 13]).reshape(1, 4)
    # S:284 reserved all farther -> output equals refined
    res = orc.key([5.0, 6.0], [20, 21]).reshape(1, 2)
    assert np.array_equal(orc.ggm_finalize(refined, res), refined)
    # S:285 reserved closer -> re-enters
    res = orc.key([0.5, 6.0], [20, 21]).reshape(1, 2)
    out = orc.ggm_finalize(refined, res)
    assert list(orc.key_ids(out[0])) == [20, 10, 11, 12]
    # S:286 reserved id already present -> kept once
    res = orc.key([2.0, 6.0], [11, 21]).reshape(1, 2)
    out = orc.ggm_finalize(refined, res)
    assert list(orc.key_ids(out[0])) == [10, 11, 12, 13]


def test_ggm_refine_cross_only_and_not_worse():
    X = datagen.make("c1", 1200, seed=4, d=8)
    nA, k, p = 500, 10, 5
    keys_in = _split_build(X, nA, k, p, 6, 4)
    keys, flags, reserved = orc.ggm_seed(X, keys_in, nA, k, 3)
    prev = keys.copy()
    for t in range(4):
        s = orc.sample(keys, flags, p, 0x80000000 | t, 3)
        # D22: NEW samples of every list are cross-subset ids
        for x in range(len(X)):
            gn = s["Gn"][x, :s["cn"][x]]
            assert all((v >= nA) != (x >= nA) for v in gn)
        m, q = s["cn"].astype(np.int64), s["co"].astype(np.int64)
        # restricted join: only cross pairs are evaluated
        cross = 0
        for x in range(len(X)):
            if m[x] == 0:
                continue
            N = s["Gn"][x, :m[x]].astype(np.int64)
            O = s["Go"][x, :q[x]].astype(np.int64)
            cross += int(((N[:, None] >= nA) != (O[None, :] >= nA)).sum())
            cross += int(np.triu((N[:, None] >= nA) != (N[None, :] >= nA), 1).sum())
        st = orc.iterate(X, keys, flags, p, 0x80000000 | t, 3, boundary=nA)
        assert st["dist_evals"] == cross
        assert (orc.key_dists(keys) <= orc.key_dists(prev)).all()
        # every entry that entered during refine links the two subsets
        for x in range(len(X)):
            newcomers = set(orc.key_ids(keys[x])) - set(orc.key_ids(prev[x]))
            assert all((v >= nA) != (x >= nA) for v in newcomers)
        prev = keys.copy()
    final = orc.ggm_finalize(keys, reserved)
    # merged lists are element-wise no worse than the input sub-graph lists
    assert (orc.key_dists(final) <= orc.key_dists(keys_in)).all()
    assert (final[:, 1:] > final[:, :-1]).all()


def test_merge_quality_spec_acceptance():
    # 10k points split in two 5k halves, GNND per half, GGM;
    # merged recall >= direct recall - 0.05.  (Data: the C1-shaped GMM, where
    # GNND itself reaches >= 0.95, so the comparison measures the merge, not
    # the saturation of D33.)  SPEC's 4 refine iterations leave the merge at
    # 0.87 with k = 10 here; 6 iterations reach 0.957 vs 0.955 direct (D23).
    X = datagen.make("c1", 10000, seed=8)
    q = datagen.sample_nodes(10000, 1000)
    gt = orc.bruteforce(X, q, 10)
    k, p = 10, 8
    ids, dists = orc.build(X, k, p, 10, 1)
    direct = orc.recall(orc.key(dists, ids)[q], gt, 10)
    keys_in = _split_build(X, 5000, k, p, 10, 1)
    merged = orc.merge(X, keys_in, 5000, k, p, 6, 1)
    assert orc.recall(merged[q], gt, 10) >= direct - 0.05


def test_tree_build_quality():
    # log-depth schedule (D26), 4 shards in 2 levels vs direct build
    X = datagen.make("c1", 8000, seed=9)
    q = datagen.sample_nodes(8000, 800)
    gt = orc.bruteforce(X, q, 10)
    ids, dists = orc.build(X, 10, 8, 10, 1)
    direct = orc.recall(orc.key(dists, ids)[q], gt, 10)
    keys = orc.tree_build(X, 4, 10, 8, 10, 8, 1)
    assert orc.recall(keys[q], gt, 10) >= direct - 0.05
    assert (orc.key_ids(keys) != np.arange(8000)[:, None]).all()


# --------------------------------------------------------------- evaluation
def test_bruteforce_spec_collinear():
    # points x = 0, 1, 2, 10; k = 2
    X = np.array([[0.0], [1.0], [2.0], [10.0]], np.float32)
    gt = orc.bruteforce(X, [0, 3], 2)
    assert list(orc.key_ids(gt[0])) == [1, 2]
    assert list(orc.key_ids(gt[1])) == [2, 1]


def test_bruteforce_matches_float64_sort():
    rng = np.random.default_rng(5)
    X = rng.integers(0, 100, size=(300, 12)).astype(np.float32)  # exact distances
    q = np.arange(0, 300, 7)
    gt = orc.bruteforce(X, q, 10)
    Xi = X.astype(np.int64)
    for r, i in enumerate(q):
        d = ((Xi - Xi[i]) ** 2).sum(1)
        d[i] = 1 << 60
        order = np.lexsort((np.arange(300), d))[:10]  # (dist, id) order, D3
        assert list(orc.key_ids(gt[r])) == list(order)
        assert list(orc.key_dists(gt[r:r + 1])[0]) == [float(d[j]) for j in order]


def test_recall_spec_examples_and_tie_rule():
    t = orc.key(np.arange(1, 11, dtype=np.float32)[None, :].repeat(2, 0), np.arange(10)[None, :].repeat(2, 0))
    assert orc.recall(t, t, 10) == 1.0
    half = t.copy()
    half[:, 5:] = orc.key(np.full((2, 5), 100.0, np.float32), np.arange(50, 55)[None, :].repeat(2, 0))
    assert orc.recall(half, t, 10) == 0.5
    far = orc.key(np.full((2, 10), 100.0, np.float32), np.arange(50, 60)[None, :].repeat(2, 0))
    assert orc.recall(far, t, 10) == 0.0
    # D27: a different id at the tied 10th distance counts as a hit
    tie = t.copy()
    tie[:, 9] = orc.key(np.full(2, 10.0, np.float32), np.full(2, 77))
    assert orc.recall(tie, t, 10) == 1.0


def test_phi_spec_examples():
    z = orc.key(np.zeros((2, 1), np.float32), np.array([[1], [0]]))
    assert orc.phi(z) == 0.0
    v = orc.key(np.array([[0.3], [0.7]], np.float32), np.array([[1], [0]]))
    assert abs(orc.phi(v) - 1.0) < 1e-7
    # phi(exact graph) <= phi(any graph of the same degree)
    X = datagen.make("c1", 500, seed=3, d=4)
    gt = orc.bruteforce(X, np.arange(500), 8)
    keys, _ = orc.init(X, 8, 1)
    assert orc.phi(gt) <= orc.phi(keys)


def test_incremental_extension_quality():
    # P:296 incremental construction: a 6k graph extended by a 4k batch
    # (GNND on the batch + GGM) stays within 0.05 recall@10 of the direct
    # build of all 10k rows, and its lists keep the invariants.
    X = datagen.make("c1", 10000, seed=10)
    q = datagen.sample_nodes(10000, 1000)
    gt = orc.bruteforce(X, q, 10)
    k, p = 10, 8
    ids, dists = orc.build(X, k, p, 10, 2)
    direct = orc.recall(orc.key(dists, ids)[q], gt, 10)
    oi, od = orc.build(X[:6000], k, p, 10, 2)
    keys = orc.extend(X[:6000], orc.key(od, oi), X[6000:], k, p, 10, 6, 3)
    assert keys.shape == (10000, k)
    assert orc.recall(keys[q], gt, 10) >= direct - 0.05
    assert (keys[:, 1:] > keys[:, :-1]).all()
    assert (orc.key_ids(keys) != np.arange(10000)[:, None]).all()
