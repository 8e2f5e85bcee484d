"""GPU parity of the adjacent rows of SURVEY.md 8(f) N4: the chi-square
metric ("K-Square"; D39) on the CUDA-core tile, and the update modes
of the paper's ablation: GNND-r1 (every pair offered),
GNND with per-segment spinlocks and GNND-r2 with one lock per list
 -- each against the oracle evaluating the same definition."""
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


MET = {"l2": orc.L2SQ, "cosine": orc.COSINE, "chi2": orc.CHI2}


def _data(shape, n, d, dtype, seed):
    if shape == "sift":
        return datagen.make("sift", n, seed=seed, dtype=dtype)
    return datagen.make(shape, n, seed=seed, d=d)


@pytest.mark.parametrize("shape,n,d,dtype,jk", [("gist", 4000, 64, "f32", 0), ("gist", 3000, 30, "f32", 0),
                                                ("sift", 3000, 128, "u8", 0), ("gist", 2000, 64, "f32", 1)])
def test_chi2_build_and_merge_bit_exact(K, shape, n, d, dtype, jk):
    X = _data(shape, n, d, dtype, 5)
    oi, od = orc.build(X, 16, 8, 5, 3, orc.CHI2)
    try:
        K.knng_set_option("join_kernel", jk)
        gi, gd = K.knng_build(dev(X), 16, 5, 8, 3, "chi2")
        assert np.array_equal(gi.cpu().numpy().view(np.uint32), oi)
        assert np.array_equal(gd.cpu().numpy(), od)
        nA = n // 2
        ia, da = orc.build(X[:nA], 16, 8, 3, 4, orc.CHI2)
        ib, db = orc.build(X[nA:], 16, 8, 3, 5, orc.CHI2)
        keys_in = np.concatenate([orc.key(da, ia), orc.key(db, ib.astype(np.uint64) + np.uint64(nA))])
        expect = orc.merge(X, keys_in, nA, 16, 8, 3, 6, level=1, metric=orc.CHI2)
        mi, md = K.knng_merge(dev(X[:nA]), dev(ia.view(np.int32)), dev(da), dev(X[nA:]), dev(ib.view(np.int32)),
                              dev(db), 16, 3, 8, seed=6, level=1, metric="chi2")
        assert np.array_equal(mi.cpu().numpy().view(np.uint32), orc.key_ids(expect))
        assert np.array_equal(md.cpu().numpy(), orc.key_dists(expect))
    finally:
        K.knng_set_option("join_kernel", 0)


def test_chi2_bruteforce_and_domain(K):
    X = datagen.make("gist", 2000, seed=7, d=48)
    q = np.arange(0, 2000, 17, dtype=np.int64)
    o = orc.bruteforce(X, q, 10, orc.CHI2)
    gi, gd = K.knng_bruteforce(dev(X), dev(q), 10, "chi2")
    assert np.array_equal(gi.cpu().numpy().view(np.uint32), orc.key_ids(o))
    assert np.array_equal(gd.cpu().numpy(), orc.key_dists(o))
    Y = X.copy()
    Y[11, 3] = -1.0
    with pytest.raises(K.KnngError) as e:
        K.knng_build(dev(Y), 16, 2, 8, 3, "chi2")
    assert e.value.status == K.KNNG_E_DOMAIN


UPDATE_CASES = [
    # (shape, n, d, k, p, dtype, metric)
    ("c1", 3000, 16, 10, 8, "f32", "l2"),
    ("sift", 3000, 128, 32, 16, "u8", "l2"),
    ("deep", 2000, 96, 16, 8, "f32", "cosine"),
    ("gist", 2000, 40, 16, 8, "f32", "chi2"),
]


@pytest.mark.parametrize("mode", [1, 2, 3])
@pytest.mark.parametrize("case", UPDATE_CASES, ids=lambda c: f"{c[0]}-{c[5]}-{c[6]}")
def test_update_modes_bit_exact(K, mode, case):
    shape, n, d, k, p, dtype, metric = case
    X = _data(shape, n, d, dtype, 8)
    m = MET[metric]
    upd = orc.UPDATE_FULL if mode == 1 else orc.UPDATE_SELECTIVE
    with orc.options(update=upd):
        oi, od, ost = orc.build(X, k, p, 5, 2, m, with_stats=True)
        nA = n // 2 + 100
        ia, da = orc.build(X[:nA], k, p, 3, 4, m)
        ib, db = orc.build(X[nA:], k, p, 3, 5, m)
        keys_in = np.concatenate([orc.key(da, ia), orc.key(db, ib.astype(np.uint64) + np.uint64(nA))])
        expect = orc.merge(X, keys_in, nA, k, p, 3, 6, level=1, metric=m)
    try:
        K.knng_set_option("update", mode)
        gi, gd = K.knng_build(dev(X), k, 5, p, 2, metric)
        st = K.knng_last_stats()
        assert np.array_equal(gi.cpu().numpy().view(np.uint32), oi)
        assert np.array_equal(gd.cpu().numpy(), od)
        for a, b in zip(st, ost):
            assert a["dist_evals"] == b["dist_evals"] and a["candidates"] == b["candidates"]
            assert a["accepted"] == b["accepted"]
        mi, md = K.knng_merge(dev(X[:nA]), dev(ia.view(np.int32)), dev(da), dev(X[nA:]), dev(ib.view(np.int32)),
                              dev(db), k, 3, p, seed=6, level=1, metric=metric)
        assert np.array_equal(mi.cpu().numpy().view(np.uint32), orc.key_ids(expect))
        assert np.array_equal(md.cpu().numpy(), orc.key_dists(expect))
    finally:
        K.knng_set_option("update", 0)
