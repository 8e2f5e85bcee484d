"""GPU parity of the GGM merge (Alg. 3) and full-size (BASELINE configs[1],
1M x 128) sampled parity of init and one iteration, through the C ABI.

Every oracle input is produced by the oracle or by datagen (never by the
CUDA path); expected values come from oracle/ only."""
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


def u64(t):
    return t.cpu().numpy().view(np.uint64)


MERGE_CASES = [
    # (shape, nA, nB, d, k, p, merge_iters, dtype, metric)
    ("c1", 1200, 1800, 16, 10, 8, 6, "f32", "l2"),
    ("sift", 2000, 2000, 128, 32, 16, 4, "f32", "l2"),
    ("sift", 1500, 1000, 128, 16, 8, 4, "u8", "l2"),
    ("c1", 700, 900, 20, 11, 5, 3, "f32", "l2"),      # odd k: keep 6, replace 5
    ("deep", 1000, 1200, 96, 16, 8, 3, "f32", "cosine"),
]


def _data(shape, n, d, dtype, seed):
    if shape == "sift":
        return datagen.make("sift", n, seed=seed, dtype=dtype)
    return datagen.make(shape, n, seed=seed, d=d)


@pytest.mark.parametrize("case", MERGE_CASES, ids=lambda c: f"{c[0]}-{c[1]}+{c[2]}-k{c[4]}-{c[7]}-{c[8]}")
def test_merge_bit_exact(K, case):
    shape, nA, nB, d, k, p, mi, dtype, metric = case
    m = orc.COSINE if metric == "cosine" else orc.L2SQ
    X = _data(shape, nA + nB, d, dtype, 4)
    XA, XB = X[:nA], X[nA:]
    ia, da = orc.build(XA, k, p, 5, 21, m)
    ib, db = orc.build(XB, k, p, 5, 22, m)
    keys_in = np.concatenate([orc.key(da, ia), orc.key(db, ib.astype(np.uint64) + np.uint64(nA))])
    expect = orc.merge(X, keys_in, nA, k, p, mi, 77, level=2, metric=m)
    gi, gd = K.knng_merge(dev(XA), dev(ia.view(np.int32)), dev(da), dev(XB), dev(ib.view(np.int32)), dev(db),
                          k, mi, p, seed=77, level=2, metric=metric)
    assert np.array_equal(gi.cpu().numpy().view(np.uint32), orc.key_ids(expect))
    assert np.array_equal(gd.cpu().numpy(), orc.key_dists(expect))


def test_merge_refine_iteration_teacher_forced(K):
    # one restricted GGM iteration (boundary = nA) from the oracle's seeded state
    X = datagen.make("c1", 3000, seed=9)
    nA, k, p = 1400, 10, 6
    ia, da = orc.build(X[:nA], k, p, 5, 1)
    ib, db = orc.build(X[nA:], k, p, 5, 2)
    keys_in = np.concatenate([orc.key(da, ia), orc.key(db, ib.astype(np.uint64) + np.uint64(nA))])
    keys, flags, _ = orc.ggm_seed(X, keys_in, nA, k, 5, level=1)
    Xd = dev(X)
    for t in range(4):
        tword = 0x80000000 | (1 << 16) | t
        gk, gf = dev(keys.view(np.int64)), dev(flags)
        st = K.knng_debug_iterate(Xd, gk, gf, p, tword, 5, nA)
        ost = orc.iterate(X, keys, flags, p, tword, 5, boundary=nA)
        assert np.array_equal(u64(gk), keys) and np.array_equal(gf.cpu().numpy(), flags)
        assert st["dist_evals"] == ost["dist_evals"] and st["accepted"] == ost["accepted"]


# ------------------------------------------------------------ full size (C2)
@pytest.fixture(scope="module")
def c2():
    X = datagen.make("sift", 1_000_000, seed=1)
    keys, flags = orc.init(X, 32, 42)
    return X, keys, flags


def test_fullsize_init_bit_exact(K, c2):
    X, keys, flags = c2
    gk, gf = K.knng_debug_init(dev(X), 32, 42)
    assert np.array_equal(u64(gk), keys)
    assert np.array_equal(gf.cpu().numpy(), flags)


def test_fullsize_iteration_sampled_targets(K, c2):
    # BASELINE configs[1] at full size, the kernels and launch configuration
    # of knng_build: one iteration from an oracle state with a seeded NEW/OLD
    # mix; the oracle evaluates the same definition on 2000 sampled targets.
    X, keys0, _ = c2
    rng = np.random.default_rng(3)
    flags0 = (rng.random(keys0.shape) < 0.4).astype(np.uint8)
    targets = datagen.sample_nodes(len(X), 2000, seed=8)
    mask = np.zeros(len(X), np.uint8)
    mask[targets] = 1
    ok, of = keys0.copy(), flags0.copy()
    orc.iterate(X, ok, of, 16, 3, 42, target_mask=mask)
    gk, gf = dev(keys0.view(np.int64)), dev(flags0)
    st = K.knng_debug_iterate(dev(X), gk, gf, 16, 3, 42)
    gk, gf = u64(gk), gf.cpu().numpy()
    assert np.array_equal(gk[targets], ok[targets])
    assert np.array_equal(gf[targets], of[targets])
    assert st["sum_q"] > 0 and st["joins"] > 900_000
    # properties that hold for every list at any size
    assert (gk[:, 1:] > gk[:, :-1]).all()
    assert (orc.key_ids(gk) != np.arange(len(X), dtype=np.uint32)[:, None]).all()
    assert (orc.key_dists(gk) <= orc.key_dists(keys0)).all()


# ------------------------------------------------- full size, float rows (C4 shape)
def test_fullsize_deep_iteration_sampled_targets(K):
    # DEEP-shaped continuous fp32 rows at 1M x 96 (the C4 shard shape; the
    # float join k_join_ws, not the exact-u8 path), one iteration from an
    # oracle state; the oracle evaluates 1500 sampled targets.
    X = datagen.make("deep", 1_000_000, seed=2)
    keys0, _ = orc.init(X, 32, 42)
    rng = np.random.default_rng(4)
    flags0 = (rng.random(keys0.shape) < 0.4).astype(np.uint8)
    targets = datagen.sample_nodes(len(X), 1500, seed=9)
    mask = np.zeros(len(X), np.uint8)
    mask[targets] = 1
    ok, of = keys0.copy(), flags0.copy()
    orc.iterate(X, ok, of, 16, 2, 42, target_mask=mask)
    gk, gf = dev(keys0.view(np.int64)), dev(flags0)
    st = K.knng_debug_iterate(dev(X), gk, gf, 16, 2, 42)
    assert K.knng_get_option("last_exact_u8") == 0
    gk, gf = u64(gk), gf.cpu().numpy()
    assert np.array_equal(gk[targets], ok[targets])
    assert np.array_equal(gf[targets], of[targets])
    assert st["joins"] > 900_000
    assert (gk[:, 1:] > gk[:, :-1]).all()
    assert (orc.key_dists(gk) <= orc.key_dists(keys0)).all()


def test_fullsize_ggm_2x500k_restricted_iteration_sampled_targets(K, c2):
    # the bench's GGM shape: C2 split into 2 x 500k.  Input graphs: each
    # half's random init (oracle), seeded by the oracle's GGM seed step; one
    # restricted refine iteration (boundary = 500k) on the GPU equals the
    # oracle's on 2000 sampled targets.
    X = c2[0]
    h = len(X) // 2
    ka, _ = orc.init(X[:h], 32, 5)
    kb, _ = orc.init(X[h:], 32, 6)
    keys_in = np.concatenate([ka, orc.key(orc.key_dists(kb), orc.key_ids(kb).astype(np.uint64) + np.uint64(h))])
    keys, flags, _ = orc.ggm_seed(X, keys_in, h, 32, 77, level=0)
    targets = datagen.sample_nodes(len(X), 2000, seed=10)
    mask = np.zeros(len(X), np.uint8)
    mask[targets] = 1
    tword = 0x80000000 | 1
    ok, of = keys.copy(), flags.copy()
    ost = orc.iterate(X, ok, of, 16, tword, 77, boundary=h, target_mask=mask)
    gk, gf = dev(keys.view(np.int64)), dev(flags)
    st = K.knng_debug_iterate(dev(X), gk, gf, 16, tword, 77, h)
    gk, gf = u64(gk), gf.cpu().numpy()
    assert np.array_equal(gk[targets], ok[targets])
    assert np.array_equal(gf[targets], of[targets])
    assert st["joins"] > 900_000 and ost["joins"] > 0
    # lists never get worse, and every entry a refine inserted is cross-subset
    assert (orc.key_dists(gk) <= orc.key_dists(keys)).all()
    for t in targets[:500]:
        fresh = set(orc.key_ids(gk[t]).tolist()) - set(orc.key_ids(keys[t]).tolist())
        assert all((v >= h) != (t >= h) for v in fresh)


@pytest.mark.parametrize("shape,dtype,metric", [("c1", "f32", "l2"), ("sift", "u8", "l2"), ("deep", "f32", "cosine")])
def test_extend_equals_oracle(K, shape, dtype, metric):
    # knng_extend = GNND on the batch + GGM into the existing graph
    m = orc.COSINE if metric == "cosine" else orc.L2SQ
    n_old, n_new, k, p = 2500, 1500, 16, 8
    X = (datagen.make("sift", n_old + n_new, seed=31, dtype=dtype) if shape == "sift"
         else datagen.make(shape, n_old + n_new, seed=31, d=32 if shape == "c1" else 96))
    oi, od = orc.build(X[:n_old], k, p, 5, 4, m)
    expect = orc.extend(X[:n_old], orc.key(od, oi), X[n_old:], k, p, 5, 4, 8, m)
    gi, gd = K.knng_extend(dev(X[:n_old]), dev(oi.view(np.int32)), dev(od), dev(X[n_old:]), k, 5, 4, p, seed=8,
                           metric=metric)
    assert np.array_equal(gi.cpu().numpy().view(np.uint32), orc.key_ids(expect))
    assert np.array_equal(gd.cpu().numpy(), orc.key_dists(expect))
    assert len(K.knng_last_stats()) == 5 + 4
