"""Parity of the CUDA path (through the C ABI) with the oracle, element by
element on seeded inputs.  Integer/index work (ids, flags, sample tables)
must match bit-exactly; distances too, because both sides evaluate the
canonical order of DESIGN.md D5/D6 (the tolerance of BASELINE.json --
1e-5 relative -- is therefore met with zero error)."""
import os

import numpy as np
import pytest

import datagen
import oracle.oracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


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


# ------------------------------------------------------------------ Philox
def test_device_philox_known_answers(K):
    rows = [l.split() for l in open(os.path.join(GOLDEN, "philox_kat.txt")) if l.strip() and not l.startswith("#")]
    for r in rows:
        if r[0] == "cxx26":
            block, seed, word, expect = (int(x) for x in r[1:])
            out = K.knng_debug_philox(dev(np.array([[block, 0, 0, 0]], np.int32)), seed)
            assert int(out.cpu().numpy().view(np.uint32)[0, word]) == expect
            continue
        v = [int(x, 16) for x in r]
        seed = v[4] | (v[5] << 32)
        ctr = dev(np.array([v[0:4]], np.uint32).view(np.int32))
        out = K.knng_debug_philox(ctr, seed).cpu().numpy().view(np.uint32)[0]
        assert list(out) == v[6:10]
    # bulk agreement with the oracle generator
    rng = np.random.default_rng(0)
    ctr = rng.integers(0, 2**32, size=(512, 4), dtype=np.uint64).astype(np.uint32)
    out = K.knng_debug_philox(dev(ctr.view(np.int32)), 0x1234_5678_9ABC).cpu().numpy().view(np.uint32)
    for i in range(0, 512, 37):
        assert list(out[i]) == list(orc.philox(ctr[i], [0x56789ABC, 0x1234]))


# ------------------------------------------------------------------ init
CASES = [
    # (shape, n, d, k, p, dtype, metric)
    ("c1", 10000, 16, 10, 8, "f32", "l2"),       # BASELINE configs[0]
    ("sift", 6000, 128, 32, 16, "f32", "l2"),    # SIFT-shaped, 4 slabs
    ("sift", 3000, 128, 32, 16, "u8", "l2"),     # uint8 path (C5 dtype)
    ("c1", 2500, 100, 20, 7, "f32", "l2"),       # ragged d (last slab partial)
    ("c1", 1500, 7, 8, 3, "f32", "l2"),          # rows not 16-B aligned
    ("deep", 3000, 96, 16, 8, "f32", "cosine"),  # cosine (D6)
    ("uniform", 40, 3, 2, 1, "f32", "l2"),       # k=2, p=1 degenerate
    ("uniform", 33, 5, 32, 16, "f32", "l2"),     # n = k + 1 (every list is all others)
]


def _data(shape, n, d, dtype, seed=3):
    if shape == "sift":
        return datagen.make("sift", n, seed=seed, dtype=dtype)
    return datagen.make(shape, n, seed=seed, d=d)


def _metric(m):
    return orc.COSINE if m == "cosine" else orc.L2SQ


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-{c[1]}-{c[2]}-{c[3]}-{c[5]}-{c[6]}" for c in CASES])
def test_init_bit_exact(K, case):
    shape, n, d, k, p, dtype, metric = case
    X = _data(shape, n, d, dtype)
    ok, of = orc.init(X, k, 42, _metric(metric))
    gk, gf = K.knng_debug_init(dev(X), k, 42, metric)
    assert np.array_equal(u64(gk), ok)
    assert np.array_equal(gf.cpu().numpy(), of)


# ------------------------------------------------------------------ sampling
@pytest.mark.parametrize("n,k,p,seed", [(2000, 10, 8, 0), (5000, 32, 16, 1), (300, 6, 2, 2), (1000, 20, 13, 3)])
def test_sample_tables_bit_exact(K, n, k, p, seed):
    rng = np.random.default_rng(seed)
    X = datagen.make("c1", n, seed=seed, d=4)
    keys, flags = orc.init(X, k, seed)
    # a mixed NEW/OLD state after two iterations, plus random flags
    for t in range(2):
        orc.iterate(X, keys, flags, p, t, seed)
    flags = (rng.random(flags.shape) < 0.5).astype(np.uint8)
    tword = 0x80000000 | 5 if seed % 2 else 3
    s = orc.sample(keys, flags, p, tword, 99)
    Gn, cn, Go, co = K.knng_debug_sample(dev(keys.view(np.int64)), dev(flags), p, tword, 99)
    cn, co = cn.cpu().numpy(), co.cpu().numpy()
    assert np.array_equal(cn, s["cn"]) and np.array_equal(co, s["co"])
    Gn, Go = Gn.cpu().numpy().view(np.uint32), Go.cpu().numpy().view(np.uint32)
    for v in range(n):
        assert np.array_equal(Gn[v, :cn[v]], s["Gn"][v, :cn[v]])
        assert np.array_equal(Go[v, :co[v]], s["Go"][v, :co[v]])


# ------------------------------------------------------ iterations (teacher forced)
@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-{c[1]}-{c[2]}-{c[3]}-{c[5]}-{c[6]}" for c in CASES])
def test_iterations_teacher_forced_bit_exact(K, case):
    shape, n, d, k, p, dtype, metric = case
    X = _data(shape, n, d, dtype)
    m = _metric(metric)
    Xd = dev(X)
    keys, flags = orc.init(X, k, 7, m)
    for t in range(6):
        gk, gf = dev(keys.view(np.int64)), dev(flags)
        st = K.knng_debug_iterate(Xd, gk, gf, p, t, 7, -1, metric)
        ost = orc.iterate(X, keys, flags, p, t, 7, m)
        assert np.array_equal(u64(gk), keys), f"keys differ at iteration {t}"
        assert np.array_equal(gf.cpu().numpy(), flags), f"flags differ at iteration {t}"
        assert st["dist_evals"] == ost["dist_evals"]
        assert st["joins"] == ost["joins"] and st["sum_m"] == ost["sum_m"] and st["sum_q"] == ost["sum_q"]
        assert st["candidates"] == ost["candidates"]
        assert st["accepted"] == ost["accepted"]


@pytest.mark.parametrize("case", CASES[:3] + CASES[5:6], ids=lambda c: f"{c[0]}-{c[1]}-{c[5]}-{c[6]}")
def test_full_build_bit_exact(K, case):
    shape, n, d, k, p, dtype, metric = case
    X = _data(shape, n, d, dtype)
    iters = 8
    oi, od = orc.build(X, k, p, iters, 11, _metric(metric))
    gi, gd = K.knng_build(dev(X), k, iters, p, 11, metric)
    assert np.array_equal(gi.cpu().numpy().view(np.uint32), oi)
    assert np.array_equal(gd.cpu().numpy(), od)  # canonical order: 0 error
    # and the end-to-end host entry point gives the same graph
    hi, hd = K.knng_build_host(np.ascontiguousarray(X), k, iters, p, 11, metric)
    assert np.array_equal(hi, oi) and np.array_equal(hd, od)


def test_c1_end_to_end_recall_matches_oracle(K):
    # BASELINE configs[0]: n=10k GMM d=16, k=10, p=8, 10 iterations
    X = datagen.make("c1", 10000, seed=1)
    q = datagen.sample_nodes(10000, 2000)
    gt = orc.bruteforce(X, q, 10)
    oi, od = orc.build(X, 10, 8, 10, 42)
    gi, gd = K.knng_build(dev(X), 10, 10, 8, 42)
    gkeys = orc.key(gd.cpu().numpy(), gi.cpu().numpy().view(np.uint32))
    r_gpu = orc.recall(gkeys[q], gt, 10)
    r_orc = orc.recall(orc.key(od, oi)[q], gt, 10)
    assert abs(r_gpu - r_orc) <= 0.005
    assert r_gpu >= 0.94


def test_determinism_two_runs(K):
    X = dev(datagen.make("sift", 20000, seed=5))
    a = K.knng_build(X, 32, 6, 16, 3)
    b = K.knng_build(X, 32, 6, 16, 3)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


# ------------------------------------------------------------------ eval
@pytest.mark.parametrize("shape,n,d,dtype,metric", [("c1", 3000, 16, "f32", "l2"), ("sift", 4000, 128, "u8", "l2"),
                                                    ("deep", 2000, 96, "f32", "cosine"), ("c1", 1000, 7, "f32", "l2")])
def test_bruteforce_bit_exact(K, shape, n, d, dtype, metric):
    X = _data(shape, n, d, dtype)
    q = np.arange(0, n, 13, dtype=np.int64)
    o = orc.bruteforce(X, q, 10, _metric(metric))
    gi, gd = K.knng_bruteforce(dev(X), dev(q), 10, metric)
    assert np.array_equal(gi.cpu().numpy().view(np.uint32), orc.key_ids(o))
    assert np.array_equal(gd.cpu().numpy(), orc.key_dists(o))


def test_exact_u8_path_is_bit_identical_to_the_float_path(K):
    # option exact_u8 (include/knng.h): integer-valued float32 data in
    # [0, 255] with d <= 258 runs on an exact uint8 copy; both paths must
    # produce the oracle's graph bit for bit.
    X = datagen.make("sift", 5000, seed=9)  # integer-valued fp32
    oi, od = orc.build(X, 32, 16, 6, 5)
    Xd = dev(X)
    try:
        for opt in (1, 0):
            K.knng_set_option("exact_u8", opt)
            gi, gd = K.knng_build(Xd, 32, 6, 16, 5)
            assert K.knng_get_option("last_exact_u8") == opt
            assert np.array_equal(gi.cpu().numpy().view(np.uint32), oi)
            assert np.array_equal(gd.cpu().numpy(), od)
        # non-integer data never takes the integer path
        K.knng_set_option("exact_u8", 1)
        Y = X + np.float32(0.5)
        K.knng_build(dev(Y), 32, 2, 16, 5)
        assert K.knng_get_option("last_exact_u8") == 0
    finally:
        K.knng_set_option("exact_u8", 1)


@pytest.mark.parametrize("jk", [0, 1, 2])
@pytest.mark.parametrize("d", [128, 64])
def test_join_kernels_u8_match(K, jk, d):
    """Every join kernel (auto = tensor-core int8 Gram tile for these uint8
    rows, legacy, warp-specialised) gives the oracle's graph bit for bit, including a
    restricted (merge) run."""
    X = datagen.make("sift", 5000, seed=8, dtype="u8", d=d)
    assert X.dtype == np.uint8 and X.shape == (5000, d)
    oi, od = orc.build(X, 16, 8, 5, 3)
    nA = 2300
    ia, da = orc.build(X[:nA], 16, 8, 3, 4)
    ib, db = orc.build(X[nA:], 16, 8, 3, 5)
    keys_in = np.concatenate([orc.key(da, ia), orc.key(db, ib.astype(np.uint64) + np.uint64(nA))])
    expect = orc.merge(X, keys_in, nA, 16, 8, 3, 6, level=1)
    try:
        K.knng_set_option("join_kernel", jk)
        gi, gd = K.knng_build(dev(X), 16, 5, 8, 3)
        assert np.array_equal(gi.cpu().numpy().view(np.uint32), oi)
        assert np.array_equal(gd.cpu().numpy(), od)
        mi, md = K.knng_merge(dev(X[:nA]), dev(ia.view(np.int32)), dev(da), dev(X[nA:]), dev(ib.view(np.int32)),
                              dev(db), 16, 3, 8, seed=6, level=1)
        assert np.array_equal(mi.cpu().numpy().view(np.uint32), orc.key_ids(expect))
        assert np.array_equal(md.cpu().numpy(), orc.key_dists(expect))
    finally:
        K.knng_set_option("join_kernel", 0)


def test_legacy_join_kernel_matches(K):
    X = datagen.make("c1", 3000, seed=4)
    oi, od = orc.build(X, 10, 8, 6, 2)
    try:
        K.knng_set_option("join_kernel", 1)
        gi, gd = K.knng_build(dev(X), 10, 6, 8, 2)
        assert np.array_equal(gi.cpu().numpy().view(np.uint32), oi)
        assert np.array_equal(gd.cpu().numpy(), od)
    finally:
        K.knng_set_option("join_kernel", 0)


@pytest.mark.parametrize("jk", [0, 3, 4])
@pytest.mark.parametrize("shape,d,metric", [("deep", 96, "l2"), ("deep", 96, "cosine"), ("gist", 128, "l2"),
                                            ("c1", 32, "l2"), ("gist", 60, "cosine")])
def test_join_kernels_f32_match(K, jk, shape, d, metric):
    """Float rows: the CUDA-core warp-specialised join (auto) and the opt-in
    tensor-core join (4: TF32 Gram tile + canonical recomputation inside the
    error-bound window) both give the oracle's graph bit for bit, in a
    plain build and in a restricted (merge) run."""
    m = _metric(metric)
    X = datagen.make(shape, 5000, seed=12, d=d)
    oi, od = orc.build(X, 16, 8, 5, 3, m)
    nA = 2600
    ia, da = orc.build(X[:nA], 16, 8, 3, 4, m)
    ib, db = orc.build(X[nA:], 16, 8, 3, 5, m)
    keys_in = np.concatenate([orc.key(da, ia), orc.key(db, ib.astype(np.uint64) + np.uint64(nA))])
    expect = orc.merge(X, keys_in, nA, 16, 8, 3, 6, level=1, metric=m)
    try:
        K.knng_set_option("join_kernel", jk)
        gi, gd = K.knng_build(dev(X), 16, 5, 8, 3, metric)
        st = K.knng_last_stats()
        assert np.array_equal(gi.cpu().numpy().view(np.uint32), oi)
        assert np.array_equal(gd.cpu().numpy(), od)
        if jk == 4:  # the window holds at least the selected key of every candidate
            assert sum(s["recomputed"] for s in st) >= sum(s["candidates"] for s in st) > 0
        mi, md = K.knng_merge(dev(X[:nA]), dev(ia.view(np.int32)), dev(da), dev(X[nA:]), dev(ib.view(np.int32)),
                              dev(db), 16, 3, 8, seed=6, level=1, metric=metric)
        assert np.array_equal(mi.cpu().numpy().view(np.uint32), orc.key_ids(expect))
        assert np.array_equal(md.cpu().numpy(), orc.key_dists(expect))
    finally:
        K.knng_set_option("join_kernel", 0)


@pytest.mark.parametrize("metric", ["l2", "cosine"])
def test_gist_960_float_join_bit_exact(K, metric):
    """BASELINE configs[2] dimensionality (d = 960: 30 row slabs per sample
    row, the stage ring wraps inside one batch) on the automatic float join,
    in a build and in a restricted (merge) run, against the oracle."""
    m = _metric(metric)
    X = datagen.make("gist", 3000, seed=15, d=960)
    assert X.shape == (3000, 960)
    oi, od = orc.build(X, 16, 8, 4, 3, m)
    gi, gd = K.knng_build(dev(X), 16, 4, 8, 3, metric)
    assert np.array_equal(gi.cpu().numpy().view(np.uint32), oi)
    assert np.array_equal(gd.cpu().numpy(), od)
    nA = 1300
    ia, da = orc.build(X[:nA], 16, 8, 3, 4, m)
    ib, db = orc.build(X[nA:], 16, 8, 3, 5, m)
    keys_in = np.concatenate([orc.key(da, ia), orc.key(db, ib.astype(np.uint64) + np.uint64(nA))])
    expect = orc.merge(X, keys_in, nA, 16, 8, 2, 6, level=1, metric=m)
    mi, md = K.knng_merge(dev(X[:nA]), dev(ia.view(np.int32)), dev(da), dev(X[nA:]), dev(ib.view(np.int32)),
                          dev(db), 16, 2, 8, seed=6, level=1, metric=metric)
    assert np.array_equal(mi.cpu().numpy().view(np.uint32), orc.key_ids(expect))
    assert np.array_equal(md.cpu().numpy(), orc.key_dists(expect))


def test_misaligned_rows_take_the_legacy_join(K):
    """Rows whose base pointer is not 16-B aligned cannot use the cp.async
    joins; the build falls back to the batched join (its staging buffer is
    allocated on demand) and still equals the oracle."""
    X = datagen.make("c1", 3000, seed=14, d=16)
    oi, od = orc.build(X, 10, 8, 4, 5)
    flat = torch.zeros(X.size + 1, dtype=torch.float32, device="cuda")
    flat[1:] = torch.from_numpy(X.reshape(-1)).cuda()
    Xm = flat[1:].view(3000, 16)
    assert Xm.data_ptr() % 16 != 0
    gi, gd = K.knng_build(Xm, 10, 4, 8, 5)
    assert np.array_equal(gi.cpu().numpy().view(np.uint32), oi)
    assert np.array_equal(gd.cpu().numpy(), od)


def test_sift_shaped_50k_end_to_end_matches_oracle(K):
    """The bench's setting (SIFT-shaped, k = 32, p = 16, 7 iterations) at 50k
    rows: the whole GPU graph equals the oracle's, so recall@10 on sampled
    nodes is the oracle's (north star: within 0.005)."""
    X = datagen.make("sift", 50000, seed=1)
    q = datagen.sample_nodes(50000, 2000)
    gt = orc.bruteforce(X, q, 10)
    oi, od = orc.build(X, 32, 16, 7, 42)
    gi, gd = K.knng_build(dev(X), 32, 7, 16, 42)
    assert np.array_equal(gi.cpu().numpy().view(np.uint32), oi)
    assert np.array_equal(gd.cpu().numpy(), od)
    assert orc.recall(orc.key(od, oi)[q], gt, 10) >= 0.95
