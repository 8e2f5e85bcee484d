"""Pins of the oracle's primitives against values fixed outside the oracle:
published known-answer vectors, SPEC worked examples, closed forms."""
import json
import os

import numpy as np
import pytest

import oracle.oracle as orc
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _kat_rows():
    rows = []
    with open(os.path.join(GOLDEN, "philox_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            rows.append(line.split())
    return rows


def test_philox_random123_kat():
    n = 0
    for row in _kat_rows():
        if row[0] == "cxx26":
            continue
        v = [int(x, 16) for x in row]
        out = orc.philox(v[0:4], v[4:6])
        assert list(out) == v[6:10]
        n += 1
    assert n == 3


def test_philox_cxx26_10000th_invocation():
    (row,) = [r for r in _kat_rows() if r[0] == "cxx26"]
    block, seed, word, expect = (int(x) for x in row[1:])
    assert orc.philox([block, 0, 0, 0], [seed, 0])[word] == expect


def test_uniform_closed_form():
    # r64 = out1:out0; uniform = floor(r64 * N / 2^64)
    assert orc.uniform([0, 0, 7, 7], 1000) == 0
    assert orc.uniform([0xFFFFFFFF, 0xFFFFFFFF, 0, 0], 1000) == 999
    assert orc.uniform([0, 0x80000000, 0, 0], 1000) == 500
    assert orc.uniform([0, 0x40000000, 0, 0], 10**9) == 250_000_000
    rng = np.random.default_rng(0)
    for _ in range(200):
        lo, hi = (int(x) for x in rng.integers(0, 2**32, size=2))
        N = int(rng.integers(1, 2**40))
        assert orc.uniform([lo, hi, 0, 0], N) == ((hi << 32 | lo) * N) >> 64


def test_uniform_is_unbiased_enough():
    # 4096 draws into 8 bins: chi-square far below the 0.1% critical value
    cnt = np.zeros(8)
    for i in range(4096):
        cnt[orc.uniform(orc.philox([1, i, 0, 0], [42, 0]), 8)] += 1
    chi2 = ((cnt - 512.0) ** 2 / 512.0).sum()
    assert chi2 < 24.3


def test_metric_spec_examples():
    ex = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))["metric_eval"]
    for e in ex:
        X = np.array([e["u"], e["v"]], dtype=np.float32)
        m = orc.L2SQ if e["metric"] == "l2sq" else orc.COSINE
        assert orc.distance(X, 0, 1, m) == e["expect"], e["cite"]


def test_l2_integer_valued_is_exact():
    # integer-valued fp32 (SIFT-like): every partial sum is an integer < 2^24,
    # so the canonical fp32 result equals the exact integer sum of squares.
    rng = np.random.default_rng(1)
    X = rng.integers(0, 256, size=(50, 128)).astype(np.float32)
    Xi = X.astype(np.int64)
    for a in range(10):
        for b in range(10):
            exact = int(((Xi[a] - Xi[b]) ** 2).sum())
            assert orc.distance(X, a, b) == float(exact)
            assert orc.distance(X.astype(np.uint8), a, b) == float(exact)


def test_l2_within_fp32_error_bound_and_symmetric():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((40, 96)).astype(np.float32)
    X64 = X.astype(np.float64)
    eps = np.finfo(np.float32).eps
    for a in range(20):
        assert orc.distance(X, a, a) == 0.0
        for b in range(20):
            dab = orc.distance(X, a, b)
            assert dab == orc.distance(X, b, a)  # bit-exact symmetry (D5)
            exact = ((X64[a] - X64[b]) ** 2).sum()
            # sequential summation bound: |err| <= (d+1) eps sum|terms|
            assert abs(dab - exact) <= 97 * eps * exact + 1e-30


def test_cosine_properties():
    rng = np.random.default_rng(3)
    X = rng.standard_normal((30, 64)).astype(np.float32)
    X64 = X.astype(np.float64)
    for a in range(15):
        assert orc.distance(X, a, a, orc.COSINE) <= 1e-6
        for b in range(15):
            d = orc.distance(X, a, b, orc.COSINE)
            assert d >= 0.0
            exact = 1.0 - X64[a] @ X64[b] / np.linalg.norm(X64[a]) / np.linalg.norm(X64[b])
            assert abs(d - max(exact, 0.0)) <= 1e-5  # D6 tolerance
    # scale invariance of the normalised form (exact for powers of two)
    Y = X.copy()
    Y[1] *= 4.0
    assert orc.distance(Y, 0, 1, orc.COSINE) == orc.distance(X, 0, 1, orc.COSINE)


def test_pair_index_spec_and_bijection():
    ex = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))["pair_index"]
    for e in ex:
        assert list(orc.pair_index(e["t"])) == e["uv"], e["cite"]
    # Eq. 1-2 enumerate each pair u > v >= 0 exactly once, t = u(u-1)/2 + v
    # (P:181 offset), for every m up to 1024.
    m = 1024
    for t in range(m * (m - 1) // 2):
        u, v = orc.pair_index(t)
        assert 0 <= v < u < m and u * (u - 1) // 2 + v == t


def _mk_list(pairs):
    keys = orc.key([d for _, d in pairs], [i for i, _ in pairs]).astype(np.uint64)
    return keys, np.zeros(len(pairs), np.uint8)


def test_list_insert_spec_examples():
    ex = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))["list_insert_single_segment"]
    for e in ex:
        keys, flags = _mk_list(e["list"])
        cid, cd = e["insert"]
        ins = orc.list_insert(keys, flags, int(orc.key([cd], [cid])[0]))
        assert ins == e["inserted"], e["cite"]
        ek, _ = _mk_list(e["expect"])
        assert np.array_equal(keys, ek), e["cite"]
        if ins:
            pos = [i for i, _ in e["expect"]].index(cid)
            assert flags[pos] == 1 and flags.sum() == 1  # inserted entry is NEW


def test_list_insert_order_independent_and_equals_k_smallest_unique():
    # D17: any order of offers ends as the k smallest unique keys of the union
    rng = np.random.default_rng(4)
    for trial in range(200):
        k = int(rng.integers(1, 33))
        ids = rng.choice(200, size=k, replace=False)
        d0 = rng.integers(0, 50, size=k).astype(np.float32)
        base = np.sort(orc.key(d0, ids))
        dist_of = {int(i): float(x) for i, x in zip(ids, d0)}
        offers = []
        for _ in range(int(rng.integers(0, 60))):
            i = int(rng.integers(0, 200))
            if i not in dist_of:
                dist_of[i] = float(rng.integers(0, 50))
            offers.append(int(orc.key([dist_of[i]], [i])[0]))
        union = sorted(set(int(x) for x in base) | set(offers))
        expect = np.array(union[:k], dtype=np.uint64)
        results = []
        for rep in range(5):
            keys = base.copy()
            flags = np.zeros(k, np.uint8)
            for o in (offers if rep == 0 else list(rng.permutation(offers))):
                orc.list_insert(keys, flags, o)
            assert np.array_equal(keys, expect)
            orig = set(int(x) for x in base)
            assert all(flags[j] == (int(keys[j]) not in orig) for j in range(k))
            results.append(keys.copy())
