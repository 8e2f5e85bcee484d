"""GPU parity of the out-of-memory all-pairs construction (D41,
knng_build_ooc through the C ABI, host buffers in and out) against
oracle.allpairs_build, bit for bit; plus usage errors.

Every expected value comes from oracle/ on datagen inputs."""
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


CASES = [
    # (shape, n, d, dtype, shards, k, p, iters, merge_iters, metric)
    ("c1", 3000, 16, "f32", 3, 10, 8, 5, 3, "l2"),          # odd shard count, float join
    ("sift", 4000, 128, "u8", 4, 16, 8, 4, 3, "l2"),       # uint8 rows: tensor-core join
    ("sift", 3001, 128, "f32", 4, 16, 8, 4, 3, "l2"),      # ragged shards, exact-u8 path
    ("deep", 2400, 96, "f32", 2, 16, 8, 4, 4, "cosine"),
    ("c1", 1500, 16, "f32", 1, 10, 8, 5, 3, "l2"),          # one shard: the direct build
]


@pytest.mark.parametrize("shape,n,d,dtype,shards,k,p,iters,mi,metric", CASES)
def test_ooc_equals_oracle_allpairs(K, shape, n, d, dtype, shards, k, p, iters, mi, metric):
    X = datagen.make(shape, n, seed=21, dtype=dtype, d=d)
    m = {"l2": orc.L2SQ, "cosine": orc.COSINE}[metric]
    expect = orc.allpairs_build(X, shards, k, p, iters, mi, 9, m)
    ids, dists = K.knng_build_ooc(np.ascontiguousarray(X), k, iters, mi, p, shards, seed=9, metric=metric)
    assert np.array_equal(ids, orc.key_ids(expect))
    assert np.array_equal(dists, orc.key_dists(expect))
    st = K.knng_last_stats()
    assert len(st) == shards * iters + (shards * (shards - 1) // 2) * mi


def test_ooc_usage_errors(K):
    X = datagen.make("c1", 100, seed=1)
    with pytest.raises(K.KnngError, match="more than k rows"):
        K.knng_build_ooc(X, 10, 3, 2, 5, 20)
    with pytest.raises(K.KnngError, match="host buffers"):
        K.knng_build_ooc(X, 10, 3, 2, 5, 2, out_ids=torch.empty((100, 10), dtype=torch.int32, device="cuda"))
