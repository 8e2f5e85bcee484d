"""Full-size C2 oracle run (SURVEY.md 8(d) "C2 runs fully once"; VERDICT r01
item 2): the single-threaded oracle GNND build of the bench's exact workload
(datagen 'sift', n = 10^6, seed 1; k 32, p 16, 7 iterations, seed 42), pinned
to one core, plus its recall@10 on the bench's 10k sampled nodes against the
oracle's own brute force (eval, run in parallel worker processes).

Writes tests/golden/c2_oracle_full.json: sha256 of the oracle graph (ids u32
and dists f32, row-major [n][k]), its recall, the build time and the host.
Only oracle/ and datagen/ are called (the stored values never come from the
CUDA path); tests/test_gpu_c2_fullsize.py compares the GPU build with it.

    python tools/oracle_c2_full.py [--workers 7]
"""
import argparse
import hashlib
import json
import multiprocessing as mp
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle.oracle as orc  # noqa: E402

N, K, P, ITERS, SEED, DATA_SEED, NODES = 1_000_000, 32, 16, 7, 42, 1, 10_000


def _gt_worker(args):
    core, queries = args
    try:
        os.sched_setaffinity(0, {core})
    except OSError:
        pass
    X = datagen.make("sift", N, seed=DATA_SEED)
    return orc.bruteforce(X, queries, 10)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c2_oracle_full.json"))
    a = ap.parse_args()
    nodes = datagen.sample_nodes(N, NODES)
    # exact ground truth on worker cores 1.. (not the timed baseline)
    chunks = np.array_split(nodes, a.workers)
    ncpu = os.cpu_count() or 1
    pool = mp.get_context("fork").Pool(a.workers)
    gt_async = pool.map_async(_gt_worker, [(1 + i % max(1, ncpu - 1), c) for i, c in enumerate(chunks)])
    # the timed oracle build, pinned to core 0
    os.sched_setaffinity(0, {0})
    X = datagen.make("sift", N, seed=DATA_SEED)
    t0 = time.perf_counter()
    ids, dists = orc.build(X, K, P, ITERS, SEED)
    build_s = time.perf_counter() - t0
    truth = np.concatenate(gt_async.get())
    pool.close()
    gkeys = orc.key(dists[nodes], ids[nodes].astype(np.uint64))
    rec = orc.recall(gkeys, truth, 10)
    out = {
        "what": "oracle GNND build of C2 (datagen 'sift' n=1e6 seed 1; k 32, p 16, iters 7, seed 42, L2); "
                "written by tools/oracle_c2_full.py (oracle/ + datagen/ only)",
        "n": N, "d": 128, "k": K, "p": P, "iters": ITERS, "seed": SEED, "data_seed": DATA_SEED,
        "sha256_ids_u32": hashlib.sha256(np.ascontiguousarray(ids, np.uint32).tobytes()).hexdigest(),
        "sha256_dists_f32": hashlib.sha256(np.ascontiguousarray(dists, np.float32).tobytes()).hexdigest(),
        "sha256_truth10": hashlib.sha256(truth.tobytes()).hexdigest(),
        "recall_at_10": rec, "recall_nodes": NODES,
        "phi": orc.phi(orc.key(dists, ids.astype(np.uint64))),
        "build_seconds_one_core": build_s, "cpu_model": cpu_model(), "nproc": os.cpu_count(),
        "pinned_core": 0,
    }
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
