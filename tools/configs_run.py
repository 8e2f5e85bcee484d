"""Measure BASELINE.json configs[2..4] shapes on one GPU (CUDA events on the
launch stream; recall@10 on 10k sampled nodes against knng_bruteforce).

  c3     GIST1M-shaped: n x 960 fp32, k = 32, p = 16, L2 and cosine
  c4     DEEP-shaped sharded tree: S shards of n/S rows (96-d, unit rows),
         GNND per shard + log-depth GGM (sharded.py at world size 1), and the
         direct build of the same set for comparison
  c5     SIFT-shaped uint8 sharded tree: k = 16, p = 8

Usage: python tools/configs_run.py c3 [--n 1000000] | c4 [--n 8000000 --shards 8] | c5 ..."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402
from paper_2103_15386_b200.sharded import knng_build_sharded  # noqa: E402


def recall(X, dists, metric, nodes=10000):
    q = datagen.sample_nodes(X.shape[0], nodes)
    _, gd = K.knng_bruteforce(X, torch.from_numpy(q), 10, metric)
    mine = dists[torch.from_numpy(q).cuda().long(), :10]
    return float((mine <= gd[:, 9:10]).float().mean().item())


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


def gen(shape, n, parts, dtype="f32"):
    t0 = time.time()
    per = n // parts
    # components: SURVEY.md section 8(d) -- SIFT-like 1000 per 10^6 rows;
    # DEEP100M: 10^4 components for 10^8 rows, SIFT1B: 10^5 for 10^9, i.e.
    # 10^4 rows per component (kept at smaller n, so every shard of 8 sees
    # ~1250 rows of a component; D38)
    comps = max(1, n // 10_000) if (shape == "deep" or dtype == "u8") else datagen.SHAPES[shape][1] * max(1, n // 1_000_000)
    X = np.concatenate([datagen.make(shape, per, seed=1, part=i, components=comps, dtype=dtype)
                        for i in range(parts)])
    return torch.from_numpy(X).cuda(), time.time() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c3", "c4", "c5"])
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--iters", default="7", help="comma list: every value is measured")
    ap.add_argument("--merge-iters", default="6", help="one count, or one per tree level (comma list)")
    ap.add_argument("--p", type=int, default=None, help="sample size (default: 16 for c3/c4, 8 for c5)")
    ap.add_argument("--no-tree", action="store_true")
    a = ap.parse_args()
    mi = [int(x) for x in str(a.merge_iters).split(",")]
    a.merge_iters = mi[0] if len(mi) == 1 else mi
    out = []
    if a.config == "c3":
        n = a.n or 1_000_000
        X, gs = gen("gist", n, 1)
        for metric, it in [(m, int(i)) for m in ["l2", "cosine"] for i in a.iters.split(",")]:
            K.knng_build(X, 32, 2, 16, 42, metric)  # warm-up
            (ids, d), ms = timed(lambda: K.knng_build(X, 32, it, 16, 42, metric))
            st = K.knng_last_stats()
            out.append({"config": "C3 GIST1M-shaped", "n": n, "d": 960, "k": 32, "p": 16, "iters": it,
                        "metric": metric, "build_ms": ms, "recall_at_10": recall(X, d, metric),
                        "dist_evals": sum(s["dist_evals"] for s in st), "datagen_s": gs})
            print(json.dumps(out[-1]), flush=True)
    else:
        c4 = a.config == "c4"
        shape, k, p = ("deep", 32, 16) if c4 else ("sift", 16, 8)
        p = a.p or p
        n = a.n or (8_000_000 if c4 else 8_000_000)
        X, gs = gen(shape, n, a.shards, "f32" if c4 else "u8")
        name = "C4 DEEP-shaped" if c4 else "C5 SIFT-shaped uint8"
        its = [int(i) for i in a.iters.split(",")]
        for it in its:
            K.knng_build(X, k, 2, p, 42)  # warm-up
            (di, dd), dms = timed(lambda: K.knng_build(X, k, it, p, 42))
            print(json.dumps({"config": name, "mode": "direct", "n": n, "d": X.shape[1], "k": k, "p": p,
                              "iters": it, "build_ms": dms, "recall_at_10": recall(X, dd, "l2"),
                              "datagen_s": gs}), flush=True)
            del di, dd
        if not a.no_tree:
            it = its[-1]
            knng_build_sharded(X, a.shards, k, 1, 1, p, 42)  # warm-up (pools, kernel attributes)
            (ids, d), ms = timed(lambda: knng_build_sharded(X, a.shards, k, it, a.merge_iters, p, 42))
            print(json.dumps({"config": name, "mode": f"tree of {a.shards} shards (one GPU)", "n": n,
                              "d": X.shape[1], "k": k, "p": p, "iters": it, "merge_iters": a.merge_iters,
                              "build_ms": ms, "recall_at_10": recall(X, d, "l2")}), flush=True)


if __name__ == "__main__":
    main()
