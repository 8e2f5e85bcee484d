"""GGM sweep on one GPU: recall@10 and time of knng_merge vs merge_iters for
SIFT-shaped halves, and of the sharded tree (all shards on one rank).
Usage: python tools/merge_sweep.py [--n-half 500000] [--tree 4]"""
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


def recall(X, ids, dists, nodes=10000):
    q = datagen.sample_nodes(X.shape[0], nodes)
    _, gd = K.knng_bruteforce(X, torch.from_numpy(q), 10)
    mine = dists[torch.from_numpy(q).cuda().long(), :10]
    return float((mine <= gd[:, 9:10]).float().mean().item())


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-half", type=int, default=500_000)
    ap.add_argument("--tree", type=int, default=4)
    ap.add_argument("--k", type=int, default=32)
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--iters", type=int, default=7)
    args = ap.parse_args()
    k, p = args.k, args.p
    nh = args.n_half
    X = torch.from_numpy(np.concatenate([datagen.make("sift", nh, seed=1, part=i, components=1000)
                                         for i in range(2)])).cuda()
    XA, XB = X[:nh], X[nh:]
    ia, da = K.knng_build(XA, k, args.iters, p, 42)
    ib, db = K.knng_build(XB, k, args.iters, p, 43)
    (gi, gd), ms = timed(lambda: K.knng_build(X, k, args.iters, p, 42))
    res = {"direct": {"ms": ms, "recall": recall(X, gi, gd)}, "merge": []}
    for mi in [2, 3, 4, 5, 6, 8]:
        (mi_ids, mi_d), ms = timed(lambda: K.knng_merge(XA, ia, da, XB, ib, db, k, mi, p, seed=42, level=0))
        st = K.knng_last_stats()
        res["merge"].append({"merge_iters": mi, "ms": ms, "recall": recall(X, mi_ids, mi_d),
                             "dist_evals": sum(s["dist_evals"] for s in st)})
        print(json.dumps(res["merge"][-1]), flush=True)
    # tree of `tree` shards of 2*nh/tree... use tree shards of nh each
    S = args.tree
    XT = torch.from_numpy(np.concatenate([datagen.make("sift", nh, seed=1, part=i, components=1000 * S // 2)
                                          for i in range(S)])).cuda()
    for mi in [4, 6, 8]:
        (ti, td), ms = timed(lambda: knng_build_sharded(XT, S, k, args.iters, mi, p, 42), reps=1)
        res.setdefault("tree", []).append({"shards": S, "n": S * nh, "merge_iters": mi, "ms": ms,
                                           "recall": recall(XT, ti, td)})
        print(json.dumps(res["tree"][-1]), flush=True)
    (di, dd), ms = timed(lambda: K.knng_build(XT, k, args.iters, p, 42), reps=1)
    res["tree_direct"] = {"ms": ms, "recall": recall(XT, di, dd)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
