"""Recall of the sharded tree vs shard count and merge iterations on one GPU
(DEEP- or SIFT-shaped), to choose merge_iters per level.
Usage: python tools/tree_levels.py --shape deep --n 8000000 --shards 2,4,8 --mi 6,10,14"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402
from paper_2103_15386_b200.sharded import knng_build_sharded  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="deep")
ap.add_argument("--n", type=int, default=8_000_000)
ap.add_argument("--parts", type=int, default=8)
ap.add_argument("--shards", default="2,4,8")
ap.add_argument("--mi", default="6,10,14")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--k", type=int, default=32)
ap.add_argument("--p", type=int, default=16)
ap.add_argument("--comps", type=int, default=0)
a = ap.parse_args()
per = a.n // a.parts
ap2 = a.n // 10_000 if a.shape == "deep" else datagen.SHAPES[a.shape][1] * max(1, a.n // 1_000_000)
comps = a.comps or ap2
X = torch.from_numpy(np.concatenate([datagen.make(a.shape, per, seed=1, part=i, components=comps)
                                     for i in range(a.parts)])).cuda()
q = datagen.sample_nodes(a.n, 10000)
_, gd = K.knng_bruteforce(X, torch.from_numpy(q), 10)
qi = torch.from_numpy(q).cuda().long()
for S in [int(s) for s in a.shards.split(",")]:
    for mi in [int(m) for m in a.mi.split(",")]:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ids, d = knng_build_sharded(X, S, a.k, a.iters, mi, a.p, 42)
        e1.record()
        torch.cuda.synchronize()
        rec = float((d[qi, :10] <= gd[:, 9:10]).float().mean())
        print(json.dumps({"shape": a.shape, "n": a.n, "shards": S, "iters": a.iters, "merge_iters": mi,
                          "ms": e0.elapsed_time(e1), "recall_at_10": rec}), flush=True)
        del ids, d
