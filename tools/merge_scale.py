"""GGM recall vs scale on one GPU: two halves built with knng_build, merged
with knng_merge; the direct build of the union for comparison.
Usage: python tools/merge_scale.py --shape deep --halves 10000,100000,1000000 --comp-per 400"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="deep")
ap.add_argument("--halves", default="10000,100000,1000000")
ap.add_argument("--comp-per", type=int, default=400, help="points per mixture component per half")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--mi", default="4,8,12")
a = ap.parse_args()
k, p = 32, 16
for h in [int(x) for x in a.halves.split(",")]:
    comps = max(1, h // a.comp_per)
    X = torch.from_numpy(np.concatenate([datagen.make(a.shape, h, seed=1, part=i, components=comps)
                                         for i in range(2)])).cuda()
    n = 2 * h
    q = datagen.sample_nodes(n, 5000)
    _, gd = K.knng_bruteforce(X, torch.from_numpy(q), 10)
    qi = torch.from_numpy(q).cuda().long()
    rec = lambda d: float((d[qi, :10] <= gd[:, 9:10]).float().mean())  # noqa: E731
    _, dd = K.knng_build(X, k, a.iters, p, 42)
    ia, da = K.knng_build(X[:h], k, a.iters, p, 42)
    ib, db = K.knng_build(X[h:], k, a.iters, p, 43)
    for mi in [int(m) for m in a.mi.split(",")]:
        _, md = K.knng_merge(X[:h], ia, da, X[h:], ib, db, k, mi, p, seed=42)
        st = K.knng_last_stats()
        print(json.dumps({"shape": a.shape, "half": h, "components": comps, "iters": a.iters, "merge_iters": mi,
                          "direct": rec(dd), "merged": rec(md),
                          "accepted_per_iter": [s["accepted"] for s in st]}), flush=True)
