"""k_join time per join_kernel option on a shape (CUDA events per launch).
Usage: python tools/join_compare.py --shape deep --n 1000000 --opts 0,2 [--metric l2]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="deep")
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=None)
ap.add_argument("--k", type=int, default=32)
ap.add_argument("--p", type=int, default=16)
ap.add_argument("--iters", type=int, default=7)
ap.add_argument("--metric", default="l2")
ap.add_argument("--opts", default="0,2")
a = ap.parse_args()
X = (torch.from_numpy(datagen.make(a.shape, a.n, seed=1, d=a.d)) if a.n <= 2_000_000 else datagen.make_device(a.shape, a.n, seed=1)).cuda()
for o in a.opts.split(","):
    K.knng_set_option("join_kernel", int(o))
    K.knng_build(X, a.k, a.iters, a.p, 42, a.metric)
    K.knng_set_timing(True)
    K.knng_reset_timing()
    K.knng_build(X, a.k, a.iters, a.p, 42, a.metric)
    K.knng_set_timing(False)
    ms, n = K.knng_kernel_time("k_join")
    st = K.knng_last_stats()
    print(f"{a.shape} d={X.shape[1]} {a.metric} join_kernel={o}: k_join {ms / max(n, 1):.3f} ms/launch over {n}; "
          f"recomputed/candidates {sum(s['recomputed'] for s in st) / max(1, sum(s['candidates'] for s in st)):.2f}",
          flush=True)
K.knng_set_option("join_kernel", 0)
