"""Sweep (sample_size p, iterations) on the C2 workload: build time and
recall@10 on 10k sampled nodes (exact GT by knng_bruteforce)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402

n = int(os.environ.get("N", 1_000_000))
X = torch.from_numpy(datagen.make("sift", n, seed=1)).cuda()
q = torch.from_numpy(datagen.sample_nodes(n, 10000))
_, gd = K.knng_bruteforce(X, q, 10)
thr = gd[:, 9:10]
qi = q.cuda().long()
for p in [int(x) for x in os.environ.get("PS", "8,10,12,16").split(",")]:
    for it in [int(x) for x in os.environ.get("ITS", "4,5,6,7,8").split(",")]:
        K.knng_build(X, 32, it, p, 42)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ids, dists = K.knng_build(X, 32, it, p, 42)
        e1.record()
        torch.cuda.synchronize()
        rec = float((dists[qi, :10] <= thr).float().mean())
        print(f"p={p:2d} iters={it} build_ms={e0.elapsed_time(e1):7.2f} recall@10={rec:.4f}", flush=True)
