"""One SIFT1M-shaped GNND build for profiling under ncu (never a bench value).

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python tools/prof_build.py
  ncu --set full --clock-control none --import-source on -k regex:k_join \
      -s 3 -c 1 -o gpurun_out/join python tools/prof_build.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--k", type=int, default=32)
ap.add_argument("--p", type=int, default=16)
ap.add_argument("--iters", type=int, default=8)
ap.add_argument("--builds", type=int, default=1)
ap.add_argument("--shape", default="sift")
ap.add_argument("--metric", default="l2")
ap.add_argument("--join-kernel", type=int, default=0)
a = ap.parse_args()
if a.shape == "sift":
    cache = f"/tmp/sift_{a.n}.npy"  # datagen takes ~25 s per 1M rows; reuse within one box session
    if os.path.exists(cache):
        Xh = np.load(cache)
    else:
        Xh = datagen.make("sift", a.n, seed=1)
        np.save(cache, Xh)
    X = torch.from_numpy(Xh).cuda()
else:
    X = datagen.make_device(a.shape, a.n, seed=1)
K.knng_set_option("join_kernel", a.join_kernel)
for _ in range(a.builds):
    K.knng_build(X, a.k, a.iters, a.p, 42, a.metric)
torch.cuda.synchronize()
print("stats", K.knng_last_stats())
