"""Per-kernel device time of one knng_merge (2 x 500k SIFT-shaped halves) per
join_kernel option.  Usage: python tools/ggm_times.py [--opts 0,5] [--mi 6]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402
from kernel_times import NAMES  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--opts", default="0,5")
ap.add_argument("--mi", type=int, default=6)
a = ap.parse_args()
X = torch.from_numpy(datagen.make("sift", 1_000_000, seed=1)).cuda()
h = 500_000
ia, da = K.knng_build(X[:h], 32, 7, 16, 42)
ib, db = K.knng_build(X[h:], 32, 7, 16, 43)
for o in a.opts.split(","):
    K.knng_set_option("join_kernel", int(o))
    K.knng_merge(X[:h], ia, da, X[h:], ib, db, 32, a.mi, 16, seed=42)
    K.knng_set_timing(True)
    K.knng_reset_timing()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    K.knng_merge(X[:h], ia, da, X[h:], ib, db, 32, a.mi, 16, seed=42)
    e1.record()
    torch.cuda.synchronize()
    K.knng_set_timing(False)
    per = {}
    for nm in NAMES:
        ms, cnt = K.knng_kernel_time(nm)
        if cnt:
            per[nm] = round(ms, 3)
    print(json.dumps({"join_kernel": int(o), "merge_ms": e0.elapsed_time(e1), "kernels": per,
                      "stats": K.knng_last_stats()}), flush=True)
K.knng_set_option("join_kernel", 0)
