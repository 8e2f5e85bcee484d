"""Per-kernel device time of one DEEP-shaped (continuous fp32, d = 96) build
generated on the GPU (datagen.make_device), CUDA events per launch.
Usage: python tools/deep_kt.py [--n 10000000] [--iters 8]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2103_15386_b200.knng as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--iters", type=int, default=8)
a = ap.parse_args()
X = datagen.make_device("deep", a.n, seed=2)
K.knng_build(X, 32, a.iters, 16, 42, "l2")
torch.cuda.synchronize()
K.knng_set_timing(True)
K.knng_reset_timing()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
K.knng_build(X, 32, a.iters, 16, 42, "l2")
e1.record()
torch.cuda.synchronize()
names = ["k_init", "k_merge_sample", "k_scan_reduce", "k_scan_bsums", "k_scan_final", "k_rev_scatter",
         "k_rev_select", "k_join", "k_merge", "k_export"]
kt = {nm: round(K.knng_kernel_time(nm)[0], 3) for nm in names}
K.knng_set_timing(False)
print(json.dumps({"n": a.n, "ms_per_build": round(e0.elapsed_time(e1), 3), "kernels_ms": kt}))
